// How many 2-CTA clusters of a 1-CTA-per-SM kernel (the paired attention's footprint: 384
// threads, ~225 KB dynamic smem) can be resident at once on this GPU?  148 SMs would allow 74
// if every GPC had an even number of usable SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  int smem = 225 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; cs *= 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148 * cs);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs resident (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
