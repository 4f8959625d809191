// select_phases.cu — phase timing of the radix select (one 1024-thread CTA per KV head) with three
// histogram variants: 0 = match.any-aggregated shared atomics, 1 = plain shared atomics,
// 2 = per-warp private histograms (32 x 256 bins) + plain atomics, merged by the 256 bin threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o select_phases select_phases.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int VAR>
__global__ void __launch_bounds__(1024) sel(const float* scores, int l_b, int lp, int32_t* out_idx, long long* t) {
  extern __shared__ uint32_t sm[];
  uint32_t* skeys = sm;                    // l_b
  uint32_t* whist = sm + l_b;              // 32 x 256 (VAR 2)
  __shared__ uint32_t hist[256];
  __shared__ uint32_t wtot[32];
  __shared__ uint32_t sh_prefix, sh_k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* s = scores + (long long)blockIdx.x * l_b;
  long long t0 = clock64();
  for (int i = tid; i < l_b; i += 1024) skeys[i] = order_key(__ldg(s + i));
  __syncthreads();
  long long tp[6];
  tp[0] = clock64();
  uint32_t prefix = 0, pmask = 0, kk = lp;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    if (tid < 256) hist[tid] = 0;
    if (VAR == 2) for (int b = lane; b < 256; b += 32) whist[warp * 256 + b] = 0;
    __syncthreads();
    for (int base = 0; base < l_b; base += 1024) {
      const int i = base + tid;
      uint32_t tag = 0xFFFFFFFFu;
      if (i < l_b) {
        const uint32_t key = skeys[i];
        if ((key & pmask) == prefix) tag = (key >> shift) & 255u;
      }
      if (VAR == 0) {
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, tag);
        if (tag != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[tag], (uint32_t)__popc(peers));
      } else if (VAR == 1) {
        if (tag != 0xFFFFFFFFu) atomicAdd(&hist[tag], 1u);
      } else {
        if (tag != 0xFFFFFFFFu) atomicAdd(&whist[warp * 256 + tag], 1u);
      }
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t g = 0;
      if (VAR == 2) { for (int w = 0; w < 32; ++w) g += whist[w * 256 + tid]; }
      else g = hist[tid];
      uint32_t incl = g;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, incl, o);
        if (lane + o < 32) incl += y;
      }
      if (lane == 0) wtot[warp] = incl;
      asm volatile("bar.sync 1, 256;");
      uint32_t above_w = 0;
      for (int w = 0; w < 8; ++w) if (w > warp) above_w += wtot[w];
      const uint32_t above = incl + above_w - g;
      if (above < kk && above + g >= kk) { sh_prefix = prefix | ((uint32_t)tid << shift); sh_k = kk - above; }
    }
    __syncthreads();
    prefix = sh_prefix; kk = sh_k; pmask |= 0xFFu << shift;
    tp[pass + 1] = clock64();
  }
  if (tid == 0) {
    t[blockIdx.x * 8 + 0] = tp[0] - t0;
    for (int p = 0; p < 4; ++p) t[blockIdx.x * 8 + 1 + p] = tp[p + 1] - tp[p];
    out_idx[blockIdx.x] = prefix;
  }
}

int main() {
  const int hk = 8, l_b = 16384, lp = 2048;
  std::vector<float> h(hk * l_b);
  std::mt19937 g(1); std::normal_distribution<float> nd;
  for (auto& x : h) x = nd(g);
  float* d; int32_t* o; long long* t;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 64 * 4); cudaMalloc(&t, hk * 8 * 8);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  for (int var = 0; var < 3; ++var) {
    const int smem = (l_b + (var == 2 ? 32 * 256 : 0)) * 4;
    auto k = var == 0 ? sel<0> : var == 1 ? sel<1> : sel<2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k<<<hk, 1024, smem>>>(d, l_b, lp, o, t);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) k<<<hk, 1024, smem>>>(d, l_b, lp, o, t);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long ht[8]; cudaMemcpy(ht, t, 64, cudaMemcpyDeviceToHost);
    printf("var %d: %.2f us/launch; clocks: stage %lld, passes %lld %lld %lld %lld  (%s)\n", var, ms * 1e3 / 20, ht[0],
           ht[1], ht[2], ht[3], ht[4], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
