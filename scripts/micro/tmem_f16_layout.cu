// Probe: TMEM layout of an f16 accumulator (tcgen05.mma kind::f16, f16 A/B, f16 D), M128 N128 K16.
// A = 1, B[n][k] = n  =>  D[m][n] = 16 n (exact in f16).  Thread 0 (lane 0 = row 0) loads 128 TMEM
// columns and prints the raw 32-bit words: packed f16x2 pairs would read (32j, 32j+16) in word j.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_f16_layout tmem_f16_layout.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../paper_2502_12085_b200/csrc/sm100.cuh"

using namespace apb::sm100;

__global__ void __launch_bounds__(128, 1) probe(uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  // K-major SW128 tiles of [128 rows][64 cols] f16; only the first 16 columns (K = 16) are used.
  __half* A = reinterpret_cast<__half*>(smem);
  __half* B = reinterpret_cast<__half*>(smem + 128 * 128);
  for (int i = threadIdx.x; i < 128 * 64; i += 128) {
    const int r = i / 64, c = i % 64;
    // SW128: 16-byte chunk index XOR (row & 7) within each 128-byte row
    const int chunk = c / 8, within = c % 8;
    const int pos = r * 64 + ((chunk ^ (r & 7)) * 8) + within;
    A[pos] = __float2half(c < 16 ? 1.f : 0.f);
    B[pos] = __float2half(c < 16 ? (float)r : 0.f);
  }
  const uint32_t bar = smem_u32(smem + 2 * 128 * 128);
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // idesc: c_format f16 (0) at [4,6), a/b format f16 (0), K-major, N>>3 at 17, M>>4 at 24
  const uint32_t idesc = ((128u >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    mma_ss(tmem, sdesc_sw128(smem_u32(A), 16, 1024), sdesc_sw128(smem_u32(B), 16, 1024), idesc, 0);
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  if (threadIdx.x < 32) {
    uint32_t r[32];
    for (int c = 0; c < 128; c += 32) {
      tmem_ld32(tmem + c, r);
      tmem_wait_ld();
      if (threadIdx.x == 0)
        for (int e = 0; e < 32; ++e) out[c + e] = r[e];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 4);
  cudaMemset(d, 0xff, 128 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * 128 + 2048);
  probe<<<1, 128, 2 * 128 * 128 + 2048>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
  uint32_t h[128];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("row 0, TMEM columns 0..15 (raw words, then as f16 lo/hi):\n");
  for (int c = 0; c < 16; ++c) {
    __half_raw lo, hi;
    lo.x = h[c] & 0xffff;
    hi.x = h[c] >> 16;
    printf("  col %3d: 0x%08x  lo %7.1f  hi %7.1f\n", c, h[c], __half2float(__half(lo)), __half2float(__half(hi)));
  }
  printf("  col  64: 0x%08x   col 127: 0x%08x\n", h[64], h[127]);
  return 0;
}
