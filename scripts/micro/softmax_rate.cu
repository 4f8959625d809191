// Microbenchmark: throughput of the attention softmax's exponential loop alone (no MMA, no TMEM):
// 8 warps per SM (two per SMSP, like the kernel's two softmax warpgroups), each thread owns a
// 128-column row; per column pair: FFMA2 (scale, subtract max), two exp2, FADD2 (row sum) and a
// bf16x2 pack.  POLY of every 16 pairs use the FMA-pipe Cody-Waite + degree-3 polynomial instead
// of MUFU.EX2 (the attention kernel's exp2_poly2).  Reports exponentials per clock per SM
// (MUFU alone: 16).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o softmax_rate softmax_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2502_12085_b200/csrc/sm100.cuh"

using namespace apb::sm100;

__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float x0, x1;
  f2_unpack(x2, x0, x1);
  x2 = f2_pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t magic = f2_pack(12582912.f, 12582912.f), nmagic = f2_pack(-12582912.f, -12582912.f);
  const uint64_t t2 = fadd2(x2, magic);
  const uint64_t j2 = fadd2(t2, nmagic);
  const uint64_t f2 = ffma2(j2, f2_pack(-1.f, -1.f), x2);
  uint64_t p2 = ffma2(f2_pack(0.05517166681468331f, 0.05517166681468331f), f2, f2_pack(0.2426111350945245f, 0.2426111350945245f));
  p2 = ffma2(p2, f2, f2_pack(0.6932609870112001f, 0.6932609870112001f));
  p2 = ffma2(p2, f2, f2_pack(0.9999280727914263f, 0.9999280727914263f));
  float t0, t1, q0, q1;
  f2_unpack(t2, t0, t1);
  f2_unpack(p2, q0, q1);
  const uint32_t r0 = __float_as_uint(t0) * (1u << 23) + __float_as_uint(q0);
  const uint32_t r1 = __float_as_uint(t1) * (1u << 23) + __float_as_uint(q1);
  return f2_pack(__uint_as_float(r0), __uint_as_float(r1));
}

template <int POLY>
__global__ void __launch_bounds__(256, 1) softmax_kernel(const float* in, unsigned long long* cycles, uint32_t* sink,
                                                         int iters) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  uint32_t chk = 0;
  uint64_t acc[4] = {0, 0, 0, 0};
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float m = 4.f + it * 1e-6f;
    const uint64_t sc2 = f2_pack(0.18f, 0.18f), nm2 = f2_pack(-m, -m);
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const uint64_t x2 = ffma2(f2_pack(s[2 * c], s[2 * c + 1]), sc2, nm2);
      float p0, p1;
      uint64_t p2;
      if ((c % 16) < POLY) {
        p2 = exp2_poly2(x2);
        f2_unpack(p2, p0, p1);
      } else {
        float x0, x1;
        f2_unpack(x2, x0, x1);
        p0 = ex2(x0);
        p1 = ex2(x1);
        p2 = f2_pack(p0, p1);
      }
      acc[c & 3] = fadd2(acc[c & 3], p2);
      chk ^= pack_bf16x2(p0, p1);
    }
  }
  const unsigned long long t1 = clock64();
  float a0, a1;
  f2_unpack(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), a0, a1);
  sink[blockIdx.x * 256 + threadIdx.x] = chk ^ __float_as_uint(a0 + a1);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int POLY>
void run(int sms, const float* in, unsigned long long* cyc, uint32_t* sink) {
  const int iters = 2000;
  softmax_kernel<POLY><<<sms, 256>>>(in, cyc, sink, iters);
  softmax_kernel<POLY><<<sms, 256>>>(in, cyc, sink, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  printf("poly %2d/16 pairs: %6.2f exp/clk/SM  (MUFU-only bound 16)\n", POLY, 256.0 * iters * 128 / c);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* in;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&in, 1024 * 4);
  cudaMalloc(&cyc, 8 * sms);
  cudaMalloc(&sink, 4 * 256 * sms);
  float hin[1024];
  for (int i = 0; i < 1024; ++i) hin[i] = (float)((i * 37) % 101) * 0.05f;
  cudaMemcpy(in, hin, sizeof(hin), cudaMemcpyHostToDevice);
  run<0>(sms, in, cyc, sink);
  run<2>(sms, in, cyc, sink);
  run<4>(sms, in, cyc, sink);
  run<6>(sms, in, cyc, sink);
  run<8>(sms, in, cyc, sink);
  return 0;
}
