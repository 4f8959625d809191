// Microbenchmark: per-SM throughput of FFMA, FFMA2, FADD2, MUFU.EX2, F2FP (bf16x2 pack), FMNMX3.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t f2(float a, float b){ uint64_t r; asm volatile("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;}
template <int OP>
__global__ void k(float* out, int iters) {
  float a[8]; uint64_t p[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; p[i] = f2(a[i], a[i] + 1); u[i] = 0x3c003c00u + i; }
  const uint64_t m = f2(0.999f, 0.998f), c = f2(1e-4f, 2e-4f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fmaf(a[i], 0.999f, 1e-4f);
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c));
      if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(c));
      if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 4) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); u[i] ^= r; a[i] += 1e-7f; }
      if (OP == 5) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i+3)&7]), "f"(a[(i+5)&7]));
      if (OP == 6) a[i] = a[i] + 1e-4f;
      if (OP == 7) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 8) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 10) { uint32_t r; asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(i+1)&7]), "f"(a[(i+2)&7])); u[i] ^= r; }
      if (OP == 11) { uint32_t r; asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                      asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a[(i+1)&7])), "r"(__float_as_uint(a[(i+2)&7]))); u[i] ^= r; }
      if (OP == 12) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c)); }
      if (OP == 13) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(i+1)&7]), "f"(a[(i+2)&7])); u[i] ^= r; }
      if (OP == 9) { uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); u[i] ^= r; a[i] += 1e-7f; }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); s += a[i] + x + y + u[i]; }
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"FFMA", "FFMA2", "FADD2", "MUFU.EX2", "F2FP.BF16x2", "FMNMX3", "FADD", "EX2.F16x2", "EX2.BF16x2", "F2FP.F16x2", "EX2+F2FP(it)", "EX2+PRMT(it)", "EX2+FFMA2(it)", "F2FP+LOP(it)"};
  const int iters = 4096;
  for (int op = 0; op < 14; ++op) {
    for (int warps : {4, 8, 16}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&]() {
        switch (op) { case 0: k<0><<<sms, 32*warps>>>(out, iters); break; case 1: k<1><<<sms, 32*warps>>>(out, iters); break;
                      case 2: k<2><<<sms, 32*warps>>>(out, iters); break; case 3: k<3><<<sms, 32*warps>>>(out, iters); break;
                      case 4: k<4><<<sms, 32*warps>>>(out, iters); break; case 5: k<5><<<sms, 32*warps>>>(out, iters); break;
                      case 6: k<6><<<sms, 32*warps>>>(out, iters); break; case 7: k<7><<<sms, 32*warps>>>(out, iters); break;
                      case 8: k<8><<<sms, 32*warps>>>(out, iters); break; case 9: k<9><<<sms, 32*warps>>>(out, iters); break;
                      case 10: k<10><<<sms, 32*warps>>>(out, iters); break; case 11: k<11><<<sms, 32*warps>>>(out, iters); break;
                      case 12: k<12><<<sms, 32*warps>>>(out, iters); break; case 13: k<13><<<sms, 32*warps>>>(out, iters); break; }
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double instr_per_sm = (double)warps * iters * 8;   // warp-instructions per SM
      double cycles = ms * 1e-3 * clk * 1e3;              // at the reported max clock
      printf("%-12s warps/SM %2d: %.2f warp-instr/clk/SM (%.1f ms)\n", names[op], warps, instr_per_sm / cycles, ms);
    }
  }
  return 0;
}
