// layer_ops.cu — the model steps of Alg. apb_prefill around the hot path (SURVEY.md 8(f)
// NEXT #2): qkv_proj and FFN of a Llama-style decoder layer.
//
//   rmsnorm_kernel  y = x / sqrt(mean(x^2) + eps) * w          HBM-bound: 4*dim B per row
//   rope_kernel     in-place rotate-half RoPE on the Q and K heads of each qkv row, 16-byte
//                   accesses (reading G19: position = caller array, or pos_offset + row)   HBM-bound
//   swiglu_kernel   a = SiLU(g) * u for [g | u] rows                      HBM-bound
//   (the projection GEMMs and their fused epilogues are in gemm_sm100.cu)
//
// All element math is fp32; every output is rounded once to bf16 (reading G9).
#include <cuda_bf16.h>


#include "internal.h"

namespace apb {
namespace layer {

__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = static_cast<uint32_t>(f2bf(f[2 * i])) | (static_cast<uint32_t>(f2bf(f[2 * i + 1])) << 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// One 256-thread CTA per row; dim % 8 == 0.  Sum of squares in fp32 (fixed-order warp + CTA
// reduction), then the row is re-read (L1/L2-hot) and normalised.
__global__ void __launch_bounds__(256) rmsnorm_kernel(const uint16_t* __restrict__ x, int64_t xs,
                                                      const uint16_t* __restrict__ w, int dim, float eps,
                                                      uint16_t* __restrict__ y, int64_t ys) {
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * xs);
  const int nv = dim / 8;
  float ss = 0.f;
  for (int i = threadIdx.x; i < nv; i += 256) {
    float f[8];
    unpack8(__ldg(xr + i), f);
#pragma unroll
    for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  __shared__ float part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot += part[i];
  const float inv = rsqrtf(tot / static_cast<float>(dim) + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * ys);
  for (int i = threadIdx.x; i < nv; i += 256) {
    float f[8], g[8];
    unpack8(__ldg(xr + i), f);
    unpack8(__ldg(wr + i), g);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = f[e] * inv * g[e];
    yr[i] = pack8(f);
  }
}

// kRopeRows rows per CTA: the d/2 inverse frequencies theta^(-2i/d) once per CTA in fp64; per row
// the angles pos * inv_freq are reduced mod 2*pi in fp64 (positions reach 10^6: fp32 angles would
// be off by O(0.1) rad), then sin/cos in fp32 (__sincosf on the reduced angle; the fused ROPE
// epilogue of apb_gemm computes the same bits).  Each thread rotates 8 consecutive pairs
// (x_i, x_{i+d/2}) of one head with 16-byte loads / stores (d % 16 == 0), else one pair.
constexpr int kRopeRows = 4;
__global__ void __launch_bounds__(256) rope_kernel(uint16_t* __restrict__ x, int64_t row_stride, int64_t rows,
                                                   int n_heads, int d, const int32_t* __restrict__ positions,
                                                   int64_t pos_offset, double log2_theta) {
  __shared__ double inv[128];
  __shared__ float cs[kRopeRows][2][128];
  const int half = d / 2;
  const int64_t r0 = (int64_t)blockIdx.x * kRopeRows;
  for (int i = threadIdx.x; i < half; i += blockDim.x) inv[i] = exp2(-log2_theta * (2.0 * i) / d);
  __syncthreads();
  for (int t = threadIdx.x; t < kRopeRows * half; t += blockDim.x) {
    const int rr = t / half, i = t % half;
    const int64_t row = r0 + rr;
    if (row >= rows) continue;
    const double pos = positions ? static_cast<double>(positions[row]) : static_cast<double>(pos_offset + row);
    double a = pos * inv[i];
    a -= rint(a * 0.15915494309189535) * 6.283185307179586;  // |a| <= pi
    float sn, c;
    __sincosf(static_cast<float>(a), &sn, &c);  // |a| <= pi: MUFU sin/cos, abs. error ~2^-21 << bf16's 2^-9
    cs[rr][0][i] = c;
    cs[rr][1][i] = sn;
  }
  __syncthreads();
  if (half % 8 == 0) {
    const int per_head = half / 8;
    for (int t = threadIdx.x; t < kRopeRows * n_heads * per_head; t += blockDim.x) {
      const int rr = t / (n_heads * per_head), rem = t % (n_heads * per_head);
      const int64_t row = r0 + rr;
      if (row >= rows) continue;
      const int h = rem / per_head, i0 = (rem % per_head) * 8;
      uint16_t* p = x + row * row_stride + (int64_t)h * d;
      float f1[8], f2[8];
      unpack8(*reinterpret_cast<const uint4*>(p + i0), f1);
      unpack8(*reinterpret_cast<const uint4*>(p + half + i0), f2);
      float o1[8], o2[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float c = cs[rr][0][i0 + e], sn = cs[rr][1][i0 + e];
        o1[e] = f1[e] * c - f2[e] * sn;
        o2[e] = f2[e] * c + f1[e] * sn;
      }
      *reinterpret_cast<uint4*>(p + i0) = pack8(o1);
      *reinterpret_cast<uint4*>(p + half + i0) = pack8(o2);
    }
  } else {
    for (int t = threadIdx.x; t < kRopeRows * n_heads * half; t += blockDim.x) {
      const int rr = t / (n_heads * half), rem = t % (n_heads * half);
      const int64_t row = r0 + rr;
      if (row >= rows) continue;
      const int h = rem / half, i = rem % half;
      uint16_t* p = x + row * row_stride + (int64_t)h * d;
      const float x1 = bf2f(p[i]), x2 = bf2f(p[i + half]);
      const float c = cs[rr][0][i], sn = cs[rr][1][i];
      p[i] = f2bf(x1 * c - x2 * sn);
      p[i + half] = f2bf(x2 * c + x1 * sn);
    }
  }
}

// a = SiLU(g) * u, 8 elements per thread (one 16-byte load of g and of u, one store), one thread
// per item over the whole grid; inter % 8 == 0.
__global__ void __launch_bounds__(256) swiglu_kernel(const uint16_t* __restrict__ gu, int64_t gs, int inter,
                                                     uint16_t* __restrict__ out, int64_t os, int64_t rows) {
  const int nv = inter / 8;
  const int64_t t = blockIdx.x * 256ll + threadIdx.x;
  if (t >= rows * nv) return;
  const int64_t r = t / nv;
  const int c = static_cast<int>(t % nv);
  const uint4* g = reinterpret_cast<const uint4*>(gu + r * gs);
  float fg[8], fu[8];
  unpack8(__ldg(g + c), fg);
  unpack8(__ldg(g + nv + c), fu);
#pragma unroll
  for (int e = 0; e < 8; ++e) fg[e] = fg[e] / (1.f + __expf(-fg[e])) * fu[e];
  reinterpret_cast<uint4*>(out + r * os)[c] = pack8(fg);
}

}  // namespace layer

apb_status launch_rmsnorm(int64_t rows, int dim, const void* x, int64_t xs, const void* w, float eps, void* y,
                          int64_t ys, cudaStream_t stream) {
  layer::rmsnorm_kernel<<<(unsigned)rows, 256, 0, stream>>>(static_cast<const uint16_t*>(x), xs,
                                                           static_cast<const uint16_t*>(w), dim, eps,
                                                           static_cast<uint16_t*>(y), ys);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("rmsnorm launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_rope(int64_t rows, int n_heads, int d, void* x, int64_t row_stride, const int32_t* positions,
                       int64_t pos_offset, double theta, cudaStream_t stream) {
  const int64_t blocks = (rows + layer::kRopeRows - 1) / layer::kRopeRows;
  layer::rope_kernel<<<(unsigned)blocks, 256, 0, stream>>>(static_cast<uint16_t*>(x), row_stride, rows, n_heads, d,
                                                          positions, pos_offset, log2(theta));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("rope launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_swiglu(int64_t rows, int inter, const void* gu, int64_t gs, void* out, int64_t os,
                         cudaStream_t stream) {
  const int64_t work = rows * (inter / 8);
  const int64_t blocks = (work + 255) / 256;
  if (blocks > 0x7fffffffLL) return fail(APB_ERR_CONFIG, "swiglu: too many rows for one launch");
  layer::swiglu_kernel<<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const uint16_t*>(gu), gs, inter,
                                                            static_cast<uint16_t*>(out), os, rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("swiglu launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace apb
