// decode.cu — APB's distributed exact decode step (Alg. apb_decode; SURVEY
// NEXT #1): on host h the t new tokens' queries attend to the host's block KV cache;
// the last host also attends to the new tokens' own keys, causally among them.  The
// partial (A_h, lse_h) of every host is gathered and merged by log-sum-exp (MergeScore,
// P:753), which makes the result exact.
//
// decode_split_kernel: memory-bound split-KV ("flash decoding") — grid (key chunks of 256, KV
// heads); a CTA stages its V chunk in shared memory with coalesced 16-byte loads, each thread
// owns one key (its K row held in registers as bf16x2), computes the logits of the t*g query
// rows of that KV head, then the rows' softmax over the chunk and the P.V product over the
// staged V.  Output: one normalised partial (O, log2-sum-exp) per chunk in the workspace.
// merge_kernel: log-sum-exp merge of n partials per row — used both to fold the chunks of one
// host and, across hosts, as MergeScore.  Fixed merge order, no atomics: deterministic.
#include "internal.h"
#include "sm100.cuh"

namespace apb {
namespace dec {

using namespace apb::sm100;

constexpr int KC = 128;        // keys per CTA
constexpr int kThreads = 128;  // == KC: one key per thread in the logit phase
constexpr int kKPad = 16;      // bytes of padding per staged K row (conflict-free per-key reads)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem_src), "r"(valid ? 16 : 0) : "memory");
}

// shared memory: K chunk [KC][D*2 + pad] bf16, V chunk [KC][D] bf16, q rows [R][D] fp32
// (pre-scaled), probabilities [R][KC] fp32, row stats [2][R]
__host__ __device__ constexpr int decode_smem_bytes(int R, int D) {
  return KC * (D * 2 + kKPad) + KC * D * 2 + R * D * 4 + R * KC * 4 + 2 * R * 4;
}

// RT: compile-time bound on the query rows each thread accumulates in the P.V phase
// (ceil(R / (kThreads / (D/2)))), so the accumulators stay in registers without predicated waste.
template <int D, int RT>
__global__ void __launch_bounds__(kThreads) decode_split_kernel(const DecodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int kRowK = D * 2 + kKPad;
  const int R = p.t * p.g;  // query rows of this KV head: r = s * g + gi  (new token s, head j*g+gi)
  uint8_t* ks = smem;
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(smem + KC * kRowK);
  float* qs = reinterpret_cast<float*>(smem + KC * kRowK + KC * D * 2);
  float* ps = qs + R * D;
  float* ms = ps + R * KC;
  float* ls = ms + R;

  const int tid = threadIdx.x;
  const int split = blockIdx.x, j = blockIdx.y;
  const int64_t k0 = (int64_t)split * KC;
  const int64_t n_keys = p.cache_len + (p.has_new ? p.t : 0);

  // stage the chunk's K and V rows: every thread issues all of its 16-byte async copies at once.
  // Thread tid always copies 16-byte column chunk c = tid % kVec of rows tid / kVec + i * kRowsPerPass.
  constexpr int kVec = D / 8;
  constexpr int kRowsPerPass = kThreads / kVec;
  {
    const int c = tid % kVec;
    const int kk0 = tid / kVec;
    const int64_t cache_in_chunk = p.cache_len - k0;  // keys [0, cache_in_chunk) of the chunk are cached
    if (cache_in_chunk >= KC) {  // fast path: the whole chunk is cached
      const __nv_bfloat16* kb = p.k_cache + (k0 + kk0) * p.cache_row_stride + (int64_t)j * D + c * 8;
      const __nv_bfloat16* vb = p.v_cache + (k0 + kk0) * p.cache_row_stride + (int64_t)j * D + c * 8;
      const int64_t step = (int64_t)kRowsPerPass * p.cache_row_stride;
#pragma unroll
      for (int i = 0; i < KC / kRowsPerPass; ++i) {
        const int kk = kk0 + i * kRowsPerPass;
        cp_async16(ks + kk * kRowK + c * 16, kb + i * step, true);
        cp_async16(reinterpret_cast<uint8_t*>(vs) + (kk * D + c * 8) * 2, vb + i * step, true);
      }
    } else {
      for (int i = 0; i < KC / kRowsPerPass; ++i) {
        const int kk = kk0 + i * kRowsPerPass;
        const int64_t key = k0 + kk;
        const bool cached = key < p.cache_len, valid = key < n_keys;
        const __nv_bfloat16* kb = cached ? p.k_cache + key * p.cache_row_stride : p.k_new + (key - p.cache_len) * p.new_row_stride;
        const __nv_bfloat16* vb = cached ? p.v_cache + key * p.cache_row_stride : p.v_new + (key - p.cache_len) * p.new_row_stride;
        cp_async16(ks + kk * kRowK + c * 16, valid ? kb + (int64_t)j * D + c * 8 : p.q, valid);
        cp_async16(reinterpret_cast<uint8_t*>(vs) + (kk * D + c * 8) * 2, valid ? vb + (int64_t)j * D + c * 8 : p.q, valid);
      }
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // queries (pre-scaled into the log2 domain) while the copies fly
  for (int idx = tid; idx < R * D; idx += kThreads) {
    const int r = idx / D, e = idx % D;
    const int s = r / p.g, qh = j * p.g + r % p.g;
    qs[idx] = __bfloat162float(p.q[((int64_t)s * p.hq + qh) * D + e]) * p.scale_log2;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  // logits: thread = key, its K row read from the padded shared-memory copy
  {
    const int64_t key = k0 + tid;
    const bool valid = key < n_keys;
    const bool is_new = key >= p.cache_len;
    const int64_t jn = key - p.cache_len;  // index among the new tokens
    const uint4* krow = reinterpret_cast<const uint4*>(ks + tid * kRowK);
    for (int r = 0; r < R; ++r) {
      float sacc = -INFINITY;
      const bool visible = valid && (!is_new || jn <= r / p.g);  // new keys: causal among new tokens
      if (visible) {
        const uint64_t* qr2 = reinterpret_cast<const uint64_t*>(qs + r * D);
        uint64_t acc0 = 0ull, acc1 = 0ull;
#pragma unroll
        for (int c = 0; c < kVec; ++c) {
          const uint4 u = krow[c];
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            // bf16x2 -> fp32x2 is two shifts/selects; the dot product runs on packed FFMA2
            const uint64_t k2 = f2_pack(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u));
            if (h & 1)
              acc1 = ffma2(qr2[c * 4 + h], k2, acc1);
            else
              acc0 = ffma2(qr2[c * 4 + h], k2, acc0);
          }
        }
        float x0, x1, y0, y1;
        f2_unpack(acc0, x0, x1);
        f2_unpack(acc1, y0, y1);
        sacc = (x0 + x1) + (y0 + y1);
      }
      ps[r * KC + tid] = sacc;
    }
  }
  __syncthreads();

  // softmax over the chunk, one warp per row
  const int warp = tid / 32, lane = tid % 32;
  for (int r = warp; r < R; r += kThreads / 32) {
    float v[KC / 32];
    float m = -INFINITY;
#pragma unroll
    for (int q = 0; q < KC / 32; ++q) {
      v[q] = ps[r * KC + q * 32 + lane];
      m = fmaxf(m, v[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float mu = (m == -INFINITY) ? 0.f : m;
    float l = 0.f;
#pragma unroll
    for (int q = 0; q < KC / 32; ++q) {
      const float e = ex2(v[q] - mu);
      ps[r * KC + q * 32 + lane] = e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      ms[r] = m;
      ls[r] = l;
    }
  }
  __syncthreads();

  // O = P V over the staged chunk: thread = (row group, head_dim pair)
  constexpr int kPairs = D / 2;
  constexpr int kGroups = kThreads / kPairs;
  const int d2 = tid % kPairs, rg = tid / kPairs;
  const int64_t rem = n_keys - k0;
  const int kmax = rem <= 0 ? 0 : (rem < KC ? (int)rem : KC);
  const int rows_total = p.t * p.hq;
  constexpr int kRowsPerThread = RT;
  float acc[kRowsPerThread][2];
#pragma unroll
  for (int q = 0; q < kRowsPerThread; ++q) acc[q][0] = acc[q][1] = 0.f;
  const int nrow = (R - rg + kGroups - 1) / kGroups;  // rows rg, rg + kGroups, ... of this thread
#pragma unroll 4
  for (int kk = 0; kk < kmax; ++kk) {
    const uint32_t vw = *reinterpret_cast<const uint32_t*>(vs + kk * D + 2 * d2);
    const float vx = __uint_as_float(vw << 16), vy = __uint_as_float(vw & 0xffff0000u);
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
      if (q < nrow) {
        const float pr = ps[(rg + q * kGroups) * KC + kk];
        acc[q][0] = fmaf(pr, vx, acc[q][0]);
        acc[q][1] = fmaf(pr, vy, acc[q][1]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kRowsPerThread; ++q) {
    if (q >= nrow) break;
    const int r = rg + q * kGroups;
    const int s = r / p.g, qh = j * p.g + r % p.g;
    const int64_t row = (int64_t)s * p.hq + qh;
    const float l = ls[r];
    const float inv = l > 0.f ? 1.f / l : 0.f;
    float2* dst = reinterpret_cast<float2*>(p.ws_o + ((int64_t)split * rows_total + row) * D) + d2;
    *dst = make_float2(acc[q][0] * inv, acc[q][1] * inv);
    if (d2 == 0) p.ws_lse[(int64_t)split * rows_total + row] = l > 0.f ? ms[r] + __log2f(l) : -INFINITY;
  }
}

// LSE merge of n partials per row (MergeScore).  lse_in_log2 selects the input log base;
// the output lse is natural.  One CTA (8 warps) per row: the weights of all parts are formed once
// in shared memory (parallel max / sum); warp w accumulates parts w, w+8, ... (lanes across
// head_dim, coalesced), and the 8 warp partials are added in a fixed order — deterministic.
constexpr int kMergeWarps = 8;
template <int D, typename OutT>
__global__ void __launch_bounds__(kMergeWarps * 32) merge_kernel(int n, int64_t rows, const float* __restrict__ parts_o,
                                                                 const float* __restrict__ parts_lse, int64_t stride_o,
                                                                 int64_t stride_lse, int lse_in_log2,
                                                                 OutT* __restrict__ out, float* __restrict__ out_lse) {
  extern __shared__ float wsm[];  // [n] weights
  __shared__ float red[kMergeWarps];
  __shared__ float part[kMergeWarps][D];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const float to2 = lse_in_log2 ? 1.f : 1.4426950408889634f;  // convert to the log2 domain
  float m = -INFINITY;
  for (int h = tid; h < n; h += kMergeWarps * 32) {
    const float l = __ldg(parts_lse + h * stride_lse + row) * to2;
    wsm[h] = l;
    m = fmaxf(m, l);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < kMergeWarps; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float z = 0.f;
  for (int h = tid; h < n; h += kMergeWarps * 32) {
    const float w = (m == -INFINITY || wsm[h] == -INFINITY) ? 0.f : ex2(wsm[h] - m);
    wsm[h] = w;
    z += w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  z = 0.f;
#pragma unroll
  for (int w = 0; w < kMergeWarps; ++w) z += red[w];
  constexpr int kPer = D / 32;
  float acc[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) acc[e] = 0.f;
  for (int h = warp; h < n; h += kMergeWarps) {
    const float w = wsm[h];
    const float* src = parts_o + h * stride_o + row * D;
#pragma unroll
    for (int e = 0; e < kPer; ++e) acc[e] = fmaf(w, __ldg(src + e * 32 + lane), acc[e]);
  }
#pragma unroll
  for (int e = 0; e < kPer; ++e) part[warp][e * 32 + lane] = acc[e];
  __syncthreads();
  for (int e = tid; e < D; e += kMergeWarps * 32) {
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < kMergeWarps; ++w) sum += part[w][e];
    const float o = z > 0.f ? sum / z : 0.f;
    if constexpr (sizeof(OutT) == 2)
      out[row * D + e] = __float2bfloat16_rn(o);
    else
      out[row * D + e] = o;
  }
  if (tid == 0 && out_lse) out_lse[row] = (z > 0.f) ? (m + __log2f(z)) * 0.69314718055994530942f : -INFINITY;
}

}  // namespace dec

size_t decode_workspace_bytes(int64_t n_keys, int t, int hq, int D) {
  const int64_t splits = (n_keys + dec::KC - 1) / dec::KC;
  const int64_t rows = (int64_t)t * hq;
  size_t o = (size_t)splits * rows * D * sizeof(float);
  o = (o + 255) & ~size_t(255);
  return o + (size_t)splits * rows * sizeof(float);
}

apb_status launch_decode(const DecodeParams& p0, float* part_o, float* part_lse, cudaStream_t stream) {
  DecodeParams p = p0;
  const int64_t n_keys = p.cache_len + (p.has_new ? p.t : 0);
  const int64_t splits = (n_keys + dec::KC - 1) / dec::KC;
  const int64_t rows = (int64_t)p.t * p.hq;
  // (splits == 0: no key at all -> the merge below of zero parts writes O = 0, lse = -inf)
  size_t o = (size_t)splits * rows * p.D * sizeof(float);
  o = (o + 255) & ~size_t(255);
  p.ws_lse = reinterpret_cast<float*>(reinterpret_cast<char*>(p.ws_o) + o);
  dim3 grid((unsigned)splits, p.hk);
  if (splits > 0) {
    const int R = p.t * p.g;
    const int smem = dec::decode_smem_bytes(R, p.D);
    const int groups = dec::kThreads / (p.D / 2);
    const int rt = (R + groups - 1) / groups;  // rows per thread in the P.V phase
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dec::decode_smem_bytes(kDecodeRowsMax, p.D));
      kern<<<grid, dec::kThreads, smem, stream>>>(p);
    };
    if (p.D == 128) {
      if (rt <= 1) launch(dec::decode_split_kernel<128, 1>);
      else if (rt <= 2) launch(dec::decode_split_kernel<128, 2>);
      else if (rt <= 4) launch(dec::decode_split_kernel<128, 4>);
      else if (rt <= 8) launch(dec::decode_split_kernel<128, 8>);
      else if (rt <= 16) launch(dec::decode_split_kernel<128, 16>);
      else launch(dec::decode_split_kernel<128, 32>);
    } else {
      if (rt <= 1) launch(dec::decode_split_kernel<64, 1>);
      else if (rt <= 2) launch(dec::decode_split_kernel<64, 2>);
      else if (rt <= 4) launch(dec::decode_split_kernel<64, 4>);
      else if (rt <= 8) launch(dec::decode_split_kernel<64, 8>);
      else launch(dec::decode_split_kernel<64, 16>);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    count_launch();
  }
  // fold the chunks: fp32 partial of this host, natural-log lse
  return launch_merge((int)splits, rows, p.D, p.ws_o, p.ws_lse, rows * p.D, rows, 1, part_o, false, part_lse, stream);
}

apb_status launch_merge(int n, int64_t rows, int D, const float* parts_o, const float* parts_lse, int64_t stride_o,
                        int64_t stride_lse, int lse_in_log2, void* out, bool out_bf16, float* out_lse,
                        cudaStream_t stream) {
  if (rows == 0) return APB_OK;
  if (D == 128) {
    if (out_bf16)
      dec::merge_kernel<128, __nv_bfloat16><<<(unsigned)rows, dec::kMergeWarps * 32, (size_t)n * sizeof(float), stream>>>(
          n, rows, parts_o, parts_lse, stride_o, stride_lse, lse_in_log2, static_cast<__nv_bfloat16*>(out), out_lse);
    else
      dec::merge_kernel<128, float><<<(unsigned)rows, dec::kMergeWarps * 32, (size_t)n * sizeof(float), stream>>>(
          n, rows, parts_o, parts_lse, stride_o, stride_lse, lse_in_log2, static_cast<float*>(out), out_lse);
  } else {
    if (out_bf16)
      dec::merge_kernel<64, __nv_bfloat16><<<(unsigned)rows, dec::kMergeWarps * 32, (size_t)n * sizeof(float), stream>>>(
          n, rows, parts_o, parts_lse, stride_o, stride_lse, lse_in_log2, static_cast<__nv_bfloat16*>(out), out_lse);
    else
      dec::merge_kernel<64, float><<<(unsigned)rows, dec::kMergeWarps * 32, (size_t)n * sizeof(float), stream>>>(
          n, rows, parts_o, parts_lse, stride_o, stride_lse, lse_in_log2, static_cast<float*>(out), out_lse);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("merge launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace apb
