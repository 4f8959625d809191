// select_topk.cu — ArgTop-l_p per KV head + KV compaction (Alg. apb_prefill lines retbeg..retend,
// PAPER.md:713-714; Top-l_p at P:180).
//
// Kernel 1 (one CTA of 1024 threads per KV head): exact radix select of the l_p'-th largest
// score on order-preserving uint32 keys (4 passes of 8-bit digits over the L2-resident score
// row, shared-memory histograms), then one ordered compaction pass: index i is kept iff
// key > T, or key == T and fewer than `need` equal keys precede it (ties -> lower index,
// reading G5).  Output indices are ascending by construction.  Bit-exact, no floating point.
// Kernel 2: gather of the selected K and V rows (256 B each at d=128) into the packed send
// slot [2][hk][l_p'][d] — vectorised 16-byte copies spread over many CTAs (HBM-bound).
#include "internal.h"

namespace apb {
namespace sel {

constexpr int kThreads = 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0.0 -> +0.0 so both compare equal
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Block-wide exclusive scan of a per-thread 0/1 flag; returns the prefix, writes the total.
__device__ __forceinline__ uint32_t block_scan_flag(bool flag, uint32_t* warp_cnt, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ballot = __ballot_sync(0xffffffffu, flag);
  const uint32_t in_warp = __popc(ballot & ((1u << lane) - 1u));
  if (lane == 0) warp_cnt[warp] = __popc(ballot);
  __syncthreads();
  if (warp == 0) {
    uint32_t c = warp_cnt[lane];
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    warp_cnt[32 + lane] = incl - c;  // exclusive
    if (lane == 31) warp_cnt[64] = incl;
  }
  __syncthreads();
  const uint32_t pre = warp_cnt[32 + warp] + in_warp;
  total = warp_cnt[64];
  __syncthreads();
  return pre;
}

__global__ void __launch_bounds__(kThreads) select_kernel(const float* __restrict__ scores, int l_b, int lp,
                                                          int32_t* __restrict__ indices) {
  const int j = blockIdx.x;
  const float* s = scores + (int64_t)j * l_b;
  __shared__ uint32_t hist[256];
  __shared__ uint32_t warp_cnt[65];
  __shared__ uint32_t sh_prefix, sh_k;
  const int tid = threadIdx.x;

  uint32_t prefix = 0, pmask = 0, k = (uint32_t)lp;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int b = tid; b < 256; b += kThreads) hist[b] = 0;
    __syncthreads();
    for (int i = tid; i < l_b; i += kThreads) {
      const uint32_t key = order_key(__ldg(s + i));
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t cum = 0;
      for (int b = 255; b >= 0; --b) {
        if (cum + hist[b] >= k) {
          sh_prefix = prefix | ((uint32_t)b << shift);
          sh_k = k - cum;
          break;
        }
        cum += hist[b];
      }
    }
    __syncthreads();
    prefix = sh_prefix;
    k = sh_k;
    pmask |= 0xFFu << shift;
  }
  const uint32_t T = prefix;  // key of the l_p'-th largest score
  const uint32_t need_eq = k; // how many keys == T are taken (lowest indices first)

  uint32_t out_base = 0, eq_base = 0;
  int32_t* out = indices + (int64_t)j * lp;
  for (int base = 0; base < l_b && out_base < (uint32_t)lp; base += kThreads) {
    const int i = base + tid;
    const uint32_t key = i < l_b ? order_key(__ldg(s + i)) : 0u;
    const bool gt = i < l_b && key > T;
    const bool eq = i < l_b && key == T;
    uint32_t eq_total, sel_total;
    const uint32_t eq_rank = eq_base + block_scan_flag(eq, warp_cnt, eq_total);
    const bool sel = gt || (eq && eq_rank < need_eq);
    const uint32_t pos = out_base + block_scan_flag(sel, warp_cnt, sel_total);
    if (sel) out[pos] = i;
    out_base += sel_total;
    eq_base += eq_total;
  }
}

// Gather the selected rows: send[kv][j][m][:] = (kv ? V : K)[L_A + idx[j][m]][j][:]
template <int D>
__global__ void __launch_bounds__(256) compact_kernel(const int32_t* __restrict__ idx, const uint16_t* __restrict__ k,
                                                      const uint16_t* __restrict__ v, int64_t kv_row_stride, int L_A,
                                                      int lp, int hk, uint16_t* __restrict__ send) {
  constexpr int kPerRow = D / 8;  // 16-byte vectors per row
  constexpr int kRowsPerBlock = 256 / kPerRow;
  const int r = blockIdx.x * kRowsPerBlock + threadIdx.x / kPerRow;
  const int c = threadIdx.x % kPerRow;
  if (r >= lp) return;
  const int j = blockIdx.y, kv = blockIdx.z;
  const int64_t src_row = L_A + __ldg(idx + (int64_t)j * lp + r);
  const uint4* src = reinterpret_cast<const uint4*>((kv ? v : k) + src_row * kv_row_stride + (int64_t)j * D) + c;
  uint4* dst = reinterpret_cast<uint4*>(send + (((int64_t)kv * hk + j) * lp + r) * D) + c;
  *dst = __ldg(src);
}

}  // namespace sel

apb_status launch_select_compact(int l_b, int lp, int hk, int D, int L_A, const float* scores, const void* k,
                                 const void* v, int64_t kv_row_stride, int32_t* indices, void* send,
                                 cudaStream_t stream) {
  sel::select_kernel<<<hk, sel::kThreads, 0, stream>>>(scores, l_b, lp, indices);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("select launch: ") + cudaGetErrorString(e));
  const int rows_per_block = 256 / (D / 8);
  dim3 grid((lp + rows_per_block - 1) / rows_per_block, hk, 2);
  if (D == 128)
    sel::compact_kernel<128><<<grid, 256, 0, stream>>>(indices, static_cast<const uint16_t*>(k),
                                                        static_cast<const uint16_t*>(v), kv_row_stride, L_A, lp, hk,
                                                        static_cast<uint16_t*>(send));
  else
    sel::compact_kernel<64><<<grid, 256, 0, stream>>>(indices, static_cast<const uint16_t*>(k),
                                                       static_cast<const uint16_t*>(v), kv_row_stride, L_A, lp, hk,
                                                       static_cast<uint16_t*>(send));
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("compact launch: ") + cudaGetErrorString(e));
  count_launch(2);
  return APB_OK;
}

// ---------------------------------------------------------------- method variants (NEXT #3)
namespace sel {

// "Rd." compressor (Table 4): a uniform score in [0,1) per
// (layer, host, KV head, block token) from the counter-based generator of DESIGN.md reading
// G17 — the (c+1)-th output of a SplitMix64 stream seeded with `seed`, top 24 bits.
__global__ void __launch_bounds__(256) random_scores_kernel(uint64_t seed, uint64_t c0, int64_t count,
                                                            float* __restrict__ scores) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < count; i += (int64_t)gridDim.x * 256) {
    uint64_t z = seed + (c0 + (uint64_t)i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    scores[i] = (float)(z >> 40) * 0x1p-24f;  // exact: a 24-bit integer times 2^-24
  }
}

// Shared index set (reading G3's alternative): every KV head's row of
// scores becomes the max over the KV heads, so the per-head select yields one common set.
__global__ void __launch_bounds__(256) share_scores_kernel(float* __restrict__ scores, int hk, int l_b) {
  for (int t = blockIdx.x * 256 + threadIdx.x; t < l_b; t += gridDim.x * 256) {
    float m = scores[t];
    for (int j = 1; j < hk; ++j) m = fmaxf(m, scores[(int64_t)j * l_b + t]);
    for (int j = 0; j < hk; ++j) scores[(int64_t)j * l_b + t] = m;
  }
}

}  // namespace sel

apb_status launch_random_scores(uint64_t seed, uint64_t c0, int64_t count, float* scores, cudaStream_t stream) {
  const int64_t blocks = (count + 255) / 256;
  sel::random_scores_kernel<<<(int)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, stream>>>(seed, c0, count, scores);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("random_scores launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_share_scores(float* scores, int hk, int l_b, cudaStream_t stream) {
  const int blocks = (l_b + 255) / 256;
  sel::share_scores_kernel<<<blocks < 148 * 4 ? blocks : 148 * 4, 256, 0, stream>>>(scores, hk, l_b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("share_scores launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace apb
