// attention_sm100.cu — APB masked attention (eq:apb, Alg. apb_prefill line
// "attn") as a warp-specialised tcgen05 kernel for sm_100a.
//
// Key sequence of host h: [anchor K_a | passing K_p | local K_h].  Mask M'
// (reading G1): anchor query rows are causal over the anchor; local query row i sees
// every anchor key, every passing key and local keys 0..i.  The kernel never builds M': each
// 128x128 (query x key) tile is classified from (segment, tile index, row) and tiles that are
// fully masked are never visited.
//
// CTA = one "work item": two 128-row query tiles of the same KV head (two GQA query heads, same
// rows) sharing every K/V tile load.  Warp roles (320 threads):
//   warps 0-3  softmax warpgroup for Q tile 0 (thread i owns query row i = TMEM lane i)
//   warps 4-7  softmax warpgroup for Q tile 1
//   warp  8    TMA producer (Q once, then a 2-stage K ring and a 2-stage V ring)
//   warp  9    tcgen05.mma issuer (one thread)
// TMEM (512 columns): S_0 [0,128)  S_1 [128,256)  O_0 [256,256+D)  O_1 [256+D, 256+2D).
// P_t (bf16) is written over the first 64 columns of S_t and consumed from TMEM as the A
// operand of O_t += P_t V (FlashAttention-4 style); S_t(j+1) is issued after PV_t(j), so the
// in-order tensor pipe never overwrites P_t(j) before it is read.
// Online softmax in the log2 domain with conditional rescaling: O_t is rescaled only when a
// row max grows by more than 8 (2^8 headroom in fp32), which after the first few tiles is rare.
#include "internal.h"
#include "sm100.cuh"

namespace apb {
namespace attn {

using namespace apb::sm100;

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KS = 2;  // K and V ring stages
constexpr int kThreads = 320;
constexpr int kLoadWarp = 8;
constexpr int kMmaWarp = 9;
constexpr float kRescaleThreshold = 8.0f;

template <int D>
struct Layout {
  static constexpr int kHalves = D / 64;           // 64-element (128 B) swizzle atoms per row
  static constexpr int kSub = BM * 128;            // bytes of one 128-row x 64-col sub-tile
  static constexpr int kTile = kHalves * kSub;     // bytes of a 128 x D bf16 tile
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + 2 * kTile;
  static constexpr int kV = kK + KS * kTile;
  static constexpr int kBar = kV + KS * kTile;
  // barriers: Qfull, Kfull[KS], Kempty[KS], Vfull[KS], Vempty[KS], Sfull[2], Pfull[2], Odone[2]
  static constexpr int kNumBars = 1 + 4 * KS + 6;
  static constexpr int kTmemPtr = kBar + kNumBars * 8;
  static constexpr int kUsed = kTmemPtr + 16;
  // keep one CTA per SM (each CTA allocates all 512 TMEM columns)
  static constexpr int kAlloc = (kUsed + 1024) > 120 * 1024 ? (kUsed + 1024) : 120 * 1024;
};

struct Item {
  int seg;  // 0 = anchor query rows, 1 = local query rows
  int rt;   // 128-row tile index inside the segment
  int j;    // KV head
  int qh0;  // first query head
  int ntiles;
  int nkv;
};

__device__ __forceinline__ Item decode_item(const AttnParams& p, int w) {
  Item it;
  const int per_rt = p.hk * p.np;
  if (w < p.n_local_items) {
    it.seg = 1;
    it.rt = p.nB_rt - 1 - w / per_rt;  // heaviest (largest causal extent) first
  } else {
    w -= p.n_local_items;
    it.seg = 0;
    it.rt = p.nA_rt - 1 - w / per_rt;
  }
  w %= per_rt;
  it.j = w / p.np;
  const int pi = w % p.np;
  it.qh0 = it.j * p.g + 2 * pi;
  it.ntiles = (2 * pi + 1 < p.g) ? 2 : 1;
  if (it.seg == 0) {
    it.nkv = it.rt + 1;
  } else {
    it.nkv = (p.phase != APB_PHASE_PASSING ? p.nA_kv + it.rt + 1 : 0) +
             (p.phase != APB_PHASE_LOCAL ? p.n_slots * p.nP_kv : 0);
  }
  return it;
}

struct KvTile {
  int kind;  // 0 = anchor keys, 1 = passing keys, 2 = local keys
  int c;     // 128-key tile index inside its segment (or slot)
  int slot;  // passing slot (host index of the sender)
};

__device__ __forceinline__ KvTile kv_tile(const AttnParams& p, const Item& it, int i) {
  if (it.seg == 0) return {0, i, 0};
  if (p.phase != APB_PHASE_PASSING) {
    if (i < p.nA_kv) return {0, i, 0};
    i -= p.nA_kv;
  }
  if (p.phase != APB_PHASE_LOCAL) {
    const int npass = p.n_slots * p.nP_kv;
    if (i < npass) return {1, i % p.nP_kv, i / p.nP_kv};
    i -= npass;
  }
  return {2, i, 0};
}

// Number of leading visible columns of a key tile for one query row (mask M', reading G1).
__device__ __forceinline__ int visible_cols(const AttnParams& p, const Item& it, const KvTile& kt, int row) {
  int ub;
  if (kt.kind == 0) {
    ub = (it.seg == 0) ? min(p.L_A, row + 1) : p.L_A;  // anchor rows: causal; local rows: all anchor keys
  } else if (kt.kind == 1) {
    ub = p.lp;                                          // passing keys: all visible to local rows
  } else {
    ub = row + 1;                                       // local keys: causal
  }
  ub -= kt.c * BN;
  return ub < 0 ? 0 : (ub > BN ? BN : ub);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    apb_attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_g,
                         const AttnParams p) {
  using L = Layout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase + L::kQ, sK = sbase + L::kK, sV = sbase + L::kV;
  const uint32_t bar0 = sbase + L::kBar;
  const uint32_t bQ = bar0;
  auto bKf = [&](int s) { return bar0 + 8u * (1 + s); };
  auto bKe = [&](int s) { return bar0 + 8u * (1 + KS + s); };
  auto bVf = [&](int s) { return bar0 + 8u * (1 + 2 * KS + s); };
  auto bVe = [&](int s) { return bar0 + 8u * (1 + 3 * KS + s); };
  auto bS = [&](int t) { return bar0 + 8u * (1 + 4 * KS + t); };
  auto bP = [&](int t) { return bar0 + 8u * (3 + 4 * KS + t); };
  auto bO = [&](int t) { return bar0 + 8u * (5 + 4 * KS + t); };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtr);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const Item it = decode_item(p, blockIdx.x);

  if (threadIdx.x == 0) {
    mbar_init(bQ, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(bKf(s), 1);
      mbar_init(bKe(s), 1);
      mbar_init(bVf(s), 1);
      mbar_init(bVe(s), 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(bS(t), 1);
      mbar_init(bP(t), BM);
      mbar_init(bO(t), 1);
    }
    fence_mbar_init();
  }
  if (warp == kLoadWarp) {
    tmem_alloc<512>(smem_u32(tmem_ptr));
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_g);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == kLoadWarp) {
    // ================================================================ TMA producer
    if (lane == 0) {
      const int qrow0 = (it.seg == 0 ? 0 : p.L_A) + it.rt * BM;
      mbar_arrive_expect_tx(bQ, it.ntiles * L::kTile);
      for (int t = 0; t < it.ntiles; ++t)
        for (int h = 0; h < L::kHalves; ++h)
          tma_load_3d(sQ + t * L::kTile + h * L::kSub, &tm_q, bQ, h * 64, it.qh0 + t, qrow0);
      for (int i = 0; i < it.nkv; ++i) {
        const int s = i % KS;
        const uint32_t ph = (i / KS) & 1;
        const KvTile kt = kv_tile(p, it, i);
        const int row0 = (kt.kind == 2 ? p.L_A : 0) + kt.c * BN;
        mbar_wait(bKe(s), ph ^ 1);
        mbar_arrive_expect_tx(bKf(s), L::kTile);
        for (int h = 0; h < L::kHalves; ++h) {
          if (kt.kind == 1)
            tma_load_4d(sK + s * L::kTile + h * L::kSub, &tm_g, bKf(s), h * 64, kt.c * BN, it.j, kt.slot * 2 + 0);
          else
            tma_load_3d(sK + s * L::kTile + h * L::kSub, &tm_k, bKf(s), h * 64, it.j, row0);
        }
        mbar_wait(bVe(s), ph ^ 1);
        mbar_arrive_expect_tx(bVf(s), L::kTile);
        for (int h = 0; h < L::kHalves; ++h) {
          if (kt.kind == 1)
            tma_load_4d(sV + s * L::kTile + h * L::kSub, &tm_g, bVf(s), h * 64, kt.c * BN, it.j, kt.slot * 2 + 1);
          else
            tma_load_3d(sV + s * L::kTile + h * L::kSub, &tm_v, bVf(s), h * 64, it.j, row0);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(BM, BN, false, false);  // S = Q K^T: both K-major
      constexpr uint32_t idPV = idesc_bf16_f32(BM, D, false, true);   // O += P V: V is MN-major
      auto issue_S = [&](int t, int s) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k / 4) * L::kSub + (k % 4) * 32;
          mma_ss(tmem + t * 128, sdesc_sw128(sQ + t * L::kTile + off, 16, 1024),
                 sdesc_sw128(sK + s * L::kTile + off, 16, 1024), idS, k > 0);
        }
      };
      auto issue_PV = [&](int t, int s, bool acc) {
#pragma unroll
        for (int k = 0; k < BN / 16; ++k) {
          mma_ts(tmem + 256 + t * D, tmem + t * 128 + k * 8, sdesc_sw128(sV + s * L::kTile + k * 2048, L::kSub, 1024),
                 idPV, (acc || k > 0) ? 1u : 0u);
        }
      };
      const bool carry = (p.phase == APB_PHASE_PASSING);
      mbar_wait(bQ, 0);
      tc_fence_after();
      for (int i = 0; i < it.nkv; ++i) {
        const int s = i % KS;
        const uint32_t ph = (i / KS) & 1;
        if (i == 0) {
          mbar_wait(bKf(s), ph);
          tc_fence_after();
          for (int t = 0; t < it.ntiles; ++t) {
            issue_S(t, s);
            mma_commit(bS(t));
          }
          mma_commit(bKe(s));
        }
        mbar_wait(bVf(s), ph);
        tc_fence_after();
        const int s1 = (i + 1) % KS;
        const uint32_t ph1 = ((i + 1) / KS) & 1;
        for (int t = 0; t < it.ntiles; ++t) {
          mbar_wait(bP(t), i & 1);
          tc_fence_after();
          issue_PV(t, s, carry || i > 0);
          if (t == it.ntiles - 1) mma_commit(bVe(s));
          if (i + 1 < it.nkv) {
            if (t == 0) {
              mbar_wait(bKf(s1), ph1);
              tc_fence_after();
            }
            issue_S(t, s1);
            mma_commit(bS(t));
            if (t == it.ntiles - 1) mma_commit(bKe(s1));
          } else {
            mma_commit(bO(t));
          }
        }
      }
    }
  } else {
    // ================================================================ softmax warpgroups
    const int t = warp / 4;
    if (t < it.ntiles) {
      const int tid = threadIdx.x % 128;
      const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const uint32_t tS = tmem + lane_base + t * 128;
      const uint32_t tO = tmem + lane_base + 256 + t * D;
      const int qh = it.qh0 + t;
      const int row = it.rt * BM + tid;  // row index inside the query segment
      const bool row_valid = it.seg == 0 ? row < p.L_A : row < p.l_b;
      const float sl2 = p.scale_log2;
      float m_run = -INFINITY, l_run = 0.f;
      bool o_valid = false;

      if (p.phase == APB_PHASE_PASSING) {
        // LSE carry-in: the LOCAL phase's normalised partial (O, m + log2 l) becomes the
        // initial online-softmax state (m = lse2, l = 1, O = O_partial) — an exact merge.
        const float* src = p.ws_o + ((int64_t)(row_valid ? row : 0) * p.hq + qh) * D;
        m_run = row_valid ? p.ws_lse[(int64_t)qh * p.l_b + row] : 0.f;
        l_run = 1.f;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            float4 f = row_valid ? *reinterpret_cast<const float4*>(src + c * 32 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
            r[e] = __float_as_uint(f.x);
            r[e + 1] = __float_as_uint(f.y);
            r[e + 2] = __float_as_uint(f.z);
            r[e + 3] = __float_as_uint(f.w);
          }
          tmem_st32(tO + c * 32, r);
        }
        tmem_wait_st();
        o_valid = true;
      }

      for (int i = 0; i < it.nkv; ++i) {
        const KvTile kt = kv_tile(p, it, i);
        const int nv = visible_cols(p, it, kt, row);
        mbar_wait(bS(t), i & 1);
        tc_fence_after();
        uint32_t sr[128];
        tmem_ld32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
        tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
        tmem_wait_ld();
        float* s = reinterpret_cast<float*>(sr);
        if (nv < BN) {
#pragma unroll
          for (int c = 0; c < BN; ++c)
            if (c >= nv) s[c] = -INFINITY;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < BN; ++c) mx = fmaxf(mx, s[c]);
        mx *= sl2;
        const float m_new = fmaxf(m_run, mx);
        const bool grow = (m_new > m_run + kRescaleThreshold) || (m_run == -INFINITY);
        float alpha = 1.f;
        if (grow) {
          alpha = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_new);
          m_run = m_new;
        }
        const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
        float rowsum = 0.f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float p0 = ex2(fmaf(s[half * 64 + 2 * c], sl2, -m_use));
            const float p1 = ex2(fmaf(s[half * 64 + 2 * c + 1], sl2, -m_use));
            rowsum += p0 + p1;
            pk[c] = pack_bf16x2(p0, p1);
          }
          tmem_st32(tS + half * 32, pk);
        }
        l_run = l_run * alpha + rowsum;
        // rescale the running O_t (PV_t(i-1) is complete: S_t(i) was issued after it)
        if (__any_sync(0xffffffffu, grow && o_valid && alpha != 1.f)) {
          const float a = o_valid ? alpha : 1.f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * a);
            tmem_st32(tO + c * 32, r);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bP(t));
        o_valid = true;
      }

      // ============================================================== epilogue
      mbar_wait(bO(t), 0);
      tc_fence_after();
      const float inv_l = 1.f / l_run;
      const bool to_ws = (it.seg == 1) && p.local_to_ws;
      const int64_t grow_idx = (it.seg == 0 ? 0 : p.L_A) + row;  // row of q/out on this host
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tO + c * 32, r);
        tmem_wait_ld();
        if (row_valid) {
          if (to_ws) {
            float* dst = p.ws_o + ((int64_t)row * p.hq + qh) * D + c * 32;
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(dst + e) =
                  make_float4(__uint_as_float(r[e]) * inv_l, __uint_as_float(r[e + 1]) * inv_l,
                              __uint_as_float(r[e + 2]) * inv_l, __uint_as_float(r[e + 3]) * inv_l);
          } else {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + grow_idx * p.out_row_stride + (int64_t)qh * D + c * 32;
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint4 v;
              v.x = pack_bf16x2(__uint_as_float(r[e]) * inv_l, __uint_as_float(r[e + 1]) * inv_l);
              v.y = pack_bf16x2(__uint_as_float(r[e + 2]) * inv_l, __uint_as_float(r[e + 3]) * inv_l);
              v.z = pack_bf16x2(__uint_as_float(r[e + 4]) * inv_l, __uint_as_float(r[e + 5]) * inv_l);
              v.w = pack_bf16x2(__uint_as_float(r[e + 6]) * inv_l, __uint_as_float(r[e + 7]) * inv_l);
              *reinterpret_cast<uint4*>(dst + e) = v;
            }
          }
        }
      }
      if (row_valid) {
        const float lse2 = m_run + __log2f(l_run);
        if (to_ws) {
          p.ws_lse[(int64_t)qh * p.l_b + row] = lse2;
        } else if (p.lse) {
          p.lse[(int64_t)qh * p.lse_ld + grow_idx] = lse2 * 0.69314718055994530942f;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kLoadWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D>
static apb_status launch_impl(const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                              const CUtensorMap& tg, cudaStream_t stream) {
  using L = Layout<D>;
  const int grid = p.n_local_items + p.n_anchor_items;
  if (grid == 0) return APB_OK;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(apb_attention_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc);
    if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    attr_set = true;
  }
  apb_attention_kernel<D><<<grid, kThreads, L::kAlloc, stream>>>(tq, tk, tv, tg, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace attn

apb_status launch_attention(int D, const AttnParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                            const CUtensorMap& tv, const CUtensorMap& tg, cudaStream_t stream) {
  if (D == 128) return attn::launch_impl<128>(p, tq, tk, tv, tg, stream);
  if (D == 64) return attn::launch_impl<64>(p, tq, tk, tv, tg, stream);
  return fail(APB_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
}

}  // namespace apb
