// decode.cu — APB's distributed exact decode step (Alg. apb_decode; SURVEY
// NEXT #1): on host h the t new tokens' queries attend to the host's block KV cache;
// the last host also attends to the new tokens' own keys, causally among them.  The
// partial (A_h, lse_h) of every host is gathered and merged by log-sum-exp (MergeScore,
// P:753), which makes the result exact.
//
// decode_mma_kernel: memory-bound split-KV ("flash decoding") — grid (splits, KV heads), ~2
// CTAs per SM, each streaming a contiguous range of 64-key chunks through a cp.async ring, both
// products on the tensor cores, online softmax across its chunks.  Output: one normalised
// partial (O, log2-sum-exp) per split in the workspace.
// merge_kernel: log-sum-exp merge of n partials per row — used both to fold the chunks of one
// host and, across hosts, as MergeScore.  Fixed merge order, no atomics: deterministic.
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace apb {
namespace dec {

using namespace apb::sm100;


__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem_src), "r"(valid ? 16 : 0) : "memory");
}

// Split plan: ~kSplitTarget CTAs over (splits x KV heads), whole 64-key chunks per split.
#ifndef APB_DEC_CTAS_PER_SM
#define APB_DEC_CTAS_PER_SM 3
#endif
constexpr int SKC = 64;                                  // keys per chunk
constexpr int kSplitTarget = APB_DEC_CTAS_PER_SM * 148;  // CTAs per launch to aim for (per SM x B200 SMs)
// The multi-host launch streams longer ranges per split; it runs faster over-subscribed (more
// CTAs than fit at once; per L8 step: 3 x 148 0.148 ms, 4 x 0.142, 5 x 0.132, 6 x 0.124, 8 x 0.124,
// 12 x 0.133 ms).
#ifndef APB_DEC_HOSTS_CTAS_PER_SM
#define APB_DEC_HOSTS_CTAS_PER_SM 9
#endif
constexpr int kHostsSplitTarget = APB_DEC_HOSTS_CTAS_PER_SM * 148;

// ---------------------------------------------------------------- tensor-core split-KV
// decode_mma_kernel: the same streaming split-KV plan, with both products on the tensor cores
// (mma.sync m16n8k16 bf16 -> fp32; R = t*g query rows padded to 16-row m-tiles — for this
// HBM-bound GEMV the point is to take the bf16 unpacking and the FMAs off the CUDA cores, not
// tensor throughput, so the legacy warp-level MMA is the right size).  Per 64-key chunk:
//   S = Q K^T: warp w owns keys [8w, 8w+8) (one n-tile), K fragments via ldmatrix from the
//              padded K rows; masks; row max over the chunk through shared memory;
//   P = 2^(S - m), written as bf16 to shared memory; row sums kept per thread;
//   O = alpha O + P V: warp w owns head_dim columns [D/8 w, D/8 (w+1)), V fragments via
//              ldmatrix.trans; O stays in registers for the whole split.
constexpr int MKC = SKC;        // keys per chunk
constexpr int kMThreads = 256;  // 8 warps
#ifndef APB_DEC_STAGES
#define APB_DEC_STAGES 2
#endif
constexpr int kMStages = APB_DEC_STAGES;

template <int D>
struct MmaSmem {
  static constexpr int kRow = D + 8;                  // padded bf16 row (Q, conflict-free ldmatrix)
  static constexpr int kKV = D * 2;                   // K / V chunk row: dense, 16-byte chunks XOR-swizzled
  static constexpr int kStage = 2 * MKC * kKV;        // K and V chunk
  static constexpr int kPRow = MKC + 8;
  __host__ __device__ static constexpr int bytes(int MT, int stages = kMStages) {
    return stages * kStage + 16 * MT * kRow * 2 + 16 * MT * kPRow * 2 + 2 * 8 * 16 * MT * 4;
  }
};
// TMA-fed variant: the K / V chunks arrive by cp.async.bulk.tensor (one elected thread issues two
// 64-column SW128 boxes per tensor per chunk) into a 3-stage ring with one mbarrier per stage;
// the tensor maps of every host of the launch sit in the parameter space.
#ifndef APB_DEC_TSTAGES
#define APB_DEC_TSTAGES 2
#endif
constexpr int kTStages = APB_DEC_TSTAGES;
struct DecMaps {
  CUtensorMap k[kDecMaxHosts], v[kDecMaxHosts];
};
template <int D>
__host__ __device__ constexpr int tma_bytes(int MT) {  // + the stage barriers + slack to align the ring at 1 KB
  return MmaSmem<D>::bytes(MT, kTStages) + 8 * kTStages + 1024;
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte offset of 16-byte chunk c of row r in a dense K / V chunk: chunk index XOR (r & 7), so the
// 8 rows an ldmatrix 8x8 reads hit 8 different bank groups
template <int D>
__device__ __forceinline__ uint32_t kv_off(int r, int c) {
  return static_cast<uint32_t>(r * (D * 2) + ((c ^ (r & 7)) << 4));
}
// the TMA (SW128) layout of a chunk: 64-column halves of [64 keys][128 B], 16-byte chunk index
// XOR (r & 7) inside each 128-byte row (the same bank spread for ldmatrix)
template <int D, bool TMA>
__device__ __forceinline__ uint32_t kv_addr(int r, int c) {
  if constexpr (TMA)
    return static_cast<uint32_t>((c >> 3) * (SKC * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
  else
    return kv_off<D>(r, c);
}

template <int D, int MT, bool TMA>
__global__ void __launch_bounds__(kMThreads) decode_mma_kernel(const DecodeParams p, const DecodeHosts hb,
                                                                 int chunks_per_split,
                                                                 const __grid_constant__ DecMaps maps) {
  using L = MmaSmem<D>;
  constexpr int kS = TMA ? kTStages : kMStages;  // ring stages
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // the TMA ring is 1 KB aligned (SW128 boxes); the cp.async ring needs 16 B
  uint8_t* smem = TMA ? smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u)
                      : smem_raw;
  constexpr int NT = D / 64;  // O n-tiles (of 8 columns) per warp: D/8 tiles over 8 warps
  // programmatic dependent launch: the merge / fold that follows may be scheduled as soon as every
  // CTA of this grid has started (it waits in griddepcontrol.wait for this grid's completion and
  // memory flush), so its launch latency and ramp overlap this grid's tail
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int R = p.t * p.g;
  __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(smem + kS * L::kStage);  // [16 MT][kRow]
  __nv_bfloat16* pss = qs + 16 * MT * L::kRow;                                       // [16 MT][kPRow]
  float* xm = reinterpret_cast<float*>(pss + 16 * MT * L::kPRow);                    // [8][16 MT]
  float* xl = xm + 8 * 16 * MT;                                                      // [8][16 MT]
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g8 = lane / 4, t4 = lane % 4;
  const int split = blockIdx.x, j = blockIdx.y;  // split: index into the workspace partials
  // multi-host launch: this split's host (its cache, length, whether it sees the new tokens)
  int split_local = split;
  const __nv_bfloat16* k_cache = p.k_cache;
  const __nv_bfloat16* v_cache = p.v_cache;
  int64_t cache_len = p.cache_len;
  int has_new = p.has_new;
  int hi = 0;  // this split's host within the launch (its tensor maps)
  if (hb.n > 0) {
    int i = 0;
    while (i + 1 < hb.n && split >= hb.split_begin[i + 1]) ++i;
    hi = i;
    split_local = split - hb.split_begin[i];
    k_cache = hb.k_cache[i];
    v_cache = hb.v_cache[i];
    cache_len = hb.cache_len[i];
    has_new = (i == hb.new_host) ? 1 : 0;
  }
  const int64_t n_keys = cache_len + (has_new ? p.t : 0);
  const int64_t c_first = (int64_t)split_local * chunks_per_split;
  const int64_t n_chunks_total = (n_keys + MKC - 1) / MKC;
  const int nch = (int)((c_first + chunks_per_split <= n_chunks_total) ? chunks_per_split
                                                                       : (n_chunks_total > c_first ? n_chunks_total - c_first : 0));
  constexpr int kVec = D / 8;
  auto stage_k = [&](int s) { return smem + s * L::kStage; };
  auto stage_v = [&](int s) { return smem + s * L::kStage + MKC * L::kKV; };
  // TMA: one barrier per stage after the Q / P / x scratch
  const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem + L::bytes(MT, kS)));
  if constexpr (TMA) {
    if (tid == 0) {
      for (int st = 0; st < kS; ++st) mbar_init(bar0 + 8u * st, 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  auto load_chunk = [&](int c, int s) {
    const int64_t k0 = (c_first + c) * MKC;
    uint8_t* ks = stage_k(s);
    uint8_t* vs = stage_v(s);
    if constexpr (TMA) {
      // the slot's previous chunk was read before the last __syncthreads; order those generic
      // reads before the async-proxy writes, then two SW128 boxes per tensor (rows past the
      // cache are zero-filled; the new tokens' rows are patched in after the wait)
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t fb = bar0 + 8u * s;
        mbar_arrive_expect_tx(fb, 2 * MKC * D * 2);
        const uint32_t ku = static_cast<uint32_t>(__cvta_generic_to_shared(ks));
        const uint32_t vu = static_cast<uint32_t>(__cvta_generic_to_shared(vs));
#pragma unroll
        for (int h = 0; h < D / 64; ++h) {
          tma_load_3d(ku + h * (MKC * 128), &maps.k[hi], fb, h * 64, j, (int)k0);
          tma_load_3d(vu + h * (MKC * 128), &maps.v[hi], fb, h * 64, j, (int)k0);
        }
      }
    } else {
      for (int idx = tid; idx < MKC * kVec; idx += kMThreads) {
      const int kk = idx / kVec, cv = idx % kVec;
      const int64_t key = k0 + kk;
      const bool cached = key < cache_len, valid = key < n_keys;
      const __nv_bfloat16* kb = cached ? k_cache + key * p.cache_row_stride
                                       : p.k_new + (key - cache_len) * p.new_row_stride;
      const __nv_bfloat16* vb = cached ? v_cache + key * p.cache_row_stride
                                       : p.v_new + (key - cache_len) * p.new_row_stride;
      cp_async16(ks + kv_off<D>(kk, cv), valid ? kb + (int64_t)j * D + cv * 8 : p.q, valid);
      cp_async16(vs + kv_off<D>(kk, cv), valid ? vb + (int64_t)j * D + cv * 8 : p.q, valid);
      }
    }
  };
  // queries as bf16 rows (16-byte async copies; rows >= R zero-filled), in the first group
  for (int idx = tid; idx < 16 * MT * kVec; idx += kMThreads) {
    const int r = idx / kVec, cv = idx % kVec;
    const int sr = r / p.g, qh = j * p.g + r % p.g;
    cp_async16(qs + r * L::kRow + cv * 8, r < R ? p.q + ((int64_t)sr * p.hq + qh) * D + cv * 8 : p.q, r < R);
  }
#pragma unroll
  for (int s = 0; s < kS - 1; ++s) {
    if (s < nch) load_chunk(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // per-thread running state for rows (mt, g8) and (mt, g8 + 8)
  float m_run[MT][2], l_run[MT][2];
  float o[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    m_run[mt][0] = m_run[mt][1] = -INFINITY;
    l_run[mt][0] = l_run[mt][1] = 0.f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[mt][nt][0] = o[mt][nt][1] = o[mt][nt][2] = o[mt][nt][3] = 0.f;
  }
  const uint32_t qs_u = static_cast<uint32_t>(__cvta_generic_to_shared(qs));
  const uint32_t ps_u = static_cast<uint32_t>(__cvta_generic_to_shared(pss));
  const float sl2 = p.scale_log2;

  for (int c = 0; c < nch; ++c) {
    const int s = c % kS;
    if (c + kS - 1 < nch) load_chunk(c + kS - 1, (c + kS - 1) % kS);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int64_t k0 = (c_first + c) * MKC;
    if constexpr (TMA) {
      asm volatile("cp.async.wait_group %0;" ::"n"(kS - 1) : "memory");  // the queries (first group)
      mbar_wait(bar0 + 8u * s, (c / kS) & 1);
      if (has_new && k0 + MKC > cache_len) {
        // the new tokens' own keys (last host) into their rows of the chunk
        for (int idx = tid; idx < MKC * kVec; idx += kMThreads) {
          const int kk = idx / kVec, cv = idx % kVec;
          const int64_t key = k0 + kk;
          if (key >= cache_len && key < n_keys) {
            const int64_t nr = (key - cache_len) * p.new_row_stride + (int64_t)j * D + cv * 8;
            *reinterpret_cast<uint4*>(stage_k(s) + kv_addr<D, true>(kk, cv)) = *reinterpret_cast<const uint4*>(p.k_new + nr);
            *reinterpret_cast<uint4*>(stage_v(s) + kv_addr<D, true>(kk, cv)) = *reinterpret_cast<const uint4*>(p.v_new + nr);
          }
        }
      }
    } else {
      asm volatile("cp.async.wait_group %0;" ::"n"(kS - 1) : "memory");
    }
    __syncthreads();
    const uint32_t ks_u = static_cast<uint32_t>(__cvta_generic_to_shared(stage_k(s)));
    const uint32_t vs_u = static_cast<uint32_t>(__cvta_generic_to_shared(stage_v(s)));
    // ---- S = Q K^T for this warp's 8 keys
    float sc[MT][4], sc2[MT][4];  // two accumulator chains (even / odd k-steps)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[mt][e] = sc2[mt][e] = 0.f;
#pragma unroll
    for (int kb = 0; kb < D / 32; ++kb) {  // two k-steps of 16 per ldmatrix.x4 of K
      uint32_t b[4];
      ldsm_x4(ks_u + kv_addr<D, TMA>(warp * 8 + (lane % 8), kb * 4 + lane / 8), b[0], b[1], b[2], b[3]);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t a[4], a2[4];
        ldsm_x4(qs_u + ((mt * 16 + (lane % 16)) * L::kRow + kb * 32 + (lane / 16) * 8) * 2, a[0], a[1], a[2], a[3]);
        ldsm_x4(qs_u + ((mt * 16 + (lane % 16)) * L::kRow + kb * 32 + 16 + (lane / 16) * 8) * 2, a2[0], a2[1], a2[2],
                a2[3]);
        mma_bf16_16816(sc[mt], a, b[0], b[1]);
        mma_bf16_16816(sc2[mt], a2, b[2], b[3]);
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[mt][e] += sc2[mt][e];
    // ---- mask, scale to the log2 domain, chunk row max (quad, then across the 8 warps)
    const int key_a = warp * 8 + 2 * t4;  // this thread's two keys inside the chunk
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = mt * 16 + g8 + (e >> 1) * 8;
        const int64_t key = k0 + key_a + (e & 1);
        const bool vis = r < R && key < n_keys && (key < cache_len || key - cache_len <= r / p.g);
        sc[mt][e] = vis ? sc[mt][e] * sl2 : -INFINITY;
      }
      float m0 = fmaxf(sc[mt][0], sc[mt][1]), m1 = fmaxf(sc[mt][2], sc[mt][3]);
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
      if (t4 == 0) {
        xm[warp * 16 * MT + mt * 16 + g8] = m0;
        xm[warp * 16 * MT + mt * 16 + g8 + 8] = m1;
      }
    }
    __syncthreads();
    // ---- P = 2^(S - m_new) (bf16 to shared memory), running state, O rescale
    float alpha[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int r = mt * 16 + g8 + hr * 8;
        float mc = xm[r];
#pragma unroll
        for (int w = 1; w < 8; ++w) mc = fmaxf(mc, xm[w * 16 * MT + r]);
        const float m_new = fmaxf(m_run[mt][hr], mc);
        const float mu = (m_new == -INFINITY) ? 0.f : m_new;
        alpha[mt][hr] = (m_run[mt][hr] == -INFINITY) ? 0.f : ex2(m_run[mt][hr] - mu);
        m_run[mt][hr] = m_new;
        const float p0 = ex2(sc[mt][2 * hr] - mu), p1 = ex2(sc[mt][2 * hr + 1] - mu);
        l_run[mt][hr] = l_run[mt][hr] * alpha[mt][hr] + (p0 + p1);
        *reinterpret_cast<uint32_t*>(pss + r * L::kPRow + key_a) = pack_bf16x2(p0, p1);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        o[mt][nt][0] *= alpha[mt][0];
        o[mt][nt][1] *= alpha[mt][0];
        o[mt][nt][2] *= alpha[mt][1];
        o[mt][nt][3] *= alpha[mt][1];
      }
    }
    __syncthreads();
    // ---- O += P V for this warp's D/8 columns
#pragma unroll
    for (int ks2 = 0; ks2 < MKC / 16; ++ks2) {
#pragma unroll
      for (int np = 0; np < NT; np += 2) {  // pairs of n-tiles per ldmatrix.x4.trans
        uint32_t b[4];
        const int col = warp * (D / 8) + np * 8 + (lane / 16) * 8;
        ldsm_x4_t(vs_u + kv_addr<D, TMA>(ks2 * 16 + (lane % 16), col / 8), b[0], b[1], b[2], b[3]);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t a[4];
          ldsm_x4(ps_u + ((mt * 16 + (lane % 16)) * L::kPRow + ks2 * 16 + (lane / 16) * 8) * 2, a[0], a[1], a[2], a[3]);
          mma_bf16_16816(o[mt][np], a, b[0], b[1]);
          if (np + 1 < NT) mma_bf16_16816(o[mt][np + 1], a, b[2], b[3]);
        }
      }
    }
    __syncthreads();  // stage s, xm and P are rewritten next chunk
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  // ---- row sums: quad, then across warps; normalised partial out
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float l = l_run[mt][hr];
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      if (t4 == 0) xl[warp * 16 * MT + mt * 16 + g8 + hr * 8] = l;
    }
  }
  __syncthreads();
  const int rows_total = p.t * p.hq;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int r = mt * 16 + g8 + hr * 8;
      if (r >= R) continue;
      float l = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) l += xl[w * 16 * MT + r];
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const int sr = r / p.g, qh = j * p.g + r % p.g;
      const int64_t row = (int64_t)sr * p.hq + qh;
      float* dst = p.ws_o + ((int64_t)split * rows_total + row) * D + warp * (D / 8) + 2 * t4;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<float2*>(dst + nt * 8) = make_float2(o[mt][nt][2 * hr] * inv, o[mt][nt][2 * hr + 1] * inv);
      if (warp == 0 && t4 == 0)
        p.ws_lse[(int64_t)split * rows_total + row] = l > 0.f ? m_run[mt][hr] + __log2f(l) : -INFINITY;
    }
  }
  // ---- the last CTA of this KV head folds its splits (LSE merge, fixed split order) into the
  // host's partial: no second launch, the split partials are read back from L2
}

// LSE merge of n partials per row (MergeScore).  lse_in_log2 selects the input log base;
// the output lse is natural.  One CTA (8 warps) per (row, block of 32 columns) — a CTA handles
// column blocks [cb0, cb0 + NCB): the weights of all parts are formed in shared memory (parallel
// max / sum, recomputed by each column block); warp w accumulates parts w, w+8, ... (lanes across
// the columns, 8 parts' loads in flight), and the 8 warp partials are added in a fixed order —
// deterministic, and the same bits whichever column split runs it.
constexpr int kMergeWarps = 8;
template <int D, typename OutT, int NCB>
__device__ __forceinline__ void merge_row(int64_t row, int cb0, int n, const float* __restrict__ parts_o,
                                          const float* __restrict__ parts_lse, int64_t stride_o, int64_t stride_lse,
                                          int lse_in_log2, OutT* __restrict__ out, float* __restrict__ out_lse) {
  extern __shared__ float wsm[];  // [n] weights
  __shared__ float red[kMergeWarps];
  __shared__ float part[kMergeWarps][NCB * 32];
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
  float acc[NCB];
#pragma unroll
  for (int e = 0; e < NCB; ++e) acc[e] = 0.f;
  const int col0 = cb0 * 32 + lane;
  int h = warp;
  // eight parts' loads in flight per warp, accumulated in the same (part-ascending) order
  constexpr int kU = NCB >= 4 ? 4 : 8;
  for (; h + (kU - 1) * kMergeWarps < n; h += kU * kMergeWarps) {
    float v[kU][NCB];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const float* src = parts_o + (h + u * kMergeWarps) * stride_o + row * D + col0;
#pragma unroll
      for (int e = 0; e < NCB; ++e) v[u][e] = __ldg(src + e * 32);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const float w = wsm[h + u * kMergeWarps];
#pragma unroll
      for (int e = 0; e < NCB; ++e) acc[e] = fmaf(w, v[u][e], acc[e]);
    }
  }
  for (; h < n; h += kMergeWarps) {
    const float w = wsm[h];
    const float* src = parts_o + h * stride_o + row * D + col0;
#pragma unroll
    for (int e = 0; e < NCB; ++e) acc[e] = fmaf(w, __ldg(src + e * 32), acc[e]);
  }
#pragma unroll
  for (int e = 0; e < NCB; ++e) part[warp][e * 32 + lane] = acc[e];
  __syncthreads();
  for (int e = tid; e < NCB * 32; e += kMergeWarps * 32) {
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < kMergeWarps; ++w) sum += part[w][e];
    const float o = z > 0.f ? sum / z : 0.f;
    if constexpr (sizeof(OutT) == 2)
      out[row * D + cb0 * 32 + e] = __float2bfloat16_rn(o);
    else
      out[row * D + cb0 * 32 + e] = o;
  }
  if (tid == 0 && cb0 == 0 && out_lse)
    out_lse[row] = (z > 0.f) ? (m + __log2f(z)) * 0.69314718055994530942f : -INFINITY;
}

template <int D, typename OutT>
__global__ void __launch_bounds__(kMergeWarps * 32) merge_kernel(int n, int64_t rows, const float* __restrict__ parts_o,
                                                                 const float* __restrict__ parts_lse, int64_t stride_o,
                                                                 int64_t stride_lse, int lse_in_log2,
                                                                 OutT* __restrict__ out, float* __restrict__ out_lse) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // no-op unless launched with PDL
  // grid (rows, D / 32): one column block per CTA
  merge_row<D, OutT, 1>(blockIdx.x, blockIdx.y, n, parts_o, parts_lse, stride_o, stride_lse, lse_in_log2, out, out_lse);
}

// Fold of a multi-host launch: CTA (row, host i) merges host i's splits (log2 lse in the
// workspace) into its partial at parts + i*part_stride (O) and + lse_offset (natural lse).
template <int D>
__global__ void __launch_bounds__(kMergeWarps * 32) fold_hosts_kernel(const DecodeHosts hb, int64_t rows,
                                                                      const float* __restrict__ ws_o,
                                                                      const float* __restrict__ ws_lse,
                                                                      float* __restrict__ parts, int64_t part_stride,
                                                                      int64_t lse_offset) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // no-op unless launched with PDL
  const int i = blockIdx.y, s0 = hb.split_begin[i];
  float* dst = parts + (int64_t)i * part_stride;
  merge_row<D, float, D / 32>(blockIdx.x, 0, hb.split_begin[i + 1] - s0, ws_o + (int64_t)s0 * rows * D, ws_lse + (int64_t)s0 * rows,
                      rows * D, rows, 1, dst, dst + lse_offset);
}

}  // namespace dec

// Launch configuration for a kernel that follows decode_mma_kernel on the same stream: with `pdl`
// it is a programmatic dependent launch (scheduled once every streaming CTA has issued
// griddepcontrol.launch_dependents; the kernel's griddepcontrol.wait then blocks until the
// streaming grid has completed and its writes are visible).
static cudaLaunchAttribute pdl_attr() {
  cudaLaunchAttribute a;
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  return a;
}
static cudaLaunchConfig_t pdl_config(dim3 grid, int threads, size_t smem, cudaStream_t stream, bool pdl) {
  cudaLaunchConfig_t c = {};
  c.gridDim = grid;
  c.blockDim = dim3(threads);
  c.dynamicSmemBytes = smem;
  c.stream = stream;
  c.numAttrs = pdl ? 1 : 0;
  return c;
}

// Split plan of the streaming kernel: ~kSplitTarget CTAs over (splits x KV heads), whole
// 64-key chunks per split.  Deterministic in the sizes only (no device query), so the
// workspace size is known without a GPU.
static void decode_plan(int64_t n_keys, int hk, int64_t* splits, int* chunks_per_split) {
  const int64_t n_chunks = (n_keys + dec::SKC - 1) / dec::SKC;
  int64_t target = (dec::kSplitTarget + hk - 1) / hk;
  if (target < 1) target = 1;
  if (n_chunks == 0) {
    *splits = 0;
    *chunks_per_split = 1;
    return;
  }
  const int64_t cps = (n_chunks + target - 1) / target;
  *chunks_per_split = (int)cps;
  *splits = (n_chunks + cps - 1) / cps;
}

// workspace: split partials O [splits][rows][D] | (256-byte aligned) lse [splits][rows]
static size_t ws_off_lse(int64_t splits, int64_t rows, int D) {
  return ((size_t)splits * rows * D * sizeof(float) + 255) & ~size_t(255);
}

size_t decode_workspace_bytes(int64_t n_keys, int t, int hq, int hk, int D) {
  int64_t splits;
  int cps;
  decode_plan(n_keys, hk, &splits, &cps);
  const int64_t rows = (int64_t)t * hq;
  return ws_off_lse(splits, rows, D) + (size_t)splits * rows * sizeof(float);
}

// Multi-host split plan: one chunk size (chunks per split) for all hosts, from the total chunk
// count and the launch's CTA target, so every split streams the same number of chunks.
static int64_t decode_hosts_plan(int n, const int64_t* n_keys, int hk, int* split_begin, int* chunks_per_split) {
  int64_t total_chunks = 0;
  for (int i = 0; i < n; ++i) total_chunks += (n_keys[i] + dec::SKC - 1) / dec::SKC;
  int64_t target = (dec::kHostsSplitTarget + hk - 1) / hk;
  if (target < 1) target = 1;
  const int64_t cps = total_chunks > 0 ? (total_chunks + target - 1) / target : 1;
  *chunks_per_split = (int)cps;
  int64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    split_begin[i] = (int)acc;
    acc += ((n_keys[i] + dec::SKC - 1) / dec::SKC + cps - 1) / cps;
  }
  split_begin[n] = (int)acc;
  return acc;
}

size_t decode_hosts_workspace_bytes(int n, const int64_t* n_keys, int t, int hq, int hk, int D) {
  int sb[kDecMaxHosts + 1];
  int cps;
  const int64_t splits = decode_hosts_plan(n, n_keys, hk, sb, &cps);
  const int64_t rows = (int64_t)t * hq;
  return ws_off_lse(splits, rows, D) + (size_t)splits * rows * sizeof(float);
}

// TMA maps of the caches of a launch's hosts ([cache_len][hk][D], row stride cache_row_stride;
// box 64 columns x 1 head x 64 keys, SW128).  An empty cache gets a 1-row map over q (its row is
// the first new token's, patched in the kernel; the rest of the chunk is out of bounds, zero).
static apb_status decode_maps(const DecodeParams& p, const DecodeHosts& hb, dec::DecMaps& m) {
  const int n = hb.n > 0 ? hb.n : 1;
  for (int i = 0; i < n; ++i) {
    const void* kc = hb.n > 0 ? hb.k_cache[i] : p.k_cache;
    const void* vc = hb.n > 0 ? hb.v_cache[i] : p.v_cache;
    const int64_t len = hb.n > 0 ? hb.cache_len[i] : p.cache_len;
    uint64_t str[2] = {(uint64_t)p.D * 2, (uint64_t)p.cache_row_stride * 2};
    uint64_t dims[3] = {(uint64_t)p.D, (uint64_t)p.hk, (uint64_t)len};
    if (len == 0 || !kc || !vc) {
      kc = vc = p.q;
      dims[2] = 1;
      str[1] = (uint64_t)p.hk * p.D * 2;
    }
    uint32_t box[3] = {64, 1, (uint32_t)dec::SKC};
    if (!make_tmap_bf16(&m.k[i], kc, 3, dims, str, box)) return APB_ERR_CUDA;
    if (!make_tmap_bf16(&m.v[i], vc, 3, dims, str, box)) return APB_ERR_CUDA;
  }
  return APB_OK;
}

// the streaming kernel over `splits` x KV heads (hb.n == 0: one host, all of p).  Default: the
// TMA-fed ring (APB_DEC_TMA=0 selects the cp.async ring, kept for A/B timing)
static apb_status launch_partials(const DecodeParams& p, const DecodeHosts& hb, int64_t splits, int cps,
                                  cudaStream_t stream) {
  dim3 grid((unsigned)splits, p.hk);
  const int R = p.t * p.g;
  const int mt = (R + 15) / 16;  // 16-row m-tiles
  // TMA ring for a launch over several hosts' caches (the N = 1 step: 0.1096 vs 0.1178 ms per L8
  // layer); a single host's 64 MiB launch streams faster through the cp.async ring (0.2065 vs
  // 0.229-0.235 ms for 8 per-host calls).  APB_DEC_TMA=1 / 0 forces either.
  const char* te = std::getenv("APB_DEC_TMA");
  const bool tma = (te && te[0] == '1') || (!(te && te[0] == '0') && hb.n > 0);
  dec::DecMaps maps;
  if (tma) {
    if (apb_status st = decode_maps(p, hb, maps)) return st;
  }
  apb_status st = APB_OK;
  auto launch = [&](auto kern, int MT, int D, bool T) {
    // one set-once device mask per kernel instantiation (D, MT, TMA)
    const int smem = T ? (D == 128 ? dec::tma_bytes<128>(MT) : dec::tma_bytes<64>(MT))
                       : (D == 128 ? dec::MmaSmem<128>::bytes(MT) : dec::MmaSmem<64>::bytes(MT));
    static std::atomic<uint64_t> smem_set[2][3][2];
    const int di = D == 128 ? 0 : 1, mi = MT <= 1 ? 0 : (MT <= 2 ? 1 : 2);
    st = set_max_smem_once(reinterpret_cast<const void*>(kern), smem, smem_set[di][mi][T ? 1 : 0]);
    if (st == APB_OK) kern<<<grid, dec::kMThreads, smem, stream>>>(p, hb, cps, maps);
  };
  if (p.D == 128) {
    if (mt <= 1) tma ? launch(dec::decode_mma_kernel<128, 1, true>, 1, 128, true) : launch(dec::decode_mma_kernel<128, 1, false>, 1, 128, false);
    else if (mt <= 2) tma ? launch(dec::decode_mma_kernel<128, 2, true>, 2, 128, true) : launch(dec::decode_mma_kernel<128, 2, false>, 2, 128, false);
    else tma ? launch(dec::decode_mma_kernel<128, 4, true>, 4, 128, true) : launch(dec::decode_mma_kernel<128, 4, false>, 4, 128, false);
  } else {
    if (mt <= 1) tma ? launch(dec::decode_mma_kernel<64, 1, true>, 1, 64, true) : launch(dec::decode_mma_kernel<64, 1, false>, 1, 64, false);
    else if (mt <= 2) tma ? launch(dec::decode_mma_kernel<64, 2, true>, 2, 64, true) : launch(dec::decode_mma_kernel<64, 2, false>, 2, 64, false);
    else tma ? launch(dec::decode_mma_kernel<64, 4, true>, 4, 64, true) : launch(dec::decode_mma_kernel<64, 4, false>, 4, 64, false);
  }
  if (st) return st;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_decode(const DecodeParams& p0, float* part_o, float* part_lse, cudaStream_t stream) {
  DecodeParams p = p0;
  const int64_t n_keys = p.cache_len + (p.has_new ? p.t : 0);
  int64_t splits;
  int cps;
  decode_plan(n_keys, p.hk, &splits, &cps);
  const int64_t rows = (int64_t)p.t * p.hq;
  char* base = reinterpret_cast<char*>(p.ws_o);
  p.ws_lse = reinterpret_cast<float*>(base + ws_off_lse(splits, rows, p.D));
  if (splits == 0)  // no key at all: the merge of zero parts writes O = 0, lse = -inf
    return launch_merge(0, rows, p.D, p.ws_o, p.ws_lse, rows * p.D, rows, 1, part_o, false, part_lse, stream, false);
  DecodeHosts hb{};
  hb.n = 0;
  hb.new_host = -1;
  if (apb_status st = launch_partials(p, hb, splits, cps, stream)) return st;
  // fold the splits (LSE merge, fixed order): the host's fp32 partial, natural-log lse
  return launch_merge((int)splits, rows, p.D, p.ws_o, p.ws_lse, rows * p.D, rows, 1, part_o, false, part_lse, stream,
                      true);
}

apb_status launch_decode_hosts(const DecodeParams& p0, DecodeHosts hb, const int64_t* n_keys, float* parts,
                               int64_t part_stride, int64_t lse_offset, void* merged_out, float* merged_lse,
                               cudaStream_t stream) {
  DecodeParams p = p0;
  int cps;
  const int64_t splits = decode_hosts_plan(hb.n, n_keys, p.hk, hb.split_begin, &cps);
  const int64_t rows = (int64_t)p.t * p.hq;
  char* base = reinterpret_cast<char*>(p.ws_o);
  p.ws_lse = reinterpret_cast<float*>(base + ws_off_lse(splits, rows, p.D));
  if (splits > 0)
    if (apb_status st = launch_partials(p, hb, splits, cps, stream)) return st;
  if (rows == 0) return APB_OK;
  if (merged_out)  // every host is here: MergeScore directly over all hosts' splits (log2 lse), bf16 out
    return launch_merge((int)splits, rows, p.D, p.ws_o, p.ws_lse, rows * p.D, rows, 1, merged_out, true, merged_lse,
                        stream, splits > 0);
  const dim3 grid((unsigned)rows, (unsigned)hb.n);
  size_t smem = 0;
  for (int i = 0; i < hb.n; ++i) {
    const size_t b = (size_t)(hb.split_begin[i + 1] - hb.split_begin[i]) * sizeof(float);
    smem = b > smem ? b : smem;
  }
  cudaLaunchConfig_t cfg = pdl_config(grid, dec::kMergeWarps * 32, smem, stream, splits > 0);
  cudaLaunchAttribute attr = pdl_attr();
  cfg.attrs = &attr;
  const float* ws_o = p.ws_o;
  const float* ws_lse = p.ws_lse;
  cudaError_t e = p.D == 128 ? cudaLaunchKernelEx(&cfg, dec::fold_hosts_kernel<128>, hb, rows, ws_o, ws_lse, parts,
                                                  part_stride, lse_offset)
                             : cudaLaunchKernelEx(&cfg, dec::fold_hosts_kernel<64>, hb, rows, ws_o, ws_lse, parts,
                                                  part_stride, lse_offset);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("fold launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_merge(int n, int64_t rows, int D, const float* parts_o, const float* parts_lse, int64_t stride_o,
                        int64_t stride_lse, int lse_in_log2, void* out, bool out_bf16, float* out_lse,
                        cudaStream_t stream, bool pdl) {
  if (rows == 0) return APB_OK;
  cudaLaunchConfig_t cfg = pdl_config(dim3((unsigned)rows, (unsigned)(D / 32)), dec::kMergeWarps * 32,
                                       (size_t)n * sizeof(float), stream, pdl);
  cudaLaunchAttribute attr = pdl_attr();
  cfg.attrs = &attr;
  __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(out);
  float* of = static_cast<float*>(out);
  cudaError_t e;
  if (D == 128)
    e = out_bf16 ? cudaLaunchKernelEx(&cfg, dec::merge_kernel<128, __nv_bfloat16>, n, rows, parts_o, parts_lse, stride_o,
                                      stride_lse, lse_in_log2, ob, out_lse)
                 : cudaLaunchKernelEx(&cfg, dec::merge_kernel<128, float>, n, rows, parts_o, parts_lse, stride_o,
                                      stride_lse, lse_in_log2, of, out_lse);
  else
    e = out_bf16 ? cudaLaunchKernelEx(&cfg, dec::merge_kernel<64, __nv_bfloat16>, n, rows, parts_o, parts_lse, stride_o,
                                      stride_lse, lse_in_log2, ob, out_lse)
                 : cudaLaunchKernelEx(&cfg, dec::merge_kernel<64, float>, n, rows, parts_o, parts_lse, stride_o,
                                      stride_lse, lse_in_log2, of, out_lse);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("merge launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace apb
