// retain_score_sm100.cu — retaining-head scoring s = R([Q_h, K_h, V_h]) (PAPER.md:171-180,
// Alg. apb_prefill line retbeg; hidden size 1024 at P:798; readings G2/G4 in DESIGN.md).
//
//   z = W1 x + b1  (tcgen05 GEMM, bf16 x bf16 -> fp32 in TMEM)
//   a = SiLU(z);  o = W2 a + b2;  s[j] = max over KV head j's group of o   (fp32 epilogue)
//
// CTA = 128 block tokens.  The A operand x_t = [Q_t | K_t | V_t] is never materialised: its
// 64-wide K blocks come straight from three TMA maps over the caller's Q, K and V rows.  The
// hidden dimension is walked in 256-wide chunks; each chunk's accumulator (128 x 256 fp32 =
// 256 TMEM columns) is double buffered so the epilogue of chunk c overlaps the MMAs of c+1.
// The W2 dot products stay in fp32 (rounding the hidden activations to bf16 changes the
// selected index sets) and are accumulated in a fixed order — no atomics, so the
// scores are bit-reproducible run to run.
// Warps 0-7: epilogue (warpgroup w handles columns [128w, 128w+128) of a chunk), warp 8: TMA,
// warp 9: MMA issuer.
// Clusters of kCluster CTAs (consecutive token tiles) share every W1 tile: each CTA fetches a
// 1/kCluster slice and multicasts it to the whole cluster, so W1 crosses L2 once per cluster
// instead of once per CTA (the kernel is otherwise bound by streaming W1 through L2).
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace apb {
namespace score {

using namespace apb::sm100;

constexpr int TM = 128;     // tokens per CTA
constexpr int TN = 256;     // hidden units per chunk (MMA N)
constexpr int TK = 64;      // K block (one 128-byte swizzle atom)
constexpr int kThreads = 320;
constexpr int kLoadWarp = 8, kMmaWarp = 9;
constexpr int kCluster = 4;
constexpr int kBSlice = TN / kCluster;  // W1 rows each CTA fetches per k block
constexpr int kABytes = TM * TK * 2;  // 16 KB
constexpr int kBBytes = TN * TK * 2;  // 32 KB

// Shared-memory plan for a pipeline depth and a W2-slice capacity (outputs).  n_out <= 32 (every
// paper config scores per query head at most 32 heads per host) leaves room for a 4th stage:
// the A rows stream from HBM (re-read once per hidden chunk), so the deeper ring hides more of
// their latency.
// PASS = 2 hidden chunks per pass over the A rows: every A tile feeds both TMEM accumulators, so
// the A rows are read d_R / 512 instead of d_R / 256 times, at the cost of the MMA/epilogue
// overlap across the pass boundary.
template <int STAGES_, int MAXOUT_, int PASS_ = 1>
struct Plan {
  static constexpr int STAGES = STAGES_;
  static constexpr int kMaxOut = MAXOUT_;
  static constexpr int PASS = PASS_;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + STAGES * kABytes;
  static constexpr int kOffW2 = kOffB + STAGES * PASS * kBBytes;  // fp32 W2 slice of one chunk [kMaxOut][TN]
  static constexpr int kOffB1 = kOffW2 + kMaxOut * TN * 4;      // fp32 b1 slice [TN]
  static constexpr int kOffBar = kOffB1 + TN * 4;
  static constexpr int kNumBars = 2 * STAGES + 4;               // full/empty per stage, acc full/empty x2
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;
  static_assert(kSmem <= 232448, "shared memory");
};

template <class PL>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    retain_score_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_w1,
                        const ScoreParams p) {
  constexpr int STAGES = PL::STAGES, kMaxOut = PL::kMaxOut, PASS = PL::PASS;
  constexpr int kStageB = PASS * kBBytes;
  constexpr int kOffA = PL::kOffA, kOffB = PL::kOffB, kOffW2 = PL::kOffW2, kOffB1 = PL::kOffB1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + PL::kOffBar;
  auto bFull = [&](int s) { return bar0 + 8u * s; };
  auto bEmpty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto bAccFull = [&](int b) { return bar0 + 8u * (2 * STAGES + b); };
  auto bAccEmpty = [&](int b) { return bar0 + 8u * (2 * STAGES + 2 + b); };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + PL::kOffTmem);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x / 32));
  const int m0 = blockIdx.x * TM;
  const int nkb = p.d_in / TK;
  const int nchunks = p.d_hidden / TN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bFull(s), 1);
      mbar_init(bEmpty(s), kCluster);  // a stage is free once every CTA of the cluster consumed it
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bAccFull(b), 1);
      mbar_init(bAccEmpty(b), 256);
    }
    fence_mbar_init();
  }
  if (warp == kLoadWarp) tmem_alloc<512>(smem_u32(tmem_ptr));
  tc_fence_before();
  cluster_sync();  // barrier inits visible cluster-wide before any multicast arrives
  tc_fence_after();
  const uint32_t crank = cluster_ctarank();
  constexpr uint16_t kMask = (1u << kCluster) - 1;
  const uint32_t tmem = warp_uniform(*tmem_ptr);  // uniform: UMMA operands stay in uniform registers

  if (warp == kLoadWarp) {
    // warp-converged producer; one elected lane issues the TMA copies
    const int row = p.L_A + m0;
    for (int pc = 0; pc < nchunks / PASS; ++pc) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int it = pc * nkb + kb, s = it % STAGES;
        mbar_wait(bEmpty(s), ((it / STAGES) & 1) ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(bFull(s), kABytes + kStageB);
          const uint32_t dA = sbase + kOffA + s * kABytes;
          if (kb < p.kq)
            tma_load_2d(dA, &tm_q, bFull(s), kb * TK, row);
          else if (kb < p.kq + p.kk)
            tma_load_2d(dA, &tm_k, bFull(s), (kb - p.kq) * TK, row);
          else
            tma_load_2d(dA, &tm_v, bFull(s), (kb - p.kq - p.kk) * TK, row);
#pragma unroll
          for (int q = 0; q < PASS; ++q)
            tma_load_2d_mc(sbase + kOffB + s * kStageB + q * kBBytes + crank * (kBSlice * 128), &tm_w1, bFull(s),
                           kb * TK, (pc * PASS + q) * TN + crank * kBSlice, kMask);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // warp-converged MMA issuer; one elected lane issues tcgen05.mma / commit
    constexpr uint32_t idesc = idesc_bf16_f32(TM, TN, false, false);
    for (int pc = 0; pc < nchunks / PASS; ++pc) {
      for (int q = 0; q < PASS; ++q) {
        const int c = pc * PASS + q;
        mbar_wait(bAccEmpty(c & 1), ((c >> 1) & 1) ^ 1);
      }
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        const int it = pc * nkb + kb, s = it % STAGES;
        mbar_wait(bFull(s), (it / STAGES) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t aA = sbase + kOffA + s * kABytes;
#pragma unroll
          for (int q = 0; q < PASS; ++q) {
            const int b = (pc * PASS + q) & 1;
            const uint32_t aB = sbase + kOffB + s * kStageB + q * kBBytes;
#pragma unroll
            for (int k = 0; k < TK / 16; ++k)
              mma_ss(tmem + b * TN, sdesc_sw128(aA + k * 32, 16, 1024), sdesc_sw128(aB + k * 32, 16, 1024), idesc,
                     (kb > 0 || k > 0) ? 1u : 0u);
          }
          mma_commit_mc(bEmpty(s), kMask);  // frees the stage in every CTA (their loads multicast here)
          if (kb == nkb - 1)
            for (int q = 0; q < PASS; ++q) mma_commit(bAccFull((pc * PASS + q) & 1));
        }
        __syncwarp();
      }
    }
  } else {
    // ================================================================ epilogue (256 threads)
    // thread = (token row r = TMEM lane, column half wg of each 256-wide chunk); the W2 partial
    // sums of the row stay in registers, summed in a fixed order (deterministic)
    const int wg = warp / 4;
    const int r = threadIdx.x % 128;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float o[kMaxOut];
#pragma unroll
    for (int oc = 0; oc < kMaxOut; ++oc) o[oc] = 0.f;
    float* w2s = reinterpret_cast<float*>(smem + kOffW2);
    float* b1s = reinterpret_cast<float*>(smem + kOffB1);
    for (int c = 0; c < nchunks; ++c) {
      const int b = c & 1;
      // this chunk's W2 columns and b1 entries -> shared memory (read back as warp broadcasts)
      for (int idx = threadIdx.x; idx < p.n_out * (TN / 4); idx += 256) {
        const int oc = idx / (TN / 4), c4 = idx % (TN / 4);
        reinterpret_cast<float4*>(w2s + oc * TN)[c4] =
            __ldg(reinterpret_cast<const float4*>(p.w2 + (size_t)oc * p.d_hidden + c * TN) + c4);
      }
      for (int idx = threadIdx.x; idx < TN; idx += 256) b1s[idx] = p.b1 ? __ldg(p.b1 + c * TN + idx) : 0.f;
      named_bar_sync(1, 256);
      mbar_wait(bAccFull(b), (c >> 1) & 1);
      tc_fence_after();
      for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t zr[32];
        tmem_ld32(tmem + lane_base + b * TN + wg * 128 + q4 * 32, zr);
        tmem_wait_ld();
        if (q4 == 3) {
          tc_fence_before();
          mbar_arrive(bAccEmpty(b));  // TMEM buffer free: the next-but-one chunk may accumulate into it
        }
#ifdef APB_DEBUG_SCORE_NO_EPILOGUE
        continue;  // timing experiment only
#endif
        const int cl = wg * 128 + q4 * 32;  // column of this piece inside the chunk
        float* a = reinterpret_cast<float*>(zr);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float z = a[e] + b1s[cl + e];
          a[e] = __fdividef(z, 1.f + __expf(-z));  // SiLU
        }
        // W2 dot on packed FFMA2 (two columns per instruction; half the issue slots of FFMA)
        uint64_t a2[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) a2[e] = f2_pack(a[2 * e], a[2 * e + 1]);
#pragma unroll
        for (int oc = 0; oc < kMaxOut; ++oc) {
          if (oc < p.n_out) {
            const ulonglong2* w = reinterpret_cast<const ulonglong2*>(w2s + oc * TN + cl);
            uint64_t acc01 = 0ull, acc23 = 0ull;
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
              const ulonglong2 wv = w[e4];
              acc01 = ffma2(wv.x, a2[2 * e4], acc01);
              acc23 = ffma2(wv.y, a2[2 * e4 + 1], acc23);
            }
            float x0, x1, y0, y1;
            f2_unpack(acc01, x0, x1);
            f2_unpack(acc23, y0, y1);
            o[oc] += (x0 + x1) + (y0 + y1);
          }
        }
      }
      named_bar_sync(1, 256);  // the slice is overwritten by the next chunk
    }
    // combine the two column halves through the (now idle) stage buffers: every MMA has
    // completed and every multicast slice has landed (each stage's full barrier was waited on)
    float* xo = reinterpret_cast<float*>(smem + kOffA);  // [kMaxOut][TM]
    named_bar_sync(1, 256);
    if (wg == 1) {
#pragma unroll
      for (int oc = 0; oc < kMaxOut; ++oc)
        if (oc < p.n_out) xo[oc * TM + r] = o[oc];
    }
    named_bar_sync(1, 256);
    if (wg == 0 && m0 + r < p.l_b) {
      const int rr = p.n_out / p.hk;
      for (int j = 0; j < p.hk; ++j) {
        float m = -INFINITY;
#pragma unroll
        for (int oc = 0; oc < kMaxOut; ++oc) {
          if (oc >= j * rr && oc < (j + 1) * rr) {
            const float v = o[oc] + xo[oc * TM + r] + (p.b2 ? __ldg(p.b2 + oc) : 0.f);
            m = fmaxf(m, v);
          }
        }
        p.scores[(int64_t)j * p.l_b + m0 + r] = m;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kLoadWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  cluster_sync();  // no CTA exits while a peer may still multicast into / arrive on its smem
}

}  // namespace score

namespace score {
template <class PL>
static apb_status launch(const ScoreParams& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const CUtensorMap& tw1, cudaStream_t stream) {
  static std::atomic<uint64_t> smem_set{0};
  if (apb_status st = set_max_smem_once(reinterpret_cast<const void*>(retain_score_kernel<PL>), PL::kSmem, smem_set))
    return st;
  int grid = (p.l_b + TM - 1) / TM;
  grid = (grid + kCluster - 1) / kCluster * kCluster;  // whole clusters
  retain_score_kernel<PL><<<grid, kThreads, PL::kSmem, stream>>>(tq, tk, tv, tw1, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("retain_score launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}
}  // namespace score

apb_status launch_retain_score(const ScoreParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                               const CUtensorMap& tv, const CUtensorMap& tw1, cudaStream_t stream) {
  // APB_SCORE_PLAN (timing experiments): "s3" forces the 3-stage plan, "p2" two chunks per pass
  // (any other value, e.g. "legacy": the default single-CTA plan)
  const char* plan = std::getenv("APB_SCORE_PLAN");
  const bool force3 = plan && plan[0] == 's' && plan[1] == '3';
  const bool pass2 = plan && plan[0] == 'p' && plan[1] == '2';
  if (pass2 && p.n_out <= 32 && (p.d_hidden / score::TN) % 2 == 0)
    return score::launch<score::Plan<2, 32, 2>>(p, tq, tk, tv, tw1, stream);
  if (!force3 && p.n_out <= 32) return score::launch<score::Plan<4, 32>>(p, tq, tk, tv, tw1, stream);
  return score::launch<score::Plan<3, 64>>(p, tq, tk, tv, tw1, stream);
}

}  // namespace apb
