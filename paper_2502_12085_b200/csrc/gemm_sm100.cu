// gemm_sm100.cu — the projection GEMMs of the APB prefill layer (qkv_proj
// P:708, O projection and FFN P:730) with their elementwise steps fused into the epilogue:
//
//   C[M][N] = A[M][K] W[N][K]^T          (bf16 in, fp32 accumulate in TMEM)
//   epilogue STORE     C = bf16(acc)
//            RESIDUAL  C = bf16(beta * C + bf16(acc))        (O / down projection + residual, G20)
//            SWIGLU    act[r][i] = bf16(SiLU(g) * u), g = bf16(acc[gate col]), u = bf16(acc[up col])
//                      (gate/up rows of W interleaved in 128-row blocks, so one 256-wide tile holds
//                      the gate and up columns of the same 128 intermediate units)
//            ROPE      C = bf16(acc), then rotate-half RoPE on the columns [0, rope_cols) (the Q and
//                      K heads of a qkv row) with the row's position — the same arithmetic as
//                      rope_kernel (fp64 angle reduction to [-pi, pi], then __sincosf), so the
//                      fused and the separate paths produce the same bits
//
// Persistent, warp-specialised, CTA pairs (cta_group::2): a pair owns a 256 x 256 output tile
// (each CTA 128 rows), each CTA loads its 128 rows of A and its half (128 rows) of the W tile per
// 64-wide K block through TMA into a 6-stage ring, and the leader CTA's single MMA thread issues
// M = 256, N = 256 tcgen05 MMAs that read both CTAs' shared memory — per SM, half of the W tile
// is loaded, which keeps the L2 -> SM operand stream at 64 B/clk at the full MMA rate.
// Accumulators are double-buffered in TMEM (2 x 256 columns), so the epilogue of one tile
// (4 warps per CTA, thread = output row = TMEM lane) overlaps the next tile's MMAs.
// Warps: 0 TMA producer, 1 MMA issuer (leader CTA), 2 TMEM allocator, 4-7 epilogue.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "internal.h"
#include "sm100.cuh"

namespace apb {
namespace gemm {

using namespace apb::sm100;

constexpr int BM = 128;              // output rows per CTA (256 per pair)
constexpr int BK = 64;               // K block: one 128-byte swizzle atom
constexpr int kThreads = 256;
constexpr int kABytes = BM * BK * 2;          // 16 KB
constexpr int kStageOut = BM * 32 * 2;        // one 128-row x 32-column bf16 output box
// Tile shape: a pair owns 256 rows x BN columns (BN = 256; the retaining-head scoring can also run
// BN = 128 — 6.9 instead of 3.5 waves, but measured slower: see score_tile_n).
template <int BN_>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr int kBBytes = (BN / 2) * BK * 2;  // this CTA's half of the W tile
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int STAGES = (192 * 1024) / kStageBytes;  // 6 (BN 256) or 8 (BN 128)
  static constexpr int kOffBar = STAGES * kStageBytes;
  static constexpr int kNumBars = 2 * STAGES + 4;  // full / empty per stage, TMEM full / empty x 2
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kOffInv = (kOffTmem + 16 + 7) / 8 * 8;  // fp64 RoPE inverse frequencies [64]
  // output staging for the TMA stores: two 128-row x 32-column bf16 boxes (64-byte swizzle)
  static constexpr int kOffStage = (kOffInv + 64 * 8 + 1023) / 1024 * 1024;
  static constexpr int kSmem = kOffStage + 2 * kStageOut + 1024;
  // retaining-head scoring (SCORE): a W2 slice [32 outputs][BN hidden] fp32 and b1 [BN]
  static constexpr int kOffW2 = kOffStage;  // the SCORE epilogue stores no tiles: reuses the staging area
  static constexpr int kOffB1 = kOffW2 + 32 * BN * 4;
  static constexpr int kSmemScore = kOffB1 + BN * 4 + 1024;
  static constexpr int kTmemCols = 2 * BN >= 512 ? 512 : 256;
  static_assert(kSmemScore <= 232448 && kSmem <= 232448, "shared memory");
};
constexpr double kL2Budget = 48.0 * (1 << 20);  // bytes of a raster group's resident operand rows
constexpr int kEpiScore = 100;                  // internal epilogue: retaining-head partial scores
constexpr int kGemmMaxHosts = 8;

// Tensor maps of one launch (kernel parameter space): A per host as up to three maps, W, C and
// the quarter-tile W map of the half-tile tail.
struct Maps {
  CUtensorMap a[kGemmMaxHosts][3];
  CUtensorMap w, c, wh;
};

struct Params {
  int64_t M;
  int N, K;
  uint16_t* c;          // output (ACT for SWIGLU) rows, ldc elements apart
  int64_t ldc;
  int epi;              // apb_gemm_epilogue
  float beta;           // RESIDUAL
  int rope_cols, head_dim;
  const int32_t* positions;
  int64_t pos_offset;
  double log2_theta;
  int num_m, num_n, num_tiles, nkb;
  int n_items, n_full;  // work items; items >= n_full are half tiles (BN/2 columns, the tail wave)
  int hint_w, hint_c;   // L2 policies: W loads evict_last, C stores evict_first (APB_GEMM_HINTS)
  int dbg;              // timing experiments only (APB_SCORE_DBG): 1 = SCORE epilogue skips the W2 products
  int raster_n, group;  // raster: groups of `group` M-tiles (N fastest... see tile_coords) or N-tiles
  // A from up to three row-aligned maps ([Q | K | V] for the retaining head): K blocks [0, kq) from
  // map 0, [kq, kqk) from map 1, the rest from map 2; A's row coordinate is a_row0[host] + row.
  // n_hosts > 1 (scoring only): the same M x N problem for several hosts in one launch, tile
  // T -> host T / tiles_per_host (its own A maps, a_row0 and partial slots part + host * part_stride)
  int kq, kqk;
  int n_hosts, tiles_per_host;
  int a_row0[kGemmMaxHosts];
  int64_t part_stride;
  // SCORE: partial[nb][n_out][row] = W2[:, nb*128 .. +128] SiLU(acc + b1[...])  (fp32)
  const float* b1;
  const float* w2;
  int n_out, d_hidden;
  float* part;
};

// Tile raster.  Row-grouped (raster_n = 0): a group of `group` M-tiles sweeps every N-tile, so its A
// rows stay in L2 while W streams through once per group.  Column-grouped (raster_n = 1): a group
// of N-tiles sweeps every M-tile (W stays, A streams once per group).  launch_params picks the
// order and group size with the smaller estimated DRAM traffic for the L2 budget.
__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mb, int& nb) {
  const int outer = p.raster_n ? p.num_n : p.num_m, inner = p.raster_n ? p.num_m : p.num_n;
  const int per_group = p.group * inner;
  const int g = t / per_group, first = g * p.group;
  const int gs = min(p.group, outer - first);
  const int r = t - g * per_group;
  const int o = first + r % gs, i = r / gs;
  mb = p.raster_n ? i : o;
  nb = p.raster_n ? o : i;
}

// Work item -> tile (+ half: -1 = the whole BN-wide tile, 0 / 1 = its left / right BN/2 columns).
// The tiles of a final partial wave are split in two halves (launch_params), so that wave is
// half as long: 256 scoring tiles on 74 pairs run in 3.5 instead of 4 tile-times.
__device__ __forceinline__ void item_coords(const Params& p, int item, int& host, int& mb, int& nb, int& half) {
  int T;
  if (item < p.n_full) {
    T = item;
    half = -1;
  } else {
    const int r = item - p.n_full;
    T = p.n_full + r / 2;
    half = r & 1;
  }
  host = T / p.tiles_per_host;
  tile_coords(p, T - host * p.tiles_per_host, mb, nb);
}

__device__ __forceinline__ float bf16_round(float x) {
  return __uint_as_float(static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(x))) << 16);
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) { return pack_bf16x2(lo, hi); }

__device__ __forceinline__ void load32(const uint16_t* src, float (&v)[32], int ncols) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = q * 8 < ncols ? s4[q] : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[8 * q + 2 * e] = __uint_as_float(w[e] << 16);
      v[8 * q + 2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
    }
  }
}

template <int BN_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ Maps tm, const Params p) {
  const CUtensorMap* tm_w = &tm.w;
  const CUtensorMap* tm_c = &tm.c;
  const CUtensorMap* tm_wh = &tm.wh;
  using C = Cfg<BN_>;
  constexpr int BN = C::BN, STAGES = C::STAGES, kBBytes = C::kBBytes, kStageBytes = C::kStageBytes;
  constexpr int kOffBar = C::kOffBar, kOffTmem = C::kOffTmem, kOffInv = C::kOffInv, kOffStage = C::kOffStage;
  constexpr int kOffW2 = C::kOffW2, kOffB1 = C::kOffB1;
  (void)kBBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + kOffBar;
  auto bFull = [&](int s) { return bar0 + 8u * s; };
  auto bEmpty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto bTFull = [&](int b) { return bar0 + 8u * (2 * STAGES + b); };
  auto bTEmpty = [&](int b) { return bar0 + 8u * (2 * STAGES + 2 + b); };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  double* inv = reinterpret_cast<double*>(smem + kOffInv);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x / 32));
  const uint32_t rank = cluster_ctarank();  // 0: the MMA-issuing (leader) CTA of the pair
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bFull(s), 1);   // leader: its own expect_tx; both CTAs' TMA bytes land here
      mbar_init(bEmpty(s), 1);  // one multicast commit from the leader's MMA thread
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bTFull(b), 1);
      mbar_init(bTEmpty(b), 8);  // leader: one lane of each of the 2 x 4 epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<C::kTmemCols>(smem_u32(tmem_ptr));
  if (p.epi == APB_EPI_ROPE && threadIdx.x < p.head_dim / 2)
    inv[threadIdx.x] = exp2(-p.log2_theta * (2.0 * threadIdx.x) / p.head_dim);
  tc_fence_before();
  cluster_sync();  // barrier inits and the TMEM address visible pair-wide
  tc_fence_after();
  const uint32_t tmem = warp_uniform(*tmem_ptr);
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0) {
    // ================================================================ TMA producer (both CTAs)
    const uint32_t full_leader0 = mapa_shared(bFull(0), 0);
    const uint64_t pol_last = policy_evict_last();
    int it = 0;
    for (int t = pair; t < p.n_items; t += npairs) {
      int host, mb, nb, half;
      item_coords(p, t, host, mb, nb, half);
      const int arow = p.a_row0[host] + mb * 2 * BM + rank * BM;
      const CUtensorMap* tma = tm.a[host];
      const int wrow = half < 0 ? nb * BN + rank * (BN / 2) : nb * BN + half * (BN / 2) + rank * (BN / 4);
      const uint32_t stage_tx = half < 0 ? 2 * kStageBytes : 2 * (kABytes + kBBytes / 2);
      for (int kb = 0; kb < p.nkb; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(bEmpty(s), ((it / STAGES) & 1) ^ 1);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bFull(s), stage_tx);
          const uint32_t st = sbase + s * kStageBytes;
          if (kb < p.kq)
            tma_load_2d_pair(st, &tma[0], full_leader0 + 8u * s, kb * BK, arow);
          else if (kb < p.kqk)
            tma_load_2d_pair(st, &tma[1], full_leader0 + 8u * s, (kb - p.kq) * BK, arow);
          else
            tma_load_2d_pair(st, &tma[2], full_leader0 + 8u * s, (kb - p.kqk) * BK, arow);
          if (half >= 0)  // this CTA's quarter of the W tile (BN/4 rows) for a half-tile item
            tma_load_2d_pair(st + kABytes, tm_wh, full_leader0 + 8u * s, kb * BK, wrow);
          else if (p.hint_w)  // the operand the raster keeps resident in L2 for the whole group
            tma_load_2d_pair_hint(st + kABytes, tm_w, full_leader0 + 8u * s, kb * BK, wrow, pol_last);
          else
            tma_load_2d_pair(st + kABytes, tm_w, full_leader0 + 8u * s, kb * BK, wrow);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (leader only)
    if (rank == 0) {
      constexpr uint32_t idesc_full = idesc_bf16_f32(2 * BM, BN, false, false);
      constexpr uint32_t idesc_half = idesc_bf16_f32(2 * BM, BN / 2, false, false);
      int it = 0, tl = 0;
      for (int t = pair; t < p.n_items; t += npairs, ++tl) {
        const uint32_t idesc = t < p.n_full ? idesc_full : idesc_half;
        const int b = tl & 1;
        mbar_wait(bTEmpty(b), ((tl >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < p.nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(bFull(s), (it / STAGES) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t aA = sbase + s * kStageBytes, aB = aA + kABytes;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_ss_pair(tmem + b * BN, sdesc_sw128(aA + k * 32, 16, 1024), sdesc_sw128(aB + k * 32, 16, 1024), idesc,
                          (kb > 0 || k > 0) ? 1u : 0u);
            mma_commit_pair_mc(bEmpty(s), 0x3);  // the stage is free in both CTAs
            if (kb == p.nkb - 1) mma_commit_pair_mc(bTFull(b), 0x3);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    // ================================================================ epilogue (128 threads)
    const int r = threadIdx.x - 128;  // row within this CTA's half = TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tempty_leader0 = mapa_shared(bTEmpty(0), 0);
    const uint32_t sstage = sbase + kOffStage;
    const uint64_t pol_first = policy_evict_first();
    int chunk_ctr = 0;
    // one 128-row x 32-column bf16 box of this CTA's rows -> shared memory (64-byte swizzle: the
    // 16-byte chunk q of row r lands at q ^ ((r >> 1) & 3), conflict-free) -> one TMA store by
    // thread 0 (out-of-range rows / columns are clipped by the tensor map).  Two buffers: a buffer
    // is rewritten only after the store issued from it two boxes earlier has read it.
    auto stage_store = [&](const float (&v)[32], int col, int row0) {
      const int buf = chunk_ctr & 1;
      if (r == 0) bulk_wait_group_read<1>();
      named_bar_sync(2, 128);
      const uint32_t rowaddr = sstage + buf * kStageOut + r * 64;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + ((q ^ ((r >> 1) & 3)) << 4)),
                     "r"(pack2(v[8 * q], v[8 * q + 1])), "r"(pack2(v[8 * q + 2], v[8 * q + 3])),
                     "r"(pack2(v[8 * q + 4], v[8 * q + 5])), "r"(pack2(v[8 * q + 6], v[8 * q + 7]))
                     : "memory");
      fence_proxy_async_smem();
      named_bar_sync(2, 128);
      if (r == 0) {
        // output lines are not re-read by this kernel: first candidates for eviction, so the
        // operand rows the raster keeps resident stay in L2
        if (p.hint_c) tma_store_2d_hint(tm_c, sstage + buf * kStageOut, col, row0, pol_first);
        else tma_store_2d(tm_c, sstage + buf * kStageOut, col, row0);
        bulk_commit_group();
      }
      ++chunk_ctr;
    };
    int tl = 0;
    for (int t = pair; t < p.n_items; t += npairs, ++tl) {
      int host, mb, nb, half;
      item_coords(p, t, host, mb, nb, half);
      const int b = tl & 1;
      const int64_t row = (int64_t)mb * 2 * BM + rank * BM + r;
      const bool row_ok = row < p.M;
      const int n0 = nb * BN + (half > 0 ? BN / 2 : 0);
      const int bne = half < 0 ? BN : BN / 2;  // columns of this item (half tiles: SCORE only)
      const uint32_t tacc = tmem + lane_base + b * BN;
      mbar_wait(bTFull(b), (tl >> 1) & 1);
      tc_fence_after();
      double posd = 0.0;
      if (p.epi == APB_EPI_ROPE)
        posd = row_ok ? (p.positions ? (double)p.positions[row] : (double)(p.pos_offset + row)) : 0.0;
      if (p.epi == kEpiScore) {
        // retaining head (reading G2): a = SiLU(z + b1) for this item's hidden units
        // (BN, or BN/2 for a half-tile item), partial o[oc] = sum_h W2[oc][h] a_h in fp32 (fixed
        // order: chunks of 32 in column order, packed FFMA2 pairs) -> part[slot][oc][row] with one
        // slot per BN/2 hidden units (a whole tile writes each half's sum to that half's slot, so
        // the slots do not depend on the tiling); score_finalize_kernel sums the slots in order.
        // 32 outputs per pass over TMEM.
        float* w2s = reinterpret_cast<float*>(smem + kOffW2);
        float* b1s = reinterpret_cast<float*>(smem + kOffB1);
        named_bar_sync(1, 128);  // the previous tile's readers of w2s / b1s are done
        for (int i = r; i < bne; i += 128) b1s[i] = p.b1 ? __ldg(p.b1 + n0 + i) : 0.f;
        const int slot = n0 / (BN / 2);
#pragma unroll 1
        for (int og = 0; og < p.n_out; og += 32) {
          const int no = min(32, p.n_out - og);
          if (og > 0) named_bar_sync(1, 128);
          for (int idx = r; idx < no * (bne / 4); idx += 128) {
            const int oc = idx / (bne / 4), c4 = idx % (bne / 4);
            reinterpret_cast<float4*>(w2s + oc * BN)[c4] =
                __ldg(reinterpret_cast<const float4*>(p.w2 + (size_t)(og + oc) * p.d_hidden + n0) + c4);
          }
          named_bar_sync(1, 128);
          float o[32];
#pragma unroll
          for (int oc = 0; oc < 32; ++oc) o[oc] = 0.f;
          float* part = p.part + host * p.part_stride;
#pragma unroll 1
          for (int c = 0; c < (p.dbg == 1 ? 0 : bne); c += 32) {
            if (c == BN / 2) {
              // a whole tile writes its first BN/2 hidden units' sum to their own slot, as the half
              // tile covering them would: the partial slots (and so the scores) do not depend on
              // which tiles of a launch run as half tiles (per-host and multi-host launches agree)
              if (row_ok) {
                float* dst = part + ((int64_t)slot * p.n_out + og) * p.M + row;
#pragma unroll
                for (int oc = 0; oc < 32; ++oc)
                  if (oc < no) dst[(int64_t)oc * p.M] = o[oc];
              }
#pragma unroll
              for (int oc = 0; oc < 32; ++oc) o[oc] = 0.f;
            }
            uint32_t zr[32];
            tmem_ld32(tacc + c, zr);
            tmem_wait_ld();
            uint64_t a2[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float z0 = __uint_as_float(zr[2 * e]) + b1s[c + 2 * e];
              const float z1 = __uint_as_float(zr[2 * e + 1]) + b1s[c + 2 * e + 1];
              a2[e] = f2_pack(__fdividef(z0, 1.f + __expf(-z0)), __fdividef(z1, 1.f + __expf(-z1)));
            }
#pragma unroll
            for (int oc = 0; oc < 32; ++oc) {
              if (oc < no) {
                const ulonglong2* w = reinterpret_cast<const ulonglong2*>(w2s + oc * BN + c);
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
          if (row_ok) {  // the (second, for a whole tile) BN/2 hidden units' slot
            float* dst = part + ((int64_t)(half < 0 ? slot + 1 : slot) * p.n_out + og) * p.M + row;
#pragma unroll
            for (int oc = 0; oc < 32; ++oc)
              if (oc < no) dst[(int64_t)oc * p.M] = o[oc];
          }
        }
      } else if (p.epi == APB_EPI_SWIGLU) {
        // gate columns [0,128) and up columns [128,256) of this tile -> act columns n0/2 + [0,128)
        const int a0 = n0 / 2;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t g[32], u[32];
          tmem_ld32(tacc + c * 32, g);
          tmem_ld32(tacc + 128 + c * 32, u);
          tmem_wait_ld();
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float gf = bf16_round(__uint_as_float(g[e])), uf = bf16_round(__uint_as_float(u[e]));
            v[e] = gf / (1.f + __expf(-gf)) * uf;
          }
          stage_store(v, a0 + c * 32, (int)(row - r));
        }
      } else if (p.epi == APB_EPI_ROPE) {
        // the angles of a row depend only on (position, i < head_dim/2): computed once per tile
        // per 32-wide i chunk and applied to every head of the tile
        const int hd = p.head_dim, half = hd / 2;
#pragma unroll 1
        for (int c = 0; c < half; c += 32) {
          float cs[32], sn[32];
          if (n0 < p.rope_cols) {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              double a = posd * inv[c + e];
              a -= rint(a * 0.15915494309189535) * 6.283185307179586;  // |a| <= pi
              __sincosf(static_cast<float>(a), &sn[e], &cs[e]);
            }
          }
#pragma unroll 1
          for (int h0 = 0; h0 < BN; h0 += hd) {
            const bool rot = n0 + h0 < p.rope_cols;  // warp-uniform
            uint32_t x1[32], x2[32];
            tmem_ld32(tacc + h0 + c, x1);
            tmem_ld32(tacc + h0 + half + c, x2);
            tmem_wait_ld();
            float o1[32], o2[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const float f1 = bf16_round(__uint_as_float(x1[e])), f2 = bf16_round(__uint_as_float(x2[e]));
              o1[e] = rot ? f1 * cs[e] - f2 * sn[e] : f1;
              o2[e] = rot ? f2 * cs[e] + f1 * sn[e] : f2;
            }
            stage_store(o1, n0 + h0 + c, (int)(row - r));
            stage_store(o2, n0 + h0 + half + c, (int)(row - r));
          }
        }
      } else {
        uint16_t* dst = p.c + row * p.ldc + n0;
#pragma unroll 1
        for (int c = 0; c < bne; c += 32) {
          const int ncols = min(32, p.N - (n0 + c));
          float old[32];
          if (p.epi == APB_EPI_RESIDUAL && row_ok && ncols > 0) load32(dst + c, old, ncols);
          uint32_t acc[32];
          tmem_ld32(tacc + c, acc);
          tmem_wait_ld();
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float prod = bf16_round(__uint_as_float(acc[e]));
            v[e] = p.epi == APB_EPI_RESIDUAL ? p.beta * old[e] + prod : prod;
          }
          if (ncols > 0) stage_store(v, n0 + c, (int)(row - r));
        }
      }
      // this tile's accumulator is in registers / stored: release the TMEM buffer to the leader
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(tempty_leader0 + 8u * b);
    }
    if (r == 0) bulk_wait_group<0>();  // every TMA store of this CTA has completed
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs done: no MMA reads the peer's smem, no arrive targets an exited CTA
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<C::kTmemCols>(tmem);
  }
}

template <int BN>
static apb_status launch_params(Params& p, Maps& m, bool halves, bool score, cudaStream_t stream) {
  using C = Cfg<BN>;
  const int smem = score ? C::kSmemScore : C::kSmem;
  if (p.n_hosts < 1) p.n_hosts = 1;
  p.num_m = (int)((p.M + 2 * BM - 1) / (2 * BM));
  p.num_n = (p.N + BN - 1) / BN;
  p.tiles_per_host = p.num_m * p.num_n;
  p.num_tiles = p.tiles_per_host * p.n_hosts;
  p.nkb = (p.K + BK - 1) / BK;
  {
    // estimated DRAM bytes: row groups read A once and W once per group; column groups the reverse
    const double row_block = 2.0 * BM * p.K * 2.0, col_block = (double)BN * p.K * 2.0;
    const int gm = std::max(1, std::min(p.num_m, (int)(kL2Budget / row_block)));
    const int gn = std::max(1, std::min(p.num_n, (int)(kL2Budget / col_block)));
    const double a_bytes = (double)p.M * p.K * 2.0, w_bytes = (double)p.N * p.K * 2.0;
    const double traf_m = a_bytes + w_bytes * ((p.num_m + gm - 1) / gm);
    const double traf_n = w_bytes + a_bytes * ((p.num_n + gn - 1) / gn);
    p.raster_n = traf_n < traf_m ? 1 : 0;
    p.group = p.raster_n ? gn : gm;
    if (const char* env = std::getenv("APB_GEMM_GROUP")) {  // timing experiments: "m8", "n4", ...
      p.raster_n = env[0] == 'n';
      p.group = std::max(1, std::atoi(env + 1));
    }
  }
  {
    const char* h = std::getenv("APB_GEMM_HINTS");  // timing experiments: "wc" (default), "w", "c", "none"
    const std::string hs = h ? h : "wc";
    p.hint_w = hs.find('w') != std::string::npos;
    p.hint_c = hs.find('c') != std::string::npos;
  }
  if (const char* dbg = std::getenv("APB_SCORE_DBG")) p.dbg = std::atoi(dbg);
  static std::atomic<uint64_t> smem_set{0};
  if (apb_status st = set_max_smem_once(reinterpret_cast<const void*>(gemm_kernel<BN>), C::kSmemScore, smem_set))
    return st;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int npairs = sms / 2;
  p.n_items = p.n_full = p.num_tiles;
  const int tail = p.num_tiles % npairs;
  const char* split_env = std::getenv("APB_GEMM_TAIL_SPLIT");  // timing experiments: "0" disables
  if (halves && tail > 0 && 2 * tail <= npairs && p.num_tiles > npairs && !(split_env && split_env[0] == '0')) {
    // a partial last wave: its tiles run as half tiles (twice as many, half as long)
    p.n_full = p.num_tiles - tail;
    p.n_items = p.n_full + 2 * tail;
  }
  const int pairs = std::min(p.n_items, npairs);
  if (!halves) m.wh = m.w;  // never dereferenced
  gemm_kernel<BN><<<2 * pairs, kThreads, smem, stream>>>(m, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

// score_finalize_kernel: o[oc] = b2[oc] + sum_nb part[nb][t][oc] (nb order), s[j][t] = max over the
// r = n_out / hk outputs of KV head j (reading G4).  One thread per block token; a token's n_out
// partials are contiguous, read as float4 when n_out % 4 == 0 (every paper config).
struct ScoreOut {
  float* s[kGemmMaxHosts];  // per host: [hk][l_b]
};
__global__ void __launch_bounds__(128) score_finalize_kernel(const float* __restrict__ part_all, int64_t part_stride,
                                                             int l_b, int n_parts, int n_out, int hk,
                                                             const float* __restrict__ b2, const __grid_constant__ ScoreOut so) {
  const int t = blockIdx.x * 128 + threadIdx.x;
  if (t >= l_b) return;
  const float* part = part_all + blockIdx.y * part_stride;  // grid.y = host of the launch
  float* scores = so.s[blockIdx.y];
  const int rr = n_out / hk;
  float m = -INFINITY;
  auto emit = [&](int oc, float o) {  // outputs arrive in oc order
    m = fmaxf(m, o + (b2 ? __ldg(b2 + oc) : 0.f));
    if ((oc + 1) % rr == 0) {
      scores[(int64_t)(oc / rr) * l_b + t] = m;
      m = -INFINITY;
    }
  };
  // partials [slot][oc][token]: consecutive threads (tokens) read consecutive words; 8 outputs x
  // 4 slots of loads in flight per thread (each output still sums its slots in ascending order)
  for (int oc0 = 0; oc0 < n_out; oc0 += 8) {
    const int no = min(8, n_out - oc0);
    float o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = 0.f;
#pragma unroll 4
    for (int nb = 0; nb < n_parts; ++nb) {
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = q < no ? __ldg(part + ((int64_t)nb * n_out + oc0 + q) * l_b + t) : 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] += v[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < no) emit(oc0 + q, o[q]);
  }
}

}  // namespace gemm

apb_status launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  using namespace gemm;
  Maps m;
  {
    uint64_t dims[2] = {(uint64_t)g.K, (uint64_t)g.M};
    uint64_t str[1] = {(uint64_t)g.lda * 2};
    uint32_t box[2] = {BK, BM};
    if (!make_tmap_bf16(&m.a[0][0], g.a, 2, dims, str, box)) return APB_ERR_CUDA;
    m.a[0][1] = m.a[0][2] = m.a[0][0];
  }
  {
    uint64_t dims[2] = {(uint64_t)g.K, (uint64_t)g.N};
    uint64_t str[1] = {(uint64_t)g.ldw * 2};
    uint32_t box[2] = {BK, 128};  // this CTA's half of a 256-column W tile
    if (!make_tmap_bf16(&m.w, g.w, 2, dims, str, box)) return APB_ERR_CUDA;
  }
  Params p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.c = static_cast<uint16_t*>(g.c);
  p.ldc = g.ldc;
  p.epi = g.epi;
  p.beta = g.beta;
  p.rope_cols = g.rope_cols;
  p.head_dim = g.head_dim > 0 ? g.head_dim : 128;
  p.positions = g.positions;
  p.pos_offset = g.pos_offset;
  p.log2_theta = g.theta > 0.f ? std::log2((double)g.theta) : 0.0;
  p.kq = p.kqk = (g.K + BK - 1) / BK;
  // STORE / RESIDUAL can run the tiles of a partial last wave as half tiles (SWIGLU's tile holds
  // gate and up halves, ROPE's whole heads: they keep whole tiles)
  const bool halves = g.epi == APB_EPI_STORE || g.epi == APB_EPI_RESIDUAL;
  if (halves) {
    uint64_t dims[2] = {(uint64_t)g.K, (uint64_t)g.N};
    uint64_t str[1] = {(uint64_t)g.ldw * 2};
    uint32_t box[2] = {BK, 64};
    if (!make_tmap_bf16(&m.wh, g.w, 2, dims, str, box)) return APB_ERR_CUDA;
  }
  {
    const uint64_t ncols = g.epi == APB_EPI_SWIGLU ? (uint64_t)g.N / 2 : (uint64_t)g.N;
    uint64_t dims[2] = {ncols, (uint64_t)g.M};
    uint64_t str[1] = {(uint64_t)g.ldc * 2};
    uint32_t box[2] = {32, BM};
    if (!make_tmap_bf16(&m.c, g.c, 2, dims, str, box, 64)) return APB_ERR_CUDA;
  }
  p.n_hosts = 1;
  return launch_params<256>(p, m, halves, false, stream);
}

// Hidden-unit tile of the scoring GEMM: 256 (default) or 128 (APB_SCORE_BN=128).  Measured on the
// L8 host: 0.176 ms with 256 vs 0.189 ms with 128 — the 128-wide tiles remove the wave
// quantisation (6.9 instead of 3.5 waves) but load 1.5x the operand bytes per FLOP.
int score_tile_n() {
  static const int bn = [] {
    const char* e = std::getenv("APB_SCORE_BN");
    return (e && std::atoi(e) == 128) ? 128 : 256;
  }();
  return bn;
}

apb_status launch_score_gemm_hosts(const ScoreParams& sp, int n, const CUtensorMap* tq, const CUtensorMap* tk,
                                   const CUtensorMap* tv, const int* L_A, float* const* scores, const CUtensorMap& tw1,
                                   const CUtensorMap& tw1h, float* part, cudaStream_t stream) {
  using namespace gemm;
  if (n < 1 || n > kGemmMaxHosts) return fail(APB_ERR_CONFIG, "1..8 hosts per scoring launch");
  Params p{};
  p.M = sp.l_b;
  p.N = sp.d_hidden;
  p.K = sp.d_in;
  p.epi = kEpiScore;
  p.kq = sp.kq;
  p.kqk = sp.kq + sp.kk;
  p.n_hosts = n;
  Maps m;
  for (int i = 0; i < n; ++i) {
    p.a_row0[i] = L_A[i];
    m.a[i][0] = tq[i];
    m.a[i][1] = tk[i];
    m.a[i][2] = tv[i];
  }
  m.w = tw1;
  m.c = tw1;  // no tile stores
  m.wh = tw1h;
  p.b1 = sp.b1;
  p.w2 = sp.w2;
  p.n_out = sp.n_out;
  p.d_hidden = sp.d_hidden;
  p.part = part;
  const int bn = score_tile_n();
  const int n_parts = (sp.d_hidden + bn / 2 - 1) / (bn / 2);  // one partial slot per bn/2 hidden units
  p.part_stride = (int64_t)n_parts * sp.l_b * sp.n_out;       // one host's partial slots
  apb_status st = bn == 128 ? launch_params<128>(p, m, true, true, stream) : launch_params<256>(p, m, true, true, stream);
  if (st) return st;
  ScoreOut so{};
  for (int i = 0; i < n; ++i) so.s[i] = scores[i];
  score_finalize_kernel<<<dim3((sp.l_b + 127) / 128, n), 128, 0, stream>>>(part, p.part_stride, sp.l_b, n_parts,
                                                                          sp.n_out, sp.hk, sp.b2, so);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("score_finalize launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_score_gemm(const ScoreParams& sp, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const CUtensorMap& tw1, const CUtensorMap& tw1h, float* part,
                             cudaStream_t stream) {
  float* scores[1] = {sp.scores};
  const int L_A[1] = {sp.L_A};
  return launch_score_gemm_hosts(sp, 1, &tq, &tk, &tv, L_A, scores, tw1, tw1h, part, stream);
}

}  // namespace apb
