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
// rows) sharing every K/V tile load.  Warp roles (384 threads):
//   warps 0-3  softmax warpgroup for Q tile 0 (thread i owns query row i = TMEM lane i)
//   warps 4-7  softmax warpgroup for Q tile 1
//   warp  8    TMA producer (Q once, then a 2-stage K ring and a 2-stage V ring)
//   warp  9    tcgen05.mma issuer (one thread);  warps 10-11 idle (complete the 3rd warpgroup
//              so setmaxnreg can move registers to the softmax warpgroups)
// TMEM (512 columns): S_0 [0,128)  S_1 [128,256)  O_0 [256,256+D)  O_1 [256+D, 256+2D).
// P_t (bf16) is written over the first 64 columns of S_t and consumed from TMEM as the A
// operand of O_t += P_t V (FlashAttention-4 style); S_t(j+1) is issued after PV_t(j), so the
// in-order tensor pipe never overwrites P_t(j) before it is read.
// Online softmax in the log2 domain with conditional rescaling: O_t is rescaled only when a
// row max grows by more than 16 (weights up to 2^16: exact range in bf16 and fp32, and the row
// sum is of the same bf16 weights, reading G21), which after the first few tiles is rare even for
// peaky logits (measured: D2 107.5 K vs 97.5 K tokens/s with the threshold at 8; D1 unchanged).
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "sm100.cuh"

namespace apb {
namespace attn {

using namespace apb::sm100;

constexpr int BM = 128;
constexpr int BN = 128;
// K and V tiles share one ring, loaded in consumption order K(0), V(0), K(1), V(1), ...;
// K(i) is released after S_1(i), V(i) after PV_1(i) — also in sequence order — so a slot is
// reused exactly kRing loads later.  Load n (= 2i for K(i), 2i+1 for V(i), counted across all the
// items a CTA runs) uses slot n % kRing.  3 slots at d = 128 leave room for the O staging tiles
// (ring depths 2..5 measured equal in round 1: the loads are not on the critical path).
template <int D>
constexpr int ring_slots() { return D == 128 ? 3 : 6; }
constexpr int kThreads = 384;  // 3 warpgroups: softmax 0, softmax 1, {TMA, MMA, 2 idle}
constexpr int kLoadWarp = 10;  // SMSP 2 (warps 0/4 on SMSP 0 would otherwise share with it)
constexpr int kMmaWarp = 9;
#ifndef APB_RESCALE_THRESHOLD
#define APB_RESCALE_THRESHOLD 16.0f
#endif
constexpr float kRescaleThreshold = APB_RESCALE_THRESHOLD;
// Of every 16 column pairs, this many are exponentiated on the FMA pipe (Cody-Waite + degree-3
// polynomial) instead of MUFU.EX2: 4 of 32 pairs per half row.  Persistent kernel, L8 bench
// (scripts/gpu/r2s2_variants.sh, same box): 0 -> 115.0 K, 1 -> 112.0 K, 2 -> 118.6 K, 3 -> 113.5 K,
// 4 -> 115.5 K, 6 -> 106.9 K tokens/s.  (Round 1 measured 2 and 4 slower with the one-item-per-CTA
// kernel; with the item gaps gone the MUFU pipe is the co-limiter and the offload pays.)
#ifndef APB_POLY_PAIRS
#define APB_POLY_PAIRS 2
#endif
// which of the 16 pair positions (bit i: pair i of every 16) use the polynomial; default the first
// APB_POLY_PAIRS positions (other placements of 2: 0x0101, 0x0011, 0xC000 measured equal or up to
// 1 % slower, 0x0300 3 % slower)
#ifndef APB_POLY_MASK
#define APB_POLY_MASK ((1u << APB_POLY_PAIRS) - 1u)
#endif
constexpr uint32_t kPolyMask = APB_POLY_MASK;
#ifndef APB_POLY_MASK1
#define APB_POLY_MASK1 APB_POLY_MASK
#endif
constexpr uint32_t kPolyMask1 = APB_POLY_MASK1;  // the second half row's positions (default: the same)

// 2^x for a pair of fp32 (x <= ~8): clamp at -126 (masked columns give ~0 denormals), split
// x = j + f with j = rint(x) via the 1.5*2^23 magic constant, 2^f by a degree-3 minimax
// polynomial on [-0.5, 0.5], then add j to the exponent field with one integer multiply-add.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  using namespace apb::sm100;
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

#ifdef APB_TRACE
// Debug instrumentation (libapb_trace.so only): clock64 stamps of one CTA's pipeline events.
// [0..): per KV step i < 64: MMA S issue (t), MMA P-half wait done (t, half), softmax S ready (t),
// softmax P-half published (t, half).
__device__ unsigned long long g_trace[64 * 32];
__device__ int g_trace_block = 0;
#define TRACE(slot, i) do { if (blockIdx.x == g_trace_block && (i) < 64) g_trace[(i) * 32 + (slot)] = clock64(); } while (0)
// per-CTA timeline of the last launch: [start globaltimer ns, end ns, smid, first S MMA issued ns,
// O final (last PV complete) ns] for blockIdx < 65536
__device__ unsigned long long g_cta_time[5 * 65536];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CTA_TIME(k) do { if (threadIdx.x == 0 && blockIdx.x < 65536) { \
    unsigned int sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); \
    g_cta_time[5 * blockIdx.x + (k)] = gtimer(); g_cta_time[5 * blockIdx.x + 2] = sm; } } while (0)
#define CTA_STAMP(k) do { if (blockIdx.x < 65536) g_cta_time[5 * blockIdx.x + (k)] = gtimer(); } while (0)
#else
#define CTA_TIME(k) do {} while (0)
#define CTA_STAMP(k) do {} while (0)
#define TRACE(slot, i) do {} while (0)
#endif

#ifdef APB_TRACE
// Hang watchdog (libapb_trace.so only): every mbarrier wait of the attention kernel is a polling
// loop that, after ~2 s, records (source line, barrier offset, parity, item seq) for its
// (CTA, warp) in mapped host memory — readable from the host while the kernel is stuck.
__device__ unsigned int* g_hang = nullptr;  // [grid][12 warps][4]
__device__ __forceinline__ void dbg_wait(uint32_t bar, uint32_t parity, uint32_t line, uint32_t bar0, int k) {
  const long long t0 = clock64();
  bool logged = false;
  for (;;) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    if (ok) return;
    if (!logged && clock64() - t0 > 4000000000ll && g_hang != nullptr) {
      logged = true;
      volatile unsigned int* h = g_hang + ((size_t)blockIdx.x * 12 + threadIdx.x / 32) * 4;
      h[0] = line;
      h[1] = bar - bar0;
      h[2] = parity;
      h[3] = (unsigned int)k;
      __threadfence_system();
    }
  }
}
#define MBW(bar, par) dbg_wait((bar), (par), __LINE__, bar0, dbg_k)
#define MBWS(bar, par) dbg_wait((bar), (par), __LINE__, bar0, dbg_k)
#else
#define MBW(bar, par) mbar_wait((bar), (par))
#define MBWS(bar, par) mbar_wait_sleep((bar), (par))
#endif

// Work counters of the persistent launches: slot [next item, CTAs done]; each launch takes the
// next slot of the ring (host side), so launches in flight on different streams never share one,
// and the launch's last CTA resets its slot for the launch that reuses it.
constexpr int kCtrSlots = 64;
__device__ unsigned int g_attn_ctr[kCtrSlots][2];
static std::atomic<uint32_t> g_launches{0};  // host: persistent launches so far (slot = count mod 64)

template <int D>
struct Layout {
  static constexpr int kHalves = D / 64;           // 64-element (128 B) swizzle atoms per row
  static constexpr int kSub = BM * 128;            // bytes of one 128-row x 64-col sub-tile
  static constexpr int kTile = kHalves * kSub;     // bytes of a 128 x D bf16 tile
  static constexpr int kRing = ring_slots<D>();
  static constexpr int kQ = 0;
  static constexpr int kR = kQ + 2 * kTile;        // the K/V ring
  static constexpr int kO = kR + kRing * kTile;    // bf16 O staging of the two tiles (TMA stores)
  static constexpr int kBar = kO + 2 * kTile;
  // barriers: Qfull, Qfree, full[kRing], empty[kRing], Sfull[2], Pfull[2][2 halves], Ofull[2],
  // Ofree[2], work[2] (next-item response landed), workfree[2] (response read by every role)
  static constexpr int kNumBars = 2 + 2 * kRing + 14;
  static_assert(14 + 2 * kRing + 1 < kNumBars, "the last barrier (workfree[1]) lies inside the barrier area");
  static constexpr int kWork = (kBar + kNumBars * 8 + 15) / 16 * 16;  // 2 x 16-byte CLC responses
  static constexpr int kTmemPtr = kWork + 32;
  static constexpr int kUsed = kTmemPtr + 16;
  static constexpr int kAlloc = kUsed + 1024;      // + alignment slack; one CTA per SM (512 TMEM columns)
  static_assert(kAlloc <= 232448, "shared memory");
};

struct Item {
  int seg;     // 0 = anchor query rows, 1 = local query rows
  int rt;      // 128-row tile index of tile 0 (the heavier one): plans the key-tile walk
  int rtt[2];  // row tile of each query tile
  int qht[2];  // query head of each query tile
  int j;       // KV head (shared by both tiles)
  int ntiles;
  int nkv;
};

// Work items: per (segment, KV head j) the units (row tile, query head of j's group) are ordered
// heaviest row tile first and paired consecutively; a pair shares every K/V tile.  For even g both
// units of a pair have the same row tile; for odd g every other pair spans two adjacent row tiles
// (the lighter tile then masks the heavier one's extra diagonal key tiles).  Item w -> pair w / hk
// of KV head w % hk, so the heaviest pairs of all heads come first.
__device__ __forceinline__ Item decode_item(const AttnParams& p, int w) {
  Item it;
  int nrt;
  if (w < p.n_local_items) {
    it.seg = 1;
    nrt = p.nB_rt;
  } else {
    w -= p.n_local_items;
    it.seg = 0;
    nrt = p.nA_rt;
  }
  const int units = nrt * p.g;
#ifdef APB_HEAD_MINOR
  it.j = w % p.hk;
  const int pidx = w / p.hk;
#else
  // KV-head-major order (heaviest row tiles first within a head): the CTAs resident at any
  // time share one or two KV heads, so the K/V tiles they walk stay L2-resident instead of
  // every head's K/V (> L2 at 128K) streaming from HBM once per item
  const int per_head = (units + 1) / 2;
  it.j = w / per_head;
  const int pidx = w % per_head;
#endif
  it.ntiles = 0;
  for (int t = 0; t < 2; ++t) {
    const int u = 2 * pidx + t;
    const int uu = u < units ? u : units - 1;
    it.rtt[t] = nrt - 1 - uu / p.g;
    it.qht[t] = it.j * p.g + uu % p.g;
    if (u < units) it.ntiles = t + 1;
  }
  it.rt = it.rtt[0];
  // key tiles reachable from query rows [128 rt, 128 rt + 128)
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

// PAIR (cluster of 2 CTAs, D = 128): the two CTAs of a cluster hold consecutive work items of the
// same KV head j and segment.  The key-tile walk depends only on (segment, phase, tile index), so
// the lighter item's walk is a prefix of the heavier one's (equal when g % 4 == 0; one diagonal
// tile shorter for odd g).  Over the shared prefix each CTA loads one 64-column half of every K/V
// tile and multicasts it to both, so the tile crosses L2 -> SM once per pair; a ring slot is
// refilled only after both CTAs' MMAs released it (empty barriers count 2, released by multicast
// commits).  Tiles past the prefix are loaded whole by the CTA that needs them and released by two
// local commits.  A pair runs one item each (no work stealing).
//
// Persistent (single CTA, one per SM): a CTA starts on item blockIdx.x, and when its TMA warp has
// issued the last load of an item it takes the next item from the launch's work counter
// (atomicAdd; items in launch order, heaviest first, so the last items go to whichever SMs free up
// first).  Every role reads the item id at the end of its current item, so the next item's
// Q / K / V loads and first S MMAs overlap the current item's last steps and epilogue, and no CTA
// launch, barrier set-up, TMEM allocation or Q-load latency sits between items.
// (A first version took items with clusterlaunchcontrol.try_cancel; both versions hung at first
// because the barrier area was two barriers short, so the 16-byte item buffer overlapped the
// workfree barriers — found with the trace build's wait watchdog, scripts/hang_repro.py.)
// Cross-item hazards: the Q tiles are reloaded after the previous item's last S MMA (Qfree), O_t
// is overwritten by the next item's first PV_t only after the softmax warps have read it (Ofree),
// the staging tile of O_t is rewritten only after its previous TMA store has read it.
template <int D, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    apb_attention_kernel(const __grid_constant__ AttnLaunch La) {
  using L = Layout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  constexpr int NR = L::kRing;
  const uint32_t sQ = sbase + L::kQ;
  const uint32_t bar0 = sbase + L::kBar;
  const uint32_t bQ = bar0, bQf = bar0 + 8u;
  auto sR = [&](int slot) { return sbase + L::kR + slot * L::kTile; };
  auto sO = [&](int t) { return sbase + L::kO + t * L::kTile; };
  auto bRf = [&](int slot) { return bar0 + 8u * (2 + slot); };
  auto bRe = [&](int slot) { return bar0 + 8u * (2 + NR + slot); };
  auto bS = [&](int t) { return bar0 + 8u * (2 + 2 * NR + t); };
  auto bP = [&](int t, int half) { return bar0 + 8u * (4 + 2 * NR + 2 * t + half); };
  auto bO = [&](int t) { return bar0 + 8u * (8 + 2 * NR + t); };
  auto bOf = [&](int t) { return bar0 + 8u * (10 + 2 * NR + t); };
  auto bW = [&](int b) { return bar0 + 8u * (12 + 2 * NR + b); };
  auto bWf = [&](int b) { return bar0 + 8u * (14 + 2 * NR + b); };
  auto sW = [&](int b) { return sbase + L::kWork + 16u * b; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtr);
  // readers of every fetched item id: the MMA warp and the 8 softmax warps; a persistent pair
  // fetches once per cluster (the leader CTA's TMA warp) and both CTAs' readers — the peer's TMA
  // warp included — report to the leader's workfree barrier
  constexpr int kWorkReaders = PAIR ? 19 : 9;

  const int warp = static_cast<int>(warp_uniform(threadIdx.x / 32));
  int dbg_k = 0;  // item sequence number of this role (hang records of the trace build)
  (void)dbg_k;
  CTA_TIME(0);

  if (threadIdx.x == 0) {
    mbar_init(bQ, 1);
    mbar_init(bQf, 1);
    for (int r = 0; r < NR; ++r) {
      mbar_init(bRf(r), 1);
      mbar_init(bRe(r), PAIR ? 2 : 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(bS(t), 1);
      mbar_init(bP(t, 0), BM);
      mbar_init(bP(t, 1), BM);
      mbar_init(bO(t), 1);
      mbar_init(bOf(t), BM);
      mbar_init(bW(t), 1);
      mbar_init(bWf(t), kWorkReaders);
    }
    fence_mbar_init();
  }
  if (warp == kLoadWarp) {
    tmem_alloc<512>(smem_u32(tmem_ptr));
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // the peer's barriers are initialised before any multicast
  tc_fence_after();
  // TMEM base broadcast from lane 0: provably warp-uniform, so every TMEM address and UMMA
  // operand below lives in uniform registers (no per-instruction waterfall loops).
  const uint32_t tmem = warp_uniform(*tmem_ptr);

  // ---- the work list: item k of this CTA is launch item `gid`; host hh, item w within the host
  struct Work {
    int hh, w;
    const AttnParams* p;
    Item it;
    int n_shared;
  };
  auto resolve = [&](int gid) {
    Work c;
    int hh = 0;
    while (hh + 1 < La.n && gid >= La.item_begin[hh + 1]) ++hh;
    c.hh = hh;
    c.w = gid - La.item_begin[hh];
    c.p = &La.p[hh];
    c.it = decode_item(*c.p, c.w);
    // K/V tiles shared with the partner CTA (PAIR): the common prefix of the two walks
    c.n_shared = PAIR ? min(c.it.nkv, decode_item(*c.p, c.w ^ 1).nkv) : 0;  // item_begin[] even
    return c;
  };
  // next item: wait for the k-th fetched item id (buffer k & 1), read it, -1 if none
  auto next_gid = [&](int k, bool reader) -> int {
    const int b = k & 1;
    if constexpr (PAIR) {
      // the leader stored the pair id into both CTAs and released it at cluster scope
      mbar_wait_acq_cluster(bW(b), (k >> 1) & 1);
    } else {
      MBWS(bW(b), (k >> 1) & 1);
    }
    const int x = *reinterpret_cast<volatile int*>(smem + L::kWork + 16 * b);
    __syncwarp();
    if (reader && (threadIdx.x & 31) == 0) {
      if constexpr (PAIR)
        mbar_arrive_cluster(mapa_shared(bWf(b), 0));
      else
        mbar_arrive(bWf(b));
    }
    if constexpr (PAIR) return x < 0 ? -1 : 2 * x + static_cast<int>(cluster_ctarank());
    return x;
  };

  // Register split: the softmax warpgroups hold a 128-wide S row per thread; the producer / MMA
  // warpgroup needs few registers.  (per SMSP: 2 x 200 + 1 x 104 regs x 32 lanes <= 16384)
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;" ::: "memory");
    if (warp == kLoadWarp) {
      // ============================================================== TMA producer (warp-converged)
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      int n0 = 0;  // ring sequence number of this item's first load
      int gid = static_cast<int>(blockIdx.x);
      for (int k = 0;; ++k) {
        dbg_k = k;
        const Work c = resolve(gid);
        const Item& it = c.it;
        const AttnParams& p = *c.p;
        const CUtensorMap* tm_q = &La.tq[c.hh];
        const CUtensorMap* tm_k = &La.tk[c.hh];
        const CUtensorMap* tm_v = &La.tv[c.hh];
        const CUtensorMap* tm_g = &La.tg;
        if (k == 0 && elect_one()) {
          tma_prefetch_desc(tm_q);
          tma_prefetch_desc(tm_k);
          tma_prefetch_desc(tm_v);
          tma_prefetch_desc(tm_g);
        }
        const int qbase = it.seg == 0 ? 0 : p.L_A;
        if (k > 0) MBWS(bQf, (k - 1) & 1);  // the previous item's last S MMA read Q
        if (elect_one()) {
          mbar_arrive_expect_tx(bQ, it.ntiles * L::kTile);
          for (int t = 0; t < it.ntiles; ++t)
            for (int h = 0; h < L::kHalves; ++h)
              tma_load_3d_hint(sQ + t * L::kTile + h * L::kSub, tm_q, bQ, h * 64, it.qht[t], qbase + it.rtt[t] * BM,
                               pol_q);
        }
        __syncwarp();
        for (int i = 0; i < it.nkv; ++i) {
          const KvTile kt = kv_tile(p, it, i);
          const int row0 = (kt.kind == 2 ? p.L_A : 0) + kt.c * BN;
#pragma unroll
          for (int kv = 0; kv < 2; ++kv) {
            const int n = n0 + 2 * i + kv, r = n % NR;
            MBWS(bRe(r), ((n / NR) & 1) ^ 1);
            if (elect_one()) {
              if (PAIR && i < c.n_shared) {
                // this CTA's half of the tile, into the same slot of both CTAs of the pair
                const int h = static_cast<int>(cluster_ctarank());
                mbar_arrive_expect_tx(bRf(r), L::kTile);
                if (kt.kind == 1)
                  tma_load_4d_mc_hint(sR(r) + h * L::kSub, tm_g, bRf(r), h * 64, kt.c * BN, it.j, kt.slot * 2 + kv, 0x3,
                                      pol_kv);
                else
                  tma_load_3d_mc_hint(sR(r) + h * L::kSub, kv ? tm_v : tm_k, bRf(r), h * 64, it.j, row0, 0x3, pol_kv);
              } else {
                mbar_arrive_expect_tx(bRf(r), L::kTile);
                for (int h = 0; h < L::kHalves; ++h) {
                  if (kt.kind == 1)
                    tma_load_4d_hint(sR(r) + h * L::kSub, tm_g, bRf(r), h * 64, kt.c * BN, it.j, kt.slot * 2 + kv,
                                     pol_kv);
                  else
                    tma_load_3d_hint(sR(r) + h * L::kSub, kv ? tm_v : tm_k, bRf(r), h * 64, it.j, row0, pol_kv);
                }
              }
            }
            __syncwarp();
          }
        }
        n0 += 2 * it.nkv;
        if (!La.persist) break;  // one item per CTA (per cluster)
        // every load of this item is issued: fetch the next item (buffer k & 1, free once the
        // readers of fetch k - 2 have read it); the CTA that finds the list empty last resets the
        // launch's counter slot.  A pair fetches a pair index once, in the leader, and stores it
        // into both CTAs.
        if (!PAIR || cluster_ctarank() == 0) {
          if constexpr (PAIR)
            mbar_wait_acq_cluster(bWf(k & 1), ((k >> 1) & 1) ^ 1);
          else
            MBWS(bWf(k & 1), ((k >> 1) & 1) ^ 1);
          if (elect_one()) {
            unsigned int* ctr = g_attn_ctr[La.ctr_slot];
            const int units = PAIR ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
            const int total = PAIR ? La.item_begin[La.n] / 2 : La.item_begin[La.n];
            const int nxt = static_cast<int>(atomicAdd(ctr, 1u)) + units;
            const int id = nxt < total ? nxt : -1;
            const uint32_t slot = sbase + L::kWork + 16u * (k & 1);
            *reinterpret_cast<volatile int*>(smem + L::kWork + 16 * (k & 1)) = id;
            if (nxt >= total && atomicAdd(ctr + 1, 1u) + 1u == static_cast<unsigned int>(units)) {
              ctr[0] = 0u;  // every CTA (cluster) has taken its last id: the slot is free for a later launch
              ctr[1] = 0u;
              __threadfence();
            }
            if constexpr (PAIR) {
              asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa_shared(slot, 1)), "r"(id) : "memory");
              mbar_arrive_cluster(mapa_shared(bW(k & 1), 1));  // release at cluster scope
              mbar_arrive_cluster(bW(k & 1));
            } else {
              mbar_arrive(bW(k & 1));  // release: the id is visible to the readers' acquire
            }
          }
          __syncwarp();
        }
        gid = next_gid(k, PAIR && cluster_ctarank() == 1);  // the peer's TMA warp is a reader
        if (gid < 0) break;
        {
          // the next item's Q tiles into L2 now: they are loaded into shared memory only once
          // this item's last S MMAs have read the current Q (Qfree), and then hit L2
          const Work nc = resolve(gid);
          const int nqb = nc.it.seg == 0 ? 0 : nc.p->L_A;
          if (elect_one())
            for (int t = 0; t < nc.it.ntiles; ++t)
              for (int h = 0; h < L::kHalves; ++h)
                tma_prefetch_3d(&La.tq[nc.hh], h * 64, nc.it.qht[t], nqb + nc.it.rtt[t] * BM);
          __syncwarp();
        }
      }
      if constexpr (PAIR) {
        // drain: every release of this CTA's slots (by both MMA warps) has landed before exit
        const int ntot = n0;
        for (int r = 0; r < NR && r < ntot; ++r) {
          const int n_last = r + ((ntot - 1 - r) / NR) * NR;
          MBWS(bRe(r), (n_last / NR) & 1);
        }
      }
    } else if (warp == kMmaWarp) {
      // ============================================================== MMA issuer (warp-converged,
      // one elected lane issues every tcgen05.mma / tcgen05.commit)
      constexpr uint32_t idS = idesc_bf16_f32(BM, BN, false, false);  // S = Q K^T: both K-major
      constexpr uint32_t idPV = idesc_bf16_f32(BM, D, false, true);   // O += P V: V is MN-major
      auto issue_S = [&](int t, int s) {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k / 4) * L::kSub + (k % 4) * 32;
            mma_ss(tmem + t * 128, sdesc_sw128(sQ + t * L::kTile + off, 16, 1024),
                   sdesc_sw128(sR(s) + off, 16, 1024), idS, k > 0);
          }
          mma_commit(bS(t));
        }
        __syncwarp();
      };
      auto commit = [&](uint32_t bar) {
        if (elect_one()) mma_commit(bar);
        __syncwarp();
      };
      int n0 = 0, gid = static_cast<int>(blockIdx.x);
      int pseq[2] = {0, 0};  // P_t steps so far (bP(t, *) phases)
      int oseq[2] = {0, 0};  // items tile t took part in so far (bO(t) / bOf(t) phases)
      for (int k = 0;; ++k) {
        dbg_k = k;
        const Work c = resolve(gid);
        const Item& it = c.it;
        const AttnParams& p = *c.p;
        // release of a ring slot: in PAIR mode on both CTAs' empty barriers
        // (tile i of the walk; past the shared prefix both arrivals are local)
        auto release = [&](int slot, int i) {
          if (elect_one()) {
            if (PAIR && i < c.n_shared) {
              mma_commit_mc(bRe(slot), 0x3);
            } else {
              mma_commit(bRe(slot));
              if (PAIR) mma_commit(bRe(slot));
            }
          }
          __syncwarp();
        };
        // O_t += P_t V in two K halves: keys [0,64) as soon as the softmax publishes the first half
        // of P_t, keys [64,128) after the second half.  The first PV_t of an item overwrites O_t:
        // the softmax warps must have read the previous item's O_t (Ofree).
        auto issue_PV = [&](int t, int s, bool acc, int step) {
          if (step == 0 && oseq[t] > 0) MBWS(bOf(t), (oseq[t] - 1) & 1);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            MBWS(bP(t, half), (pseq[t] + step) & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kk = half * (BN / 32); kk < (half + 1) * (BN / 32); ++kk) {
                mma_ts(tmem + 256 + t * D, tmem + t * 128 + kk * 8, sdesc_sw128(sR(s) + kk * 2048, L::kSub, 1024), idPV,
                       (acc || kk > 0) ? 1u : 0u);
              }
            }
            __syncwarp();
          }
        };
        const bool carry = (p.phase == APB_PHASE_PASSING);
        MBWS(bQ, k & 1);
        tc_fence_after();
        for (int i = 0; i < it.nkv; ++i) {
          const int nK = n0 + 2 * i, nV = nK + 1, nK1 = nK + 2;  // ring sequence numbers
          if (i == 0) {
            MBWS(bRf(nK % NR), (nK / NR) & 1);
            tc_fence_after();
            if (elect_one()) CTA_STAMP(3);
            __syncwarp();
            for (int t = 0; t < it.ntiles; ++t) {
              TRACE(t, 0);
              issue_S(t, nK % NR);
            }
            release(nK % NR, 0);
            if (it.nkv == 1) commit(bQf);  // the item's last S MMAs are issued: Q may be reloaded
          }
          MBWS(bRf(nV % NR), (nV / NR) & 1);
          TRACE(12, i);
          tc_fence_after();
          for (int t = 0; t < it.ntiles; ++t) {
            issue_PV(t, nV % NR, carry || i > 0, i);
            if (t == it.ntiles - 1) release(nV % NR, i);
            if (i + 1 < it.nkv) {
              if (t == 0) {
                MBWS(bRf(nK1 % NR), (nK1 / NR) & 1);
                TRACE(13, i + 1);
                tc_fence_after();
              }
              TRACE(t, i + 1);
              issue_S(t, nK1 % NR);
              if (t == it.ntiles - 1) {
                release(nK1 % NR, i + 1);
                if (i + 2 == it.nkv) commit(bQf);  // the item's last S MMAs are issued
              }
            } else {
              commit(bO(t));
            }
          }
        }
        for (int t = 0; t < it.ntiles; ++t) {
          pseq[t] += it.nkv;
          ++oseq[t];
        }
        n0 += 2 * it.nkv;
        if (!La.persist) break;
        gid = next_gid(k, true);
        if (gid < 0) break;
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;" ::: "memory");
    // ================================================================ softmax warpgroups
    const int t = warp / 4;
    const int tid = threadIdx.x % 128;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + 256 + t * D;
    int sseq = 0;  // S_t steps so far (bS(t) phases)
    int oseq = 0;  // items this tile took part in (bO(t) phases)
    int gid = static_cast<int>(blockIdx.x);
    for (int k = 0;; ++k) {
      dbg_k = k;
      const Work c = resolve(gid);
      const Item& it = c.it;
      const AttnParams& p = *c.p;
      if (t < it.ntiles) {
        const int qh = it.qht[t];
        const int row = it.rtt[t] * BM + tid;  // row index inside the query segment
        const bool row_valid = it.seg == 0 ? row < p.L_A : row < p.l_b;
        const float sl2 = p.scale_log2;
        float m_run = -INFINITY, l_run = 0.f;
        bool o_valid = false;

        if (p.phase == APB_PHASE_PASSING) {
          // LSE carry-in: the LOCAL phase's normalised partial (O, m + log2 l) becomes the
          // initial online-softmax state (m = lse2, l = 1, O = O_partial) — an exact merge.
          // (O_t of this tile's previous item was read by these threads' epilogue.)
          const float* src = p.ws_o + ((int64_t)(row_valid ? row : 0) * p.hq + qh) * D;
          m_run = row_valid ? p.ws_lse[(int64_t)qh * p.l_b + row] : 0.f;
          l_run = 1.f;
#pragma unroll
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t r[32];
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              float4 f = row_valid ? *reinterpret_cast<const float4*>(src + cc * 32 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
              r[e] = __float_as_uint(f.x);
              r[e + 1] = __float_as_uint(f.y);
              r[e + 2] = __float_as_uint(f.z);
              r[e + 3] = __float_as_uint(f.w);
            }
            tmem_st32(tO + cc * 32, r);
          }
          tmem_wait_st();
          o_valid = true;
        }

        for (int i = 0; i < it.nkv; ++i) {
          const KvTile kt = kv_tile(p, it, i);
          const int nv = visible_cols(p, it, kt, row);
          MBW(bS(t), (sseq + i) & 1);
          if (tid == 0) TRACE(6 + t, i);
          tc_fence_after();
          uint32_t sr[128];
          tmem_ld32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
          tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
          tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
          tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
          tmem_wait_ld();
          float* s = reinterpret_cast<float*>(sr);
          if (tid == 0) TRACE(16 + t * 4, i);
          if (nv < BN) {
#pragma unroll
            for (int cc = 0; cc < BN; ++cc)
              if (cc >= nv) s[cc] = -INFINITY;
          }
          // 2^(s*scale*log2e - m) for the 64 columns of one half; packed FFMA2 for the argument;
          // the kPolyMask pairs of every 16 on the FMA pipe (Cody-Waite + degree-3 polynomial,
          // rel. error 7.5e-5 << bf16's 3.9e-3), the rest on MUFU.EX2.
          auto exp_half = [&](int half, float m_use, uint32_t (&pk)[32], uint64_t (&acc2)[4]) {
            const uint64_t sc2 = f2_pack(sl2, sl2), nm2 = f2_pack(-m_use, -m_use);
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
              const int col = half * 64 + 2 * cc;
              const uint64_t x2 = ffma2(f2_pack(s[col], s[col + 1]), sc2, nm2);
              float p0, p1;
              if ((((half == 0) ? kPolyMask : kPolyMask1) >> (cc % 16)) & 1u) {
                const uint64_t p2 = exp2_poly2(x2);
                f2_unpack(p2, p0, p1);
              } else {
                float x0, x1;
                f2_unpack(x2, x0, x1);
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              pk[cc] = pack_bf16x2(p0, p1);
              // the row sum adds the bf16 weights the PV MMA actually uses, so the normalisation
              // matches them (with the lazy rescale the row max's weight is 2^delta, not 1, and
              // bf16-rounding it alone would bias O by up to 2^-9 relative; reading G21)
              acc2[cc & 3] = f2_add_bf16x2(acc2[cc & 3], pk[cc]);
            }
          };
          // Speculation: the running max m_run only moves when a row max grows by more than the
          // threshold, so the first half's exponentials are computed against m_run on the
          // MUFU/FMA pipes while the ALU pipe reduces the new row max; the (rare) rows whose max
          // grew redo the half with the new max.
          uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
          uint32_t pk[32];
          const bool have_m = (m_run != -INFINITY);
          const float m_spec = have_m ? m_run : 0.f;
          exp_half(0, m_spec, pk, acc2);
          float mx8[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) mx8[q] = fmax3(s[2 * q], s[2 * q + 1], s[16 + 2 * q]);
#pragma unroll
          for (int cc = 32; cc < BN; cc += 16) {
#pragma unroll
            for (int q = 0; q < 8; ++q) mx8[q] = fmax3(mx8[q], s[cc + 2 * q], s[cc + 2 * q + 1]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], s[16 + 2 * q + 1]);
          const float mx = sl2 * fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
          const bool grow = !have_m || (mx > m_run + kRescaleThreshold);
          float alpha = 1.f;
          if (tid == 0) TRACE(17 + t * 4, i);
          if (__any_sync(0xffffffffu, grow)) {
            if (grow) {
              const float m_new = fmaxf(m_run, mx);
              alpha = have_m ? ex2(m_run - m_new) : 0.f;
              m_run = m_new;
              const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
              acc2[0] = acc2[1] = acc2[2] = acc2[3] = 0ull;
              exp_half(0, m_use, pk, acc2);
            }
            // rescale the running O_t before any PV_t(i) MMA (PV_t(i-1) is complete: S_t(i) was
            // issued after it)
            if (__any_sync(0xffffffffu, grow && o_valid && alpha != 1.f)) {
              const float a = (grow && o_valid) ? alpha : 1.f;
#pragma unroll
              for (int cc = 0; cc < D / 16; ++cc) {
                uint32_t r[16];
                tmem_ld16(tO + cc * 16, r);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * a);
                tmem_st16(tO + cc * 16, r);
              }
            }
          }
          const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
          if (tid == 0) TRACE(18 + t * 4, i);
          tmem_st32(tS, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bP(t, 0));
          if (tid == 0) TRACE(8 + 2 * t, i);
          exp_half(1, m_use, pk, acc2);
          tmem_st32(tS + 32, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bP(t, 1));
          if (tid == 0) TRACE(9 + 2 * t, i);
          if ((tid & 31) == 0) TRACE(24 + t * 4 + (tid >> 5), i);
          float r0, r1, r2, r3;
          f2_unpack(fadd2(acc2[0], acc2[1]), r0, r1);
          f2_unpack(fadd2(acc2[2], acc2[3]), r2, r3);
          l_run = l_run * alpha + ((r0 + r1) + (r2 + r3));
          o_valid = true;
        }
        sseq += it.nkv;

        // ============================================================== epilogue
        MBW(bO(t), oseq & 1);
        ++oseq;
        tc_fence_after();
        if (tid == 0 && t == 0) CTA_STAMP(4);
        const float inv_l = 1.f / l_run;
        const bool to_ws = (it.seg == 1) && p.local_to_ws;
        const int64_t grow_idx = (it.seg == 0 ? 0 : p.L_A) + row;  // row of q/out on this host
        uint32_t o[D];
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tmem_ld32(tO + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[cc * 32]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(bOf(t));  // O_t is in registers: the next item's first PV_t may overwrite it
        if (!to_ws) {
          // bf16 O tile -> shared memory (SW128, the Q tile layout) -> TMA store(s) by one thread.
          // Rows past the segment's end are clipped by the output map (anchor and block rows are
          // separate maps).  The staging tile is rewritten only after its previous store read it.
          const uint32_t stg = sO(t);
          if (tid == 0) bulk_wait_group_read<0>();
          named_bar_sync(3 + t, 128);
#pragma unroll
          for (int cc = 0; cc < D / 32; ++cc) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int e = cc * 32 + q4 * 8, chunk = (cc & 1) * 4 + q4;
              const uint32_t a = stg + (cc >> 1) * L::kSub + tid * 128 + ((chunk ^ (tid & 7)) << 4);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                           "r"(pack_bf16x2(__uint_as_float(o[e]) * inv_l, __uint_as_float(o[e + 1]) * inv_l)),
                           "r"(pack_bf16x2(__uint_as_float(o[e + 2]) * inv_l, __uint_as_float(o[e + 3]) * inv_l)),
                           "r"(pack_bf16x2(__uint_as_float(o[e + 4]) * inv_l, __uint_as_float(o[e + 5]) * inv_l)),
                           "r"(pack_bf16x2(__uint_as_float(o[e + 6]) * inv_l, __uint_as_float(o[e + 7]) * inv_l))
                           : "memory");
            }
          }
          fence_proxy_async_smem();  // the generic-proxy writes are visible to the TMA engine
          named_bar_sync(3 + t, 128);
          if (tid == 0) {
            const CUtensorMap* to = it.seg == 0 ? &La.to_a[c.hh] : &La.to_b[c.hh];
#pragma unroll
            for (int h = 0; h < L::kHalves; ++h) tma_store_3d(to, stg + h * L::kSub, h * 64, qh, it.rtt[t] * BM);
            bulk_commit_group();
          }
        } else if (row_valid) {
          float* dst = p.ws_o + ((int64_t)row * p.hq + qh) * D;
#pragma unroll
          for (int e = 0; e < D; e += 4)
            *reinterpret_cast<float4*>(dst + e) =
                make_float4(__uint_as_float(o[e]) * inv_l, __uint_as_float(o[e + 1]) * inv_l,
                            __uint_as_float(o[e + 2]) * inv_l, __uint_as_float(o[e + 3]) * inv_l);
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
      if (!La.persist) break;
      gid = next_gid(k, true);
      if (gid < 0) break;
    }
    if (tid == 0) bulk_wait_group_read<0>();  // the last TMA store has read its staging tile
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // neither CTA exits while the peer may still write to it
  CTA_TIME(1);
  if (warp == kLoadWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Launch policy.  Default: the persistent single-CTA kernel for every phase (one CTA per SM taking
// items from the launch's work counter, so no launch / set-up / Q-load gap sits between items):
// L8 bench 113.1 K tokens/s (e2e 110.7 K) vs 111.1 K for round 2's one-item-per-cluster paired
// kernel, 32K 383 K vs 364 K, Qwen-14B 60.1 K vs 59.1 K (scripts/gpu/r2s2_persist2.sh).
// APB_ATTN_PERSIST=0: one item per CTA everywhere, =1: persistent LOCAL too; APB_ATTN_PAIR=1: the paired 2-CTA kernel (multicast K/V,
// ~50 W less, one item per cluster) for every phase where it applies; APB_ATTN_PAIR=all: paired
// for PHASE_ALL only (round 2's default).
// The LOCAL launch of the split schedule (N > 1) stays one item per CTA by default: it overlaps
// the side stream's scoring / selection / exchange, whose kernels get SMs as LOCAL's CTAs retire
// (persistent CTAs would hold every SM until LOCAL ends and serialise the compression behind it).
static bool persist_enabled(int phase) {
  const char* pe = std::getenv("APB_ATTN_PERSIST");
  if (pe && pe[0] == '0') return false;
  if (pe && pe[0] == '1') return true;
  return phase != APB_PHASE_LOCAL;
}
static bool pair_enabled(int phase) {
  const char* e = std::getenv("APB_ATTN_PAIR");
  if (e && e[0] == '1') return true;
  if (e && e[0] == 'a') return phase == APB_PHASE_ALL;
  return false;
}

template <int D, bool PAIR>
static apb_status launch_impl(const AttnLaunch& La_in, int phase, cudaStream_t stream) {
  using L = Layout<D>;
  const int items = La_in.item_begin[La_in.n];
  if (items == 0) return APB_OK;
  AttnLaunch La = La_in;
  int grid = items;  // not persistent: one item per CTA
  La.persist = 0;
  // a persistent pair needs equal partner walks for every item pair (its two rings advance
  // together): g % 4 == 0, where both items of a pair cover the same row tile
  bool equal_walks = true;
  for (int i = 0; i < La.n; ++i) equal_walks = equal_walks && La.p[i].g % 4 == 0;
  if (persist_enabled(phase) && (!PAIR || equal_walks)) {
    La.persist = 1;
    La.ctr_slot = static_cast<int>(g_launches.fetch_add(1) % kCtrSlots);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = items < sms ? items : sms;  // persistent: one CTA per SM, the rest from the counter
    if (PAIR) grid &= ~1;              // whole clusters (items is even for a paired launch)
  }
  static std::atomic<uint64_t> smem_set{0};
  if (apb_status st = set_max_smem_once(reinterpret_cast<const void*>(apb_attention_kernel<D, PAIR>), L::kAlloc, smem_set))
    return st;
  cudaError_t e;
  if constexpr (PAIR) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L::kAlloc;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, apb_attention_kernel<D, PAIR>, La);
  } else {
    apb_attention_kernel<D, PAIR><<<grid, kThreads, L::kAlloc, stream>>>(La);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace attn

#ifdef APB_TRACE
extern "C" int apb_debug_trace(unsigned long long* out, int n, int block) {
  if (block >= 0) {
    return cudaMemcpyToSymbol(attn::g_trace_block, &block, sizeof(int)) == cudaSuccess ? 0 : 1;
  }
  return cudaMemcpyFromSymbol(out, attn::g_trace, sizeof(unsigned long long) * (n < 2048 ? n : 2048)) == cudaSuccess ? 0 : 1;
}
// Mapped host buffer for the hang watchdog records ([grid][12][4] uint32), 0 = nothing recorded.
extern "C" int apb_debug_hang_buffer(unsigned int** host_ptr, int n_words) {
  unsigned int* h = nullptr;
  if (cudaHostAlloc(&h, sizeof(unsigned int) * n_words, cudaHostAllocMapped) != cudaSuccess) return 1;
  memset(h, 0, sizeof(unsigned int) * n_words);
  unsigned int* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return 2;
  if (cudaMemcpyToSymbol(attn::g_hang, &d, sizeof(d)) != cudaSuccess) return 3;
  *host_ptr = h;
  return 0;
}
extern "C" int apb_debug_cta_times(unsigned long long* out, int n_ctas) {
  const int n = 5 * (n_ctas < 65536 ? n_ctas : 65536);
  return cudaMemcpyFromSymbol(out, attn::g_cta_time, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif

apb_status launch_attention_hosts(int D, const AttnLaunch& La, int phase, cudaStream_t stream) {
  static_assert(sizeof(AttnLaunch) <= 32764, "kernel parameter space");
  if (La.n < 1 || La.n > kAttnMaxHosts) return fail(APB_ERR_CONFIG, "1..8 hosts per attention launch");
#ifndef APB_PSMEM
  // clusters pair items 2c and 2c+1: both must belong to the same host and (segment, KV head), i.e.
  // every host's segments hold an even number of items per KV head (decode_item: per_head =
  // ceil(units / 2)) — then every host's item range starts at an even index
  bool even_heads = true;
  for (int i = 0; i < La.n; ++i) {
    const AttnParams& p = La.p[i];
    even_heads = even_heads && (p.n_local_items / p.hk) % 2 == 0 && (p.n_anchor_items / p.hk) % 2 == 0;
  }
  if (D == 128 && even_heads && attn::pair_enabled(phase))
    return attn::launch_impl<128, true>(La, phase, stream);
#endif
  if (D == 128) return attn::launch_impl<128, false>(La, phase, stream);
  if (D == 64) return attn::launch_impl<64, false>(La, phase, stream);
  return fail(APB_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
}

}  // namespace apb
