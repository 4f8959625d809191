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
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

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

// ---------------------------------------------------------------- fast select + PDL gather
// select_fast_kernel: one 1024-thread CTA per KV head.  The l_b order-preserving keys are staged
// in shared memory once (else re-read from L2 when they do not fit), then 4 radix passes of 8-bit
// digits run on the CTA's histogram: warp-aggregated (match.any: the first digit holds the sign +
// exponent, so most keys share a handful of bins and plain shared atomics would serialise on
// them), and the 256-bin suffix scan is parallel (8 warps of shuffles), not one thread's loop.
// The ordered compaction is warp-local: warp w owns a contiguous index range, counts its
// (> T, == T) keys, one block scan of the 32 warp counts gives every warp its output offset and
// tie rank, and each warp writes its ascending indices with ballots — one block barrier instead of
// two block scans per 1024 elements.  It then triggers the dependent launch.
// gather_kernel (programmatic dependent launch, many CTAs): copies the selected K/V rows into the
// send slot, 8 x 16-byte loads in flight per thread.  Both are bit-exact integer logic.
namespace sel {
constexpr int kFT = 1024;                 // threads of the select CTA
constexpr int kMaxSmemKeys = 40 * 1024;   // 160 KB of staged keys; beyond that keys come from L2
constexpr int kCand = 8192;               // candidate keys kept after the first digit (32 KB)

// Suffix search over `nb` histogram bins (nb = 1024 or 2048; thread t holds bins [t*bpt, t*bpt+bpt)):
// the bin b with above(b) < kk <= above(b) + hist[b], above(b) = count in bins > b.
__device__ __forceinline__ void find_bin(const uint32_t* hist, int nb, uint32_t kk, uint32_t* wtot,
                                         uint32_t* sh_bin, uint32_t* sh_k) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bpt = nb / kFT;  // 1 or 2
  uint32_t c[2] = {hist[tid * bpt], bpt > 1 ? hist[tid * bpt + 1] : 0u};
  const uint32_t mine = c[0] + c[1];
  uint32_t incl = mine;  // suffix within the warp (lanes >= lane)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, incl, o);
    if (lane + o < 32) incl += y;
  }
  if (lane == 0) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {  // suffix over the 32 warp totals, exclusive
    const uint32_t wt = wtot[lane];
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, wi, o);
      if (lane + o < 32) wi += y;
    }
    wtot[32 + lane] = wi - wt;
  }
  __syncthreads();
  uint32_t above = incl - mine + wtot[32 + warp];  // keys in bins above this thread's bins
  for (int q = bpt - 1; q >= 0; --q) {
    if (above < kk && above + c[q] >= kk) {
      *sh_bin = (uint32_t)(tid * bpt + q);
      *sh_k = kk - above;
    }
    above += c[q];
  }
  __syncthreads();
}

template <bool kSmemKeys>
__global__ void __launch_bounds__(kFT) select_fast_kernel(const float* __restrict__ scores, int l_b, int lp,
                                                          int32_t* __restrict__ indices) {
  extern __shared__ uint32_t dyn[];
  uint32_t* skeys = dyn;                      // [l_b] (kSmemKeys)
  uint32_t* cand = dyn + (kSmemKeys ? l_b : 0);  // [kCand]
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t wtot[64];
  __shared__ uint32_t sh_bin, sh_k, n_cand;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = blockIdx.x;
  const float* s = scores + (int64_t)j * l_b;
  auto key_at = [&](int i) -> uint32_t {
    if constexpr (kSmemKeys) return skeys[i];
    else return order_key(__ldg(s + i));
  };
  for (int b = tid; b < 2048; b += kFT) hist[b] = 0;
  if (tid == 0) n_cand = 0;
  __syncthreads();
  // ---- stage the keys: loads only, so the compiler keeps many in flight (one HBM latency, not
  // one per iteration as when each load is followed by a shared atomic)
  if constexpr (kSmemKeys) {
#pragma unroll 8
    for (int i = tid; i < l_b; i += kFT) skeys[i] = order_key(__ldg(s + i));
    __syncthreads();
  }
  // ---- digit 1 (key bits 31..21, 2048 bins)
  for (int i = tid; i < l_b; i += kFT) atomicAdd(&hist[key_at(i) >> 21], 1u);
  __syncthreads();
  find_bin(hist, 2048, (uint32_t)lp, wtot, &sh_bin, &sh_k);
  uint32_t prefix = sh_bin << 21, kk = sh_k;
  // ---- candidates: the keys in that bin (unordered; selection only needs their values)
  for (int b = tid; b < 2048; b += kFT) hist[b] = 0;
  for (int base = 0; base < l_b; base += kFT) {
    const int i = base + tid;
    const bool m = i < l_b && (key_at(i) >> 21) == (prefix >> 21);
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
    uint32_t off = 0;
    if (lane == 0 && bal) off = atomicAdd(&n_cand, (uint32_t)__popc(bal));
    off = __shfl_sync(0xFFFFFFFFu, off, 0);
    const uint32_t slot = off + __popc(bal & ((1u << lane) - 1u));
    if (m && slot < (uint32_t)kCand) cand[slot] = key_at(i);
  }
  __syncthreads();
  const uint32_t nc = n_cand;
  const bool use_cand = nc <= (uint32_t)kCand;
  const int n2 = use_cand ? (int)nc : l_b;
  // ---- digit 2 (bits 20..10, 2048 bins) and digit 3 (bits 9..0, 1024 bins) over the candidates
  for (int pass = 0; pass < 2; ++pass) {
    const int shift = pass == 0 ? 10 : 0;
    const uint32_t pmask = pass == 0 ? 0xFFE00000u : 0xFFFFFC00u;
    const uint32_t dmask = pass == 0 ? 0x7FFu : 0x3FFu;
    if (pass == 1) {
      for (int b = tid; b < 2048; b += kFT) hist[b] = 0;
      __syncthreads();
    }
    for (int i = tid; i < n2; i += kFT) {
      const uint32_t key = use_cand ? cand[i] : key_at(i);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    find_bin(hist, pass == 0 ? 2048 : 1024, kk, wtot, &sh_bin, &sh_k);
    prefix |= sh_bin << shift;
    kk = sh_k;
  }
  const uint32_t T = prefix, need_eq = kk;  // key of the l_p'-th largest score; ties taken

  // ---- warp-local ordered compaction: warp w owns [w*per, (w+1)*per), per a multiple of 32
  __shared__ uint32_t wg[32], we[32];
  const int per = ((l_b + 31) / 32 + 31) / 32 * 32;
  const int w0 = min(l_b, warp * per), w1 = min(l_b, w0 + per);
  uint32_t gt = 0, eq = 0;
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    const uint32_t key = i < w1 ? key_at(i) : 0u;
    gt += __popc(__ballot_sync(0xFFFFFFFFu, i < w1 && key > T));
    eq += __popc(__ballot_sync(0xFFFFFFFFu, i < w1 && key == T));
  }
  if (lane == 0) {
    wg[warp] = gt;
    we[warp] = eq;
  }
  __syncthreads();
  uint32_t g_before = 0, e_before = 0;
  for (int w = 0; w < warp; ++w) {
    g_before += wg[w];
    e_before += we[w];
  }
  // selected before this warp: its > T keys plus the ties of lower warps that are taken
  uint32_t pos = g_before + min(need_eq, e_before);
  uint32_t erank = e_before;
  int32_t* out = indices + (int64_t)j * lp;
  const uint32_t lt = (1u << lane) - 1u;
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    const uint32_t key = i < w1 ? key_at(i) : 0u;
    const bool is_eq = i < w1 && key == T;
    const uint32_t eqb = __ballot_sync(0xFFFFFFFFu, is_eq);
    const bool sel = (i < w1 && key > T) || (is_eq && erank + __popc(eqb & lt) < need_eq);
    const uint32_t selb = __ballot_sync(0xFFFFFFFFu, sel);
    if (sel) out[pos + __popc(selb & lt)] = i;
    pos += __popc(selb);
    erank += __popc(eqb);
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Block exclusive scan of one 32-bit value per thread (1024 threads); returns the prefix.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wtot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wt = wtot[lane];
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    wtot[32 + lane] = wi - wt;
  }
  __syncthreads();
  return incl - v + wtot[32 + warp];
}

// Block exclusive scan of one 32-bit value per thread (NT threads, NT/32 <= 32 warps).
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_n(uint32_t v, uint32_t* wtot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kW = NT / 32;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wt = lane < kW ? wtot[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kW) wtot[32 + lane] = wi - wt;
  }
  __syncthreads();
  const uint32_t r = incl - v + wtot[32 + warp];
  __syncthreads();  // wtot may be reused right after
  return r;
}

// Register variant (l_b <= 1024 * KPT, every paper config): thread t holds the keys of indices
// [t*KPT, (t+1)*KPT) in registers.  Digit 1 (bits 31..21) histograms every key; the keys in the
// chosen bin are then compacted into a shared candidate list (one block scan, no contended
// counter), and digits 2 and 3 (11 + 10 bits) histogram only those.  The ordered compaction is one
// block scan of the per-thread (> T, == T) counts; each thread writes its ascending indices to a
// shared staging buffer, copied out coalesced.
constexpr int kCandReg = 4096;  // candidate list capacity (else digits 2-3 scan the registers)
constexpr int kOutStage = 4096; // staged output indices (else written straight to global)

template <int KPT>
__global__ void __launch_bounds__(kFT) select_reg_kernel(const __grid_constant__ SelHosts sh, int l_b, int lp) {
  const float* __restrict__ scores = sh.scores[blockIdx.y];  // grid.y = host of the launch
  int32_t* __restrict__ indices = sh.indices[blockIdx.y];
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t wtot[64];
  __shared__ uint32_t cand[kCandReg];  // candidate keys; reused as the staged output indices
  __shared__ uint32_t sh_bin, sh_k, sh_nc;
  const int tid = threadIdx.x;
  const int j = blockIdx.x;
  const float* s = scores + (int64_t)j * l_b;
  const int e0 = tid * KPT;
  uint32_t key[KPT];
  if (e0 + KPT <= l_b && (l_b & 3) == 0) {
#pragma unroll
    for (int e = 0; e < KPT; e += 4) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(s + e0 + e));
      key[e] = order_key(f.x);
      key[e + 1] = order_key(f.y);
      key[e + 2] = order_key(f.z);
      key[e + 3] = order_key(f.w);
    }
  } else {
#pragma unroll
    for (int e = 0; e < KPT; ++e) key[e] = e0 + e < l_b ? order_key(__ldg(s + e0 + e)) : 0u;
  }
  const int nmine = max(0, min(KPT, l_b - e0));
  for (int b = tid; b < 2048; b += kFT) hist[b] = 0;
  __syncthreads();
#pragma unroll
  for (int e = 0; e < KPT; ++e)
    if (e < nmine) atomicAdd(&hist[key[e] >> 21], 1u);
  __syncthreads();
  find_bin(hist, 2048, (uint32_t)lp, wtot, &sh_bin, &sh_k);
  uint32_t prefix = sh_bin << 21, kk = sh_k;
  // ---- candidate list: the keys of the chosen digit-1 bin
  uint32_t nm = 0;
#pragma unroll
  for (int e = 0; e < KPT; ++e) nm += (e < nmine && (key[e] >> 21) == sh_bin);
  uint32_t cpos = block_excl_scan(nm, wtot);
  if (tid == kFT - 1) sh_nc = cpos + nm;
  for (int b = tid; b < 2048; b += kFT) hist[b] = 0;
  __syncthreads();
  const uint32_t nc = sh_nc;
  const bool use_cand = nc <= (uint32_t)kCandReg;
  if (use_cand) {
#pragma unroll
    for (int e = 0; e < KPT; ++e)
      if (e < nmine && (key[e] >> 21) == (prefix >> 21)) cand[cpos++] = key[e];
  }
  __syncthreads();
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int shift = pass == 0 ? 10 : 0;
    const uint32_t pmask = pass == 0 ? 0xFFE00000u : 0xFFFFFC00u;
    const uint32_t dmask = pass == 0 ? 0x7FFu : 0x3FFu;
    if (pass == 1) {
      for (int b = tid; b < 1024; b += kFT) hist[b] = 0;
      __syncthreads();
    }
    if (use_cand) {
      for (int i = tid; i < (int)nc; i += kFT) {
        const uint32_t c = cand[i];
        if ((c & pmask) == prefix) atomicAdd(&hist[(c >> shift) & dmask], 1u);
      }
    } else {
#pragma unroll
      for (int e = 0; e < KPT; ++e)
        if (e < nmine && (key[e] & pmask) == prefix) atomicAdd(&hist[(key[e] >> shift) & dmask], 1u);
    }
    __syncthreads();
    find_bin(hist, pass == 0 ? 2048 : 1024, kk, wtot, &sh_bin, &sh_k);
    prefix |= sh_bin << shift;
    kk = sh_k;
  }
  const uint32_t T = prefix, need_eq = kk;  // key of the l_p'-th largest score; ties taken
  // ---- ordered compaction: block exclusive scan of (gt << 16 | eq) (both <= 1024 * KPT < 2^16)
  uint32_t gt = 0, eq = 0;
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    gt += (e < nmine && key[e] > T);
    eq += (e < nmine && key[e] == T);
  }
  const uint32_t before = block_excl_scan((gt << 16) | eq, wtot);
  const uint32_t g_before = before >> 16, e_before = before & 0xFFFFu;
  uint32_t pos = g_before + min(need_eq, e_before);
  uint32_t erank = e_before;
  int32_t* out = indices + (int64_t)j * lp;
  const bool stage = lp <= kOutStage;
  int32_t* dst = stage ? reinterpret_cast<int32_t*>(cand) : out;  // the candidates are no longer read
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    if (e < nmine) {
      bool sel = key[e] > T;
      if (key[e] == T) sel = erank++ < need_eq;
      if (sel) dst[pos++] = e0 + e;
    }
  }
  if (stage) {
    __syncthreads();
    for (int i = tid; i < lp; i += kFT) out[i] = dst[i];
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// send[kv][j][m][:] = (kv ? V : K)[L_A + idx[j][m]][j][:]; grid (ceil(lp / rows_per_cta), hk, 2).
// With a peer push (GatherDst.n > 1 or flags set) every row is stored into the same slot of every
// rank's buffer (CUDA IPC mappings: NVLink / NVSwitch stores) — the AllGather fused into the
// compaction — and the launch's last CTA then publishes `epoch` in every rank's flag word for this
// slot (release at system scope, after every CTA's stores were fenced at system scope).
template <int D>
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ SelHosts sh, int64_t kv_row_stride,
                                                     int lp, int hk, const __grid_constant__ GatherDst dst) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the select grid's indices are visible
  const int host = blockIdx.z >> 1;                   // grid.z = 2 x hosts of the launch
  const int32_t* __restrict__ idx = sh.indices[host];
  const uint16_t* __restrict__ k = sh.k[host];
  const uint16_t* __restrict__ v = sh.v[host];
  const int L_A = sh.L_A[host];
  constexpr int kVec = D / 8;                         // 16-byte vectors per row
  constexpr int kBatch = 8;
  constexpr int kRows = 256 * kBatch / kVec;          // rows per CTA
  const int j = blockIdx.y, kv = blockIdx.z & 1;
  const int r0 = blockIdx.x * kRows;
  const uint16_t* src = (kv ? v : k) + (int64_t)j * D;
  const int64_t off = (((int64_t)kv * hk + j) * lp) * D;  // elements into a slot
  uint4 buf[kBatch];
  int rr[kBatch];
#pragma unroll
  for (int q = 0; q < kBatch; ++q) {
    const int u = q * 256 + threadIdx.x;
    const int r = r0 + u / kVec, c = u % kVec;
    rr[q] = r < lp ? r : -1;
    if (r < lp)
      buf[q] = __ldg(reinterpret_cast<const uint4*>(src + (L_A + (int64_t)__ldg(idx + (int64_t)j * lp + r)) * kv_row_stride) + c);
  }
  // destinations: the push list (one host, peer exchange) or this host's own slot
  const int nd = dst.n > 0 ? dst.n : 1;
  for (int d = 0; d < nd; ++d) {
    uint4* out = reinterpret_cast<uint4*>((dst.n > 0 ? dst.send[d] : sh.send[host]) + off);
#pragma unroll
    for (int q = 0; q < kBatch; ++q)
      if (rr[q] >= 0) out[(int64_t)rr[q] * kVec + (q * 256 + threadIdx.x) % kVec] = buf[q];
  }
  if (dst.flag[0] != nullptr) {
    __threadfence_system();  // this thread's peer stores are visible system-wide
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t n_ctas = gridDim.x * gridDim.y * gridDim.z;
      const uint32_t done = atomicAdd(dst.counter, 1u) + 1u;
      if (done % n_ctas == 0) {  // the last CTA of this launch: every CTA's stores are fenced
        __threadfence_system();
        for (int d = 0; d < dst.n; ++d)
          asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(dst.flag[d]), "r"(dst.epoch) : "memory");
      }
    }
  }
}

// ---------------------------------------------------------------- cluster select + fused gather
// select_cluster_kernel<KPT>: one cluster of kCC = 8 CTAs (512 threads each) per KV head; CTA c of
// the cluster owns the contiguous index range [c*per, (c+1)*per) of the head's l_b scores, KPT
// order-preserving keys per thread in registers.  The three radix digits (bits 31..21, 20..10,
// 9..0) are counted in a private shared histogram per CTA; after one cluster barrier every CTA
// sums the 8 histograms through distributed shared memory (ld.shared::cluster.v4, fixed order, so
// every CTA derives the same bin) and runs the suffix search locally — no CTA waits on another
// beyond the barrier.  The ordered output: per-CTA (> T, == T) totals are exchanged the same way,
// each thread writes its ascending indices at its global position (ties -> lower index, reading
// G5), and after a last cluster barrier (release / acquire at cluster scope: the indices written
// to global by the other CTAs are visible) CTA c copies rows [c*lp/8, (c+1)*lp/8) of the send slot
// — the gather is spread evenly over the cluster whatever the positions of the selected keys.
// One launch replaces select + gather; 8 * hk CTAs share the select's latency-bound phases and the
// 2 * hk * l_p' * d * 2 B copy.
using namespace apb::sm100;
constexpr int kCC = 8;     // CTAs per cluster (one cluster per KV head)
constexpr int kCT = 512;   // threads per CTA

// Suffix search over nb = kCT * BPT bins whose counts thread t holds for bins [t*BPT, t*BPT+BPT).
template <int BPT>
__device__ __forceinline__ void find_bin_regs(const uint32_t (&c)[BPT], uint32_t kk, uint32_t* wtot, uint32_t* sh_bin,
                                              uint32_t* sh_k) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = kCT / 32;
  uint32_t mine = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) mine += c[q];
  uint32_t incl = mine;  // suffix within the warp (lanes >= lane)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, incl, o);
    if (lane + o < 32) incl += y;
  }
  if (lane == 0) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {  // exclusive suffix over the warp totals
    const uint32_t wt = lane < kW ? wtot[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, wi, o);
      if (lane + o < 32) wi += y;
    }
    if (lane < kW) wtot[32 + lane] = wi - wt;
  }
  __syncthreads();
  uint32_t above = incl - mine + wtot[32 + warp];  // keys in bins above this thread's bins
#pragma unroll
  for (int q = BPT - 1; q >= 0; --q) {
    if (above < kk && above + c[q] >= kk) {
      *sh_bin = (uint32_t)(tid * BPT + q);
      *sh_k = kk - above;
    }
    above += c[q];
  }
  __syncthreads();
}

__device__ __forceinline__ uint4 ld_dsmem_v4(uint32_t cluster_addr) {
  uint4 r;
  // not volatile / no memory clobber: the cluster barriers order these loads, and the compiler may
  // then keep several in flight
  asm("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(cluster_addr));
  return r;
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t cluster_addr) {
  uint32_t r;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(r) : "r"(cluster_addr) : "memory");
  return r;
}

template <int KPT, int D>
__global__ void __cluster_dims__(kCC, 1, 1) __launch_bounds__(kCT, 1)
    select_cluster_kernel(const float* __restrict__ scores, int l_b, int lp, int32_t* __restrict__ indices,
                          const uint16_t* __restrict__ k, const uint16_t* __restrict__ v, int64_t kv_row_stride,
                          int L_A, int hk, const GatherDst dst) {
  __shared__ __align__(16) uint32_t hist[3][2048];
  __shared__ uint32_t wtot[64];
  __shared__ uint32_t tot[2];  // this CTA's (> T, == T) counts
  __shared__ uint32_t sh_bin, sh_k;
  const int tid = threadIdx.x;
  const uint32_t c = cluster_ctarank();
  const int j = blockIdx.y;
  const float* s = scores + (int64_t)j * l_b;
  const int per = ((l_b + kCC - 1) / kCC + 3) & ~3;
  const int lo = min(l_b, (int)c * per), hi = min(l_b, lo + per);
  const int e0 = lo + tid * KPT;
  uint32_t key[KPT];
  if (e0 + KPT <= hi && (l_b & 3) == 0) {
#pragma unroll
    for (int e = 0; e < KPT; e += 4) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(s + e0 + e));
      key[e] = order_key(f.x);
      key[e + 1] = order_key(f.y);
      key[e + 2] = order_key(f.z);
      key[e + 3] = order_key(f.w);
    }
  } else {
#pragma unroll
    for (int e = 0; e < KPT; ++e) key[e] = e0 + e < hi ? order_key(__ldg(s + e0 + e)) : 0u;
  }
  const int nmine = max(0, min(KPT, hi - e0));
  for (int b = tid; b < 3 * 2048; b += kCT) (&hist[0][0])[b] = 0;
  __syncthreads();

  uint32_t prefix = 0, kk = (uint32_t)lp;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int shift = d == 0 ? 21 : (d == 1 ? 10 : 0);
    const uint32_t pmask = d == 0 ? 0u : (d == 1 ? 0xFFE00000u : 0xFFFFFC00u);
    const uint32_t dmask = d == 2 ? 0x3FFu : 0x7FFu;
#pragma unroll
    for (int e = 0; e < KPT; ++e)
      if (e < nmine && (key[e] & pmask) == prefix) atomicAdd(&hist[d][(key[e] >> shift) & dmask], 1u);
    cluster_sync();  // every CTA's digit-d histogram is complete
    constexpr int kBpt = 4;  // 2048 bins / 512 threads (digit 3: 1024 bins, the upper half stays 0)
    uint32_t cnt[kBpt] = {0u, 0u, 0u, 0u};
    const uint32_t local = smem_u32(&hist[d][tid * kBpt]);
    uint4 q[kCC];  // all 8 remote loads in flight before the first add
#pragma unroll
    for (int r = 0; r < kCC; ++r) q[r] = ld_dsmem_v4(mapa_shared(local, (uint32_t)r));
#pragma unroll
    for (int r = 0; r < kCC; ++r) {
      cnt[0] += q[r].x;
      cnt[1] += q[r].y;
      cnt[2] += q[r].z;
      cnt[3] += q[r].w;
    }
    find_bin_regs<kBpt>(cnt, kk, wtot, &sh_bin, &sh_k);
    prefix |= sh_bin << shift;
    kk = sh_k;
  }
  const uint32_t T = prefix, need_eq = kk;  // key of the l_p'-th largest score; ties taken

  // ---- ordered output: this CTA's position among the cluster's (> T, == T) counts
  uint32_t gt = 0, eq = 0;
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    gt += (e < nmine && key[e] > T);
    eq += (e < nmine && key[e] == T);
  }
  const uint32_t before = block_excl_scan_n<kCT>((gt << 16) | eq, wtot);
  if (tid == kCT - 1) {
    tot[0] = (before >> 16) + gt;
    tot[1] = (before & 0xFFFFu) + eq;
  }
  cluster_sync();
  uint32_t g_cta = 0, e_cta = 0;
  if (tid < 32) {  // the totals of the CTAs before this one
    uint32_t gg = 0, ee = 0;
    if (tid < (int)c) {
      gg = ld_dsmem_u32(mapa_shared(smem_u32(&tot[0]), (uint32_t)tid));
      ee = ld_dsmem_u32(mapa_shared(smem_u32(&tot[1]), (uint32_t)tid));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gg += __shfl_xor_sync(0xFFFFFFFFu, gg, o);
      ee += __shfl_xor_sync(0xFFFFFFFFu, ee, o);
    }
    if (tid == 0) {
      wtot[0] = gg;
      wtot[1] = ee;
    }
  }
  __syncthreads();
  g_cta = wtot[0];
  e_cta = wtot[1];
  const uint32_t e_before = e_cta + (before & 0xFFFFu);
  uint32_t pos = g_cta + (before >> 16) + min(need_eq, e_before);
  uint32_t erank = e_before;
  int32_t* out = indices + (int64_t)j * lp;
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    if (e < nmine) {
      bool sel = key[e] > T;
      if (key[e] == T) sel = erank++ < need_eq;
      if (sel) out[pos++] = e0 + e;
    }
  }
  cluster_sync();  // release / acquire at cluster scope: every CTA's indices are visible

  // ---- gather: output rows [c*lp/8, (c+1)*lp/8) of K and V of head j into every destination
  constexpr int kVec = D / 8;  // 16-byte vectors per row
  constexpr int kBatch = 16;   // vectors per thread in flight (one batch at L8: 2 x 256 rows x 16)
  const int r_lo = (int)(((int64_t)lp * c) / kCC), r_hi = (int)(((int64_t)lp * (c + 1)) / kCC);
  const int nr = r_hi - r_lo;
  const int n_vec = 2 * nr * kVec;  // K rows then V rows
  for (int u0 = 0; u0 < n_vec; u0 += kBatch * kCT) {
    int32_t src[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {  // the batch's source indices first: one L2 latency
      const int u = u0 + q * kCT + tid;
      const int w = u < nr * kVec ? u : u - nr * kVec;
      src[q] = u < n_vec ? __ldcg(out + r_lo + w / kVec) : 0;
    }
    uint4 buf[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {  // then every row load: one HBM latency
      const int u = u0 + q * kCT + tid;
      if (u < n_vec) {
        const int kv = u >= nr * kVec;
        const int cv = u % kVec;
        const uint16_t* row = (kv ? v : k) + (L_A + (int64_t)src[q]) * kv_row_stride + (int64_t)j * D;
        buf[q] = __ldg(reinterpret_cast<const uint4*>(row) + cv);
      }
    }
    for (int dd = 0; dd < dst.n; ++dd) {
      uint4* o = reinterpret_cast<uint4*>(dst.send[dd]);
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        const int u = u0 + q * kCT + tid;
        if (u < n_vec) {
          const int kv = u >= nr * kVec;
          const int w = kv ? u - nr * kVec : u;
          o[((((int64_t)kv * hk + j) * lp + r_lo) * D) / 8 + w] = buf[q];
        }
      }
    }
  }
  if (dst.flag[0] != nullptr) {
    __threadfence_system();  // this thread's peer stores are visible system-wide
    __syncthreads();
    if (tid == 0) {
      const uint32_t n_ctas = gridDim.x * gridDim.y * gridDim.z;
      const uint32_t done = atomicAdd(dst.counter, 1u) + 1u;
      if (done % n_ctas == 0) {  // the last CTA of this launch: every CTA's stores are fenced
        __threadfence_system();
        for (int dd = 0; dd < dst.n; ++dd)
          asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(dst.flag[dd]), "r"(dst.epoch) : "memory");
      }
    }
  }
}

template <int KPT>
static cudaError_t launch_cluster(int D, const float* scores, int l_b, int lp, int hk, int32_t* indices,
                                  const void* k, const void* v, int64_t kv_row_stride, int L_A, const GatherDst& dst,
                                  cudaStream_t stream) {
  const dim3 grid(kCC, hk);
  if (D == 128)
    select_cluster_kernel<KPT, 128><<<grid, kCT, 0, stream>>>(scores, l_b, lp, indices, static_cast<const uint16_t*>(k),
                                                             static_cast<const uint16_t*>(v), kv_row_stride, L_A, hk, dst);
  else
    select_cluster_kernel<KPT, 64><<<grid, kCT, 0, stream>>>(scores, l_b, lp, indices, static_cast<const uint16_t*>(k),
                                                            static_cast<const uint16_t*>(v), kv_row_stride, L_A, hk, dst);
  return cudaGetLastError();
}

template <bool kSmem>
static apb_status launch_fast(const float* scores, int l_b, int lp, int hk, int32_t* indices, cudaStream_t stream) {
  static std::atomic<uint64_t> smem_set{0};
  const int smem = ((kSmem ? l_b : 0) + kCand) * 4;
  apb_status st = set_max_smem_once(reinterpret_cast<const void*>(select_fast_kernel<kSmem>),
                                    (kMaxSmemKeys + kCand) * 4, smem_set);
  if (st) return st;
  select_fast_kernel<kSmem><<<hk, kFT, smem, stream>>>(scores, l_b, lp, indices);
  return APB_OK;
}

template <int D>
static cudaError_t launch_gather(const SelHosts& sh, int64_t kv_row_stride, int lp, int hk, const GatherDst& dst,
                                 cudaStream_t stream) {
  constexpr int kRows = 256 * 8 / (D / 8);
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3((lp + kRows - 1) / kRows, hk, 2 * sh.n);
  c.blockDim = dim3(256);
  c.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  c.attrs = &attr;
  c.numAttrs = 1;
  return cudaLaunchKernelEx(&c, gather_kernel<D>, sh, kv_row_stride, lp, hk, dst);
}

}  // namespace sel

apb_status launch_select_compact(int l_b, int lp, int hk, int D, int L_A, const float* scores, const void* k,
                                 const void* v, int64_t kv_row_stride, int32_t* indices, void* send,
                                 cudaStream_t stream, const GatherDst* push) {
  const char* env = std::getenv("APB_SELECT");
  GatherDst local{};
  if (!push) {
    local.n = 1;
    local.send[0] = static_cast<uint16_t*>(send);
  }
  const GatherDst& dst = push ? *push : local;
  // l_b > 32K (the 512K / 1M configs): one launch, an 8-CTA cluster per KV head (select + gather;
  // 1M host: 30.8 vs 106.6 us for the staged single-CTA select + gather).  Up to 32K the single-CTA
  // register select + PDL gather is faster (L8: 14.6 vs 21.8 us queued): the cluster's three
  // distributed-shared-memory histogram reductions (8 x 2048 bins read by every CTA) cost ~2 us
  // each, more than the single CTA's extra keys.  APB_SELECT=reg / legacy force the other paths.
  const int per = ((l_b + sel::kCC - 1) / sel::kCC + 3) & ~3;  // keys per cluster CTA
  if (!(env && (env[0] == 'l' || env[0] == 'r')) && l_b > 32 * sel::kFT && per <= 32 * sel::kCT &&
      (D == 128 || D == 64)) {
    cudaError_t e = per <= 16 * sel::kCT
                        ? sel::launch_cluster<16>(D, scores, l_b, lp, hk, indices, k, v, kv_row_stride, L_A, dst, stream)
                        : sel::launch_cluster<32>(D, scores, l_b, lp, hk, indices, k, v, kv_row_stride, L_A, dst, stream);
    if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("select_cluster launch: ") + cudaGetErrorString(e));
    count_launch(1);
    return APB_OK;
  }
  if (push || !(env && env[0] == 'l')) {
    apb_status st = APB_OK;
    SelHosts sh{};
    sh.n = 1;
    sh.scores[0] = scores;
    sh.indices[0] = indices;
    sh.k[0] = static_cast<const uint16_t*>(k);
    sh.v[0] = static_cast<const uint16_t*>(v);
    sh.send[0] = static_cast<uint16_t*>(send);
    sh.L_A[0] = L_A;
    if (l_b <= 16 * sel::kFT)
      sel::select_reg_kernel<16><<<hk, sel::kFT, 0, stream>>>(sh, l_b, lp);
    else if (l_b <= 32 * sel::kFT)
      sel::select_reg_kernel<32><<<hk, sel::kFT, 0, stream>>>(sh, l_b, lp);
    else
      st = l_b <= sel::kMaxSmemKeys ? sel::launch_fast<true>(scores, l_b, lp, hk, indices, stream)
                                    : sel::launch_fast<false>(scores, l_b, lp, hk, indices, stream);
    if (st) return st;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("select launch: ") + cudaGetErrorString(e));
    const char* dbg = std::getenv("APB_SELECT_DBG");  // timing experiments only: 1 = no gather
    if (dbg && dbg[0] == '1' && !push) {
      count_launch(1);
      return APB_OK;
    }
    const GatherDst none{};  // n = 0: each host's own slot sh.send[host]
    const GatherDst& gd = push ? *push : none;
    e = D == 128 ? sel::launch_gather<128>(sh, kv_row_stride, lp, hk, gd, stream)
                 : sel::launch_gather<64>(sh, kv_row_stride, lp, hk, gd, stream);
    if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("gather launch: ") + cudaGetErrorString(e));
    count_launch(2);
    return APB_OK;
  }
  // APB_SELECT=legacy: the round-1 two-kernel path (serial bin scan, one block scan per
  // 1024 elements, one 16-byte copy per thread), kept for A/B timing; both are bit-exact
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

apb_status launch_select_compact_hosts(int l_b, int lp, int hk, int D, const SelHosts& sh, int64_t kv_row_stride,
                                       cudaStream_t stream) {
  const char* env = std::getenv("APB_SELECT");
  if (sh.n < 1 || sh.n > kSelMaxHosts) return fail(APB_ERR_CONFIG, "1..8 hosts per select launch");
  if (l_b > 32 * sel::kFT || (env && env[0] == 'l') || (D != 128 && D != 64)) {
    for (int i = 0; i < sh.n; ++i) {  // one launch (pair) per host
      apb_status st = launch_select_compact(l_b, lp, hk, D, sh.L_A[i], sh.scores[i], sh.k[i], sh.v[i], kv_row_stride,
                                            sh.indices[i], sh.send[i], stream);
      if (st) return st;
    }
    return APB_OK;
  }
  // every host's KV heads in one select launch (grid hk x n) and one PDL gather launch
  if (l_b <= 16 * sel::kFT)
    sel::select_reg_kernel<16><<<dim3(hk, sh.n), sel::kFT, 0, stream>>>(sh, l_b, lp);
  else
    sel::select_reg_kernel<32><<<dim3(hk, sh.n), sel::kFT, 0, stream>>>(sh, l_b, lp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("select launch: ") + cudaGetErrorString(e));
  const GatherDst none{};
  e = D == 128 ? sel::launch_gather<128>(sh, kv_row_stride, lp, hk, none, stream)
               : sel::launch_gather<64>(sh, kv_row_stride, lp, hk, none, stream);
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("gather launch: ") + cudaGetErrorString(e));
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
