// internal.h — declarations shared by libapb's translation units (not part of the ABI).
#pragma once
#include <atomic>
#include <cstdint>
#include <cstddef>
#include <string>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include "../../include/apb.h"

namespace apb {

// thread-local error detail for apb_last_error()
void set_error(const std::string& msg);
apb_status fail(apb_status s, const std::string& msg);
void count_launch(int n = 1);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (call site, device): the attribute
// is per device, so a process that drives several GPUs needs it on each.  `done` is a per-call-
// site bitmask of devices already configured.
apb_status set_max_smem_once(const void* func, int bytes, std::atomic<uint64_t>& done);

// TMA descriptor encoding through the driver entry point (no -lcuda at link time).
// Returns false (and sets the error) if the driver call fails.
bool make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                    const uint64_t* strides_bytes, const uint32_t* box, int swizzle_bytes = 128);

// ---------------------------------------------------------------- attention
struct AttnParams {
  int L_A, l_b, lp, n_slots;  // n_slots = host: passing slots 0..host-1
  int hq, hk, g, np;          // np = ceil(g/2) (unused by the unit pairing; kept for the ABI struct layout)
  int nA_rt, nB_rt;           // 128-row query tiles of the anchor / local segment
  int nA_kv, nP_kv;           // 128-key tiles of the anchor segment / of one passing slot
  int n_local_items, n_anchor_items;
  int phase;                  // apb_phase
  int local_to_ws;            // LOCAL phase: local rows -> fp32 partial in ws
  float scale_log2;           // softmax_scale * log2(e)
  void* out;
  int64_t out_row_stride;
  float* lse;
  int64_t lse_ld;
  float* ws_o;                // [l_b][hq][D] fp32
  float* ws_lse;              // [hq][l_b] fp32, log2 domain
  int dbg_skip;               // unused (round-1 timing experiments; kept for the struct layout)
};
// Several hosts' attention in ONE launch (the hosts a rank owns, same phase): per-host tensor maps
// and parameters in the kernel's parameter space (~4.4 KB, CUDA >= 12.1 large kernel parameters);
// the grid is the concatenation of the hosts' work items, host i's items at
// [item_begin[i], item_begin[i+1]) in that host's own order.
constexpr int kAttnMaxHosts = 8;
struct AttnLaunch {
  CUtensorMap tq[kAttnMaxHosts], tk[kAttnMaxHosts], tv[kAttnMaxHosts];
  // bf16 output of the anchor rows [0, L_A) and of the block rows [L_A, L_A + l_b) as two maps
  // (d, heads, rows), so a TMA store of a ragged last tile is clipped at its own segment's end
  CUtensorMap to_a[kAttnMaxHosts], to_b[kAttnMaxHosts];
  CUtensorMap tg;  // the gathered passing slots (shared by every host of the launch)
  AttnParams p[kAttnMaxHosts];
  int item_begin[kAttnMaxHosts + 1];
  int n;
  int ctr_slot;  // persistent launches: this launch's work-counter slot (set by launch_attention_hosts)
  int persist;   // 1: persistent CTAs take further items from the counter; 0: one item per CTA
};
// phase: the launch's phase for the pairing policy (a host without passing keys runs LOCAL as ALL)
apb_status launch_attention_hosts(int D, const AttnLaunch& L, int phase, cudaStream_t stream);

// ---------------------------------------------------------------- retaining-head scoring
struct ScoreParams {
  int l_b, L_A, hq, hk, D, d_in, d_hidden, n_out;
  int kq, kk;                 // number of 64-wide K blocks coming from Q and from K (rest from V)
  const float* b1;
  const float* w2;
  const float* b2;
  float* scores;              // [hk][l_b]
};
apb_status launch_retain_score(const ScoreParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                               const CUtensorMap& tv, const CUtensorMap& tw1, cudaStream_t stream);
// CTA-pair GEMM form (gemm_sm100.cu): partials [d_hidden/(BN/2)][n_out][l_b] in `part`, then a
// fixed-order finalize (tw1: box {64, BN/2}, tw1h: box {64, BN/4} for the half tiles of the last
// wave; BN = score_tile_n())
int score_tile_n();  // hidden units per scoring GEMM tile (128 or 256)
apb_status launch_score_gemm(const ScoreParams& p, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const CUtensorMap& tw1, const CUtensorMap& tw1h, float* part,
                             cudaStream_t stream);
// n (1..8) hosts' scoring in one GEMM launch + one finalize launch: host i's [Q|K|V] maps tq/tk/tv[i],
// anchor rows L_A[i], scores[i]; `part` holds n consecutive per-host partial areas (the retain
// workspace of one host, n times).  p's L_A and scores fields are ignored.
apb_status launch_score_gemm_hosts(const ScoreParams& p, int n, const CUtensorMap* tq, const CUtensorMap* tk,
                                   const CUtensorMap* tv, const int* L_A, float* const* scores, const CUtensorMap& tw1,
                                   const CUtensorMap& tw1h, float* part, cudaStream_t stream);

// ---------------------------------------------------------------- selection + compaction
apb_status launch_rmsnorm(int64_t rows, int dim, const void* x, int64_t xs, const void* w, float eps, void* y,
                          int64_t ys, cudaStream_t stream);
apb_status launch_rope(int64_t rows, int n_heads, int d, void* x, int64_t row_stride, const int32_t* positions,
                       int64_t pos_offset, double theta, cudaStream_t stream);
apb_status launch_swiglu(int64_t rows, int inter, const void* gu, int64_t gs, void* out, int64_t os,
                         cudaStream_t stream);
struct GemmArgs {
  int64_t M;
  int N, K;
  const void* a;
  int64_t lda;
  const void* w;
  int64_t ldw;
  void* c;
  int64_t ldc;
  int epi;  // apb_gemm_epilogue
  float beta;
  int rope_cols, head_dim;
  float theta;
  const int32_t* positions;
  int64_t pos_offset;
};
apb_status launch_gemm(const GemmArgs& g, cudaStream_t stream);
apb_status launch_random_scores(uint64_t seed, uint64_t c0, int64_t count, float* scores, cudaStream_t stream);
apb_status launch_share_scores(float* scores, int hk, int l_b, cudaStream_t stream);
// Destinations of the compaction: one local slot, or (peer exchange) the same slot in every rank's
// IPC-mapped buffer plus a completion flag per rank.
constexpr int kMaxPeers = 8;
struct GatherDst {
  int n;
  uint16_t* send[kMaxPeers];  // slot base ([2][hk][l_p'][d]) in each destination
  int32_t* flag[kMaxPeers];   // nullptr: no signal; else set to `epoch` once the launch's stores landed
  uint32_t* counter;          // CTA-completion counter (this rank's device memory)
  int32_t epoch;
};
// Several hosts' selection + compaction in one select launch and one gather launch (same l_b, l_p,
// hk; per-host pointers and anchor lengths).  l_b > 32K: one launch pair per host.
constexpr int kSelMaxHosts = 8;
struct SelHosts {
  int n;
  const float* scores[kSelMaxHosts];
  int32_t* indices[kSelMaxHosts];
  const uint16_t* k[kSelMaxHosts];
  const uint16_t* v[kSelMaxHosts];
  uint16_t* send[kSelMaxHosts];
  int L_A[kSelMaxHosts];
};
apb_status launch_select_compact_hosts(int l_b, int lp, int hk, int D, const SelHosts& sh, int64_t kv_row_stride,
                                       cudaStream_t stream);
apb_status launch_select_compact(int l_b, int lp, int hk, int D, int L_A, const float* scores,
                                 const void* k, const void* v, int64_t kv_row_stride, int32_t* indices,
                                 void* send, cudaStream_t stream, const GatherDst* push = nullptr);
// peer exchange helpers (peers.cu)
apb_status launch_wait_flags(const int32_t* flags, int n, int32_t epoch, cudaStream_t stream);
apb_status launch_publish(int32_t* const* dsts, int n, int32_t epoch, cudaStream_t stream);

// ---------------------------------------------------------------- decode (Alg. apb_decode)
constexpr int kDecodeRowsMax = 64;  // t_new * (n_heads / n_kv_heads) per KV head
struct DecodeParams {
  int t, hq, hk, g, D, has_new;
  int64_t cache_len, cache_row_stride, new_row_stride;
  float scale_log2;
  const __nv_bfloat16* q;        // [t][hq][D]
  const __nv_bfloat16* k_cache;  // [cache_len][hk][D] (row stride cache_row_stride)
  const __nv_bfloat16* v_cache;
  const __nv_bfloat16* k_new;    // [t][hk][D] (row stride new_row_stride), last host only
  const __nv_bfloat16* v_new;
  float* ws_o;                   // [splits][t*hq][D] then (256-B aligned) ws_lse [splits][t*hq]
  float* ws_lse;
};
// Several hosts' partials in one launch (the hosts one rank owns): per-host cache pointers and
// lengths; host i's splits are [split_begin[i], split_begin[i+1]) of the launch's split axis.
constexpr int kDecMaxHosts = 16;
struct DecodeHosts {
  int n;         // 0: single-host launch (DecodeParams alone)
  int new_host;  // index i of the host that also attends to the new tokens (-1: none)
  int split_begin[kDecMaxHosts + 1];
  int64_t cache_len[kDecMaxHosts];
  const __nv_bfloat16* k_cache[kDecMaxHosts];
  const __nv_bfloat16* v_cache[kDecMaxHosts];
};
size_t decode_workspace_bytes(int64_t n_keys, int t, int hq, int hk, int D);
size_t decode_hosts_workspace_bytes(int n, const int64_t* n_keys, int t, int hq, int hk, int D);
apb_status launch_decode(const DecodeParams& p, float* part_o, float* part_lse, cudaStream_t stream);
// p: common fields (q, k_new/v_new, strides, scale, ws); n hosts with keys n_keys[i] (cache plus
// the new tokens for hb.new_host); host i's partial -> parts + i*part_stride (O), + lse_offset (lse);
// or, with merged_out != NULL (all hosts present), the merged bf16 output and natural lse directly
apb_status launch_decode_hosts(const DecodeParams& p, DecodeHosts hb, const int64_t* n_keys, float* parts,
                               int64_t part_stride, int64_t lse_offset, void* merged_out, float* merged_lse,
                               cudaStream_t stream);
apb_status launch_merge(int n, int64_t rows, int D, const float* parts_o, const float* parts_lse, int64_t stride_o,
                        int64_t stride_lse, int lse_in_log2, void* out, bool out_bf16, float* out_lse,
                        cudaStream_t stream, bool pdl = false);  // pdl: follows decode_mma_kernel on `stream`

}  // namespace apb
