// apb_api.cu — the C ABI of libapb (include/apb.h): argument validation, workspace sizing, TMA
// descriptor construction, NCCL exchange (dlopen'ed, no link-time dependency) and dispatch to
// the sm_100a kernels.  No exception crosses the ABI; every failure is an apb_status plus a
// thread-local detail string.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>

#include "internal.h"

namespace apb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
apb_status fail(apb_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                    const uint64_t* strides_bytes, const uint32_t* box, int swizzle_bytes) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
    return false;
  }
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
  }
  for (int i = 0; i + 1 < rank; ++i) s[i] = strides_bytes[i];
  const CUtensorMapSwizzle swz = swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : swizzle_bytes == 0  ? CU_TENSOR_MAP_SWIZZLE_NONE
                                                       : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, b, e,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed, CUresult " + std::to_string((int)r));
    return false;
  }
  return true;
}

// ---------------------------------------------------------------- validation helpers
static int64_t L_A_of(const apb_dims* d) { return d->host == 0 ? 0 : (int64_t)d->l_q + d->l_a; }
static int64_t lpp_of(const apb_dims* d) { return d->l_p < d->l_b ? d->l_p : d->l_b; }
apb_status set_max_smem_once(const void* func, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return APB_OK;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  done.fetch_or(bit, std::memory_order_acq_rel);
  return APB_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static apb_status check_dims(const apb_dims* d) {
  if (!d) return fail(APB_ERR_CONTRACT, "dims is NULL");
  if (d->H < 1) return fail(APB_ERR_CONFIG, "H must be >= 1");
  if (d->host < 0 || d->host >= d->H) return fail(APB_ERR_CONFIG, "host must be in [0, H)");
  if (d->l_q < 0 || d->l_a < 0 || d->l_p < 0 || d->l_b < 1) return fail(APB_ERR_CONFIG, "negative length");
  if (d->n != (int64_t)d->H * d->l_b) return fail(APB_ERR_CONFIG, "n must equal H * l_b (reading G15)");
  if (d->l_a > d->n) return fail(APB_ERR_CONFIG, "l_a must be <= n");
  if (d->n_heads < 1 || d->n_kv_heads < 1 || d->n_heads % d->n_kv_heads)
    return fail(APB_ERR_CONFIG, "n_heads must be a positive multiple of n_kv_heads");
  if (d->head_dim != 64 && d->head_dim != 128) return fail(APB_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  const int64_t rows = L_A_of(d) + d->l_b;
  if (rows > (int64_t)1 << 30) return fail(APB_ERR_CONFIG, "too many rows on one host");
  if ((int64_t)d->H * lpp_of(d) > ((int64_t)1 << 30)) return fail(APB_ERR_CONFIG, "passing too long");
  return APB_OK;
}

static apb_status check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  static int cached_major = -1, cached_minor = -1, cached_dev = -1;
  if (cached_dev != dev) {
    cudaDeviceGetAttribute(&cached_major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&cached_minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached_dev = dev;
  }
  if (cached_major != 10 || cached_minor != 0)
    return fail(APB_ERR_UNSUPPORTED, "libapb is built for sm_100a (B200); device is sm_" +
                                         std::to_string(cached_major) + std::to_string(cached_minor));
  return APB_OK;
}

static apb_status check_rows(const void* p, int64_t stride, int64_t min_stride, const char* what) {
  if (!p) return fail(APB_ERR_CONTRACT, std::string(what) + " is NULL");
  if (!aligned16(p)) return fail(APB_ERR_CONTRACT, std::string(what) + " is not 16-byte aligned");
  if (stride < min_stride || stride % 8) return fail(APB_ERR_CONTRACT, std::string(what) + " row stride invalid");
  return APB_OK;
}

}  // namespace apb

using namespace apb;

// ---------------------------------------------------------------- plumbing
extern "C" const char* apb_status_string(apb_status s) {
  switch (s) {
    case APB_OK: return "APB_OK";
    case APB_ERR_CONFIG: return "APB_ERR_CONFIG";
    case APB_ERR_CONTRACT: return "APB_ERR_CONTRACT";
    case APB_ERR_UNSUPPORTED: return "APB_ERR_UNSUPPORTED";
    case APB_ERR_CUDA: return "APB_ERR_CUDA";
    case APB_ERR_NCCL: return "APB_ERR_NCCL";
  }
  return "APB_ERR_UNKNOWN";
}
extern "C" const char* apb_last_error(void) { return g_last_error.c_str(); }
extern "C" int32_t apb_version(void) { return 100; }
extern "C" int64_t apb_launch_count(void) { return g_launches.load(); }
extern "C" apb_status apb_check_dims(const apb_dims* d) { return check_dims(d); }

extern "C" apb_status apb_workspace_size(const apb_dims* d, apb_ws_kind which, size_t* bytes) {
  if (!bytes) return fail(APB_ERR_CONTRACT, "bytes is NULL");
  apb_status st = check_dims(d);
  if (st) return st;
  *bytes = 0;
  if (which == APB_WS_ATTENTION) {
    if (d->host > 0 && lpp_of(d) > 0) {
      size_t o = (size_t)d->l_b * d->n_heads * d->head_dim * sizeof(float);
      o = (o + 255) & ~size_t(255);
      *bytes = o + (size_t)d->n_heads * d->l_b * sizeof(float);
    }
  } else if (which != APB_WS_RETAIN && which != APB_WS_SELECT) {
    return fail(APB_ERR_CONTRACT, "unknown workspace kind");
  }
  return APB_OK;
}

// ---------------------------------------------------------------- step 4: attention
// Validation and launch parameters of one host's attention (apb_attention_fwd and each host of
// apb_attention_fwd_hosts).  *skip: nothing to compute (PASSING without passing keys).
static apb_status attention_setup(const apb_dims* d, const void* q, const void* k, const void* v, int64_t q_row_stride,
                                  int64_t kv_row_stride, const void* gathered, void* out, int64_t out_row_stride,
                                  float* lse, apb_phase phase, void* ws, size_t ws_bytes, AttnLaunch& La, int slot,
                                  CUtensorMap& tg, bool* skip) {
  AttnParams& p = La.p[slot];
  CUtensorMap &tq = La.tq[slot], &tk = La.tk[slot], &tv = La.tv[slot];
  *skip = false;
  apb_status st = check_dims(d);
  if (st) return st;
  if (phase != APB_PHASE_ALL && phase != APB_PHASE_LOCAL && phase != APB_PHASE_PASSING)
    return fail(APB_ERR_CONTRACT, "unknown phase");
  const int D = d->head_dim, hq = d->n_heads, hk = d->n_kv_heads;
  if ((st = check_rows(q, q_row_stride, (int64_t)hq * D, "q"))) return st;
  if ((st = check_rows(k, kv_row_stride, (int64_t)hk * D, "k"))) return st;
  if ((st = check_rows(v, kv_row_stride, (int64_t)hk * D, "v"))) return st;
  if ((st = check_rows(out, out_row_stride, (int64_t)hq * D, "out"))) return st;
  if (lse && (reinterpret_cast<uintptr_t>(lse) & 3)) return fail(APB_ERR_CONTRACT, "lse misaligned");
  const int64_t L_A = L_A_of(d), lpp = lpp_of(d), rows = L_A + d->l_b;
  const int n_slots = d->host;
  const bool has_pass = n_slots > 0 && lpp > 0;
  if (has_pass && phase != APB_PHASE_LOCAL) {
    if (!gathered) return fail(APB_ERR_CONTRACT, "gathered is NULL but host > 0 and l_p > 0");
    if (!aligned16(gathered)) return fail(APB_ERR_CONTRACT, "gathered is not 16-byte aligned");
  }
  size_t need = 0;
  apb_workspace_size(d, APB_WS_ATTENTION, &need);
  const bool use_ws = has_pass && phase != APB_PHASE_ALL;
  if (use_ws && (ws == nullptr || ws_bytes < need || !aligned16(ws)))
    return fail(APB_ERR_CONTRACT, "attention workspace missing, too small or misaligned");
  if (phase == APB_PHASE_PASSING && !has_pass) {  // nothing to merge
    *skip = true;
    return APB_OK;
  }

  p = AttnParams{};
  p.L_A = (int)L_A;
  p.l_b = d->l_b;
  p.lp = (int)lpp;
  p.n_slots = has_pass ? n_slots : 0;
  p.hq = hq;
  p.hk = hk;
  p.g = hq / hk;
  p.np = (p.g + 1) / 2;
  p.nA_rt = (int)((L_A + 127) / 128);
  p.nB_rt = (d->l_b + 127) / 128;
  p.nA_kv = p.nA_rt;
  p.nP_kv = (int)((lpp + 127) / 128);
  p.phase = (int)phase;
  if (!has_pass && phase == APB_PHASE_LOCAL) p.phase = APB_PHASE_ALL;  // LOCAL == ALL without passing
  p.local_to_ws = (phase == APB_PHASE_LOCAL && has_pass) ? 1 : 0;
  // work items: pairs of (row tile, query head) units per KV head (see decode_item)
  p.n_local_items = (p.nB_rt * p.g + 1) / 2 * hk;
  p.n_anchor_items = (phase == APB_PHASE_PASSING) ? 0 : (p.nA_rt * p.g + 1) / 2 * hk;
  const float scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt((float)D);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.out_row_stride = out_row_stride;
  p.lse = lse;
  p.lse_ld = rows;
  if (use_ws) {
    size_t o = (size_t)d->l_b * hq * D * sizeof(float);
    o = (o + 255) & ~size_t(255);
    p.ws_o = static_cast<float*>(ws);
    p.ws_lse = reinterpret_cast<float*>(static_cast<char*>(ws) + o);
  }

  {
    uint64_t dims[3] = {(uint64_t)D, (uint64_t)hq, (uint64_t)rows};
    uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)q_row_stride * 2};
    uint32_t box[3] = {64, 1, 128};
    if (!make_tmap_bf16(&tq, q, 3, dims, str, box)) return APB_ERR_CUDA;
  }
  {
    uint64_t dims[3] = {(uint64_t)D, (uint64_t)hk, (uint64_t)rows};
    uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)kv_row_stride * 2};
    uint32_t box[3] = {64, 1, 128};
    if (!make_tmap_bf16(&tk, k, 3, dims, str, box)) return APB_ERR_CUDA;
    if (!make_tmap_bf16(&tv, v, 3, dims, str, box)) return APB_ERR_CUDA;
  }
  {
    // the bf16 output, anchor rows and block rows as separate maps (TMA stores clip at each end)
    uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)out_row_stride * 2};
    uint32_t box[3] = {64, 1, 128};
    uint64_t da[3] = {(uint64_t)D, (uint64_t)hq, (uint64_t)(L_A > 0 ? L_A : 1)};
    uint64_t db[3] = {(uint64_t)D, (uint64_t)hq, (uint64_t)d->l_b};
    if (!make_tmap_bf16(&La.to_a[slot], out, 3, da, str, box)) return APB_ERR_CUDA;
    if (!make_tmap_bf16(&La.to_b[slot], static_cast<char*>(out) + L_A * out_row_stride * 2, 3, db, str, box))
      return APB_ERR_CUDA;
  }
  if (p.n_slots > 0 && phase != APB_PHASE_LOCAL) {
    uint64_t dims[4] = {(uint64_t)D, (uint64_t)lpp, (uint64_t)hk, (uint64_t)2 * d->H};
    uint64_t str[3] = {(uint64_t)D * 2, (uint64_t)lpp * D * 2, (uint64_t)hk * lpp * D * 2};
    uint32_t box[4] = {64, 128, 1, 1};
    if (!make_tmap_bf16(&tg, gathered, 4, dims, str, box)) return APB_ERR_CUDA;
  } else {
    tg = tk;  // never dereferenced
  }
  return APB_OK;
}

extern "C" apb_status apb_attention_fwd(const apb_dims* d, const void* q, const void* k, const void* v,
                                        int64_t q_row_stride, int64_t kv_row_stride, const void* gathered, void* out,
                                        int64_t out_row_stride, float* lse, apb_phase phase, void* ws, size_t ws_bytes,
                                        apb_stream_t stream) {
  AttnLaunch La{};
  bool skip = false;
  apb_status st = attention_setup(d, q, k, v, q_row_stride, kv_row_stride, gathered, out, out_row_stride, lse, phase,
                                  ws, ws_bytes, La, 0, La.tg, &skip);
  if (st) return st;
  if ((st = check_device())) return st;
  if (skip) return APB_OK;
  La.n = 1;
  La.item_begin[0] = 0;
  La.item_begin[1] = La.p[0].n_local_items + La.p[0].n_anchor_items;
  return launch_attention_hosts(d->head_dim, La, (int)phase, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_attention_fwd_hosts(int32_t n, const apb_dims* dims, const void* const* q,
                                              const void* const* k, const void* const* v, int64_t q_row_stride,
                                              int64_t kv_row_stride, const void* gathered, void* const* out,
                                              int64_t out_row_stride, float* const* lse, apb_phase phase,
                                              void* const* ws, const size_t* ws_bytes, apb_stream_t stream) {
  if (n < 1 || n > kAttnMaxHosts) return fail(APB_ERR_CONFIG, "n must be in [1, 8]");
  if (!dims || !q || !k || !v || !out) return fail(APB_ERR_CONTRACT, "dims/q/k/v/out array is NULL");
  // every host of one launch shares the problem (only `host` differs) and no host appears twice
  for (int i = 0; i < n; ++i) {
    const apb_dims& a = dims[i];
    const apb_dims& b = dims[0];
    if (a.n != b.n || a.H != b.H || a.l_q != b.l_q || a.l_a != b.l_a || a.l_p != b.l_p || a.n_heads != b.n_heads ||
        a.n_kv_heads != b.n_kv_heads || a.head_dim != b.head_dim || a.softmax_scale != b.softmax_scale)
      return fail(APB_ERR_CONFIG, "the hosts of one launch must share every dimension but `host`");
    for (int j = 0; j < i; ++j)
      if (dims[j].host == a.host) return fail(APB_ERR_CONFIG, "a host appears twice");
  }
  // heaviest host first (host h attends to h * l_p' passing keys): the lightest items form the tail
  int order[kAttnMaxHosts];
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order, order + n, [&](int x, int y) { return dims[x].host > dims[y].host; });
  AttnLaunch La{};
  La.n = 0;
  La.item_begin[0] = 0;
  bool have_g = false;
  for (int oi = 0; oi < n; ++oi) {
    const int i = order[oi];
    CUtensorMap tg;
    bool skip = false;
    apb_status st = attention_setup(&dims[i], q[i], k[i], v[i], q_row_stride, kv_row_stride, gathered, out[i],
                                    out_row_stride, lse ? lse[i] : nullptr, phase, ws ? ws[i] : nullptr,
                                    ws_bytes ? ws_bytes[i] : 0, La, La.n, tg, &skip);
    if (st) return st;
    if (skip) continue;
    if (La.p[La.n].n_slots > 0 && phase != APB_PHASE_LOCAL) {
      La.tg = tg;
      have_g = true;
    }
    La.item_begin[La.n + 1] = La.item_begin[La.n] + La.p[La.n].n_local_items + La.p[La.n].n_anchor_items;
    ++La.n;
  }
  if (!have_g) La.tg = La.tk[0];  // never dereferenced
  apb_status st = check_device();
  if (st) return st;
  if (La.n == 0) return APB_OK;
  return launch_attention_hosts(dims[0].head_dim, La, (int)phase, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- step 1: scoring
static size_t retain_ws_bytes(const apb_dims* d, const apb_retain_weights* w) {
  // one fp32 partial slot per half tile of hidden units (score_tile_n() / 2 = 128 by default)
  const int unit = score_tile_n() / 2;
  return (size_t)((w->d_hidden + unit - 1) / unit) * (size_t)d->l_b * (size_t)w->n_out * sizeof(float);
}

static apb_status check_retain_weights(const apb_dims* d, const apb_retain_weights* w) {
  if (!w) return fail(APB_ERR_CONTRACT, "weights is NULL");
  const int D = d->head_dim, hq = d->n_heads, hk = d->n_kv_heads;
  if (w->d_in != (hq + 2 * hk) * D) return fail(APB_ERR_CONFIG, "d_in must equal (n_heads + 2 n_kv_heads) * head_dim");
  if (w->n_out != hk && w->n_out != hq) return fail(APB_ERR_CONFIG, "n_out must be n_kv_heads or n_heads");
  if (w->d_hidden < 256 || w->d_hidden % 256) return fail(APB_ERR_UNSUPPORTED, "d_hidden must be a multiple of 256");
  if (w->n_out > 64) return fail(APB_ERR_UNSUPPORTED, "n_out must be <= 64");
  return APB_OK;
}

extern "C" apb_status apb_retain_workspace_size(const apb_dims* d, const apb_retain_weights* w, size_t* bytes) {
  if (!bytes) return fail(APB_ERR_CONTRACT, "bytes is NULL");
  apb_status st = check_dims(d);
  if (st) return st;
  if ((st = check_retain_weights(d, w))) return st;
  *bytes = retain_ws_bytes(d, w);
  return APB_OK;
}

extern "C" apb_status apb_retain_score(const apb_dims* d, const apb_retain_weights* w, const void* q, const void* k,
                                       const void* v, int64_t q_row_stride, int64_t kv_row_stride, float* scores,
                                       void* ws, size_t ws_bytes, apb_stream_t stream) {
  apb_status st = check_dims(d);
  if (st) return st;
  if ((st = check_retain_weights(d, w))) return st;
  const int D = d->head_dim, hq = d->n_heads, hk = d->n_kv_heads;
  if (!w->w1 || !aligned16(w->w1) || !w->w2) return fail(APB_ERR_CONTRACT, "w1/w2 NULL or misaligned");
  if ((st = check_rows(q, q_row_stride, (int64_t)hq * D, "q"))) return st;
  if ((st = check_rows(k, kv_row_stride, (int64_t)hk * D, "k"))) return st;
  if ((st = check_rows(v, kv_row_stride, (int64_t)hk * D, "v"))) return st;
  if (!scores || (reinterpret_cast<uintptr_t>(scores) & 15)) return fail(APB_ERR_CONTRACT, "scores NULL or misaligned");
  if ((st = check_device())) return st;
  const int64_t L_A = L_A_of(d), rows = L_A + d->l_b;
  ScoreParams p{};
  p.l_b = d->l_b;
  p.L_A = (int)L_A;
  p.hq = hq;
  p.hk = hk;
  p.D = D;
  p.d_in = w->d_in;
  p.d_hidden = w->d_hidden;
  p.n_out = w->n_out;
  p.kq = hq * D / 64;
  p.kk = hk * D / 64;
  p.b1 = w->b1;
  p.w2 = w->w2;
  p.b2 = w->b2;
  p.scores = scores;
  CUtensorMap tq, tk, tv, tw;
  uint32_t box[2] = {64, 128};
  {
    uint64_t dims[2] = {(uint64_t)hq * D, (uint64_t)rows};
    uint64_t str[1] = {(uint64_t)q_row_stride * 2};
    if (!make_tmap_bf16(&tq, q, 2, dims, str, box)) return APB_ERR_CUDA;
  }
  {
    uint64_t dims[2] = {(uint64_t)hk * D, (uint64_t)rows};
    uint64_t str[1] = {(uint64_t)kv_row_stride * 2};
    if (!make_tmap_bf16(&tk, k, 2, dims, str, box)) return APB_ERR_CUDA;
    if (!make_tmap_bf16(&tv, v, 2, dims, str, box)) return APB_ERR_CUDA;
  }
  // the CTA-pair GEMM (pair = 256 tokens x 256 hidden units, partials reduced by a fixed-order
  // finalize) whenever the caller provides its workspace, unless APB_SCORE_PLAN selects one of the
  // round-1 single-CTA plans ("legacy" / "s3" / "p2", kept for A/B timing)
  const char* plan = std::getenv("APB_SCORE_PLAN");
  const bool legacy = plan && plan[0] != '\0';
  if (!legacy && ws && ws_bytes >= retain_ws_bytes(d, w) && aligned16(ws)) {
    uint64_t dims[2] = {(uint64_t)w->d_in, (uint64_t)w->d_hidden};
    uint64_t str[1] = {(uint64_t)w->d_in * 2};
    uint32_t wbox[2] = {64, (uint32_t)score_tile_n() / 2};  // this CTA's half of a W1 tile
    if (!make_tmap_bf16(&tw, w->w1, 2, dims, str, wbox)) return APB_ERR_CUDA;
    CUtensorMap twh;
    uint32_t whbox[2] = {64, (uint32_t)score_tile_n() / 4};  // ... of a half tile (the tail wave)
    if (!make_tmap_bf16(&twh, w->w1, 2, dims, str, whbox)) return APB_ERR_CUDA;
    return launch_score_gemm(p, tq, tk, tv, tw, twh, static_cast<float*>(ws), reinterpret_cast<cudaStream_t>(stream));
  }
  {
    uint64_t dims[2] = {(uint64_t)w->d_in, (uint64_t)w->d_hidden};
    uint64_t str[1] = {(uint64_t)w->d_in * 2};
    uint32_t wbox[2] = {64, 64};  // one quarter of a 256-row W1 tile per CTA of a 4-CTA cluster (multicast)
    if (!make_tmap_bf16(&tw, w->w1, 2, dims, str, wbox)) return APB_ERR_CUDA;
  }
  return launch_retain_score(p, tq, tk, tv, tw, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_retain_score_hosts(int32_t n, const apb_dims* dims, const apb_retain_weights* w,
                                             const void* const* q, const void* const* k, const void* const* v,
                                             int64_t q_row_stride, int64_t kv_row_stride, float* const* scores,
                                             void* ws, size_t ws_bytes, apb_stream_t stream) {
  if (n < 1 || n > 8) return fail(APB_ERR_CONFIG, "n must be in [1, 8]");
  if (!dims || !q || !k || !v || !scores) return fail(APB_ERR_CONTRACT, "dims/q/k/v/scores array is NULL");
  apb_status st;
  for (int i = 0; i < n; ++i) {
    const apb_dims& a = dims[i];
    const apb_dims& b = dims[0];
    if ((st = check_dims(&a))) return st;
    if (a.n != b.n || a.H != b.H || a.l_q != b.l_q || a.l_a != b.l_a || a.l_p != b.l_p || a.n_heads != b.n_heads ||
        a.n_kv_heads != b.n_kv_heads || a.head_dim != b.head_dim)
      return fail(APB_ERR_CONFIG, "the hosts of one launch must share every dimension but `host`");
  }
  const apb_dims* d = &dims[0];
  if ((st = check_retain_weights(d, w))) return st;
  const int D = d->head_dim, hq = d->n_heads, hk = d->n_kv_heads;
  if (!w->w1 || !aligned16(w->w1) || !w->w2) return fail(APB_ERR_CONTRACT, "w1/w2 NULL or misaligned");
  const size_t per = retain_ws_bytes(d, w);
  if (!ws || ws_bytes < per * (size_t)n || !aligned16(ws))
    return fail(APB_ERR_CONTRACT, "workspace missing, misaligned or smaller than n x apb_retain_workspace_size");
  CUtensorMap tq[8], tk[8], tv[8];
  int L_A[8];
  uint32_t box[2] = {64, 128};
  for (int i = 0; i < n; ++i) {
    if ((st = check_rows(q[i], q_row_stride, (int64_t)hq * D, "q"))) return st;
    if ((st = check_rows(k[i], kv_row_stride, (int64_t)hk * D, "k"))) return st;
    if ((st = check_rows(v[i], kv_row_stride, (int64_t)hk * D, "v"))) return st;
    if (!scores[i] || (reinterpret_cast<uintptr_t>(scores[i]) & 15))
      return fail(APB_ERR_CONTRACT, "scores NULL or misaligned");
    L_A[i] = (int)L_A_of(&dims[i]);
    const int64_t rows = L_A[i] + d->l_b;
    uint64_t qd[2] = {(uint64_t)hq * D, (uint64_t)rows}, qs[1] = {(uint64_t)q_row_stride * 2};
    uint64_t kd[2] = {(uint64_t)hk * D, (uint64_t)rows}, ks[1] = {(uint64_t)kv_row_stride * 2};
    if (!make_tmap_bf16(&tq[i], q[i], 2, qd, qs, box)) return APB_ERR_CUDA;
    if (!make_tmap_bf16(&tk[i], k[i], 2, kd, ks, box)) return APB_ERR_CUDA;
    if (!make_tmap_bf16(&tv[i], v[i], 2, kd, ks, box)) return APB_ERR_CUDA;
  }
  if ((st = check_device())) return st;
  ScoreParams p{};
  p.l_b = d->l_b;
  p.hq = hq;
  p.hk = hk;
  p.D = D;
  p.d_in = w->d_in;
  p.d_hidden = w->d_hidden;
  p.n_out = w->n_out;
  p.kq = hq * D / 64;
  p.kk = hk * D / 64;
  p.b1 = w->b1;
  p.w2 = w->w2;
  p.b2 = w->b2;
  CUtensorMap tw, twh;
  uint64_t wd[2] = {(uint64_t)w->d_in, (uint64_t)w->d_hidden};
  uint64_t ws_[1] = {(uint64_t)w->d_in * 2};
  uint32_t wbox[2] = {64, (uint32_t)score_tile_n() / 2}, whbox[2] = {64, (uint32_t)score_tile_n() / 4};
  if (!make_tmap_bf16(&tw, w->w1, 2, wd, ws_, wbox)) return APB_ERR_CUDA;
  if (!make_tmap_bf16(&twh, w->w1, 2, wd, ws_, whbox)) return APB_ERR_CUDA;
  return launch_score_gemm_hosts(p, n, tq, tk, tv, L_A, scores, tw, twh, static_cast<float*>(ws),
                                 reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- step 2: select + compact
extern "C" apb_status apb_select_topk(const apb_dims* d, const float* scores, const void* k, const void* v,
                                      int64_t kv_row_stride, int32_t* indices, void* send, void* ws, size_t ws_bytes,
                                      apb_stream_t stream) {
  (void)ws;
  (void)ws_bytes;
  apb_status st = check_dims(d);
  if (st) return st;
  const int D = d->head_dim, hk = d->n_kv_heads;
  const int64_t lpp = lpp_of(d);
  if (lpp == 0) return APB_OK;
  if (!scores || !indices) return fail(APB_ERR_CONTRACT, "scores/indices NULL");
  if ((st = check_rows(k, kv_row_stride, (int64_t)hk * D, "k"))) return st;
  if ((st = check_rows(v, kv_row_stride, (int64_t)hk * D, "v"))) return st;
  if (!send || !aligned16(send)) return fail(APB_ERR_CONTRACT, "send NULL or misaligned");
  if ((st = check_device())) return st;
  return launch_select_compact(d->l_b, (int)lpp, hk, D, (int)L_A_of(d), scores, k, v, kv_row_stride, indices, send,
                               reinterpret_cast<cudaStream_t>(stream));
}


extern "C" apb_status apb_select_topk_hosts(int32_t n, const apb_dims* dims, const float* const* scores,
                                            const void* const* k, const void* const* v, int64_t kv_row_stride,
                                            int32_t* const* indices, void* const* send, apb_stream_t stream) {
  if (n < 1 || n > kSelMaxHosts) return fail(APB_ERR_CONFIG, "n must be in [1, 8]");
  if (!dims || !scores || !k || !v || !indices || !send) return fail(APB_ERR_CONTRACT, "an array argument is NULL");
  apb_status st;
  const apb_dims* d = &dims[0];
  const int D = d->head_dim, hk = d->n_kv_heads;
  SelHosts sh{};
  sh.n = n;
  for (int i = 0; i < n; ++i) {
    const apb_dims& a = dims[i];
    if ((st = check_dims(&a))) return st;
    if (a.n != d->n || a.H != d->H || a.l_q != d->l_q || a.l_a != d->l_a || a.l_p != d->l_p ||
        a.n_heads != d->n_heads || a.n_kv_heads != hk || a.head_dim != D)
      return fail(APB_ERR_CONFIG, "the hosts of one launch must share every dimension but `host`");
    if (!scores[i] || !indices[i]) return fail(APB_ERR_CONTRACT, "scores/indices NULL");
    if ((st = check_rows(k[i], kv_row_stride, (int64_t)hk * D, "k"))) return st;
    if ((st = check_rows(v[i], kv_row_stride, (int64_t)hk * D, "v"))) return st;
    if (!send[i] || !aligned16(send[i])) return fail(APB_ERR_CONTRACT, "send NULL or misaligned");
    sh.scores[i] = scores[i];
    sh.indices[i] = indices[i];
    sh.k[i] = static_cast<const uint16_t*>(k[i]);
    sh.v[i] = static_cast<const uint16_t*>(v[i]);
    sh.send[i] = static_cast<uint16_t*>(send[i]);
    sh.L_A[i] = (int)L_A_of(&a);
  }
  const int64_t lpp = lpp_of(d);
  if (lpp == 0) return APB_OK;
  if ((st = check_device())) return st;
  return launch_select_compact_hosts(d->l_b, (int)lpp, hk, D, sh, kv_row_stride, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- method variants (NEXT #3)
extern "C" apb_status apb_random_scores(const apb_dims* d, uint64_t seed, int32_t layer, float* scores,
                                        apb_stream_t stream) {
  apb_status st = check_dims(d);
  if (st) return st;
  if (layer < 0) return fail(APB_ERR_CONFIG, "layer must be >= 0");
  if (!scores) return fail(APB_ERR_CONTRACT, "scores NULL");
  if ((st = check_device())) return st;
  const int64_t per_host = (int64_t)d->n_kv_heads * d->l_b;
  const uint64_t c0 = ((uint64_t)layer * (uint64_t)d->H + (uint64_t)d->host) * (uint64_t)per_host;
  return launch_random_scores(seed, c0, per_host, scores, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_share_scores(const apb_dims* d, float* scores, apb_stream_t stream) {
  apb_status st = check_dims(d);
  if (st) return st;
  if (!scores) return fail(APB_ERR_CONTRACT, "scores NULL");
  if ((st = check_device())) return st;
  return launch_share_scores(scores, d->n_kv_heads, d->l_b, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- model layer (NEXT #2)
namespace {
apb_status check_bf16_rows(const void* p, int64_t rows, int64_t stride, int64_t width, const char* what) {
  if (rows == 0) return APB_OK;
  if (!p || !aligned16(p)) return fail(APB_ERR_CONTRACT, std::string(what) + " NULL or not 16-byte aligned");
  if (stride % 8 != 0 || stride < width)
    return fail(APB_ERR_CONTRACT, std::string(what) + " row stride must be a multiple of 8 elements and >= width");
  return APB_OK;
}
}  // namespace

extern "C" apb_status apb_rmsnorm(int64_t rows, int32_t dim, const void* x, int64_t x_stride, const void* w, float eps,
                                  void* out, int64_t out_stride, apb_stream_t stream) {
  if (rows < 0 || dim <= 0 || dim % 8 != 0 || !(eps >= 0.f)) return fail(APB_ERR_CONFIG, "rmsnorm: rows >= 0, dim % 8 == 0, eps >= 0");
  apb_status st;
  if ((st = check_bf16_rows(x, rows, x_stride, dim, "x"))) return st;
  if ((st = check_bf16_rows(out, rows, out_stride, dim, "out"))) return st;
  if (!w || !aligned16(w)) return fail(APB_ERR_CONTRACT, "w NULL or not 16-byte aligned");
  if (rows == 0) return APB_OK;
  if ((st = check_device())) return st;
  return launch_rmsnorm(rows, dim, x, x_stride, w, eps, out, out_stride, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_rope(int64_t rows, int32_t n_heads, int32_t head_dim, void* x, int64_t row_stride,
                               const int32_t* positions, int64_t pos_offset, float theta, apb_stream_t stream) {
  if (rows < 0 || n_heads < 0 || head_dim <= 0 || head_dim % 2 != 0 || head_dim > 256 || !(theta > 0.f))
    return fail(APB_ERR_CONFIG, "rope: rows, n_heads >= 0, even head_dim <= 256, theta > 0");
  if (rows == 0 || n_heads == 0) return APB_OK;
  if (!x) return fail(APB_ERR_CONTRACT, "x NULL");
  if (row_stride < (int64_t)n_heads * head_dim) return fail(APB_ERR_CONTRACT, "row_stride < n_heads * head_dim");
  apb_status st;
  if ((st = check_device())) return st;
  return launch_rope(rows, n_heads, head_dim, x, row_stride, positions, pos_offset, (double)theta,
                     reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_swiglu(int64_t rows, int32_t inter, const void* gu, int64_t gu_stride, void* out,
                                 int64_t out_stride, apb_stream_t stream) {
  if (rows < 0 || inter <= 0 || inter % 8 != 0) return fail(APB_ERR_CONFIG, "swiglu: rows >= 0, inter % 8 == 0");
  apb_status st;
  if ((st = check_bf16_rows(gu, rows, gu_stride, 2 * (int64_t)inter, "gu"))) return st;
  if ((st = check_bf16_rows(out, rows, out_stride, inter, "out"))) return st;
  if (rows == 0) return APB_OK;
  if ((st = check_device())) return st;
  return launch_swiglu(rows, inter, gu, gu_stride, out, out_stride, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_gemm(int64_t M, int32_t N, int32_t K, const void* a, int64_t lda, const void* w,
                               int64_t ldw, void* c, int64_t ldc, const apb_gemm_epi* epi, apb_stream_t stream) {
  if (!epi) return fail(APB_ERR_CONTRACT, "gemm: epi is NULL");
  if (M < 0 || N <= 0 || K <= 0 || N % 8 != 0 || K % 8 != 0)
    return fail(APB_ERR_CONFIG, "gemm: M >= 0, N and K positive multiples of 8");
  const int e = epi->epilogue;
  if (e < APB_EPI_STORE || e > APB_EPI_ROPE) return fail(APB_ERR_CONFIG, "gemm: unknown epilogue");
  if (e == APB_EPI_SWIGLU && N % 256 != 0)
    return fail(APB_ERR_CONFIG, "gemm: SWIGLU needs N % 256 == 0 (gate/up rows interleaved in 128-row blocks)");
  if (e == APB_EPI_ROPE) {
    if (epi->head_dim != 64 && epi->head_dim != 128) return fail(APB_ERR_UNSUPPORTED, "gemm: ROPE head_dim must be 64 or 128");
    if (epi->rope_cols < 0 || epi->rope_cols > N || epi->rope_cols % epi->head_dim || N % epi->head_dim)
      return fail(APB_ERR_CONFIG, "gemm: ROPE needs rope_cols <= N, both multiples of head_dim");
    if (!(epi->theta > 0.f)) return fail(APB_ERR_CONFIG, "gemm: ROPE theta must be > 0");
  }
  apb_status st;
  if ((st = check_bf16_rows(a, M, lda, K, "a"))) return st;
  if ((st = check_bf16_rows(w, N, ldw, K, "w"))) return st;
  if ((st = check_bf16_rows(c, M, ldc, e == APB_EPI_SWIGLU ? N / 2 : N, "c"))) return st;
  if (M == 0) return APB_OK;
  if ((st = check_device())) return st;
  GemmArgs g{M, N, K, a, lda, w, ldw, c, ldc, e, epi->beta, epi->rope_cols, epi->head_dim, epi->theta,
             epi->positions, epi->pos_offset};
  return launch_gemm(g, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_gemm_bf16(int64_t M, int32_t N, int32_t K, const void* a, int64_t lda, const void* w,
                                    int64_t ldw, void* c, int64_t ldc, float beta, void* ws, size_t ws_bytes,
                                    apb_stream_t stream) {
  (void)ws;
  (void)ws_bytes;
  apb_gemm_epi epi{};
  epi.epilogue = beta != 0.f ? APB_EPI_RESIDUAL : APB_EPI_STORE;
  epi.beta = beta;
  return apb_gemm(M, N, K, a, lda, w, ldw, c, ldc, &epi, stream);
}

// ---------------------------------------------------------------- step 3: exchange (NCCL)
struct apb_comm {
  ncclComm_t comm;
  int32_t nranks, rank;
};

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
};
NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // Prefer the NCCL already loaded into the process (torch's), else the system one.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.commGetAsyncError = reinterpret_cast<decltype(api.commGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    api.commAbort = reinterpret_cast<decltype(api.commAbort)>(dlsym(h, "ncclCommAbort"));
    if (api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather) api.h = h;
  });
  return api.h ? &api : nullptr;
}
apb_status nccl_fail(NcclApi* api, ncclResult_t r, const char* what) {
  return fail(APB_ERR_NCCL, std::string(what) + ": " + (api->getErrorString ? api->getErrorString(r) : "nccl error"));
}
}  // namespace

extern "C" apb_status apb_comm_get_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(APB_ERR_CONTRACT, "id_out is NULL");
  NcclApi* api = nccl();
  if (!api) return fail(APB_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId id;
  ncclResult_t r = api->getUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
  static_assert(sizeof(id.internal) == 128, "NCCL unique id is 128 bytes");
  std::memcpy(id_out, id.internal, 128);
  return APB_OK;
}

extern "C" apb_status apb_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, apb_comm** out) {
  if (!id || !out) return fail(APB_ERR_CONTRACT, "id/out is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(APB_ERR_CONFIG, "bad nranks/rank");
  *out = nullptr;
  apb_comm* c = new apb_comm{nullptr, nranks, rank};
  if (nranks > 1) {
    NcclApi* api = nccl();
    if (!api) {
      delete c;
      return fail(APB_ERR_NCCL, "libnccl.so.2 not found");
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ncclResult_t r = api->commInitRank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      return nccl_fail(api, r, "ncclCommInitRank");
    }
  }
  *out = c;
  return APB_OK;
}

extern "C" apb_status apb_comm_destroy(apb_comm* c) {
  if (!c) return APB_OK;
  apb_status st = APB_OK;
  if (c->comm) {
    NcclApi* api = nccl();
    if (api) {
      ncclResult_t r = api->commDestroy(c->comm);
      if (r != ncclSuccess) st = nccl_fail(api, r, "ncclCommDestroy");
    }
  }
  delete c;
  return st;
}

// The exchange plan: the in-place AllGather rounds for rank `rank` of `nranks` (element offsets
// into gathered [H][2][hk][l_p'][d]).  BLOCK ownership is one round over contiguous per-rank slot
// ranges; CYCLIC ownership is H/N rounds, round k gathering slots [k*N, (k+1)*N) one per rank.
// apb_exchange_passing{,_cyclic} enqueue exactly these rounds (the CPU multi-rank tests drive
// their gloo all-gathers from the same function).
static apb_status exchange_plan(const apb_dims* d, int32_t nranks, int32_t rank, int32_t layout, int32_t max_rounds,
                                int64_t* send_off, int64_t* recv_off, int64_t* count, int32_t* n_rounds) {
  apb_status st = check_dims(d);
  if (st) return st;
  if (!n_rounds) return fail(APB_ERR_CONTRACT, "n_rounds is NULL");
  *n_rounds = 0;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(APB_ERR_CONFIG, "bad nranks/rank");
  if (d->H % nranks) return fail(APB_ERR_CONFIG, "comm nranks must divide H");
  if (layout != APB_LAYOUT_BLOCK && layout != APB_LAYOUT_CYCLIC) return fail(APB_ERR_CONFIG, "unknown host layout");
  const int64_t lpp = lpp_of(d);
  if (nranks == 1 || lpp == 0) return APB_OK;  // nothing to exchange
  const int64_t slot = (int64_t)2 * d->n_kv_heads * lpp * d->head_dim;  // bf16 elements per host slot
  const int32_t rounds = layout == APB_LAYOUT_BLOCK ? 1 : d->H / nranks;
  if (max_rounds < rounds) return fail(APB_ERR_CONTRACT, "plan arrays hold fewer than H/nranks rounds");
  if (!send_off || !recv_off || !count) return fail(APB_ERR_CONTRACT, "plan arrays are NULL");
  if (layout == APB_LAYOUT_BLOCK) {
    count[0] = slot * (d->H / nranks);
    recv_off[0] = 0;
    send_off[0] = (int64_t)rank * count[0];
  } else {
    for (int32_t k = 0; k < rounds; ++k) {
      count[k] = slot;
      recv_off[k] = (int64_t)k * nranks * slot;
      send_off[k] = recv_off[k] + (int64_t)rank * slot;
    }
  }
  *n_rounds = rounds;
  return APB_OK;
}

extern "C" apb_status apb_exchange_plan(const apb_dims* d, int32_t nranks, int32_t rank, apb_host_layout layout,
                                        int32_t max_rounds, int64_t* send_offset, int64_t* recv_offset,
                                        int64_t* count, int32_t* n_rounds) {
  return exchange_plan(d, nranks, rank, layout, max_rounds, send_offset, recv_offset, count, n_rounds);
}

// Poll the communicator for an asynchronous NCCL failure (a peer died, a network error): such
// errors surface only here, never as a return code of the enqueueing call.
static apb_status comm_async_check(NcclApi* api, apb_comm* c) {
  if (!c || !c->comm || !api->commGetAsyncError) return APB_OK;
  ncclResult_t async = ncclSuccess;
  ncclResult_t r = api->commGetAsyncError(c->comm, &async);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommGetAsyncError");
  if (async != ncclSuccess && async != ncclInProgress) return nccl_fail(api, async, "NCCL asynchronous error");
  return APB_OK;
}

extern "C" apb_status apb_comm_check(apb_comm* c) {
  if (!c || !c->comm) return APB_OK;
  NcclApi* api = nccl();
  if (!api) return fail(APB_ERR_NCCL, "libnccl.so.2 not found");
  return comm_async_check(api, c);
}

extern "C" apb_status apb_comm_abort(apb_comm* c) {
  if (!c) return APB_OK;
  apb_status st = APB_OK;
  if (c->comm) {
    NcclApi* api = nccl();
    if (api && api->commAbort) {
      ncclResult_t r = api->commAbort(c->comm);
      if (r != ncclSuccess) st = nccl_fail(api, r, "ncclCommAbort");
    }
  }
  delete c;
  return st;
}

static apb_status exchange_impl(apb_comm* c, const apb_dims* d, int32_t layout, void* gathered, apb_stream_t stream) {
  apb_status st = check_dims(d);
  if (st) return st;
  if (!c || c->nranks == 1) return APB_OK;
  const int32_t max_rounds = d->H;
  std::vector<int64_t> send_off(max_rounds), recv_off(max_rounds), count(max_rounds);
  int32_t rounds = 0;
  if ((st = exchange_plan(d, c->nranks, c->rank, layout, max_rounds, send_off.data(), recv_off.data(), count.data(),
                          &rounds)))
    return st;
  if (rounds == 0) return APB_OK;
  if (!gathered || !aligned16(gathered)) return fail(APB_ERR_CONTRACT, "gathered NULL or misaligned");
  NcclApi* api = nccl();
  if (!api) return fail(APB_ERR_NCCL, "libnccl.so.2 not found");
  if ((st = comm_async_check(api, c))) return st;
  char* base = static_cast<char*>(gathered);
  for (int32_t k = 0; k < rounds; ++k) {
    ncclResult_t r = api->allGather(base + send_off[k] * 2, base + recv_off[k] * 2, (size_t)count[k], ncclBfloat16,
                                    c->comm, reinterpret_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return nccl_fail(api, r, layout == APB_LAYOUT_BLOCK ? "ncclAllGather" : "ncclAllGather (cyclic round)");
  }
  return comm_async_check(api, c);
}

extern "C" apb_status apb_exchange_passing(apb_comm* c, const apb_dims* d, void* gathered, apb_stream_t stream) {
  return exchange_impl(c, d, APB_LAYOUT_BLOCK, gathered, stream);
}

extern "C" apb_status apb_exchange_passing_cyclic(apb_comm* c, const apb_dims* d, void* gathered,
                                                  apb_stream_t stream) {
  return exchange_impl(c, d, APB_LAYOUT_CYCLIC, gathered, stream);
}

// ---------------------------------------------------------------- decode step (NEXT #1)
static apb_status check_decode_dims(const apb_decode_dims* d) {
  if (!d) return fail(APB_ERR_CONTRACT, "dims is NULL");
  if (d->H < 1 || d->host < 0 || d->host >= d->H) return fail(APB_ERR_CONFIG, "host must be in [0, H)");
  if (d->t_new < 1 || d->cache_len < 0) return fail(APB_ERR_CONFIG, "t_new >= 1 and cache_len >= 0 required");
  if (d->n_heads < 1 || d->n_kv_heads < 1 || d->n_heads % d->n_kv_heads)
    return fail(APB_ERR_CONFIG, "n_heads must be a positive multiple of n_kv_heads");
  if (d->head_dim != 64 && d->head_dim != 128) return fail(APB_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if ((int64_t)d->t_new * (d->n_heads / d->n_kv_heads) > kDecodeRowsMax)
    return fail(APB_ERR_UNSUPPORTED, "t_new * (n_heads / n_kv_heads) must be <= 64: chunk the new tokens");
  return APB_OK;
}

static int64_t decode_keys(const apb_decode_dims* d) {
  return d->cache_len + (d->host == d->H - 1 ? d->t_new : 0);
}

extern "C" apb_status apb_decode_workspace_size(const apb_decode_dims* d, size_t* bytes) {
  if (!bytes) return fail(APB_ERR_CONTRACT, "bytes is NULL");
  apb_status st = check_decode_dims(d);
  if (st) return st;
  *bytes = decode_workspace_bytes(decode_keys(d), d->t_new, d->n_heads, d->n_kv_heads, d->head_dim);
  return APB_OK;
}

extern "C" apb_status apb_decode_attention(const apb_decode_dims* d, const void* q, const void* k_cache,
                                           const void* v_cache, int64_t cache_row_stride, const void* k_new,
                                           const void* v_new, int64_t new_row_stride, float* part_o, float* part_lse,
                                           void* ws, size_t ws_bytes, apb_stream_t stream) {
  apb_status st = check_decode_dims(d);
  if (st) return st;
  const int D = d->head_dim, hq = d->n_heads, hk = d->n_kv_heads;
  const bool last = d->host == d->H - 1;
  if (!q || !aligned16(q)) return fail(APB_ERR_CONTRACT, "q NULL or misaligned");
  if (d->cache_len > 0) {
    if ((st = check_rows(k_cache, cache_row_stride, (int64_t)hk * D, "k_cache"))) return st;
    if ((st = check_rows(v_cache, cache_row_stride, (int64_t)hk * D, "v_cache"))) return st;
  }
  if (last) {
    if ((st = check_rows(k_new, new_row_stride, (int64_t)hk * D, "k_new"))) return st;
    if ((st = check_rows(v_new, new_row_stride, (int64_t)hk * D, "v_new"))) return st;
  }
  if (!part_o || !part_lse || !aligned16(part_o)) return fail(APB_ERR_CONTRACT, "part_o/part_lse NULL or misaligned");
  const size_t need = decode_workspace_bytes(decode_keys(d), d->t_new, hq, d->n_kv_heads, D);
  if (need && (!ws || ws_bytes < need || !aligned16(ws))) return fail(APB_ERR_CONTRACT, "decode workspace missing or too small");
  if ((st = check_device())) return st;
  DecodeParams p{};
  p.t = d->t_new;
  p.hq = hq;
  p.hk = hk;
  p.g = hq / hk;
  p.D = D;
  p.has_new = last ? 1 : 0;
  p.cache_len = d->cache_len;
  p.cache_row_stride = cache_row_stride;
  p.new_row_stride = new_row_stride;
  const float scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt((float)D);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k_cache = static_cast<const __nv_bfloat16*>(k_cache);
  p.v_cache = static_cast<const __nv_bfloat16*>(v_cache);
  p.k_new = static_cast<const __nv_bfloat16*>(k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(v_new);
  p.ws_o = static_cast<float*>(ws);
  return launch_decode(p, part_o, part_lse, reinterpret_cast<cudaStream_t>(stream));
}

static apb_status check_decode_hosts(const apb_decode_dims* d, int32_t n, const int64_t* cache_lens) {
  apb_status st = check_decode_dims(d);
  if (st) return st;
  if (n < 1 || n > kDecMaxHosts || d->host + n > d->H) return fail(APB_ERR_CONFIG, "n_hosts must be in [1, 16] and host + n_hosts <= H");
  if (!cache_lens) return fail(APB_ERR_CONTRACT, "cache_lens is NULL");
  for (int i = 0; i < n; ++i)
    if (cache_lens[i] < 0) return fail(APB_ERR_CONFIG, "cache_lens[i] >= 0 required");
  return APB_OK;
}

static void decode_hosts_keys(const apb_decode_dims* d, int32_t n, const int64_t* cache_lens, int64_t* keys) {
  for (int i = 0; i < n; ++i) keys[i] = cache_lens[i] + (d->host + i == d->H - 1 ? d->t_new : 0);
}

extern "C" apb_status apb_decode_hosts_workspace_size(const apb_decode_dims* d, int32_t n, const int64_t* cache_lens,
                                                      size_t* bytes) {
  if (!bytes) return fail(APB_ERR_CONTRACT, "bytes is NULL");
  apb_status st = check_decode_hosts(d, n, cache_lens);
  if (st) return st;
  int64_t keys[kDecMaxHosts];
  decode_hosts_keys(d, n, cache_lens, keys);
  *bytes = decode_hosts_workspace_bytes(n, keys, d->t_new, d->n_heads, d->n_kv_heads, d->head_dim);
  return APB_OK;
}

static apb_status decode_hosts_impl(const apb_decode_dims* d, int32_t n, const int64_t* cache_lens,
                                                 const void* const* k_caches, const void* const* v_caches,
                                                 int64_t cache_row_stride, const void* q, const void* k_new,
                                                 const void* v_new, int64_t new_row_stride, float* parts,
                                                 int64_t part_stride, int64_t lse_offset, void* merged_out,
                                                 float* merged_lse, void* ws, size_t ws_bytes, apb_stream_t stream) {
  apb_status st = check_decode_hosts(d, n, cache_lens);
  if (st) return st;
  const int D = d->head_dim, hq = d->n_heads, hk = d->n_kv_heads;
  if (!q || !aligned16(q)) return fail(APB_ERR_CONTRACT, "q NULL or misaligned");
  if (!k_caches || !v_caches) return fail(APB_ERR_CONTRACT, "k_caches/v_caches is NULL");
  DecodeHosts hb{};
  hb.n = n;
  hb.new_host = -1;
  for (int i = 0; i < n; ++i) {
    if (cache_lens[i] > 0) {
      if ((st = check_rows(k_caches[i], cache_row_stride, (int64_t)hk * D, "k_caches[i]"))) return st;
      if ((st = check_rows(v_caches[i], cache_row_stride, (int64_t)hk * D, "v_caches[i]"))) return st;
    }
    hb.cache_len[i] = cache_lens[i];
    hb.k_cache[i] = static_cast<const __nv_bfloat16*>(k_caches[i]);
    hb.v_cache[i] = static_cast<const __nv_bfloat16*>(v_caches[i]);
    if (d->host + i == d->H - 1) hb.new_host = i;
  }
  if (hb.new_host >= 0) {
    if ((st = check_rows(k_new, new_row_stride, (int64_t)hk * D, "k_new"))) return st;
    if ((st = check_rows(v_new, new_row_stride, (int64_t)hk * D, "v_new"))) return st;
  }
  const int64_t rows = (int64_t)d->t_new * hq;
  if (merged_out) {
    if (!aligned16(merged_out)) return fail(APB_ERR_CONTRACT, "out misaligned");
  } else {
    if (!parts || !aligned16(parts)) return fail(APB_ERR_CONTRACT, "parts NULL or misaligned");
    if (part_stride < rows * D + rows || lse_offset < rows * D || lse_offset + rows > part_stride)
      return fail(APB_ERR_CONTRACT, "part_stride / lse_offset do not hold O [rows][head_dim] and lse [rows]");
  }
  int64_t keys[kDecMaxHosts];
  decode_hosts_keys(d, n, cache_lens, keys);
  const size_t need = decode_hosts_workspace_bytes(n, keys, d->t_new, hq, hk, D);
  if (need && (!ws || ws_bytes < need || !aligned16(ws))) return fail(APB_ERR_CONTRACT, "decode workspace missing or too small");
  if ((st = check_device())) return st;
  DecodeParams p{};
  p.t = d->t_new;
  p.hq = hq;
  p.hk = hk;
  p.g = hq / hk;
  p.D = D;
  p.cache_row_stride = cache_row_stride;
  p.new_row_stride = new_row_stride;
  const float scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt((float)D);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k_new = static_cast<const __nv_bfloat16*>(k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(v_new);
  p.ws_o = static_cast<float*>(ws);
  return launch_decode_hosts(p, hb, keys, parts, part_stride, lse_offset, merged_out, merged_lse,
                             reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_decode_attention_hosts(const apb_decode_dims* d, int32_t n, const int64_t* cache_lens,
                                                 const void* const* k_caches, const void* const* v_caches,
                                                 int64_t cache_row_stride, const void* q, const void* k_new,
                                                 const void* v_new, int64_t new_row_stride, float* parts,
                                                 int64_t part_stride, int64_t lse_offset, void* ws, size_t ws_bytes,
                                                 apb_stream_t stream) {
  return decode_hosts_impl(d, n, cache_lens, k_caches, v_caches, cache_row_stride, q, k_new, v_new, new_row_stride,
                           parts, part_stride, lse_offset, nullptr, nullptr, ws, ws_bytes, stream);
}

extern "C" apb_status apb_decode_step_hosts(const apb_decode_dims* d, const int64_t* cache_lens,
                                            const void* const* k_caches, const void* const* v_caches,
                                            int64_t cache_row_stride, const void* q, const void* k_new,
                                            const void* v_new, int64_t new_row_stride, void* out, float* out_lse,
                                            void* ws, size_t ws_bytes, apb_stream_t stream) {
  if (d && (d->host != 0 || d->H > kDecMaxHosts))
    return fail(APB_ERR_CONFIG, "apb_decode_step_hosts needs every host: host == 0 and H <= 16");
  if (!out) return fail(APB_ERR_CONTRACT, "out is NULL");
  return decode_hosts_impl(d, d ? d->H : 0, cache_lens, k_caches, v_caches, cache_row_stride, q, k_new, v_new,
                           new_row_stride, nullptr, 0, 0, out, out_lse, ws, ws_bytes, stream);
}

extern "C" apb_status apb_merge_partials(int32_t n_parts, int64_t rows, int32_t head_dim, const float* parts_o,
                                         int64_t part_stride_o, const float* parts_lse, int64_t part_stride_lse,
                                         void* out, float* out_lse, apb_stream_t stream) {
  if (n_parts < 1 || rows < 0) return fail(APB_ERR_CONFIG, "n_parts >= 1 and rows >= 0 required");
  if (head_dim != 64 && head_dim != 128) return fail(APB_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (!parts_o || !parts_lse || !out) return fail(APB_ERR_CONTRACT, "NULL buffer");
  if (part_stride_o < rows * head_dim || part_stride_lse < rows) return fail(APB_ERR_CONTRACT, "part stride too small");
  apb_status st = check_device();
  if (st) return st;
  return launch_merge(n_parts, rows, head_dim, parts_o, parts_lse, part_stride_o, part_stride_lse, 0, out, true,
                      out_lse, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_exchange_partials(apb_comm* c, int64_t count_per_rank, float* buf, apb_stream_t stream) {
  if (!c || c->nranks == 1 || count_per_rank == 0) return APB_OK;
  if (count_per_rank < 0) return fail(APB_ERR_CONFIG, "count_per_rank < 0");
  if (!buf || !aligned16(buf)) return fail(APB_ERR_CONTRACT, "buf NULL or misaligned");
  NcclApi* api = nccl();
  if (!api) return fail(APB_ERR_NCCL, "libnccl.so.2 not found");
  ncclResult_t r = api->allGather(buf + (size_t)c->rank * count_per_rank, buf, (size_t)count_per_rank, ncclFloat32,
                                  c->comm, reinterpret_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllGather (partials)");
  return APB_OK;
}

extern "C" apb_status apb_exchange_partials_cyclic(apb_comm* c, int32_t H, int64_t slot_count, float* buf,
                                                   apb_stream_t stream) {
  if (!c || c->nranks == 1 || slot_count == 0) return APB_OK;
  if (slot_count < 0 || H < 1 || H % c->nranks) return fail(APB_ERR_CONFIG, "slot_count >= 0 and nranks | H required");
  if (!buf || !aligned16(buf)) return fail(APB_ERR_CONTRACT, "buf NULL or misaligned");
  NcclApi* api = nccl();
  if (!api) return fail(APB_ERR_NCCL, "libnccl.so.2 not found");
  apb_status st = comm_async_check(api, c);
  if (st) return st;
  for (int32_t k = 0; k < H / c->nranks; ++k) {  // round k: slots k*N .. k*N+N-1, one per rank
    float* round = buf + (size_t)k * c->nranks * slot_count;
    ncclResult_t r = api->allGather(round + (size_t)c->rank * slot_count, round, (size_t)slot_count, ncclFloat32,
                                    c->comm, reinterpret_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllGather (partials, cyclic round)");
  }
  return comm_async_check(api, c);
}
