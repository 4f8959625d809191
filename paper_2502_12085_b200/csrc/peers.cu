// peers.cu — the passing-block exchange (Alg. apb_prefill) over peer
// memory instead of NCCL: every rank's exchange buffer is mapped into every other rank's address
// space (CUDA IPC; NVLink / NVSwitch loads and stores between the GPUs of one node), and the
// compaction kernel stores each selected K/V row straight into that host's slot of EVERY rank's
// buffer — the AllGather fused into the gather (select_topk.cu, GatherDst).
//
// Buffer of one rank (one cudaMalloc, one IPC handle):
//   gathered[2]  two [H][2][hk][l_p'][d] bf16 buffers, alternated by layer parity
//   filled[2][H] int32: epoch of the data present in slot s of gathered[parity]
//   consumed[N]  int32: the last epoch rank r has finished reading (released)
// A writer may refill gathered[e & 1] for epoch e only once every rank has released epoch e-2
// (apb_peers_release after its PASSING launch); a reader's PASSING launch waits until the slots
// it reads carry epoch e (apb_peers_wait).  No cycle: releases follow reads, which follow the
// writers' earlier-epoch pushes.
#include <cstring>

#include "internal.h"

struct apb_peers {
  int nranks, rank, H, hk, lpp, D;
  int64_t slot_bytes;      // one host slot of gathered
  size_t gathered_bytes;   // one parity buffer: H slots
  size_t flags_off, bytes;
  char* local;             // this rank's allocation
  char* peer[apb::kMaxPeers];  // every rank's allocation as mapped here (peer[rank] == local)
  uint32_t* counter;       // [H] CTA-completion counters of the gather launches (local only)
  bool opened;
};

namespace apb {
namespace peers {

__global__ void wait_flags_kernel(const int32_t* flags, int n, int32_t epoch) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int32_t v;
    while (true) {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
      if (v >= epoch) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
}

struct PublishArgs {
  int32_t* dst[kMaxPeers];
};
__global__ void publish_kernel(const PublishArgs a, int n, int32_t epoch) {
  __threadfence_system();  // every prior read of this rank's stream is complete (stream order) and ordered
  if (threadIdx.x < n)
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(a.dst[threadIdx.x]), "r"(epoch) : "memory");
}

}  // namespace peers

apb_status launch_wait_flags(const int32_t* flags, int n, int32_t epoch, cudaStream_t stream) {
  if (n <= 0) return APB_OK;
  peers::wait_flags_kernel<<<1, 32, 0, stream>>>(flags, n, epoch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("peer wait launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

apb_status launch_publish(int32_t* const* dsts, int n, int32_t epoch, cudaStream_t stream) {
  peers::PublishArgs a{};
  for (int i = 0; i < n; ++i) a.dst[i] = dsts[i];
  peers::publish_kernel<<<1, 32, 0, stream>>>(a, n, epoch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("peer publish launch: ") + cudaGetErrorString(e));
  count_launch();
  return APB_OK;
}

}  // namespace apb

using apb::fail;

static int32_t* filled_ptr(const apb_peers* p, int r, int parity, int slot) {
  return reinterpret_cast<int32_t*>(p->peer[r] + p->flags_off) + parity * p->H + slot;
}
static int32_t* consumed_ptr(const apb_peers* p, int r, int reader) {
  return reinterpret_cast<int32_t*>(p->peer[r] + p->flags_off) + 2 * p->H + reader;
}

extern "C" apb_status apb_peers_create(const apb_dims* d, int32_t nranks, int32_t rank, apb_peers** out,
                                       uint8_t ipc_handle[64]) {
  if (!out || !ipc_handle) return fail(APB_ERR_CONTRACT, "out/ipc_handle is NULL");
  *out = nullptr;
  apb_status st = apb_check_dims(d);
  if (st) return st;
  if (nranks < 1 || nranks > apb::kMaxPeers || rank < 0 || rank >= nranks)
    return fail(APB_ERR_CONFIG, "nranks must be in [1, 8] and 0 <= rank < nranks");
  if (d->H % nranks) return fail(APB_ERR_CONFIG, "nranks must divide H");
  apb_peers* p = new apb_peers{};
  p->nranks = nranks;
  p->rank = rank;
  p->H = d->H;
  p->hk = d->n_kv_heads;
  p->lpp = d->l_p < d->l_b ? d->l_p : d->l_b;
  p->D = d->head_dim;
  p->slot_bytes = (int64_t)2 * p->hk * p->lpp * p->D * 2;
  p->gathered_bytes = (size_t)p->H * (size_t)p->slot_bytes;
  p->flags_off = (2 * p->gathered_bytes + 255) / 256 * 256;
  p->bytes = p->flags_off + (size_t)(2 * p->H + apb::kMaxPeers) * 4;
  cudaError_t e = cudaMalloc(&p->local, p->bytes);
  if (e == cudaSuccess) e = cudaMemset(p->local + p->flags_off, 0, p->bytes - p->flags_off);
  if (e == cudaSuccess) e = cudaMalloc(&p->counter, (size_t)p->H * 4);
  if (e == cudaSuccess) e = cudaMemset(p->counter, 0, (size_t)p->H * 4);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p->local);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (p->local) cudaFree(p->local);
    if (p->counter) cudaFree(p->counter);
    delete p;
    return fail(APB_ERR_CUDA, std::string("apb_peers_create: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  std::memcpy(ipc_handle, &h, 64);
  p->peer[rank] = p->local;
  *out = p;
  return APB_OK;
}

extern "C" apb_status apb_peers_open(apb_peers* p, const uint8_t* handles) {
  if (!p || !handles) return fail(APB_ERR_CONTRACT, "peers/handles is NULL");
  if (p->opened) return fail(APB_ERR_CONTRACT, "apb_peers_open called twice");
  for (int r = 0; r < p->nranks; ++r) {
    if (r == p->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * r, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(APB_ERR_CUDA, "apb_peers_open: rank " + std::to_string(r) + ": " + cudaGetErrorString(e));
    p->peer[r] = static_cast<char*>(ptr);
  }
  p->opened = true;
  return APB_OK;
}

extern "C" apb_status apb_peers_gathered(const apb_peers* p, int32_t parity, void** gathered) {
  if (!p || !gathered) return fail(APB_ERR_CONTRACT, "peers/gathered is NULL");
  *gathered = p->local + (size_t)(parity & 1) * p->gathered_bytes;
  return APB_OK;
}

extern "C" apb_status apb_select_topk_peers(const apb_dims* d, const float* scores, const void* k, const void* v,
                                            int64_t kv_row_stride, int32_t* indices, apb_peers* p, int32_t epoch,
                                            apb_stream_t stream) {
  apb_status st = apb_check_dims(d);
  if (st) return st;
  if (!p || !p->opened) return fail(APB_ERR_CONTRACT, "peers not opened (apb_peers_open)");
  if (epoch < 1) return fail(APB_ERR_CONFIG, "epoch must be >= 1");
  const int lpp = d->l_p < d->l_b ? d->l_p : d->l_b;
  if (d->H != p->H || d->n_kv_heads != p->hk || lpp != p->lpp || d->head_dim != p->D)
    return fail(APB_ERR_CONFIG, "dims do not match the peer buffers");
  if (lpp == 0) return APB_OK;
  if (!scores || !indices) return fail(APB_ERR_CONTRACT, "scores/indices NULL");
  if (!k || !v || kv_row_stride < (int64_t)p->hk * p->D || kv_row_stride % 8)
    return fail(APB_ERR_CONTRACT, "k/v NULL or bad row stride");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int parity = epoch & 1;
  // gathered[parity] may be refilled once every rank released epoch - 2 (the last use of it)
  if (epoch > 2) {
    if ((st = apb::launch_wait_flags(consumed_ptr(p, p->rank, 0), p->nranks, epoch - 2, s))) return st;
  }
  apb::GatherDst dst{};
  dst.n = p->nranks;
  for (int r = 0; r < p->nranks; ++r) {
    dst.send[r] = reinterpret_cast<uint16_t*>(p->peer[r] + (size_t)parity * p->gathered_bytes +
                                              (size_t)d->host * p->slot_bytes);
    dst.flag[r] = filled_ptr(p, r, parity, d->host);
  }
  dst.counter = p->counter + d->host;
  dst.epoch = epoch;
  const int64_t L_A = d->host == 0 ? 0 : (int64_t)d->l_q + d->l_a;
  return apb::launch_select_compact(d->l_b, lpp, p->hk, p->D, (int)L_A, scores, k, v, kv_row_stride, indices, nullptr,
                                    s, &dst);
}

extern "C" apb_status apb_peers_wait(apb_peers* p, int32_t n_slots, int32_t epoch, apb_stream_t stream) {
  if (!p) return fail(APB_ERR_CONTRACT, "peers is NULL");
  if (n_slots < 0 || n_slots > p->H) return fail(APB_ERR_CONFIG, "n_slots must be in [0, H]");
  if (p->lpp == 0) return APB_OK;
  return apb::launch_wait_flags(filled_ptr(p, p->rank, epoch & 1, 0), n_slots, epoch,
                                reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_peers_release(apb_peers* p, int32_t epoch, apb_stream_t stream) {
  if (!p || !p->opened) return fail(APB_ERR_CONTRACT, "peers not opened (apb_peers_open)");
  int32_t* dsts[apb::kMaxPeers];
  for (int r = 0; r < p->nranks; ++r) dsts[r] = consumed_ptr(p, r, p->rank);
  return apb::launch_publish(dsts, p->nranks, epoch, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" apb_status apb_peers_destroy(apb_peers* p) {
  if (!p) return APB_OK;
  cudaError_t e = cudaDeviceSynchronize();
  for (int r = 0; r < p->nranks; ++r)
    if (r != p->rank && p->peer[r]) cudaIpcCloseMemHandle(p->peer[r]);
  if (p->local) cudaFree(p->local);
  if (p->counter) cudaFree(p->counter);
  delete p;
  if (e != cudaSuccess) return fail(APB_ERR_CUDA, std::string("apb_peers_destroy: ") + cudaGetErrorString(e));
  return APB_OK;
}
