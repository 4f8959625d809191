/*
 * apb.h — C ABI of libapb, the B200 (sm_100a) implementation of APB's per-layer
 * sequence-parallel prefill hot path (arXiv 2502.12085, "APB: Accelerating Distributed
 * Long-Context Inference by Passing Compressed Context Blocks across GPUs").
 *
 * Citations are PAPER.md line numbers of the paper's LaTeX source (P:<line>) plus the
 * algorithm / equation label.  Readings of points the paper leaves open (G1..G16) are
 * listed in DESIGN.md.
 *
 * Per layer, on every host h = host + 1 (one host = one GPU in deployment; several hosts
 * may be emulated on one GPU), Alg. apb_prefill runs four steps:
 *   1. apb_retain_score      s = R([Q_h, K_h, V_h])
 *   2. apb_select_topk       idx = ArgTop-l_p(s); K^C, V^C = K_h[idx], V_h[idx]
 *   3. apb_exchange_passing  AllGather(K^C_h, V^C_h)
 *   4. apb_attention_fwd     Attention([Q_a,Q_h], [K_a,K_p,K_h], [V_a,V_p,V_h])  (eq:apb)
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Tensors are caller-owned DEVICE memory (e.g. torch tensors).  libapb never allocates,
 *    frees or retains them beyond the call's stream work.  Workspace is caller-provided;
 *    query its size with apb_workspace_size().
 *  - bf16 tensors are passed as `const void*` of 16-bit IEEE bfloat16 values.
 *  - Host-local rows: L_A = (host == 0) ? 0 : l_q + l_a anchor rows, then
 *    l_b = n / H block rows.  Q is [L_A + l_b][n_heads][head_dim] with a row stride of
 *    q_row_stride ELEMENTS (>= n_heads*head_dim, multiple of 8); K and V are
 *    [L_A + l_b][n_kv_heads][head_dim] with row stride kv_row_stride.  head_dim is
 *    contiguous; heads are head_dim apart.
 *  - l_p' = min(l_p, l_b) (reading G6).  P_h = host * l_p' passing keys.
 *  - Every call validates synchronously, then enqueues on `stream` and returns without a
 *    host synchronisation.  Ordering across calls/streams is the caller's job (events).
 *  - Errors: no exception crosses the ABI and nothing aborts.  The return value is an
 *    apb_status; apb_last_error() gives a thread-local detail string.
 *      APB_ERR_CONFIG      inconsistent sizes (n != H*l_b, host out of range, ...)
 *      APB_ERR_CONTRACT    NULL / misaligned (16 B) pointer, bad stride, missing buffer
 *      APB_ERR_UNSUPPORTED head_dim not in {64,128}, device not sm_100, d_hidden % 128 != 0
 *      APB_ERR_CUDA        a CUDA call failed (launch error, no device, ...)
 *      APB_ERR_NCCL        NCCL missing or an NCCL call failed
 */
#ifndef APB_H_
#define APB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* apb_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    APB_OK = 0,
    APB_ERR_CONFIG = 1,
    APB_ERR_CONTRACT = 2,
    APB_ERR_UNSUPPORTED = 3,
    APB_ERR_CUDA = 4,
    APB_ERR_NCCL = 5
} apb_status;

/* Problem statement of one host's layer.
 *  n           document length l_d (tokens) — the query part is counted in l_q
 *  H           number of hosts; host in [0, H) is this call's host (h = host + 1)
 *  l_q, l_a    query length and anchor length; anchor = [q_1..q_lq, d_1..d_la] on host >= 1
 *  l_b         block length; must equal n / H exactly (reading G15)
 *  l_p         passing length per host (clamped to l_b)
 *  n_heads, n_kv_heads, head_dim   GQA: query head qh reads KV head qh / (n_heads/n_kv_heads)
 *  softmax_scale   <= 0 selects 1/sqrt(head_dim) (1/sqrt(d_m))            */
typedef struct {
    int64_t n;
    int32_t H, host, l_q, l_a, l_b, l_p;
    int32_t n_heads, n_kv_heads, head_dim;
    float softmax_scale;
} apb_dims;

/* Retaining-head weights of one layer (hidden size d_hidden = 1024 at P:798).
 *   z = W1 x + b1,  a = SiLU(z),  o = W2 a + b2,  s[j] = max_{c in group j} o[c]   (G2, G4)
 *  d_in      must equal (n_heads + 2 n_kv_heads) * head_dim (x = [Q_t | K_t | V_t])
 *  d_hidden  multiple of 256
 *  n_out     n_kv_heads (identity pool) or n_heads (max over each KV head's query group)
 *  w1  bf16 [d_hidden][d_in] row-major (device);  b1 fp32 [d_hidden] or NULL;
 *  w2  fp32 [n_out][d_hidden] row-major;          b2 fp32 [n_out] or NULL.            */
typedef struct {
    int32_t d_in, d_hidden, n_out;
    const void* w1;
    const float* b1;
    const float* w2;
    const float* b2;
} apb_retain_weights;

typedef enum {
    APB_PHASE_ALL = 0,     /* whole eq:apb in one launch                                         */
    APB_PHASE_LOCAL = 1,   /* anchor rows (final) + local rows over anchor and local keys;
                              local rows go to the workspace as an (O, lse) partial when P_h > 0,
                              else straight to `out` (no passing needed)                         */
    APB_PHASE_PASSING = 2  /* local rows over the passing keys, merged with the LOCAL partial by
                              its log-sum-exp (exact online-softmax merge, P:753 MergeScore);
                              writes the final `out` rows [L_A, L_A+l_b).  No-op if P_h == 0.   */
} apb_phase;

typedef enum { APB_WS_RETAIN = 0, APB_WS_SELECT = 1, APB_WS_ATTENTION = 2 } apb_ws_kind;

/* ---------------------------------------------------------------- step 1: scoring
 * scores[j][t] (fp32 [n_kv_heads][l_b]) for block rows t = L_A .. L_A+l_b-1 of q/k/v.
 * Kernel: tcgen05 GEMM (A = [Q|K|V] rows via three TMA maps, B = W1) with a fused fp32
 * epilogue (b1, SiLU, W2 dot), then b2 and the group max.  Deterministic (no atomics).
 * ws: caller-owned device workspace of apb_retain_workspace_size() bytes (16-byte aligned;
 * fp32 partial W2 sums [d_hidden/128][n_out][l_b]: one slot per 128 hidden units).  With it the CTA-pair GEMM runs (each
 * pair 256 tokens x 256 hidden units, the [Q|K|V] rows read from HBM about once); with ws ==
 * NULL (or too small) a single-CTA kernel (128 tokens x all of d_hidden) computes the same
 * definition in its own fixed summation order.  d_hidden % 256 == 0 and n_out <= 64, else
 * APB_ERR_UNSUPPORTED.                                                                   */
apb_status apb_retain_score(const apb_dims* dims, const apb_retain_weights* w,
                            const void* q, const void* k, const void* v,
                            int64_t q_row_stride, int64_t kv_row_stride,
                            float* scores, void* ws, size_t ws_bytes, apb_stream_t stream);
apb_status apb_retain_workspace_size(const apb_dims* dims, const apb_retain_weights* w, size_t* bytes);
/* The scoring of n (1..8) hosts of one rank in ONE GEMM launch (plus one finalize launch) — the
 * same scores, bit for bit, as n apb_retain_score calls with the CTA-pair GEMM (Alg. apb_prefill
 * line "retain", runs on every host; a rank owning several hosts runs them all).
 *  dims[i]  host i's dims (every field equal across entries except `host`, else APB_ERR_CONFIG)
 *  q/k/v/scores: HOST arrays of n per-host device pointers as in apb_retain_score; strides shared
 *  ws       n x apb_retain_workspace_size() bytes (host i's partials at i x that size), required */
apb_status apb_retain_score_hosts(int32_t n, const apb_dims* dims, const apb_retain_weights* w,
                                  const void* const* q, const void* const* k, const void* const* v,
                                  int64_t q_row_stride, int64_t kv_row_stride, float* const* scores,
                                  void* ws, size_t ws_bytes, apb_stream_t stream);

/* ---------------------------------------------------------------- step 2: select + compact
 * For each KV head j: idx[j] = the l_p' block indices with the largest scores[j][.]
 * (ties -> lower index, reading G5), written ASCENDING to indices (int32 [n_kv_heads][l_p']),
 * then send[0][j][m] = K[L_A + idx[j][m]][j][:], send[1][j][m] = V[...] (bf16
 * [2][n_kv_heads][l_p'][head_dim], contiguous).  -0.0 and +0.0 compare equal.
 * `send` may alias gathered + host * slot (the in-place AllGather layout); no other aliasing. */
apb_status apb_select_topk(const apb_dims* dims, const float* scores,
                           const void* k, const void* v, int64_t kv_row_stride,
                           int32_t* indices, void* send, void* ws, size_t ws_bytes,
                           apb_stream_t stream);
/* The selection + compaction of n (1..8) hosts of one rank in one select launch and one gather
 * launch (l_b <= 32K; above, one launch per host) — bit-identical to n apb_select_topk calls.
 *  dims[i]  host i's dims (every field equal across entries except `host`, else APB_ERR_CONFIG)
 *  scores/k/v/indices/send: HOST arrays of n per-host device pointers as in apb_select_topk */
apb_status apb_select_topk_hosts(int32_t n, const apb_dims* dims, const float* const* scores,
                                 const void* const* k, const void* const* v, int64_t kv_row_stride,
                                 int32_t* const* indices, void* const* send, apb_stream_t stream);

/* ---------------------------------------------------------------- method variants (NEXT #3)
 * Compressor and selection variants of the ablation lattice (Table 4).
 *
 * apb_random_scores — the random selector "Rd.": writes
 * scores[j][t] (fp32 [n_kv_heads][l_b]) = uniform in [0,1) drawn from counter
 *   c = ((layer * H + host) * n_kv_heads + j) * l_b + t
 * as the top 24 bits (times 2^-24) of the (c+1)-th output of a SplitMix64 stream seeded with
 * `seed` (reading G17).  Feeding these to apb_select_topk picks a uniformly random
 * l_p'-subset per KV head.  Deterministic; layer >= 0 (else APB_ERR_CONFIG).
 *
 * apb_share_scores — the shared-index-set reading (one index list per host,
 * Alg. apb_prefill): in place, every row j of scores (fp32 [n_kv_heads][l_b]) becomes
 * max over KV heads of scores[.][t]; apb_select_topk then returns the same set for every head.
 * Both: caller-owned device buffer, enqueued on `stream`, APB_ERR_CONTRACT on NULL.        */
apb_status apb_random_scores(const apb_dims* dims, uint64_t seed, int32_t layer, float* scores,
                             apb_stream_t stream);
apb_status apb_share_scores(const apb_dims* dims, float* scores, apb_stream_t stream);

/* ---------------------------------------------------------------- model layer (NEXT #2)
 * The model steps of Alg. apb_prefill around the hot path: qkv_proj and
 * FFN of a Llama-style decoder layer (the paper's backbones).  All tensors
 * are caller-owned bf16 device rows (16-byte aligned, row strides in ELEMENTS, multiples of
 * 8); element math is fp32 and each output is rounded once to bf16 (reading G9).  rows == 0
 * is a no-op.  Errors: APB_ERR_CONFIG for bad sizes, APB_ERR_CONTRACT for bad pointers or
 * strides (both before any launch), APB_ERR_CUDA for launch failures.
 *
 * apb_rmsnorm — out[r] = x[r] / sqrt(mean(x[r]^2) + eps) * w   (w: bf16 [dim]; dim % 8 == 0).
 *   x and out may alias (same rows, same stride).
 * apb_rope — in place on rows of x: for each of the n_heads consecutive heads (head_dim
 *   elements each) of row r, the pairs (x_i, x_{i+d/2}), i < d/2, are rotated by angle
 *   pos(r) * theta^(-2i/d) (rotate-half RoPE as in Llama).  pos(r) = positions[r] (int32
 *   device array) or, if positions == NULL, pos_offset + r (reading G19: the host's local row
 *   index, so the anchor gets the starting positions 0..l_q+l_a-1 of P:160).  Angles are
 *   reduced in fp64.  head_dim even and <= 256.
 * apb_swiglu — out[r][c] = SiLU(gu[r][c]) * gu[r][inter + c]   (inter % 8 == 0).
 * apb_gemm_bf16 — C[M][N] = A[M][K] W[N][K]^T + beta * C (fp32 accumulate; beta = 1 adds the
 *   residual in place): apb_gemm with the STORE (beta == 0) or RESIDUAL epilogue.  ws and
 *   ws_bytes are ignored (kept for ABI compatibility).
 *   With beta != 0 the result is bf16(beta * C + bf16(A W^T)) — the product is rounded before
 *   the add, exactly as a bf16 PyTorch residual add (reading G20).
 * apb_gemm — the same product on libapb's tcgen05 GEMM (CTA pairs, 256 x 256 tiles, TMA,
 *   TMEM double buffering) with an elementwise step fused into its epilogue (P:708 qkv_proj +
 *   RoPE, P:730 FFN):
 *     STORE     C = bf16(A W^T)
 *     RESIDUAL  C = bf16(beta * C + bf16(A W^T))                              (in place, G20)
 *     SWIGLU    W's rows are [gate; up] interleaved in 128-row blocks (rows 256b..256b+127 =
 *               gate rows 128b.., rows 256b+128.. = up rows 128b..); C is the activation
 *               [M][N/2]: C[r][128b+i] = bf16(SiLU(g) * u), g, u the bf16-rounded products.
 *               N % 256 == 0.
 *     ROPE      C = bf16(A W^T), then the columns [0, rope_cols) (whole heads of head_dim 64 or
 *               128, e.g. the Q and K heads of a qkv row) are rotated exactly as apb_rope does
 *               with pos(r) = positions[r] or pos_offset + r.
 *   M >= 0; N, K multiples of 8; A, W, C 16-byte aligned with row strides (elements) multiples
 *   of 8.  C must not alias A or W.  Errors as above, plus APB_ERR_UNSUPPORTED for a ROPE
 *   head_dim outside {64, 128}.                                                           */
apb_status apb_rmsnorm(int64_t rows, int32_t dim, const void* x, int64_t x_stride, const void* w, float eps,
                       void* out, int64_t out_stride, apb_stream_t stream);
apb_status apb_rope(int64_t rows, int32_t n_heads, int32_t head_dim, void* x, int64_t row_stride,
                    const int32_t* positions, int64_t pos_offset, float theta, apb_stream_t stream);
apb_status apb_swiglu(int64_t rows, int32_t inter, const void* gu, int64_t gu_stride, void* out,
                      int64_t out_stride, apb_stream_t stream);
apb_status apb_gemm_bf16(int64_t M, int32_t N, int32_t K, const void* a, int64_t lda, const void* w,
                         int64_t ldw, void* c, int64_t ldc, float beta, void* ws, size_t ws_bytes,
                         apb_stream_t stream);
typedef enum { APB_EPI_STORE = 0, APB_EPI_RESIDUAL = 1, APB_EPI_SWIGLU = 2, APB_EPI_ROPE = 3 } apb_gemm_epilogue;
typedef struct {
    int32_t epilogue;          /* apb_gemm_epilogue                                        */
    float beta;                /* RESIDUAL                                                 */
    int32_t rope_cols;         /* ROPE: rotated columns [0, rope_cols)                     */
    int32_t head_dim;          /* ROPE: 64 or 128                                          */
    float theta;               /* ROPE: base                                               */
    const int32_t* positions;  /* ROPE: int32 [M] device array, or NULL                    */
    int64_t pos_offset;        /* ROPE: pos(r) = pos_offset + r when positions == NULL     */
} apb_gemm_epi;
apb_status apb_gemm(int64_t M, int32_t N, int32_t K, const void* a, int64_t lda, const void* w, int64_t ldw,
                    void* c, int64_t ldc, const apb_gemm_epi* epi, apb_stream_t stream);

/* ---------------------------------------------------------------- step 3: exchange
 * One in-place AllGather of the packed compressed blocks over NCCL (the
 * paper's two AllGathers of K and V are fused into one, reading G11).
 * gathered: bf16 [H][2][n_kv_heads][l_p'][head_dim].  The comm's nranks must divide H; rank
 * r owns (and must already have written) slots [r*H/nranks, (r+1)*H/nranks).  After the
 * call (in stream order) every slot holds that host's payload on every rank.  A comm with
 * nranks == 1 (or comm == NULL) makes this a no-op.  dims->host is not used.           */
typedef struct apb_comm apb_comm;
apb_status apb_comm_get_unique_id(uint8_t id_out[128]);
apb_status apb_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, apb_comm** out);
apb_status apb_comm_destroy(apb_comm* comm);
apb_status apb_exchange_passing(apb_comm* comm, const apb_dims* dims, void* gathered,
                                apb_stream_t stream);
/* The same exchange for CYCLIC host ownership (N < H ranks, work-balanced: the later hosts carry
 * more passing keys, so rank r owning hosts r, r+N, r+2N, ... levels the per-rank attention
 * work that contiguous blocks skew towards the last rank).  H/N in-place AllGathers, round k
 * gathering slots [k*N, (k+1)*N) in host order.  Same buffer, same result; equal to
 * apb_exchange_passing when N == H.                                                      */
apb_status apb_exchange_passing_cyclic(apb_comm* comm, const apb_dims* dims, void* gathered,
                                       apb_stream_t stream);

/* Host ownership of a multi-rank run: BLOCK = rank r owns hosts
 * [r*H/N, (r+1)*H/N); CYCLIC = rank r owns hosts r, r+N, r+2N, ...                        */
typedef enum { APB_LAYOUT_BLOCK = 0, APB_LAYOUT_CYCLIC = 1 } apb_host_layout;

/* The exchange plan (host-only, no GPU needed): the in-place AllGather rounds that
 * apb_exchange_passing (BLOCK) / apb_exchange_passing_cyclic (CYCLIC) enqueue for rank `rank`
 * of `nranks`.  Round i gathers count[i] bf16 ELEMENTS per rank: this rank's payload is
 * gathered[send_offset[i] .. + count[i]) and the round fills gathered[recv_offset[i] ..
 * + nranks*count[i]) with rank r's payload at recv_offset[i] + r*count[i].  The arrays are
 * caller-owned with max_rounds entries (H/nranks always suffices); *n_rounds gets the number of
 * rounds (0 when nranks == 1 or l_p' == 0: nothing to exchange).  Errors: APB_ERR_CONFIG for
 * bad dims / nranks not dividing H / unknown layout; APB_ERR_CONTRACT for NULL arrays or
 * max_rounds too small.  P:194-197.                                            */
apb_status apb_exchange_plan(const apb_dims* dims, int32_t nranks, int32_t rank, apb_host_layout layout,
                             int32_t max_rounds, int64_t* send_offset, int64_t* recv_offset, int64_t* count,
                             int32_t* n_rounds);

/* ---- the exchange over peer memory (one node: NVLink / NVSwitch P2P through CUDA IPC) ----
 * An alternative to apb_exchange_passing that fuses the AllGather into the compaction
 * (P:194-197): libapb allocates each rank's exchange buffer — two `gathered` buffers
 * bf16 [H][2][n_kv_heads][l_p'][head_dim] alternated by layer parity (epoch & 1), plus flag words
 * — and apb_select_topk_peers stores every selected K/V row of host `dims->host` straight into
 * that slot of EVERY rank's buffer, then publishes `epoch` in every rank's flag for the slot.
 *   apb_peers_create  allocate this rank's buffer; returns its 64-byte CUDA IPC handle
 *   apb_peers_open    map every other rank's buffer from the [nranks][64] handles (the caller
 *                     all-gathers the handles, e.g. torch.distributed.all_gather_object)
 *   apb_peers_gathered  this rank's gathered buffer for a parity (device pointer, library-owned)
 *   apb_select_topk_peers  apb_select_topk with the fused push; epoch >= 1 increases by one per
 *                     layer; it first waits until every rank released epoch - 2 (same buffer)
 *   apb_peers_wait    enqueue a wait until slots [0, n_slots) of gathered[epoch & 1] hold epoch
 *                     (before the PASSING attention that reads them)
 *   apb_peers_release enqueue "this rank finished reading epoch" on every rank (after PASSING)
 *   apb_peers_destroy free (after a barrier: no rank may still write into this buffer)
 * Ownership: the buffers are library-owned; callers read gathered through the returned pointer.
 * Errors: APB_ERR_CONFIG (nranks outside [1, 8], not dividing H, dims not matching), APB_ERR_CONTRACT
 * (NULL / unopened), APB_ERR_CUDA (allocation, IPC, launch).  Waits are device-side spins: every
 * rank must keep issuing its pushes and releases, as in any collective.                        */
typedef struct apb_peers apb_peers;
apb_status apb_peers_create(const apb_dims* dims, int32_t nranks, int32_t rank, apb_peers** out,
                            uint8_t ipc_handle[64]);
apb_status apb_peers_open(apb_peers* peers, const uint8_t* handles);
apb_status apb_peers_gathered(const apb_peers* peers, int32_t parity, void** gathered);
apb_status apb_select_topk_peers(const apb_dims* dims, const float* scores, const void* k, const void* v,
                                 int64_t kv_row_stride, int32_t* indices, apb_peers* peers, int32_t epoch,
                                 apb_stream_t stream);
apb_status apb_peers_wait(apb_peers* peers, int32_t n_slots, int32_t epoch, apb_stream_t stream);
apb_status apb_peers_release(apb_peers* peers, int32_t epoch, apb_stream_t stream);
apb_status apb_peers_destroy(apb_peers* peers);

/* Polls the communicator for an asynchronous NCCL error (ncclCommGetAsyncError): a failure of
 * an already-enqueued collective (peer lost, network error) surfaces here as APB_ERR_NCCL with
 * the NCCL message in apb_last_error().  apb_exchange_passing{,_cyclic} poll before and after
 * they enqueue.  APB_OK for a NULL or 1-rank comm.                                          */
apb_status apb_comm_check(apb_comm* comm);
/* Aborts (ncclCommAbort: does not wait for pending collectives) and frees the comm — the
 * recovery path after apb_comm_check reported an error.                                   */
apb_status apb_comm_abort(apb_comm* comm);

/* ---------------------------------------------------------------- step 4: masked attention
 * eq:apb: for query head qh and query row r in [0, L_A + l_b), with the key
 * sequence [anchor rows of k | passing P_h | block rows of k] (passing = slots 0..host-1 of
 * gathered, host order then ascending index):
 *   r <  L_A : keys 0..r                                     (anchor: causal over the anchor)
 *   r >= L_A : all L_A anchor keys, all P_h passing keys, block keys 0..r-L_A   (reading G1)
 *   out[r][qh] = sum softmax(scale q.k) v (bf16), lse[qh][r] = log sum exp (fp32, natural log)
 * gathered may be NULL iff P_h == 0 or phase == APB_PHASE_LOCAL.
 * out: bf16 rows with out_row_stride elements (multiple of 8).  lse: NULL or [n_heads][L_A+l_b].
 * ws: APB_WS_ATTENTION bytes, shared by the LOCAL and PASSING calls of one layer.
 * Kernel: warp-specialised tcgen05 (TMEM accumulators, TMA loads, online softmax),
 * fully masked tiles never visited; persistent (one CTA per SM taking work items from a
 * per-launch counter slot, 64 slots per device) for APB_PHASE_ALL / PASSING, so at most 64
 * attention launches may run concurrently on one device (launches on one stream never do).  */
apb_status apb_attention_fwd(const apb_dims* dims, const void* q, const void* k, const void* v,
                             int64_t q_row_stride, int64_t kv_row_stride, const void* gathered,
                             void* out, int64_t out_row_stride, float* lse, apb_phase phase,
                             void* ws, size_t ws_bytes, apb_stream_t stream);

/* The same attention for n (1..8) hosts of ONE rank in one kernel launch — exactly the n
 * apb_attention_fwd calls, with one grid over every host's work items, so the per-host launch
 * ramp and tail are paid once (Alg. apb_prefill P:728 runs on every host; a rank that owns
 * several hosts, N < H, runs them all).
 *  dims[i]    host i's dims: every field equal across the n entries except `host`, and no host
 *             twice (else APB_ERR_CONFIG).
 *  q/k/v/out/lse/ws/ws_bytes: HOST arrays of n per-host values, each as in apb_attention_fwd
 *             (lse and ws/ws_bytes may be NULL arrays: no lse / no workspace); strides shared.
 *  gathered   the one passing buffer every host reads (its own slots 0..host-1).
 * Validation is per host, as apb_attention_fwd; nothing is launched unless every host passes.
 * Items run heaviest host first (the lightest host's items form the launch's tail).
 * Outputs are bit-identical to the per-host calls.                                           */
apb_status apb_attention_fwd_hosts(int32_t n, const apb_dims* dims, const void* const* q,
                                   const void* const* k, const void* const* v, int64_t q_row_stride,
                                   int64_t kv_row_stride, const void* gathered, void* const* out,
                                   int64_t out_row_stride, float* const* lse, apb_phase phase,
                                   void* const* ws, const size_t* ws_bytes, apb_stream_t stream);

/* ---------------------------------------------------------------- decode step
 * Alg. apb_decode ("Accu"): after prefill every host holds its block's KV cache
 * (P:675-678).  For t new tokens (t = 1 when generating; the whole query chunk on the first
 * decoding iteration) host h computes a partial attention of their queries over its cache
 * (P:745-746); the last host (host == H-1) also attends to the new tokens' own keys, causally
 * among them.  The partials are gathered and merged by log-sum-exp
 * (MergeScore) — exact attention over [B_1 .. B_H | new tokens].
 *  cache_len      rows of this host's cache (K/V: [cache_len][n_kv_heads][head_dim], row stride
 *                 cache_row_stride elements, multiple of 8; may be 0)
 *  t_new          new tokens; t_new * (n_heads / n_kv_heads) must be <= 64 (else
 *                 APB_ERR_UNSUPPORTED: chunk the query)                                       */
typedef struct {
    int32_t H, host, t_new;
    int64_t cache_len;
    int32_t n_heads, n_kv_heads, head_dim;
    float softmax_scale;  /* <= 0 selects 1/sqrt(head_dim) */
} apb_decode_dims;

/* Partial attention of host `host`: q bf16 [t_new][n_heads][head_dim]; k_new/v_new bf16
 * [t_new][n_kv_heads][head_dim] (row stride new_row_stride; read only when host == H-1, may be
 * NULL otherwise).  Writes part_o fp32 [t_new][n_heads][head_dim] (normalised) and part_lse fp32
 * [t_new][n_heads] (natural log; -inf for a row that sees no key).  ws: apb_decode_workspace_size
 * bytes; one workspace per concurrently running call.
 * Kernels: split-KV over ~2 CTAs per SM x KV heads, each streaming 64-key chunks through a
 * cp.async ring with both products on the tensor cores (mma.sync bf16, fp32 accumulate) and an
 * online softmax across its chunks; then a log-sum-exp fold of the splits (fixed order:
 * deterministic).                                                                              */
apb_status apb_decode_attention(const apb_decode_dims* dims, const void* q, const void* k_cache,
                                const void* v_cache, int64_t cache_row_stride, const void* k_new,
                                const void* v_new, int64_t new_row_stride, float* part_o,
                                float* part_lse, void* ws, size_t ws_bytes, apb_stream_t stream);
apb_status apb_decode_workspace_size(const apb_decode_dims* dims, size_t* bytes);

/* The partials of the n_hosts consecutive hosts one rank owns (dims->host .. dims->host +
 * n_hosts - 1; N < H ranks emulate several hosts per GPU), in ONE launch of the streaming kernel
 * and ONE fold launch instead of n_hosts of each.  Host i has its own cache k_caches[i] /
 * v_caches[i] of cache_lens[i] rows (row stride cache_row_stride; dims->cache_len is ignored);
 * the host with index H-1, if in range, also attends to k_new/v_new.  Host i's partial is
 * written to parts + i*part_stride: O fp32 [t_new][n_heads][head_dim] at float offset 0 and lse
 * fp32 [t_new][n_heads] (natural log) at float offset lse_offset.  k_caches, v_caches and
 * cache_lens are HOST arrays of n_hosts entries, 1 <= n_hosts <= 16 (else APB_ERR_CONFIG);
 * ws: apb_decode_hosts_workspace_size bytes.  Same partials as n_hosts calls of
 * apb_decode_attention up to the split plan (the fp32 summation order).                       */
apb_status apb_decode_attention_hosts(const apb_decode_dims* dims, int32_t n_hosts, const int64_t* cache_lens,
                                      const void* const* k_caches, const void* const* v_caches,
                                      int64_t cache_row_stride, const void* q, const void* k_new,
                                      const void* v_new, int64_t new_row_stride, float* parts,
                                      int64_t part_stride, int64_t lse_offset, void* ws, size_t ws_bytes,
                                      apb_stream_t stream);
apb_status apb_decode_hosts_workspace_size(const apb_decode_dims* dims, int32_t n_hosts, const int64_t* cache_lens,
                                           size_t* bytes);
/* The whole decode step when ONE rank holds every host (N = 1; dims->host == 0, H <= 16 caches,
 * host arrays as above): the partial streaming launch of apb_decode_attention_hosts followed by
 * MergeScore directly over every host's splits — no per-host partials, no Gather (the
 * log-sum-exp merge is associative, so the grouping does not change the result beyond fp32
 * summation order).  out bf16 [t_new][n_heads][head_dim]; out_lse fp32 [t_new][n_heads] (natural
 * log) or NULL.  ws: apb_decode_hosts_workspace_size(dims, H, cache_lens) bytes.               */
apb_status apb_decode_step_hosts(const apb_decode_dims* dims, const int64_t* cache_lens, const void* const* k_caches,
                                 const void* const* v_caches, int64_t cache_row_stride, const void* q,
                                 const void* k_new, const void* v_new, int64_t new_row_stride, void* out,
                                 float* out_lse, void* ws, size_t ws_bytes, apb_stream_t stream);

/* MergeScore: out[r] = sum_h parts_o[h][r] * exp(parts_lse[h][r] - L[r]),
 * L[r] = log sum_h exp(parts_lse[h][r]).  parts_o fp32 with part stride part_stride_o floats
 * (rows x head_dim each), parts_lse fp32 with part stride part_stride_lse; out bf16 [rows][head_dim];
 * out_lse fp32 [rows] or NULL.  Deterministic (fixed host order).                            */
apb_status apb_merge_partials(int32_t n_parts, int64_t rows, int32_t head_dim, const float* parts_o,
                              int64_t part_stride_o, const float* parts_lse, int64_t part_stride_lse,
                              void* out, float* out_lse, apb_stream_t stream);

/* Gather of the partials: in-place AllGather of fp32 buffer [nranks][count_per_rank]
 * (rank r owns block r).  No-op for comm == NULL or a 1-rank comm.                             */
apb_status apb_exchange_partials(apb_comm* comm, int64_t count_per_rank, float* buf, apb_stream_t stream);

/* The same Gather for CYCLIC host ownership (rank r owns hosts r, r+N, ...): buf is fp32
 * [H][slot_count], host h's partial in slot h; H/N in-place AllGather rounds, round k gathering
 * slots [k*N, (k+1)*N) (one per rank), so every slot ends in host order on every rank.  No-op
 * for comm == NULL or a 1-rank comm; APB_ERR_CONFIG unless nranks divides H.                */
apb_status apb_exchange_partials_cyclic(apb_comm* comm, int32_t H, int64_t slot_count, float* buf,
                                        apb_stream_t stream);

/* ---------------------------------------------------------------- plumbing */
apb_status apb_workspace_size(const apb_dims* dims, apb_ws_kind which, size_t* bytes);
/* Validates dims alone (APB_ERR_CONFIG / APB_ERR_UNSUPPORTED) without touching a GPU. */
apb_status apb_check_dims(const apb_dims* dims);
const char* apb_status_string(apb_status s);
const char* apb_last_error(void);
int32_t apb_version(void);

/* Counts of kernel launches issued by this process (for the bench's gpu_launches claim). */
int64_t apb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* APB_H_ */
