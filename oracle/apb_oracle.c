/*
 * apb_oracle.c — plain, slow, fp64 CPU oracle for the APB prefill hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2502_12085_b200/csrc).
 *
 * Every function follows the paper's definition step by step, in fp64, with no
 * blocking, fusion or reordering beyond what the definition states.  Citations:
 * PAPER.md line numbers (P:<line>) inside arXiv 2502.12085's LaTeX source.
 *
 *   oracle_retain_score  P:171-180 (retaining heads R take [Q,K,V], output
 *                        importance scores), P:712 (Alg. apb_prefill line retbeg),
 *                        P:798 (intermediate size 1024).  Readings G2/G3/G4 of
 *                        2-layer MLP with SiLU, per-KV-head max-pool of
 *                        the n_out outputs.
 *   oracle_select_topk   P:180 (Top-l_p), P:713 (ArgTop-l_p).  Reading G5: ties go to
 *                        the lower index; returned ascending.
 *   oracle_attention     P:112 (softmax(M . QK^T/sqrt(d_m)) V), P:203-221 and
 *                        eq:apb (Q = [Q_a, Q_h], K = [K_a, K_p, K_h]), reading G1 of
 *                        DESIGN.md for M' (anchor rows causal over the anchor; local
 *                        rows see all anchor + all passing keys + causal local keys).
 *                        Two-pass softmax, not online.
 *
 * Compaction, AllGather and passing-block construction (P:177-178, P:194-197,
 * P:714-723) are pure indexing/concatenation and live in oracle/__init__.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ scoring */
/* x: [l_b][d_in] = per block token t, concat(Q[t, 0..hq-1, :], K[t, 0..hk-1, :], V[t, 0..hk-1, :])
 * w1: [d_hidden][d_in], b1: [d_hidden] (may be NULL), w2: [n_out][d_hidden], b2: [n_out] (may be NULL)
 * s:  [hk][l_b] output.   n_out must be a multiple of hk; r = n_out / hk.
 *   z_u = sum_i W1[u][i] x_i + b1[u]          (u < d_hidden)
 *   a_u = z_u / (1 + exp(-z_u))               (SiLU)
 *   o_c = sum_u W2[c][u] a_u + b2[c]
 *   s[j][t] = max_{c in [j r, (j+1) r)} o_c
 */
int oracle_retain_score(int64_t l_b, int32_t d_in, int32_t d_hidden, int32_t n_out, int32_t hk,
                        const double* x, const double* w1, const double* b1,
                        const double* w2, const double* b2, double* s) {
    if (l_b < 0 || d_in <= 0 || d_hidden <= 0 || hk <= 0 || n_out <= 0 || n_out % hk) return 1;
    const int32_t r = n_out / hk;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < l_b; ++t) {
        const double* xt = x + t * (int64_t)d_in;
        double* a = (double*)malloc(sizeof(double) * (size_t)d_hidden);
        double* o = (double*)malloc(sizeof(double) * (size_t)n_out);
        for (int32_t u = 0; u < d_hidden; ++u) {
            double z = 0.0;
            const double* wu = w1 + (int64_t)u * d_in;
            for (int32_t i = 0; i < d_in; ++i) z += wu[i] * xt[i];
            if (b1) z += b1[u];
            a[u] = z / (1.0 + exp(-z));
        }
        for (int32_t c = 0; c < n_out; ++c) {
            double acc = 0.0;
            const double* wc = w2 + (int64_t)c * d_hidden;
            for (int32_t u = 0; u < d_hidden; ++u) acc += wc[u] * a[u];
            if (b2) acc += b2[c];
            o[c] = acc;
        }
        for (int32_t j = 0; j < hk; ++j) {
            double m = o[j * r];
            for (int32_t c = 1; c < r; ++c)
                if (o[j * r + c] > m) m = o[j * r + c];
            s[(int64_t)j * l_b + t] = m;
        }
        free(a);
        free(o);
    }
    return 0;
}

/* ------------------------------------------------------------------ selection */
typedef struct { double v; int64_t i; } oracle_kv;

/* order: larger score first; equal scores -> lower index first (reading G5) */
static int cmp_desc_then_index(const void* pa, const void* pb) {
    const oracle_kv* a = (const oracle_kv*)pa;
    const oracle_kv* b = (const oracle_kv*)pb;
    if (a->v > b->v) return -1;
    if (a->v < b->v) return 1;
    return (a->i < b->i) ? -1 : (a->i > b->i);
}

static int cmp_int32_asc(const void* pa, const void* pb) {
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    return (a > b) - (a < b);
}

/* One KV head: indices of the min(l_p, l_b) largest scores, ascending. */
int oracle_select_topk(int64_t l_b, int64_t l_p, const double* s, int32_t* idx) {
    if (l_b < 0 || l_p < 0) return 1;
    int64_t k = l_p < l_b ? l_p : l_b;
    if (k == 0) return 0;
    oracle_kv* all = (oracle_kv*)malloc(sizeof(oracle_kv) * (size_t)l_b);
    for (int64_t i = 0; i < l_b; ++i) { all[i].v = s[i]; all[i].i = i; }
    qsort(all, (size_t)l_b, sizeof(oracle_kv), cmp_desc_then_index);
    for (int64_t m = 0; m < k; ++m) idx[m] = (int32_t)all[m].i;
    qsort(idx, (size_t)k, sizeof(int32_t), cmp_int32_asc);
    free(all);
    return 0;
}

/* ------------------------------------------------------------------ attention */
/* Q:    [L_A + l_b][hq][d]            query rows [anchor | local block]
 * K, V: [L_A + P + l_b][hk][d]        key sequence [anchor | passing | local block]
 * rows: n_rows query-row indices to evaluate (NULL -> all L_A + l_b rows, n_rows ignored)
 * O:    [n_rows][hq][d], lse: [n_rows][hq] (natural log)
 * Visible set of query row r (reading G1):
 *   r <  L_A:  keys k with k <= r                         (anchor causal over the anchor)
 *   r >= L_A:  i = r - L_A; keys k < L_A + P (all anchor + all passing)
 *              and local keys L_A + P + m with m <= i    (causal over the local block)
 * Query head qh reads KV head qh / (hq / hk) (GQA).
 */
/* q_subset != 0: Q holds only the requested rows, in the order of `rows` (row x of Q is query
 * row rows[x]) — for sampled checks at sizes whose full Q would not fit in host memory as fp64.
 * The arithmetic is identical. */
int oracle_attention_ex(int64_t L_A, int64_t P, int64_t l_b, int32_t hq, int32_t hk, int32_t d,
                        double scale, const double* Q, const double* K, const double* V,
                        int64_t n_rows, const int64_t* rows, double* O, double* lse, int q_subset) {
    if (L_A < 0 || P < 0 || l_b < 0 || hq <= 0 || hk <= 0 || hq % hk || d <= 0) return 1;
    const int64_t n_q = L_A + l_b, n_k = L_A + P + l_b;
    const int32_t g = hq / hk;
    if (!rows) n_rows = n_q;
    if (q_subset && !rows) return 3;
    for (int64_t x = 0; x < n_rows; ++x) {
        int64_t r = rows ? rows[x] : x;
        if (r < 0 || r >= n_q) return 2;
    }
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int64_t x = 0; x < n_rows; ++x) {
        for (int32_t qh = 0; qh < hq; ++qh) {
            const int64_t r = rows ? rows[x] : x;
            const int32_t j = qh / g;
            const double* q = Q + ((q_subset ? x : r) * hq + qh) * (int64_t)d;
            double* logit = (double*)malloc(sizeof(double) * (size_t)(n_k > 0 ? n_k : 1));
            unsigned char* vis = (unsigned char*)malloc((size_t)(n_k > 0 ? n_k : 1));
            for (int64_t k = 0; k < n_k; ++k) {
                int visible;
                if (r < L_A) {
                    visible = (k <= r);
                } else {
                    int64_t i = r - L_A;
                    visible = (k < L_A + P) || (k - (L_A + P) <= i);
                }
                vis[k] = (unsigned char)visible;
                if (visible) {
                    const double* kk = K + (k * hk + j) * (int64_t)d;
                    double dot = 0.0;
                    for (int32_t c = 0; c < d; ++c) dot += q[c] * kk[c];
                    logit[k] = scale * dot;
                }
            }
            /* pass 1: max over the visible set */
            double m = -INFINITY;
            for (int64_t k = 0; k < n_k; ++k)
                if (vis[k] && logit[k] > m) m = logit[k];
            /* pass 2: weights, normaliser, weighted sum of values */
            double Z = 0.0;
            double* o = O + (x * hq + qh) * (int64_t)d;
            for (int32_t c = 0; c < d; ++c) o[c] = 0.0;
            for (int64_t k = 0; k < n_k; ++k) {
                if (!vis[k]) continue;
                double w = exp(logit[k] - m);
                Z += w;
                const double* vv = V + (k * hk + j) * (int64_t)d;
                for (int32_t c = 0; c < d; ++c) o[c] += w * vv[c];
            }
            for (int32_t c = 0; c < d; ++c) o[c] /= Z;
            lse[x * hq + qh] = m + log(Z);
            free(logit);
            free(vis);
        }
    }
    return 0;
}

int oracle_attention(int64_t L_A, int64_t P, int64_t l_b, int32_t hq, int32_t hk, int32_t d,
                     double scale, const double* Q, const double* K, const double* V,
                     int64_t n_rows, const int64_t* rows, double* O, double* lse) {
    return oracle_attention_ex(L_A, P, l_b, hq, hk, d, scale, Q, K, V, n_rows, rows, O, lse, 0);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count for the timing legs (bench.py cpu_baseline reports a single-thread rate too);
 * the arithmetic does not depend on it (each output is computed by one thread, fixed order). */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ decode (NEXT #1) */
/* Alg. apb_decode: the t new tokens' queries attend on host h to its block KV cache
 * (P:745-746); the last host also attends to the new tokens' own keys, causally among
 * them (new token s sees new tokens 0..s).  Returns the host's partial attention A_h and lse_h.
 * Q: [t][hq][d]; Kc, Vc: [c][hk][d]; Kn, Vn: [t][hk][d] or NULL (hosts other than the last).
 * O: [t][hq][d]; lse: [t][hq] (natural log; -inf when a row sees no key).                    */
int oracle_decode_partial(int64_t t, int64_t c, int32_t hq, int32_t hk, int32_t d, double scale,
                          const double* Q, const double* Kc, const double* Vc, const double* Kn,
                          const double* Vn, double* O, double* lse) {
    if (t < 0 || c < 0 || hq <= 0 || hk <= 0 || hq % hk || d <= 0) return 1;
    const int32_t g = hq / hk;
    const int64_t nmax = c + t;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int64_t s = 0; s < t; ++s) {
        for (int32_t qh = 0; qh < hq; ++qh) {
            const int32_t j = qh / g;
            const double* q = Q + (s * hq + qh) * (int64_t)d;
            double* logit = (double*)malloc(sizeof(double) * (size_t)(nmax > 0 ? nmax : 1));
            const double** vrow = (const double**)malloc(sizeof(double*) * (size_t)(nmax > 0 ? nmax : 1));
            int64_t n = 0;
            for (int64_t k = 0; k < c; ++k) {            /* every cached key precedes the new tokens */
                const double* kk = Kc + (k * hk + j) * (int64_t)d;
                double dot = 0.0;
                for (int32_t e = 0; e < d; ++e) dot += q[e] * kk[e];
                logit[n] = scale * dot;
                vrow[n++] = Vc + (k * hk + j) * (int64_t)d;
            }
            if (Kn) {
                for (int64_t k = 0; k <= s; ++k) {       /* new tokens: causal among themselves */
                    const double* kk = Kn + (k * hk + j) * (int64_t)d;
                    double dot = 0.0;
                    for (int32_t e = 0; e < d; ++e) dot += q[e] * kk[e];
                    logit[n] = scale * dot;
                    vrow[n++] = Vn + (k * hk + j) * (int64_t)d;
                }
            }
            double* o = O + (s * hq + qh) * (int64_t)d;
            for (int32_t e = 0; e < d; ++e) o[e] = 0.0;
            if (n == 0) {
                lse[s * hq + qh] = -INFINITY;
            } else {
                double m = -INFINITY;
                for (int64_t k = 0; k < n; ++k) if (logit[k] > m) m = logit[k];
                double Z = 0.0;
                for (int64_t k = 0; k < n; ++k) {
                    double w = exp(logit[k] - m);
                    Z += w;
                    for (int32_t e = 0; e < d; ++e) o[e] += w * vrow[k][e];
                }
                for (int32_t e = 0; e < d; ++e) o[e] /= Z;
                lse[s * hq + qh] = m + log(Z);
            }
            free(logit);
            free(vrow);
        }
    }
    return 0;
}

/* MergeScore: A = sum_h A_h exp(lse_h - L), L = log sum_h exp(lse_h).
 * parts_o: [n][rows][d], parts_lse: [n][rows]; out: [rows][d], out_lse: [rows].              */
int oracle_merge_score(int32_t n, int64_t rows, int32_t d, const double* parts_o, const double* parts_lse,
                       double* out, double* out_lse) {
    if (n <= 0 || rows < 0 || d <= 0) return 1;
    for (int64_t r = 0; r < rows; ++r) {
        double m = -INFINITY;
        for (int32_t h = 0; h < n; ++h) if (parts_lse[h * rows + r] > m) m = parts_lse[h * rows + r];
        double Z = 0.0;
        for (int32_t h = 0; h < n; ++h)
            if (parts_lse[h * rows + r] > -INFINITY) Z += exp(parts_lse[h * rows + r] - m);
        const double L = (m == -INFINITY) ? -INFINITY : m + log(Z);
        out_lse[r] = L;
        for (int32_t e = 0; e < d; ++e) {
            double acc = 0.0;
            for (int32_t h = 0; h < n; ++h) {
                const double l = parts_lse[h * rows + r];
                if (l > -INFINITY) acc += parts_o[(h * rows + r) * (int64_t)d + e] * exp(l - L);
            }
            out[r * (int64_t)d + e] = acc;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ method variants
 * Random selector "Rd." (Table 4), reading G17: a
 * SplitMix64 stream seeded with `seed`, advanced to position c0, emits `count` outputs;
 * score = top 24 bits * 2^-24 (uniform in [0,1), exact in fp32 and fp64).  Written as the
 * textbook sequential generator (state += golden gamma; mix) — one output per step. */
int oracle_random_scores(uint64_t seed, uint64_t c0, int64_t count, double* out) {
  uint64_t state = seed + c0 * 0x9E3779B97F4A7C15ull; /* = seed after c0 steps */
  for (int64_t i = 0; i < count; ++i) {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    out[i] = (double)(z >> 40) / 16777216.0;
  }
  return 0;
}
