"""fp64 CPU oracle for the APB prefill hot path (arXiv 2502.12085).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs are the only callers.  The product package never imports this.
It shares no code with the CUDA path; only `synth` (seeded inputs, no method arithmetic)
feeds both.

The numeric kernels (scoring, top-l_p, masked attention) are plain C in apb_oracle.c
(fp64, two-pass softmax, OpenMP over rows).  This file holds the pure indexing steps of
Alg. apb_prefill in the paper's order:

    s = R([Q_h, K_h, V_h])                       P:712   -> retain_score
    indices = ArgTop-l_p(s)                       P:713   -> select_topk
    K^C_h, V^C_h = K_h[indices], V_h[indices]     P:714   -> compact
    (K^C_1..H, V^C_1..H) = AllGather(K^C_h, ...)  P:719-720 -> all_gather
    K_p, V_p = concat of hosts 1..h-1             P:722-723 -> passing
    Attention([Q_a,Q_h], [K_a,K_p,K_h], ...)      P:728   -> attention

Parity pins: every function here is checked against something other than itself in
tests/test_oracle.py (torch fp64 SDPA, brute force, closed forms, the SPEC worked mask
example, the hand-evaluated scorer value tanh(1/2)).  No function is "parity unpinned".
"""
from __future__ import annotations

import concurrent.futures
import ctypes
import os
import subprocess
import threading

import numpy as np

from synth import bf16_bits_to_f64

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "apb_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile apb_oracle.c with gcc (-O2, OpenMP).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            dp, ip, lp = (ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32),
                          ctypes.POINTER(ctypes.c_int64))
            i64, i32 = ctypes.c_int64, ctypes.c_int32
            lib.oracle_retain_score.argtypes = [i64, i32, i32, i32, i32, dp, dp, dp, dp, dp, dp]
            lib.oracle_select_topk.argtypes = [i64, i64, dp, ip]
            lib.oracle_attention.argtypes = [i64, i64, i64, i32, i32, i32, ctypes.c_double,
                                             dp, dp, dp, i64, lp, dp, dp]
            lib.oracle_attention_ex.argtypes = [i64, i64, i64, i32, i32, i32, ctypes.c_double,
                                                dp, dp, dp, i64, lp, dp, dp, ctypes.c_int]
            lib.oracle_decode_partial.argtypes = [i64, i64, i32, i32, i32, ctypes.c_double,
                                                  dp, dp, dp, dp, dp, dp, dp]
            lib.oracle_merge_score.argtypes = [i32, i64, i32, dp, dp, dp, dp]
            lib.oracle_random_scores.argtypes = [ctypes.c_uint64, ctypes.c_uint64, i64, dp]
            for f in (lib.oracle_retain_score, lib.oracle_select_topk, lib.oracle_attention, lib.oracle_attention_ex,
                      lib.oracle_decode_partial, lib.oracle_merge_score, lib.oracle_random_scores):
                f.restype = ctypes.c_int
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
            lib.oracle_set_num_threads.restype = None
            _lib = lib
    return _lib


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the C oracle (timing legs only; results do not depend on it)."""
    _load().oracle_set_num_threads(int(n))


def _as_f64(x):
    x = np.asarray(x)
    if x.dtype == np.uint16:  # bf16 bit patterns
        return bf16_bits_to_f64(x)
    return np.ascontiguousarray(x, dtype=np.float64)


# ----------------------------------------------------------------------------- steps

def retain_score(q, k, v, L_A: int, w1, b1, w2, b2, hk: int) -> np.ndarray:
    """s[j][t] for the block rows t in [L_A, L_A + l_b).

    q: [L_A+l_b][hq][d], k/v: [L_A+l_b][hk][d] (bf16 bits or floats); w1: [d_hidden][d_in];
    b1: [d_hidden] or None; w2: [n_out][d_hidden]; b2: [n_out] or None.  Returns fp64 [hk][l_b].
    """
    q, k, v = _as_f64(q), _as_f64(k), _as_f64(v)
    l_b = q.shape[0] - L_A
    # x_t = [Q_t | K_t | V_t], heads then head_dim (reading G2)
    x = np.ascontiguousarray(np.concatenate(
        [q[L_A:].reshape(l_b, -1), k[L_A:].reshape(l_b, -1), v[L_A:].reshape(l_b, -1)], axis=1))
    w1 = np.ascontiguousarray(_as_f64(w1))
    w2 = np.ascontiguousarray(_as_f64(w2))
    b1 = None if b1 is None else np.ascontiguousarray(_as_f64(b1))
    b2 = None if b2 is None else np.ascontiguousarray(_as_f64(b2))
    d_hidden, d_in = w1.shape
    n_out = w2.shape[0]
    assert x.shape[1] == d_in
    s = np.empty((hk, l_b), np.float64)
    rc = _load().oracle_retain_score(l_b, d_in, d_hidden, n_out, hk, _p(x), _p(w1), _p(b1),
                                     _p(w2), _p(b2), _p(s))
    if rc:
        raise ValueError(f"oracle_retain_score rc={rc}")
    return s


def select_topk(s_row, l_p: int) -> np.ndarray:
    """ArgTop-l_p of one KV head's scores: min(l_p, l_b) indices, ascending,
    ties to the lower index (reading G5).  Decisions are taken in the precision of the
    values passed (fp32 scores upcast to fp64 compare identically)."""
    s_row = np.ascontiguousarray(s_row, dtype=np.float64)
    k = min(l_p, s_row.shape[0])
    idx = np.empty(max(k, 0), np.int32)
    rc = _load().oracle_select_topk(s_row.shape[0], l_p, _p(s_row), _p(idx, ctypes.c_int32))
    if rc:
        raise ValueError(f"oracle_select_topk rc={rc}")
    return idx


def random_scores(seed: int, layer: int, H: int, host: int, hk: int, l_b: int) -> np.ndarray:
    """The random compressor "Rd." (Table 4) for one host and layer:
    [hk][l_b] uniform scores in [0,1), counter c = ((layer*H + host)*hk + j)*l_b + t of the
    SplitMix64 stream seeded with `seed` (reading G17)."""
    out = np.empty((hk, l_b), np.float64)
    c0 = ((layer * H + host) * hk * l_b) % (1 << 64)
    _load().oracle_random_scores(ctypes.c_uint64(seed % (1 << 64)), ctypes.c_uint64(c0), hk * l_b, _p(out))
    return out


def share_scores(s) -> np.ndarray:
    """Shared index set (SPEC S:255, S:294 — one index list per host, as Alg. apb_prefill
    writes it): every KV head's score row is replaced by the max over KV heads."""
    s = np.asarray(s, np.float64)
    return np.broadcast_to(s.max(axis=0, keepdims=True), s.shape).copy()


def select_all_heads(s, l_p: int) -> np.ndarray:
    return np.stack([select_topk(s[j], l_p) for j in range(s.shape[0])]) if s.shape[0] else \
        np.zeros((0, 0), np.int32)


def compact(k, v, L_A: int, idx) -> np.ndarray:
    """K^C_h, V^C_h = K_h[indices], V_h[indices], per KV head j.

    Returns the packed payload [2][hk][l_p'][d] in the dtype of k/v (bit-exact copies)."""
    k, v = np.asarray(k), np.asarray(v)
    hk, lp = idx.shape
    out = np.empty((2, hk, lp, k.shape[2]), k.dtype)
    for j in range(hk):
        for m in range(lp):
            out[0, j, m] = k[L_A + idx[j, m], j]
            out[1, j, m] = v[L_A + idx[j, m], j]
    return out


def all_gather(sends) -> np.ndarray:
    """AllGather: every host ends with [C_1, ..., C_H] in host order."""
    return np.stack(list(sends))


def passing(gathered, host: int):
    """P_h = concat(K^C_1..K^C_{h-1}), host order then ascending
    index; later hosts' blocks are ignored.  Returns (PK, PV): [P_h][hk][d] each."""
    hk, lp, d = gathered.shape[2], gathered.shape[3], gathered.shape[4]
    if host == 0 or lp == 0:
        e = np.zeros((0, hk, d), gathered.dtype)
        return e, e.copy()
    pk = np.concatenate([gathered[s, 0].transpose(1, 0, 2) for s in range(host)], axis=0)
    pv = np.concatenate([gathered[s, 1].transpose(1, 0, 2) for s in range(host)], axis=0)
    return pk, pv


def attention(q, k, v, L_A: int, pk, pv, scale: float | None = None, rows=None, q_subset: bool = False):
    """[A_a, A_h] = softmax(M' . Q K^T / sqrt(d_m)) V  (eq:apb).

    q: [L_A+l_b][hq][d]; k, v: [L_A+l_b][hk][d]; pk, pv: [P][hk][d].
    Key sequence: [K_a ; K_p ; K_h].  rows: optional query-row subset.
    q_subset: q holds only the rows listed in `rows`, in that order (same arithmetic; for
    sampled checks at sizes whose full Q does not fit in host memory as fp64).
    Returns (O [rows][hq][d] fp64, lse [rows][hq] fp64)."""
    q, k, v = _as_f64(q), _as_f64(k), _as_f64(v)
    pk, pv = _as_f64(pk), _as_f64(pv)
    _, hq, d = q.shape
    n_q = k.shape[0]
    if not q_subset and q.shape[0] != n_q:
        raise ValueError("q and k must have the same number of rows")
    if q_subset and (rows is None or len(rows) != q.shape[0]):
        raise ValueError("q_subset needs rows with one entry per q row")
    hk = k.shape[1]
    l_b = n_q - L_A
    P = pk.shape[0]
    kseq = np.ascontiguousarray(np.concatenate([k[:L_A], pk.reshape(P, hk, d), k[L_A:]], axis=0))
    vseq = np.ascontiguousarray(np.concatenate([v[:L_A], pv.reshape(P, hk, d), v[L_A:]], axis=0))
    if scale is None:
        scale = 1.0 / np.sqrt(d)  # 1/sqrt(d_m), d_m = per-head hidden size
    q = np.ascontiguousarray(q)
    if rows is None:
        n_rows, rp = n_q, None
    else:
        rp = np.ascontiguousarray(rows, dtype=np.int64)
        n_rows = rp.shape[0]
    O = np.empty((n_rows, hq, d), np.float64)
    lse = np.empty((n_rows, hq), np.float64)
    rc = _load().oracle_attention_ex(L_A, P, l_b, hq, hk, d, float(scale), _p(q), _p(kseq), _p(vseq),
                                     n_rows, _p(rp, ctypes.c_int64) if rp is not None else None,
                                     _p(O), _p(lse), int(q_subset))
    if rc:
        raise ValueError(f"oracle_attention rc={rc}")
    return O, lse


# ----------------------------------------------------------------------------- full-size forms
# The same two definitions with fp64 LIBRARY matmuls (numpy / OpenBLAS) as steps, for checks at
# the bench's full sizes (a retaining head is ~207 GFLOP per L8 host, ~100x the C loops' speed
# is needed to check every token).  No blocking beyond row chunks, no reordering of the math:
# each output is the plain definition.  Pinned like the C forms (tests/test_oracle.py,
# *_blas pins): hand value, SiLU closed form, torch fp64 Linear, torch fp64 SDPA, closed-form
# lse counts, rows sum to one, one-hot probes.

def retain_score_blas(q, k, v, L_A: int, w1, b1, w2, b2, hk: int, chunk: int = 2048) -> np.ndarray:
    """s[j][t] (readings G2/G4): z = W1 x_t + b1, a = SiLU(z) = z / (1 + e^-z),
    o = W2 a + b2, s[j] = max over KV head j's r = n_out/hk outputs.  x_t = [Q_t | K_t | V_t].
    Arguments as retain_score; returns fp64 [hk][l_b]."""
    q, k, v = np.asarray(q), np.asarray(k), np.asarray(v)
    l_b = q.shape[0] - L_A
    w1 = _as_f64(w1)
    w2 = _as_f64(w2)
    b1 = np.zeros(w1.shape[0]) if b1 is None else _as_f64(b1)
    b2 = np.zeros(w2.shape[0]) if b2 is None else _as_f64(b2)
    n_out = w2.shape[0]
    r = n_out // hk
    s = np.empty((hk, l_b), np.float64)
    for t0 in range(0, l_b, chunk):
        t1 = min(l_b, t0 + chunk)
        x = np.concatenate([_as_f64(a[L_A + t0:L_A + t1]).reshape(t1 - t0, -1) for a in (q, k, v)], axis=1)
        z = x @ w1.T + b1
        with np.errstate(over="ignore"):
            a_ = z / (1.0 + np.exp(-z))
        o = a_ @ w2.T + b2
        s[:, t0:t1] = o.reshape(t1 - t0, hk, r).max(axis=2).T
    return s


def attention_blas(q, k, v, L_A: int, pk, pv, rows, scale: float | None = None, q_subset: bool = False,
                   chunk: int = 256):
    """eq:apb for the query rows `rows`, with fp64 matmuls for q.k and p.v.
    Key sequence [K_a ; K_p ; K_h].  vis(r) (reading G1): anchor row r < L_A sees
    keys 0..r; local row r = L_A + i sees all L_A anchor keys, all P passing keys and local keys
    0..i — in both cases the first lim(r) keys of the sequence, lim = r+1 (anchor) or
    L_A + P + i + 1 (local).  Two-pass softmax: m = max, w = e^(l - m), Z = sum w,
    O = sum w v / Z, lse = m + ln Z.  Arguments as attention(); returns (O [rows][hq][d], lse [rows][hq])."""
    q, k, v = np.asarray(q), np.asarray(k), np.asarray(v)
    pk, pv = np.asarray(pk), np.asarray(pv)
    hq, d = q.shape[1], q.shape[2]
    hk = k.shape[1]
    g = hq // hk
    L_A = int(L_A)
    P = pk.shape[0]
    rows = np.asarray(rows, np.int64)
    if q_subset and len(rows) != q.shape[0]:
        raise ValueError("q_subset needs rows with one entry per q row")
    if scale is None:
        scale = 1.0 / np.sqrt(d)  # 1/sqrt(d_m)
    lim = np.where(rows < L_A, rows + 1, P + rows + 1)
    order = np.argsort(lim, kind="stable")
    O = np.empty((len(rows), hq, d), np.float64)
    lse = np.empty((len(rows), hq), np.float64)
    def head(j):  # KV head j and its g query heads (independent of every other head)
        kseq = np.concatenate([_as_f64(k[:L_A, j]), _as_f64(pk[:, j]).reshape(P, d), _as_f64(k[L_A:, j])], 0)
        vseq = np.concatenate([_as_f64(v[:L_A, j]), _as_f64(pv[:, j]).reshape(P, d), _as_f64(v[L_A:, j])], 0)
        for c0 in range(0, len(rows), chunk):
            sel = order[c0:c0 + chunk]
            src = sel if q_subset else rows[sel]
            Qc = _as_f64(q[src, j * g:(j + 1) * g]).reshape(len(sel) * g, d)
            lim_c = np.repeat(lim[sel], g)
            kmax = int(lim_c.max())
            logits = Qc @ kseq[:kmax].T
            logits *= scale
            for i in np.nonzero(lim_c < kmax)[0]:  # keys past lim(r) are not visible
                logits[i, lim_c[i]:] = -np.inf
            m = logits.max(axis=1, keepdims=True)
            logits -= m
            w = np.exp(logits, out=logits)
            Z = w.sum(axis=1, keepdims=True)
            Oc = (w @ vseq[:kmax]) / Z
            O[sel, j * g:(j + 1) * g] = Oc.reshape(len(sel), g, d)
            lse[sel, j * g:(j + 1) * g] = (m + np.log(Z)).reshape(len(sel), g)

    # heads in parallel threads (numpy's elementwise passes are single-threaded and release the GIL)
    with concurrent.futures.ThreadPoolExecutor(max_workers=min(hk, os.cpu_count() or 1)) as ex:
        list(ex.map(head, range(hk)))
    return O, lse


# ----------------------------------------------------------------------------- decode (NEXT #1)

def decode_partial(q, k_cache, v_cache, k_new=None, v_new=None, scale: float | None = None):
    """Alg. apb_decode lines attnl / attnh: host h's partial attention of the t new
    tokens over its block cache, plus (last host only) the new tokens' own keys, causally.
    q: [t][hq][d]; k/v_cache: [c][hk][d]; k/v_new: [t][hk][d] or None.
    Returns (A_h [t][hq][d] fp64, lse_h [t][hq] fp64, natural log)."""
    q = np.ascontiguousarray(_as_f64(q))
    kc, vc = np.ascontiguousarray(_as_f64(k_cache)), np.ascontiguousarray(_as_f64(v_cache))
    kn = None if k_new is None else np.ascontiguousarray(_as_f64(k_new))
    vn = None if v_new is None else np.ascontiguousarray(_as_f64(v_new))
    t, hq, d = q.shape
    c, hk = kc.shape[0], kc.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    O = np.empty((t, hq, d), np.float64)
    lse = np.empty((t, hq), np.float64)
    rc = _load().oracle_decode_partial(t, c, hq, hk, d, float(scale), _p(q), _p(kc), _p(vc), _p(kn), _p(vn),
                                       _p(O), _p(lse))
    if rc:
        raise ValueError(f"oracle_decode_partial rc={rc}")
    return O, lse


def merge_score(parts_o, parts_lse):
    """MergeScore: merge partial attentions by their log-sum-exp.
    parts_o: [n][rows...][d], parts_lse: [n][rows...].  Returns (A [rows...][d], L [rows...])."""
    po = np.ascontiguousarray(parts_o, dtype=np.float64)
    pl = np.ascontiguousarray(parts_lse, dtype=np.float64)
    n, d = po.shape[0], po.shape[-1]
    rows = int(np.prod(po.shape[1:-1]))
    out = np.empty(po.shape[1:], np.float64)
    out_lse = np.empty(pl.shape[1:], np.float64)
    rc = _load().oracle_merge_score(n, rows, d, _p(po), _p(pl), _p(out), _p(out_lse))
    if rc:
        raise ValueError(f"oracle_merge_score rc={rc}")
    return out, out_lse


def decode_step(q, caches, k_new, v_new, scale: float | None = None):
    """One Accu attention (Alg. apb_decode) over H hosts: per-host partials (the last
    host includes the new tokens' keys), Gather, MergeScore.  caches: list of (k_cache, v_cache)
    in host order.  Returns (A [t][hq][d], L [t][hq], partials list)."""
    parts = []
    for h, (kc, vc) in enumerate(caches):
        last = h == len(caches) - 1
        parts.append(decode_partial(q, kc, vc, k_new if last else None, v_new if last else None, scale))
    A, L = merge_score(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]))
    return A, L, parts


# ----------------------------------------------------------------------------- pipeline

def prefill_layer(hosts_qkv, weights, l_p: int, scale: float | None = None, rows_per_host=None,
                  scores_override=None):
    """Alg. apb_prefill for ONE layer on every host h = 1..H, in the paper's order.

    hosts_qkv: list over hosts of dict(q, k, v, L_A) (bf16 bits); weights: dict(w1,b1,w2,b2)
    or None when scores_override (list of [hk][l_b] arrays) is given.
    Returns dict with per-host scores, indices, sends, the gathered buffer, O and lse."""
    H = len(hosts_qkv)
    hk = hosts_qkv[0]["k"].shape[1]
    scores, idxs, sends = [], [], []
    for h in range(H):
        x = hosts_qkv[h]
        if scores_override is not None:
            s = np.asarray(scores_override[h], np.float64)
        else:
            s = retain_score(x["q"], x["k"], x["v"], x["L_A"], weights["w1"], weights.get("b1"),
                             weights["w2"], weights.get("b2"), hk)
        idx = select_all_heads(s, l_p)
        scores.append(s)
        idxs.append(idx)
        sends.append(compact(x["k"], x["v"], x["L_A"], idx))
    gathered = all_gather(sends)
    outs, lses = [], []
    for h in range(H):
        x = hosts_qkv[h]
        pk, pv = passing(gathered, h)
        rows = None if rows_per_host is None else rows_per_host[h]
        O, lse = attention(x["q"], x["k"], x["v"], x["L_A"], pk, pv, scale, rows)
        outs.append(O)
        lses.append(lse)
    return {"scores": scores, "indices": idxs, "sends": sends, "gathered": gathered,
            "O": outs, "lse": lses}
