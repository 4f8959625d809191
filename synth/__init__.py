"""Seeded synthetic inputs for the APB hot path — shared by the oracle and the GPU path.

This module holds NO arithmetic of the method (no scoring, selection, masking or
softmax).  It only draws seeded random numbers, rounds them to bf16 once (so the
oracle and the kernels consume bit-identical values) and lays them out the way
APB's context splitting places tokens on hosts (§3.3 "Context
Splitting"; the layout itself is index bookkeeping, not the method's math).

Recipe:
  * seeds: numpy SeedSequence([2502, 12085, cfg_id, layer, tensor_id, chunk]) — any
    row range of the document can be regenerated independently, so one host's
    block (or a sampled row) never needs the whole 128K-token document in memory;
  * D1 "flat":   Q, K, V ~ N(0, 1)            (the paper's timing input is "synthetic
                 random input")
  * D2 "peaky":  Q, K ~ N(0, 2^2), V ~ N(0, 1)
  * D3 "sink":   D2 + a shared per-KV-group direction mu added to every query, document
                 key row 0 set to 2 mu (an attention sink) + 16 needle key rows per
                 host block scaled x3 (retrieval structure of
                 the paper's RULER / InfiniteBench tasks)
  * retaining-head weights: W1 ~ N(0, 1/d_in) (bf16), b1 ~ N(0, 0.02^2),
    W2 ~ N(0, 1/d_hidden), b2 = 0 (fp32)   — random init, no trained heads exist here.
  * consistent anchor (default): with l_q = 0 the anchor rows of hosts >= 2 are the
    document's first l_a rows, exactly what a real model produces.
"""
from __future__ import annotations

import dataclasses
import numpy as np

CHUNK = 1024  # rows per independently seeded chunk
_T_Q, _T_K, _T_V, _T_QQ, _T_W1, _T_B1, _T_W2, _T_NEEDLE, _T_SCORES = range(9)


# ----------------------------------------------------------------------------- bf16 data

def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even), returned as uint16 bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    rounding = ((u >> 16) & np.uint32(1)) + np.uint32(0x7FFF)  # finite inputs never overflow
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(b).astype(np.float64)


# ----------------------------------------------------------------------------- configs

@dataclasses.dataclass(frozen=True)
class Config:
    """One APB workload (symbols as SURVEY.md §8: n, H, l_a, l_p, hq, hk, d)."""
    name: str
    cfg_id: int
    n: int
    H: int
    l_a: int
    l_p: int
    hq: int
    hk: int
    d: int
    layers: int = 1
    l_q: int = 0
    d_hidden: int = 1024
    dist: str = "D1"

    @property
    def l_b(self) -> int:
        return self.n // self.H

    @property
    def l_pp(self) -> int:  # l_p' = min(l_p, l_b)
        return min(self.l_p, self.l_b)

    @property
    def d_in(self) -> int:
        return (self.hq + 2 * self.hk) * self.d

    def L_A(self, host: int) -> int:
        return 0 if host == 0 else self.l_q + self.l_a

    def P(self, host: int) -> int:
        return host * self.l_pp

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: toy single layer (emulated 4 hosts)
    "toy": Config("toy", 1, n=2048, H=4, l_a=128, l_p=64, hq=4, hk=2, d=64),
    # configs[1]: Llama-3.1-8B-shaped, 128K, paper defaults l_a=4K, l_p=2K
    "llama8b-128k": Config("llama8b-128k", 2, n=131072, H=8, l_a=4096, l_p=2048,
                           hq=32, hk=8, d=128, layers=32),
    "llama8b-32k": Config("llama8b-32k", 6, n=32768, H=8, l_a=1024, l_p=512,
                          hq=32, hk=8, d=128, layers=32),
    # configs[2]: Qwen-2.5-14B-shaped
    "qwen14b-128k": Config("qwen14b-128k", 3, n=131072, H=8, l_a=4096, l_p=2048,
                           hq=40, hk=8, d=128, layers=48),
    # configs[3]: Yi-34B-200K-shaped
    "yi34b-200k": Config("yi34b-200k", 4, n=204800, H=8, l_a=4096, l_p=2048,
                         hq=56, hk=8, d=128, layers=60),
    # configs[4]: Llama-3-8B-1M-shaped
    "llama8b-512k": Config("llama8b-512k", 5, n=524288, H=8, l_a=8192, l_p=8192,
                           hq=32, hk=8, d=128, layers=32),
    "llama8b-1m": Config("llama8b-1m", 7, n=1048576, H=8, l_a=4096, l_p=2048,
                         hq=32, hk=8, d=128, layers=32),
}


# ----------------------------------------------------------------------------- generators

def _rng(cfg: Config, layer: int, tensor_id: int, chunk: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([2502, 12085, cfg.cfg_id, layer, tensor_id, chunk]))


def _scale(cfg: Config, tensor_id: int) -> float:
    if cfg.dist in ("D2", "D3") and tensor_id in (_T_Q, _T_K, _T_QQ):
        return 2.0
    return 1.0


def doc_rows(cfg: Config, layer: int, which: str, r0: int, r1: int) -> np.ndarray:
    """fp32 values of document rows [r0, r1) of Q ('q'), K ('k') or V ('v'): [rows][heads][d]."""
    tid = {"q": _T_Q, "k": _T_K, "v": _T_V}[which]
    heads = cfg.hq if which == "q" else cfg.hk
    out = np.empty((r1 - r0, heads, cfg.d), np.float32)
    c0, c1 = r0 // CHUNK, (r1 - 1) // CHUNK if r1 > r0 else r0 // CHUNK - 1
    for c in range(c0, c1 + 1):
        g = _rng(cfg, layer, tid, c).standard_normal((CHUNK, heads, cfg.d), dtype=np.float32)
        g *= _scale(cfg, tid)
        lo, hi = max(r0, c * CHUNK), min(r1, (c + 1) * CHUNK)
        out[lo - r0:hi - r0] = g[lo - c * CHUNK:hi - c * CHUNK]
    if cfg.dist == "D3":
        _plant_structure(cfg, layer, which, r0, r1, out)
    return out


def _plant_structure(cfg: Config, layer: int, which: str, r0: int, r1: int, out: np.ndarray) -> None:
    """D3: a shared query direction mu (per KV group) added to every query row, an attention
    sink at document key row 0 (= 2 mu, logit ~ 2|mu|^2/sqrt(d) >> others) and 16 needle key
    rows per host block scaled x3."""
    mu = _rng(cfg, layer, _T_NEEDLE, 0).standard_normal((cfg.hk, cfg.d), dtype=np.float32)
    if which == "q":
        g = cfg.hq // cfg.hk
        out += np.repeat(mu, g, axis=0)[None]
        return
    if which != "k":
        return
    if r0 == 0 and r1 > 0:
        out[0] = 2.0 * mu
    for h in range(cfg.H):
        b0 = h * cfg.l_b
        if b0 >= r1 or b0 + cfg.l_b <= r0:
            continue
        pos = _rng(cfg, layer, _T_NEEDLE, 1 + h).choice(cfg.l_b, size=min(16, cfg.l_b), replace=False)
        for p in pos:
            r = b0 + int(p)
            if r0 <= r < r1:
                out[r - r0] *= 3.0


def query_rows(cfg: Config, layer: int, which: str) -> np.ndarray:
    """fp32 rows of the query part q (l_q tokens) embedded at the front of the anchor."""
    heads = cfg.hq if which == "q" else cfg.hk
    tid = _T_QQ * 8 + {"q": 0, "k": 1, "v": 2}[which]
    g = _rng(cfg, layer, tid, 0).standard_normal((cfg.l_q, heads, cfg.d), dtype=np.float32)
    return g * _scale(cfg, _T_QQ)


def host_qkv(cfg: Config, layer: int, host: int, rows: slice | None = None) -> dict:
    """bf16 bit patterns of host `host`'s [anchor | block] Q, K, V.

    Row layout on host h (0-based): rows [0, L_A) = anchor A = [q_1..q_{l_q}, d_1..d_{l_a}]
    (empty on host 0), rows [L_A, L_A + l_b) = block B_h = d_{h*l_b+1} .. d_{(h+1)*l_b}.
    Returns dict(q=[rows][hq][d] uint16, k=[rows][hk][d] uint16, v=..., L_A=int).
    """
    L_A = cfg.L_A(host)
    total = L_A + cfg.l_b
    rows = rows or slice(0, total)
    r0, r1 = rows.start, min(rows.stop, total)
    out = {"L_A": L_A}
    for which in ("q", "k", "v"):
        heads = cfg.hq if which == "q" else cfg.hk
        buf = np.empty((r1 - r0, heads, cfg.d), np.float32)
        # anchor part
        if L_A > 0:
            a0, a1 = r0, min(r1, L_A)
            if a1 > a0:
                lq = cfg.l_q
                if lq > 0:
                    qq = query_rows(cfg, layer, which)
                    q0, q1 = a0, min(a1, lq)
                    if q1 > q0:
                        buf[q0 - r0:q1 - r0] = qq[q0:q1]
                d0, d1 = max(a0, lq), a1
                if d1 > d0:
                    buf[d0 - r0:d1 - r0] = doc_rows(cfg, layer, which, d0 - lq, d1 - lq)
        b0, b1 = max(r0, L_A), r1
        if b1 > b0:
            base = host * cfg.l_b - L_A
            buf[b0 - r0:b1 - r0] = doc_rows(cfg, layer, which, base + b0, base + b1)
        out[which] = f32_to_bf16_bits(buf)
    return out


def retain_weights(cfg: Config, layer: int, n_out: int | None = None) -> dict:
    """Random-init retaining-head weights (hidden size 1024 at PAPER.md:798)."""
    n_out = cfg.hq if n_out is None else n_out
    g1 = _rng(cfg, layer, _T_W1, 0)
    w1 = g1.standard_normal((cfg.d_hidden, cfg.d_in), dtype=np.float32) / np.sqrt(cfg.d_in)
    b1 = (_rng(cfg, layer, _T_B1, 0).standard_normal(cfg.d_hidden, dtype=np.float32) * 0.02).astype(np.float32)
    w2 = (_rng(cfg, layer, _T_W2, 0).standard_normal((n_out, cfg.d_hidden), dtype=np.float32)
          / np.sqrt(cfg.d_hidden)).astype(np.float32)
    b2 = np.zeros(n_out, np.float32)
    return {"w1": f32_to_bf16_bits(w1), "b1": b1, "w2": w2, "b2": b2, "n_out": n_out}


def random_scores(cfg: Config, layer: int, host: int, ties: bool = False) -> np.ndarray:
    """fp32 scores [hk][l_b] for exercising selection alone (SPEC 'Rd.' selector idea).

    ties=True quantises to a coarse grid so many exact ties exist (tie rule G5)."""
    s = _rng(cfg, layer, _T_SCORES, host).standard_normal((cfg.hk, cfg.l_b), dtype=np.float32)
    if ties:
        s = np.round(s * 4.0).astype(np.float32) / 4.0
    return s


# ----------------------------------------------------------------------------- model layer (NEXT #2)
_T_HID, _T_QHID, _T_MW = 40, 41, 50  # hidden rows, query hidden rows, model weights (+0..5)


def model_weights(cfg: Config, layer: int, hidden: int, inter: int) -> dict:
    """Random-init Llama-style decoder-layer weights (bf16 bits, nn.Linear layout [out][in]):
    projections ~ N(0, 1/fan_in) so activations stay O(1); norm weights ~ 1 + N(0, 0.1^2)."""
    hq, hk, d = cfg.hq, cfg.hk, cfg.d

    def lin(k, n_out, n_in):
        w = _rng(cfg, layer, _T_MW + k, 0).standard_normal((n_out, n_in), dtype=np.float32) / np.sqrt(n_in)
        return f32_to_bf16_bits(w)

    def norm(k):
        return f32_to_bf16_bits(1.0 + 0.1 * _rng(cfg, layer, _T_MW + k, 0).standard_normal(hidden, dtype=np.float32))

    return {"attn_norm": norm(0), "w_qkv": lin(1, (hq + 2 * hk) * d, hidden), "w_o": lin(2, hidden, hq * d),
            "ffn_norm": norm(3), "w_gu": lin(4, 2 * inter, hidden), "w_down": lin(5, hidden, inter)}


def host_hidden(cfg: Config, host: int, hidden: int) -> np.ndarray:
    """bf16 bits [L_A + l_b][hidden] of host `host`'s input hidden states [A; B_h] (the layout of
    host_qkv: anchor = query rows then the document's first l_a rows, block = its document
    block).  Document and query rows ~ N(0, 1), chunked by CHUNK rows like doc_rows."""
    L_A = cfg.L_A(host)

    def doc(r0, r1):
        out = np.empty((r1 - r0, hidden), np.float32)
        for c in range(r0 // CHUNK, (r1 - 1) // CHUNK + 1 if r1 > r0 else 0):
            g = _rng(cfg, 0, _T_HID, c).standard_normal((CHUNK, hidden), dtype=np.float32)
            lo, hi = max(r0, c * CHUNK), min(r1, (c + 1) * CHUNK)
            out[lo - r0:hi - r0] = g[lo - c * CHUNK:hi - c * CHUNK]
        return out

    parts = []
    if L_A:
        if cfg.l_q:
            parts.append(_rng(cfg, 0, _T_QHID, 0).standard_normal((cfg.l_q, hidden), dtype=np.float32))
        parts.append(doc(0, cfg.l_a))
    parts.append(doc(host * cfg.l_b, (host + 1) * cfg.l_b))
    return f32_to_bf16_bits(np.concatenate(parts))
