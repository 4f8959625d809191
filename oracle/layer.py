"""fp64 oracle for the APB prefill LAYER around the hot path:
Alg. apb_prefill with its model steps written out — qkv_proj,
the hot path (`oracle.prefill_layer`), and FFN — for a Llama-style
decoder layer (the paper's backbones: Llama-3.1, Qwen-2.5, Yi).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): tests/ and bench's cpu_baseline are the
only callers.  Shares no code with the CUDA path; `synth` supplies the bf16 rounding of the
storage points only.

The layer, per host, on the rows [A; B_h] of that host (reading G19: a row's RoPE position is
its index in the host's local sequence, so the anchor gets the starting positions
0..l_q+l_a-1 of P:160):

    h   = RMSNorm(x) * w_attn_norm                 (Llama RMSNorm, eps)
    qkv = h W_qkv^T ;  Q, K <- RoPE(Q, K, pos)     (rotate-half RoPE, base theta)
    O   = APB attention hot path (scores, top-l_p, AllGather, masked attention)
    x'  = x + O W_o^T
    g|u = RMSNorm(x') * w_ffn_norm  W_gu^T ;  a = SiLU(g) * u
    out = x' + a W_down^T

`rnd=True` rounds to bf16 at the points where the GPU path stores bf16 (readings G9, G20:
every linear output, norm output, activation and residual sum, as in a bf16 PyTorch Llama
layer); with
`rnd=False` every step is exact fp64 (the form pinned against transformers' LlamaDecoderLayer
in tests/test_oracle_layer.py).
"""
from __future__ import annotations

import numpy as np

import oracle
from synth import bf16_bits_to_f64, f32_to_bf16_bits


def bf16(x) -> np.ndarray:
    """Round to the nearest bf16 (via fp32), returned as fp64."""
    return bf16_bits_to_f64(f32_to_bf16_bits(np.asarray(x, np.float32)))


def _r(x, rnd: bool):
    return bf16(x) if rnd else np.asarray(x, np.float64)


def rmsnorm(x, w, eps: float) -> np.ndarray:
    """RMSNorm (Zhang & Sennrich 2019, as in Llama): x / sqrt(mean(x^2) + eps) * w, per row."""
    x = np.asarray(x, np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * np.asarray(w, np.float64)


def rope(x, positions, theta: float) -> np.ndarray:
    """Rotary position embedding, rotate-half form (Llama): for i < d/2 the pair
    (x_i, x_{i+d/2}) is rotated by angle pos * theta^(-2i/d).  x: [rows][heads][d]."""
    x = np.asarray(x, np.float64)
    d = x.shape[-1]
    inv = theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)          # [d/2]
    ang = np.asarray(positions, np.float64)[:, None] * inv[None, :]     # [rows][d/2]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(z):
    z = np.asarray(z, np.float64)
    return z / (1.0 + np.exp(-z))


def swiglu(gu, inter: int) -> np.ndarray:
    """SwiGLU (Shazeer 2020): SiLU(g) * u with [g | u] = gu along the last axis."""
    gu = np.asarray(gu, np.float64)
    return silu(gu[..., :inter]) * gu[..., inter:]


def attn_in(x, lw: dict, hq: int, hk: int, d: int, positions, rnd: bool = True) -> np.ndarray:
    """qkv_proj of Alg. apb_prefill with the pre-attention RMSNorm and RoPE on Q and K.
    Returns qkv [rows][hq+2hk][d] (Q heads, then K heads, then V heads — the row layout the
    hot path reads with row stride (hq+2hk)*d)."""
    h = _r(rmsnorm(x, lw["attn_norm"], lw["eps"]), rnd)
    qkv = _r(h @ np.asarray(lw["w_qkv"], np.float64).T, rnd).reshape(h.shape[0], hq + 2 * hk, d)
    qk = _r(rope(qkv[:, : hq + hk], positions, lw["theta"]), rnd)
    return np.concatenate([qk, qkv[:, hq + hk:]], axis=1)


def attn_out_ffn(x, attn, lw: dict, rnd: bool = True) -> np.ndarray:
    """O projection + residual, then the FFN of Alg. apb_prefill + residual.
    attn: [rows][hq][d] attention output."""
    x = np.asarray(x, np.float64)
    a = np.asarray(attn, np.float64).reshape(x.shape[0], -1)
    # reading G20: as in a bf16 PyTorch Llama layer, each projection output is a bf16 tensor
    # that is then added to the bf16 residual (two roundings per residual add)
    x1 = _r(x + _r(a @ np.asarray(lw["w_o"], np.float64).T, rnd), rnd)
    h2 = _r(rmsnorm(x1, lw["ffn_norm"], lw["eps"]), rnd)
    gu = _r(h2 @ np.asarray(lw["w_gu"], np.float64).T, rnd)
    act = _r(swiglu(gu, gu.shape[-1] // 2), rnd)
    return _r(x1 + _r(act @ np.asarray(lw["w_down"], np.float64).T, rnd), rnd)


def apb_layer(hosts_x, L_As, lw: dict, retain: dict, l_p: int, hq: int, hk: int, d: int, rnd: bool = True,
              compressor_scores=None):
    """One APB prefill layer (Alg. apb_prefill) on every host, in the paper's order.

    hosts_x: per host [L_A+l_b][hidden] hidden states (rows [A; B_h]); L_As: per host L_A.
    retain: retaining-head weights dict(w1 (bf16 bits), b1, w2, b2); compressor_scores:
    optional per-host [hk][l_b] scores replacing R (e.g. the "Rd." selector).
    Returns dict(out=per-host outputs, qkv=..., attn=..., layer=oracle.prefill_layer result)."""
    qkvs = [attn_in(x, lw, hq, hk, d, np.arange(x.shape[0]), rnd) for x in hosts_x]
    hosts = []
    for qkv, L_A in zip(qkvs, L_As):
        hosts.append({"q": qkv[:, :hq], "k": qkv[:, hq:hq + hk], "v": qkv[:, hq + hk:], "L_A": L_A})
    res = oracle.prefill_layer(hosts, retain, l_p, scores_override=compressor_scores)
    attn = [_r(o, rnd) for o in res["O"]]
    outs = [attn_out_ffn(x, a, lw, rnd) for x, a in zip(hosts_x, attn)]
    return {"out": outs, "qkv": qkvs, "attn": attn, "layer": res}
