"""Work accounting for the APB hot path (metrics only; no numerics of the method).

Useful attention FLOPs are counted from the mask M' (reading G13): 4 * d * hq per
visible (query row, key) pair — the paper's own 2 n^2 d causal convention (tab:flops,
PAPER.md:927) — with, per host h (0-based) and P_h = h * l_p' passing keys:
    anchor rows: L_A (L_A + 1) / 2 pairs;  local rows: l_b (L_A + P_h) + l_b (l_b + 1) / 2 pairs.
"""
from __future__ import annotations


def visible_pairs(L_A: int, P: int, l_b: int) -> int:
    return L_A * (L_A + 1) // 2 + l_b * (L_A + P) + l_b * (l_b + 1) // 2


def host_L_A(host: int, l_q: int, l_a: int) -> int:
    return 0 if host == 0 else l_q + l_a


def attention_flops(n: int, H: int, host: int, l_a: int, l_p: int, hq: int, d: int, l_q: int = 0) -> int:
    l_b = n // H
    lpp = min(l_p, l_b)
    return 4 * d * hq * visible_pairs(host_L_A(host, l_q, l_a), host * lpp, l_b)


def attention_executed_flops(n: int, H: int, host: int, l_a: int, l_p: int, hq: int, d: int, l_q: int = 0,
                             tile: int = 128) -> int:
    """MMA FLOPs the attention kernel executes: whole tile x tile (query x key) tiles, every tile
    a row tile reaches (anchor rows: anchor key tiles up to the diagonal; local rows: all anchor
    tiles, every passing slot's tiles, local tiles up to the diagonal).  useful / executed is the
    tile efficiency."""
    l_b = n // H
    lpp = min(l_p, l_b)
    L_A = host_L_A(host, l_q, l_a)
    cdiv = lambda a: (a + tile - 1) // tile  # noqa: E731
    nA, nB, nP = cdiv(L_A), cdiv(l_b), cdiv(lpp)
    visits = nA * (nA + 1) // 2 + nB * (nA + host * nP) + nB * (nB + 1) // 2
    return 4 * d * hq * tile * tile * visits


def attention_flops_split(n, H, host, l_a, l_p, hq, d, l_q=0):
    """(LOCAL-phase FLOPs, PASSING-phase FLOPs) of one host's layer."""
    l_b = n // H
    lpp = min(l_p, l_b)
    L_A = host_L_A(host, l_q, l_a)
    local = 4 * d * hq * (L_A * (L_A + 1) // 2 + l_b * L_A + l_b * (l_b + 1) // 2)
    passing = 4 * d * hq * l_b * host * lpp
    return local, passing


def score_flops(l_b: int, d_in: int, d_hidden: int, n_out: int) -> int:
    return l_b * (2 * d_in * d_hidden + 2 * d_hidden * n_out)


def attention_compulsory_bytes(L_A: int, P: int, l_b: int, hq: int, hk: int, d: int) -> int:
    """Q + O (bf16) + anchor/local K, V + passing K, V read once."""
    rows = L_A + l_b
    return 2 * rows * hq * d * 2 + 2 * rows * hk * d * 2 + 2 * P * hk * d * 2
