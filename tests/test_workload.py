"""Work accounting used by bench.py (host logic, CPU): useful FLOPs from the mask (reading G13)
and the executed whole-tile MMA FLOPs (SURVEY 8(d) tile efficiency)."""
import itertools

import numpy as np

from paper_2502_12085_b200 import workload


def _mask_pairs(L_A, P, l_b):
    """Visible (row, key) pairs by brute force over an explicit mask M' (reading G1)."""
    n_k = L_A + P + l_b
    m = np.zeros((L_A + l_b, n_k), bool)
    for r in range(L_A):
        m[r, : r + 1] = True
    for i in range(l_b):
        m[L_A + i, : L_A + P + i + 1] = True
    return int(m.sum())


def test_visible_pairs_brute_force():
    for L_A, P, l_b in itertools.product([0, 1, 3, 7], [0, 2, 5], [1, 4, 9]):
        assert workload.visible_pairs(L_A, P, l_b) == _mask_pairs(L_A, P, l_b)


def test_executed_flops_bounds_and_unit_tile():
    for n, H, l_a, l_p in [(2048, 4, 128, 64), (131072, 8, 4096, 2048), (1536, 3, 200, 100), (1000, 5, 37, 300)]:
        for h in range(H):
            u = workload.attention_flops(n, H, h, l_a, l_p, 4, 64)
            e = workload.attention_executed_flops(n, H, h, l_a, l_p, 4, 64)
            assert e >= u
            # with 1 x 1 tiles the kernel would execute exactly the visible pairs
            assert workload.attention_executed_flops(n, H, h, l_a, l_p, 4, 64, tile=1) == u


def test_executed_flops_l8_tile_efficiency():
    n, H, l_a, l_p, hq, d = 131072, 8, 4096, 2048, 32, 128
    eff = [workload.attention_flops(n, H, h, l_a, l_p, hq, d) / workload.attention_executed_flops(n, H, h, l_a, l_p, hq, d)
           for h in range(H)]
    assert all(0.99 < e <= 1.0 for e in eff)
