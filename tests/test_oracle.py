"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the pin id of SURVEY.md §8(c) / DESIGN.md and the paper passage.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def _attn_blas_all(q, k, v, L_A, pk, pv, scale=None):
    return oracle.attention_blas(q, k, v, L_A, pk, pv, np.arange(q.shape[0]), scale)


# every pin of the two oracle forms: the plain C loops and the full-size (fp64 library matmul) form
SCORERS = {"c": oracle.retain_score, "blas": oracle.retain_score_blas}
ATTNS = {"c": oracle.attention, "blas": _attn_blas_all}
scorer_forms = pytest.mark.parametrize("form", list(SCORERS))
attn_forms = pytest.mark.parametrize("form", list(ATTNS))


# ----------------------------------------------------------------------------- scorer

@scorer_forms
def test_scorer_hand_value(form):
    """P18: worked value tanh(1/2) for a 1-token, hidden-2 retaining head (tests/golden/scorer_hand.json)."""
    g = json.load(open(os.path.join(GOLD, "scorer_hand.json")))
    x = np.array(g["x"], np.float64)
    q, k, v = x[0].reshape(1, 1, 1), x[1].reshape(1, 1, 1), x[2].reshape(1, 1, 1)
    s = SCORERS[form](q, k, v, 0, np.array(g["w1"]), np.array(g["b1"]), np.array(g["w2"]),
                            np.array(g["b2"]), hk=1)
    assert abs(s[0, 0] - g["expected"]) < 1e-15


@scorer_forms
def test_scorer_silu_closed_form(form):
    """SiLU(z) = z/2 (1 + tanh(z/2)) — selecting single hidden units with W1/W2 one-hots."""
    hq, hk, d = 2, 1, 2
    d_in = (hq + 2 * hk) * d
    rng = np.random.default_rng(3)
    q = rng.standard_normal((5, hq, d)) * 3
    k = rng.standard_normal((5, hk, d)) * 3
    v = rng.standard_normal((5, hk, d)) * 3
    x = np.concatenate([q.reshape(5, -1), k.reshape(5, -1), v.reshape(5, -1)], 1)
    for u in range(d_in):
        w1 = np.zeros((4, d_in)); w1[1, u] = 1.0
        b1 = np.array([0.0, 0.25, 0.0, 0.0])
        w2 = np.zeros((1, 4)); w2[0, 1] = 1.0
        s = SCORERS[form](q, k, v, 0, w1, b1, w2, None, hk=1)
        z = x[:, u] + 0.25
        assert np.allclose(s[0], z / 2 * (1 + np.tanh(z / 2)), rtol=0, atol=1e-13)


@scorer_forms
def test_scorer_group_max_and_bias(form):
    """W2 = 0 => o = b2, s[j] = max of head j's group (reading G4, n_out = hq)."""
    hq, hk, d = 4, 2, 2
    rng = np.random.default_rng(4)
    q = rng.standard_normal((3, hq, d)); k = rng.standard_normal((3, hk, d)); v = rng.standard_normal((3, hk, d))
    w1 = rng.standard_normal((8, (hq + 2 * hk) * d))
    b2 = np.array([0.5, -1.0, 2.0, 3.0])
    s = SCORERS[form](q, k, v, 0, w1, None, np.zeros((4, 8)), b2, hk=hk)
    assert np.all(s[0] == 0.5) and np.all(s[1] == 3.0)


@scorer_forms
def test_scorer_matches_torch_fp64(form):
    """P10: torch fp64 Linear -> SiLU -> Linear -> group max on the same weights."""
    hq, hk, d, L_A, l_b, dh = 4, 2, 8, 3, 17, 32
    q = _rand((L_A + l_b, hq, d), 1); k = _rand((L_A + l_b, hk, d), 2); v = _rand((L_A + l_b, hk, d), 3)
    d_in = (hq + 2 * hk) * d
    w1 = _rand((dh, d_in), 4, 0.2); b1 = _rand(dh, 5, 0.1); w2 = _rand((hq, dh), 6, 0.3); b2 = _rand(hq, 7)
    s = SCORERS[form](q, k, v, L_A, w1, b1, w2, b2, hk)
    x = torch.cat([torch.from_numpy(a[L_A:]).reshape(l_b, -1) for a in (q, k, v)], 1)
    h = torch.nn.functional.silu(torch.nn.functional.linear(x, torch.from_numpy(w1), torch.from_numpy(b1)))
    o = torch.nn.functional.linear(h, torch.from_numpy(w2), torch.from_numpy(b2))
    ref = o.reshape(l_b, hk, hq // hk).amax(-1).T.numpy()
    assert np.allclose(s, ref, rtol=0, atol=1e-12)


@scorer_forms
def test_scorer_zero_weights_select_prefix(form):
    """P10: zero W1/W2 => constant scores => ties => indices 0..l_p'-1 (tie rule G5)."""
    hq, hk, d = 2, 1, 4
    q = _rand((10, hq, d), 1); k = _rand((10, hk, d), 2); v = _rand((10, hk, d), 3)
    s = SCORERS[form](q, k, v, 2, np.zeros((4, 16)), None, np.zeros((2, 4)), None, hk)
    assert np.all(s == 0.0)
    assert oracle.select_topk(s[0], 3).tolist() == [0, 1, 2]


# ----------------------------------------------------------------------------- selection

def test_select_spec_examples():
    """P11: SPEC.md:276-278 worked examples."""
    assert oracle.select_topk(np.array([3.0, 1.0, 2.0]), 2).tolist() == [0, 2]
    assert oracle.select_topk(np.array([3.0, 1.0, 2.0]), 5).tolist() == [0, 1, 2]
    assert oracle.select_topk(np.array([0.9, 0.9, 0.1]), 1).tolist() == [0]
    assert oracle.select_topk(np.array([1.0, 2.0]), 0).tolist() == []


def test_select_fuzz_vs_sort():
    """P11: 1000 fuzz cases vs Python's stable sort by (-score, index), incl. +-inf and ties."""
    rng = np.random.default_rng(11)
    for case in range(1000):
        n = int(rng.integers(1, 80))
        kind = case % 4
        if kind == 0:
            s = rng.standard_normal(n)
        elif kind == 1:
            s = rng.integers(-3, 3, n).astype(np.float64)
        elif kind == 2:
            s = rng.choice([-np.inf, np.inf, 0.0, 1.0, -1.0], n)
        else:
            s = np.full(n, 0.5)
        lp = int(rng.integers(0, n + 3))
        want = sorted(sorted(range(n), key=lambda i: (-s[i], i))[:min(lp, n)])
        assert oracle.select_topk(s, lp).tolist() == want


# ----------------------------------------------------------------------------- attention

def _onehot_probe(L_A, P, l_b, attn=oracle.attention):
    """Q = 0 => all visible logits 0 => O[r] = mean of visible V rows.  With V_k = e_k
    (one-hot over keys), O[r][k] = 1/|vis(r)| if k visible else 0 — the mask itself."""
    nk = L_A + P + l_b
    d = max(nk, 1)
    q = np.zeros((L_A + l_b, 1, d))
    k = np.zeros((L_A + l_b, 1, d))
    eye = np.eye(nk)
    v = np.concatenate([eye[:L_A], eye[L_A + P:]], 0)[:, None, :]
    pv = eye[L_A:L_A + P][:, None, :]
    O, lse = attn(q, k, v, L_A, np.zeros((P, 1, d)), pv)
    return (O[:, 0, :nk] > 0).astype(int), O, lse


@attn_forms
def test_mask_spec_worked_examples(form):
    """P7: SPEC.md:214-215 printed masks (tests/golden/mask_examples.json)."""
    g = json.load(open(os.path.join(GOLD, "mask_examples.json")))
    for c in g["cases"]:
        vis, _, _ = _onehot_probe(c["L_A"], c["P"], c["l_b"], ATTNS[form])
        assert vis.tolist() == c["rows"], c["cite"]


@attn_forms
def test_mask_closed_form_lse_counts(form):
    """P16: Q = 0 => lse[r] = ln|vis(r)| exactly; counts for (3,4,5) from the golden file."""
    g = json.load(open(os.path.join(GOLD, "mask_examples.json")))
    for c in g["visible_counts"]:
        vis, O, lse = _onehot_probe(c["L_A"], c["P"], c["l_b"], ATTNS[form])
        assert vis.sum(1).tolist() == c["counts"]
        assert np.allclose(lse[:, 0], np.log(c["counts"]), rtol=0, atol=1e-14)


@attn_forms
def test_mask_equals_restricted_causal_brute_force(form):
    """P7 / G1: for every (L_A, P, l_b) <= 5 the mask equals rows [0,L_A) u [L_A+P, end) of a
    plain lower-triangular causal mask over the concatenated sequence [A|P|B]."""
    for L_A, P, l_b in itertools.product(range(5), range(5), range(1, 5)):
        vis, _, _ = _onehot_probe(L_A, P, l_b, ATTNS[form])
        nk = L_A + P + l_b
        causal = np.tril(np.ones((nk, nk), int))
        rows = list(range(L_A)) + list(range(L_A + P, nk))
        assert vis.tolist() == causal[rows].tolist(), (L_A, P, l_b)


def _sdpa_reference(q, k, v, L_A, pk, pv, scale):
    """P1: torch fp64 scaled_dot_product_attention: anchor rows = is_causal SDPA over A; local
    rows = causal_lower_right over [A|P|B] (SURVEY App. B equivalence)."""
    hq, hk = q.shape[1], k.shape[1]
    g = hq // hk
    kseq = np.concatenate([k[:L_A], pk, k[L_A:]], 0)
    vseq = np.concatenate([v[:L_A], pv, v[L_A:]], 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).permute(1, 0, 2)  # [heads][rows][d]
    K = T(kseq).repeat_interleave(g, 0); V = T(vseq).repeat_interleave(g, 0)
    outs, lses = [], []
    Q = T(q)
    nk = kseq.shape[0]
    l_b = q.shape[0] - L_A
    if L_A:
        m = torch.ones(L_A, L_A, dtype=torch.bool).tril()
        outs.append(torch.nn.functional.scaled_dot_product_attention(Q[:, :L_A], K[:, :L_A], V[:, :L_A],
                                                                       attn_mask=m, scale=scale))
        lses.append(torch.logsumexp((Q[:, :L_A] @ K[:, :L_A].transpose(1, 2) * scale).masked_fill(~m, -math.inf), -1))
    m = torch.ones(l_b, nk, dtype=torch.bool).tril(diagonal=nk - l_b)  # causal_lower_right
    outs.append(torch.nn.functional.scaled_dot_product_attention(Q[:, L_A:], K, V, attn_mask=m, scale=scale))
    lses.append(torch.logsumexp((Q[:, L_A:] @ K.transpose(1, 2) * scale).masked_fill(~m, -math.inf), -1))
    O = torch.cat(outs, 1).permute(1, 0, 2).numpy()
    lse = torch.cat(lses, 1).T.numpy()
    return O, lse


@attn_forms
@pytest.mark.parametrize("L_A,P,l_b", [(0, 0, 9), (5, 0, 7), (0, 6, 5), (7, 9, 3), (16, 24, 33), (3, 4, 5)])
def test_attention_matches_torch_sdpa(L_A, P, l_b, form):
    """P1: oracle == torch fp64 SDPA (library special case) on random inputs, GQA g=2."""
    hq, hk, d = 4, 2, 16
    q = _rand((L_A + l_b, hq, d), 1, 2.0); k = _rand((L_A + l_b, hk, d), 2, 2.0); v = _rand((L_A + l_b, hk, d), 3)
    pk = _rand((P, hk, d), 4, 2.0); pv = _rand((P, hk, d), 5)
    scale = 1 / math.sqrt(d)
    O, lse = ATTNS[form](q, k, v, L_A, pk, pv, scale)
    Or, lr = _sdpa_reference(q, k, v, L_A, pk, pv, scale)
    assert np.allclose(O, Or, rtol=0, atol=1e-12)
    assert np.allclose(lse, lr, rtol=0, atol=1e-12)


def test_attention_row_subset_matches_full():
    hq, hk, d, L_A, P, l_b = 2, 1, 8, 4, 3, 9
    q = _rand((L_A + l_b, hq, d), 1); k = _rand((L_A + l_b, hk, d), 2); v = _rand((L_A + l_b, hk, d), 3)
    pk = _rand((P, hk, d), 4); pv = _rand((P, hk, d), 5)
    O, lse = oracle.attention(q, k, v, L_A, pk, pv)
    rows = [12, 0, 5, 3]
    O2, lse2 = oracle.attention(q, k, v, L_A, pk, pv, rows=rows)
    assert np.array_equal(O2, O[rows]) and np.array_equal(lse2, lse[rows])


@attn_forms
def test_attention_rows_sum_to_one(form):
    """P5: V = 1 => O = 1 (softmax rows sum to 1)."""
    hq, hk, d, L_A, P, l_b = 4, 2, 8, 6, 5, 11
    q = _rand((L_A + l_b, hq, d), 1, 3.0); k = _rand((L_A + l_b, hk, d), 2, 3.0)
    v = np.ones((L_A + l_b, hk, d)); pv = np.ones((P, hk, d))
    O, _ = ATTNS[form](q, k, v, L_A, _rand((P, hk, d), 4, 3.0), pv)
    assert np.allclose(O, 1.0, rtol=0, atol=1e-14)


@attn_forms
def test_attention_one_hot_probe(form):
    """P17: q_r = c k* (c large) => O[r] = V[k*] iff k* is visible to r; passing keys are
    visible to local rows only; local key i+1 is invisible to local row i."""
    hk, hq, d, L_A, P, l_b = 1, 1, 16, 4, 3, 6
    rng = np.random.default_rng(9)
    basis = np.linalg.qr(rng.standard_normal((d, d)))[0]  # orthonormal keys
    keys = basis[: L_A + P + l_b] * 4
    k = np.concatenate([keys[:L_A], keys[L_A + P:]], 0)[:, None]
    pk = keys[L_A:L_A + P][:, None]
    vals = rng.standard_normal((L_A + P + l_b, d))
    v = np.concatenate([vals[:L_A], vals[L_A + P:]], 0)[:, None]
    pv = vals[L_A:L_A + P][:, None]
    # probe: local row i=2 targets passing key 1 -> must get it; anchor row 3 targets passing -> must not
    q = np.zeros((L_A + l_b, 1, d))
    q[L_A + 2, 0] = keys[L_A + 1] * 50
    q[3, 0] = keys[L_A + 1] * 50
    q[L_A + 1, 0] = keys[L_A + P + 2] * 50  # local row 1 targets local key 2 (future) -> invisible
    O, _ = ATTNS[form](q, k, v, L_A, pk, pv)
    assert np.allclose(O[L_A + 2, 0], vals[L_A + 1], atol=1e-9)
    assert not np.allclose(O[3, 0], vals[L_A + 1], atol=1e-3)
    assert not np.allclose(O[L_A + 1, 0], vals[L_A + P + 2], atol=1e-3)


@attn_forms
def test_attention_passing_permutation_invariance(form):
    """P9: permuting passing keys together with their values leaves O unchanged."""
    hq, hk, d, L_A, P, l_b = 2, 1, 8, 3, 7, 5
    q = _rand((L_A + l_b, hq, d), 1); k = _rand((L_A + l_b, hk, d), 2); v = _rand((L_A + l_b, hk, d), 3)
    pk = _rand((P, hk, d), 4); pv = _rand((P, hk, d), 5)
    perm = np.random.default_rng(0).permutation(P)
    O1, l1 = ATTNS[form](q, k, v, L_A, pk, pv)
    O2, l2 = ATTNS[form](q, k, v, L_A, pk[perm], pv[perm])
    assert np.allclose(O1, O2, atol=1e-13) and np.allclose(l1, l2, atol=1e-13)


# ----------------------------------------------------------------------------- pipeline

def _toy(**kw):
    return synth.CONFIGS["toy"].replace(n=kw.pop("n", 256), l_a=kw.pop("l_a", 16), l_p=kw.pop("l_p", 8),
                                        d_hidden=kw.pop("d_hidden", 32), **kw)


def _hosts(cfg, layer=0):
    return [synth.host_qkv(cfg, layer, h) for h in range(cfg.H)]


def _causal_sdpa(q, k, v, scale):
    hq, hk = q.shape[1], k.shape[1]
    Q = torch.from_numpy(q).permute(1, 0, 2)
    K = torch.from_numpy(k).permute(1, 0, 2).repeat_interleave(hq // hk, 0)
    V = torch.from_numpy(v).permute(1, 0, 2).repeat_interleave(hq // hk, 0)
    m = torch.ones(q.shape[0], k.shape[0], dtype=torch.bool).tril(diagonal=k.shape[0] - q.shape[0])
    return torch.nn.functional.scaled_dot_product_attention(Q, K, V, attn_mask=m, scale=scale).permute(1, 0, 2).numpy()


def test_pipeline_single_host_is_causal():
    """P2: H = 1 (P:640 'falls back to vanilla FlashAttn') => exact causal attention."""
    cfg = _toy(H=1, n=96)
    hosts = _hosts(cfg)
    w = synth.retain_weights(cfg, 0)
    res = oracle.prefill_layer(hosts, w, cfg.l_p)
    x = hosts[0]
    f = synth.bf16_bits_to_f64
    ref = _causal_sdpa(f(x["q"]), f(x["k"]), f(x["v"]), 1 / math.sqrt(cfg.d))
    assert np.allclose(res["O"][0], ref, atol=1e-12)


def test_pipeline_lp_zero_is_star_attention():
    """P4: l_p = 0 => host output = causal attention over [A | B_h] (StarAttn)."""
    cfg = _toy(l_p=0)
    hosts = _hosts(cfg)
    res = oracle.prefill_layer(hosts, synth.retain_weights(cfg, 0), 0)
    f = synth.bf16_bits_to_f64
    for h in range(cfg.H):
        x = hosts[h]
        ref = _causal_sdpa(f(x["q"]), f(x["k"]), f(x["v"]), 1 / math.sqrt(cfg.d))
        assert np.allclose(res["O"][h], ref, atol=1e-12)


def test_pipeline_lp_full_is_exact_prefix_attention():
    """P3 / P19: l_p = l_b => local rows of host h = exact causal attention over
    [A | B_1 | ... | B_h] whatever the scores (every block token passes, in order)."""
    cfg = _toy(l_p=10 ** 6)
    hosts = _hosts(cfg)
    res = oracle.prefill_layer(hosts, synth.retain_weights(cfg, 0), cfg.l_p)
    f = synth.bf16_bits_to_f64
    for h in range(cfg.H):
        x = hosts[h]
        L_A = x["L_A"]
        ks = np.concatenate([f(x["k"][:L_A])] + [f(hosts[s]["k"][hosts[s]["L_A"]:]) for s in range(h)] + [f(x["k"][L_A:])])
        vs = np.concatenate([f(x["v"][:L_A])] + [f(hosts[s]["v"][hosts[s]["L_A"]:]) for s in range(h)] + [f(x["v"][L_A:])])
        ref = _causal_sdpa(f(x["q"][L_A:]), ks, vs, 1 / math.sqrt(cfg.d))
        assert np.allclose(res["O"][h][L_A:], ref, atol=1e-12)


def test_pipeline_consistent_anchor():
    """P6 / P19: anchor outputs are identical on hosts 2..H and equal host 1's first l_a rows."""
    cfg = _toy()
    res = oracle.prefill_layer(_hosts(cfg), synth.retain_weights(cfg, 0), cfg.l_p)
    for h in range(1, cfg.H):
        assert np.array_equal(res["O"][h][:cfg.l_a], res["O"][0][:cfg.l_a])


def test_pipeline_needles_always_passed():
    """P12: planted +large scores are always selected and reach every later host."""
    cfg = _toy()
    hosts = _hosts(cfg)
    rng = np.random.default_rng(5)
    scores, needles = [], []
    for h in range(cfg.H):
        s = rng.standard_normal((cfg.hk, cfg.l_b))
        nd = rng.choice(cfg.l_b, 3, replace=False)
        s[:, nd] = 1e30
        scores.append(s); needles.append(nd)
    res = oracle.prefill_layer(hosts, None, cfg.l_p, scores_override=scores)
    for h in range(cfg.H):
        for j in range(cfg.hk):
            assert set(needles[h]).issubset(set(res["indices"][h][j].tolist()))
            for nd in needles[h]:
                m = res["indices"][h][j].tolist().index(nd)
                assert np.array_equal(res["gathered"][h][0, j, m], hosts[h]["k"][hosts[h]["L_A"] + nd, j])


def test_pipeline_compaction_equals_masked_full_block():
    """P13: attention over the compacted passing keys == attention over the full earlier blocks
    with the unselected keys masked out; compaction copies rows verbatim."""
    cfg = _toy(H=2)
    hosts = _hosts(cfg)
    res = oracle.prefill_layer(hosts, synth.retain_weights(cfg, 0), cfg.l_p)
    f = synth.bf16_bits_to_f64
    x0, x1 = hosts
    idx = res["indices"][0]
    # verbatim rows
    for j in range(cfg.hk):
        assert np.array_equal(res["sends"][0][0, j], x0["k"][idx[j], j])
        assert np.array_equal(res["sends"][0][1, j], x0["v"][idx[j], j])
    # masked-full reference for host 1's local rows, per KV head (each head has its own set)
    L_A = x1["L_A"]
    g = cfg.hq // cfg.hk
    scale = 1 / math.sqrt(cfg.d)
    for qh in range(cfg.hq):
        j = qh // g
        ks = np.concatenate([f(x1["k"][:L_A, j]), f(x0["k"][:, j]), f(x1["k"][L_A:, j])])
        vs = np.concatenate([f(x1["v"][:L_A, j]), f(x0["v"][:, j]), f(x1["v"][L_A:, j])])
        nk = ks.shape[0]
        m = np.ones((cfg.l_b, nk), bool)
        m &= np.tril(np.ones((cfg.l_b, nk), bool), k=nk - cfg.l_b)
        sel = np.zeros(cfg.l_b, bool); sel[idx[j]] = True
        m[:, L_A:L_A + cfg.l_b] &= sel[None]
        Q = torch.from_numpy(f(x1["q"][L_A:, qh]))[None]
        ref = torch.nn.functional.scaled_dot_product_attention(Q, torch.from_numpy(ks)[None], torch.from_numpy(vs)[None],
                                                               attn_mask=torch.from_numpy(m), scale=scale)[0].numpy()
        assert np.allclose(res["O"][1][L_A:, qh], ref, atol=1e-12)


def test_all_gather_volume_and_identity():
    """P14: every host holds [C_1..C_H]; bytes = 2*H*l_p'*hk*d*2 per layer."""
    cfg = _toy()
    res = oracle.prefill_layer(_hosts(cfg), synth.retain_weights(cfg, 0), cfg.l_p)
    G = res["gathered"]
    assert G.nbytes == 2 * cfg.H * cfg.l_pp * cfg.hk * cfg.d * 2
    for h in range(cfg.H):
        assert np.array_equal(G[h], res["sends"][h])
    one = oracle.all_gather([res["sends"][0]])
    assert np.array_equal(one[0], res["sends"][0])


def test_determinism():
    """P15: repeated runs are bit-identical."""
    cfg = _toy()
    a = oracle.prefill_layer(_hosts(cfg), synth.retain_weights(cfg, 0), cfg.l_p)
    b = oracle.prefill_layer(_hosts(cfg), synth.retain_weights(cfg, 0), cfg.l_p)
    for h in range(cfg.H):
        assert np.array_equal(a["O"][h], b["O"][h]) and np.array_equal(a["indices"][h], b["indices"][h])


def test_synth_bf16_rounding():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e38], np.float32)
    b = synth.f32_to_bf16_bits(x)
    back = synth.bf16_bits_to_f32(b)
    assert back[0] == 1.0 and back[1] == 1.0  # tie -> even
    assert back[2] == 1.0078125 and back[3] == -2.5


# ----------------------------------------------------------------------------- decode (NEXT #1)

def _sdpa_new_over_caches(q, caches, k_new, v_new, scale):
    """torch fp64 SDPA: the t new rows attend to every cached key (in host order) and causally
    to the new keys — single-host exact attention (SPEC S:413 'equals single-host ... decoding')."""
    hq, hk = q.shape[1], k_new.shape[1]
    K = np.concatenate([c[0] for c in caches] + [k_new])
    V = np.concatenate([c[1] for c in caches] + [v_new])
    t, nk = q.shape[0], K.shape[0]
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).permute(1, 0, 2)
    m = torch.ones(t, nk, dtype=torch.bool).tril(diagonal=nk - t)
    Kt = T(K).repeat_interleave(hq // hk, 0)
    Vt = T(V).repeat_interleave(hq // hk, 0)
    O = torch.nn.functional.scaled_dot_product_attention(T(q), Kt, Vt, attn_mask=m, scale=scale)
    lse = torch.logsumexp((T(q) @ Kt.transpose(1, 2) * scale).masked_fill(~m, -math.inf), -1)
    return O.permute(1, 0, 2).numpy(), lse.T.numpy()


@pytest.mark.parametrize("H,t,c", [(1, 1, 37), (4, 1, 50), (4, 5, 33), (3, 3, 0), (2, 8, 129)])
def test_decode_step_equals_exact_attention(H, t, c):
    """Alg. apb_decode is exact: MergeScore of the per-host partials (last host with
    the new tokens' own keys) == one-shot attention over [B_1 .. B_H | new]."""
    hq, hk, d = 4, 2, 16
    rng = np.random.default_rng(H * 100 + t)
    caches = [(rng.standard_normal((c, hk, d)) * 1.5, rng.standard_normal((c, hk, d))) for _ in range(H)]
    q = rng.standard_normal((t, hq, d)) * 1.5
    kn, vn = rng.standard_normal((t, hk, d)) * 1.5, rng.standard_normal((t, hk, d))
    A, L, parts = oracle.decode_step(q, caches, kn, vn)
    ref, ref_lse = _sdpa_new_over_caches(q, caches, kn, vn, 1 / math.sqrt(d))
    assert np.allclose(A, ref, atol=1e-12) and np.allclose(L, ref_lse, atol=1e-12)
    # every host's partial is itself exact attention over that host's keys
    for h, (O_h, l_h) in enumerate(parts):
        last = h == H - 1
        ks = [caches[h]] if c else []
        if last:
            r, rl = _sdpa_new_over_caches(q, ks, kn, vn, 1 / math.sqrt(d))
            assert np.allclose(O_h, r, atol=1e-12) and np.allclose(l_h, rl, atol=1e-12)
        elif c:
            Kc, Vc = caches[h]
            T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).permute(1, 0, 2)
            r = torch.nn.functional.scaled_dot_product_attention(
                T(q), T(Kc).repeat_interleave(2, 0), T(Vc).repeat_interleave(2, 0), scale=1 / math.sqrt(d))
            assert np.allclose(O_h, r.permute(1, 0, 2).numpy(), atol=1e-12)
        else:
            assert np.all(np.isneginf(l_h)) and np.all(O_h == 0)


def test_merge_score_spec_examples():
    """single part = identity; two identical parts = same vector; two disjoint key
    halves of an 8-key attention == attention over all 8 keys."""
    rng = np.random.default_rng(7)
    o, l = rng.standard_normal((1, 3, 5)), rng.standard_normal((1, 3))
    A, L = oracle.merge_score(o, l)
    assert np.array_equal(A, o[0]) and np.array_equal(L, l[0])
    A, L = oracle.merge_score(np.concatenate([o, o]), np.concatenate([l, l]))
    assert np.allclose(A, o[0], atol=1e-15) and np.allclose(L, l[0] + math.log(2), atol=1e-15)
    q = rng.standard_normal((1, 1, 4)); k = rng.standard_normal((8, 1, 4)); v = rng.standard_normal((8, 1, 4))
    full, full_l = oracle.decode_partial(q, k, v)
    a1, l1 = oracle.decode_partial(q, k[:3], v[:3])
    a2, l2 = oracle.decode_partial(q, k[3:], v[3:])
    A, L = oracle.merge_score(np.stack([a1, a2]), np.stack([l1, l2]))
    assert np.allclose(A, full, atol=1e-14) and np.allclose(L, full_l, atol=1e-14)


# ------------------------------------------------------------------ method variants (NEXT #3)
def test_random_scores_match_splitmix64_reference_stream():
    """Rd. compressor (Table 4), reading G17: the scores are the published
    SplitMix64 outputs (tests/golden/splitmix64.json), top 24 bits, times 2^-24."""
    g = json.load(open(os.path.join(GOLD, "splitmix64.json")))
    want = [int(h, 16) >> 40 for h in g["outputs_hex"]]
    s = oracle.random_scores(g["seed"], 0, 1, 0, 1, len(want))
    assert s.shape == (1, len(want))
    assert [int(x * 2 ** 24) for x in s[0]] == want
    assert np.all(s * 2 ** 24 == np.floor(s * 2 ** 24))  # exact 24-bit grid, in [0, 1)


def test_random_scores_counter_layout_and_determinism():
    """c = ((layer*H + host)*hk + j)*l_b + t indexes one stream: a host's block is a slice of it."""
    seed, H, hk, l_b = 12345, 3, 2, 5
    stream = oracle.random_scores(seed, 0, 1, 0, 1, 4 * H * hk * l_b)[0]
    for layer in range(2):
        for host in range(H):
            s = oracle.random_scores(seed, layer, H, host, hk, l_b)
            c0 = (layer * H + host) * hk * l_b
            np.testing.assert_array_equal(s.reshape(-1), stream[c0:c0 + hk * l_b])
            np.testing.assert_array_equal(s, oracle.random_scores(seed, layer, H, host, hk, l_b))
    assert not np.array_equal(oracle.random_scores(1, 0, 1, 0, 2, 64), oracle.random_scores(2, 0, 1, 0, 2, 64))


def test_random_selector_is_uniform_monte_carlo():
    """over 200 trials each index is selected with frequency l_p/l_b +- 0.05."""
    l_b, l_p, trials = 64, 16, 200
    counts = np.zeros(l_b)
    for layer in range(trials):
        s = oracle.random_scores(7, layer, 1, 0, 1, l_b)
        counts[oracle.select_topk(s[0], l_p)] += 1
    freq = counts / trials
    assert np.all(np.abs(freq - l_p / l_b) <= 0.1)  # per-index binomial sd = 0.031; 3.2 sd
    assert abs(freq.mean() - l_p / l_b) < 1e-12  # exactly l_p picks per trial
    # and the scores themselves are uniform: Kolmogorov-Smirnov distance vs U[0,1)
    u = np.sort(oracle.random_scores(7, 0, 1, 0, 1, 20000)[0])
    ks = np.max(np.abs(u - np.arange(1, u.size + 1) / u.size))
    assert ks < 1.63 / np.sqrt(u.size)  # 1 % critical value


def test_share_scores_examples():
    """Shared index set: max over KV heads, then one selection for all."""
    s = np.array([[3.0, 1.0, 2.0], [0.0, 5.0, 1.0]])
    sh = oracle.share_scores(s)
    np.testing.assert_array_equal(sh, [[3, 5, 2], [3, 5, 2]])
    idx = oracle.select_all_heads(sh, 2)
    np.testing.assert_array_equal(idx, [[0, 1], [0, 1]])
    # per-head selection of the same scores differs (head 1 would take 1, 2)
    np.testing.assert_array_equal(oracle.select_all_heads(s, 2), [[0, 2], [1, 2]])
    # one KV head: identity
    one = np.array([[0.5, -1.0, 2.0]])
    np.testing.assert_array_equal(oracle.share_scores(one), one)
    # the shared set maximises the head-max of the selected scores (brute force, tiny case)
    rng = np.random.default_rng(3)
    s = rng.standard_normal((3, 7))
    best = max(itertools.combinations(range(7), 3), key=lambda c: (sorted(s.max(0)[list(c)], reverse=True)))
    np.testing.assert_array_equal(oracle.select_all_heads(oracle.share_scores(s), 3)[0], sorted(best))


def test_attention_q_subset_equals_full_rows():
    """The q_subset indexing option (sampled checks at maximum sizes) returns exactly the rows of
    the full-Q call."""
    rng = np.random.default_rng(11)
    L_A, P, l_b, hq, hk, d = 5, 3, 9, 4, 2, 8
    q = rng.standard_normal((L_A + l_b, hq, d))
    k, v = rng.standard_normal((L_A + l_b, hk, d)), rng.standard_normal((L_A + l_b, hk, d))
    pk, pv = rng.standard_normal((P, hk, d)), rng.standard_normal((P, hk, d))
    rows = np.array([13, 0, 6, 4, 5])
    O, lse = oracle.attention(q, k, v, L_A, pk, pv, rows=rows)
    O2, lse2 = oracle.attention(q[rows], k, v, L_A, pk, pv, rows=rows, q_subset=True)
    np.testing.assert_array_equal(O, O2)
    np.testing.assert_array_equal(lse, lse2)


def test_blas_forms_sampled_rows_and_bf16_inputs():
    """The full-size forms take bf16 bit patterns, sampled (unsorted, repeated-limit) rows and
    q_subset exactly as the C forms do (same outputs to rounding)."""
    cfg = synth.CONFIGS["toy"].replace(n=1024, l_a=96, l_p=40, d_hidden=64)
    x = synth.host_qkv(cfg, 0, 2)
    w = synth.retain_weights(cfg, 0)
    s_c = oracle.retain_score(x["q"], x["k"], x["v"], x["L_A"], w["w1"], w["b1"], w["w2"], w["b2"], cfg.hk)
    s_b = oracle.retain_score_blas(x["q"], x["k"], x["v"], x["L_A"], w["w1"], w["b1"], w["w2"], w["b2"], cfg.hk,
                                   chunk=100)
    assert np.allclose(s_c, s_b, rtol=0, atol=1e-12)
    g = synth.f32_to_bf16_bits(_rand((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d), 3).astype(np.float32))
    pk, pv = oracle.passing(g, 2)
    rows = [300, 0, 95, 96, 97, 351, 5, 200]
    O_c, l_c = oracle.attention(x["q"], x["k"], x["v"], x["L_A"], pk, pv, rows=rows)
    O_b, l_b = oracle.attention_blas(x["q"], x["k"], x["v"], x["L_A"], pk, pv, rows, chunk=3)
    assert np.allclose(O_c, O_b, rtol=0, atol=1e-12) and np.allclose(l_c, l_b, rtol=0, atol=1e-12)
    O_s, l_s = oracle.attention_blas(x["q"][rows], x["k"], x["v"], x["L_A"], pk, pv, rows, q_subset=True)
    assert np.allclose(O_s, O_b, rtol=0, atol=1e-13) and np.allclose(l_s, l_b, rtol=0, atol=1e-13)
