"""GPU parity: libapb (sm_100a, through the C ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star, made precise in SURVEY.md 8(c) / DESIGN.md):
  attention  max|O - O_or| <= 2e-2, mean|O - O_or| <= 2e-3, |lse - lse_or| <= 1e-2
  scores     |s - s_or| <= 1e-2 * max(|s_or|, rms_j(s_or))
  indices    bit-exact vs the oracle's stable sort of the SAME fp32 scores; end to end, every
             index in the symmetric difference has an oracle score within 1e-3 of the cut
  compaction / gathered buffer: bit-exact
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ATOL_MAX, ATOL_MEAN, LSE_TOL = 2e-2, 2e-3, 1e-2


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_12085_b200 import apb, build
    build.build()
    apb.load()


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def to_bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def dims_of(cfg, host):
    from paper_2502_12085_b200 import apb
    return apb.Dims(n=cfg.n, H=cfg.H, host=host, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq,
                    n_kv_heads=cfg.hk, head_dim=cfg.d, l_q=cfg.l_q)


def weights_dev(w):
    from paper_2502_12085_b200 import apb
    return apb.RetainWeights(w1=dev(w["w1"]), w2=torch.from_numpy(w["w2"]).cuda(),
                             b1=torch.from_numpy(w["b1"]).cuda(), b2=torch.from_numpy(w["b2"]).cuda())


def check_attention(O, lse, O_ref, lse_ref, what):
    err = np.abs(O - O_ref)
    lerr = np.abs(lse - lse_ref)
    msg = f"{what}: max {err.max():.3e} mean {err.mean():.3e} lse {lerr.max():.3e}"
    print(msg)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN and lerr.max() <= LSE_TOL, msg


def run_attention(cfg, host, x, gathered_bits, phase):
    """x: synth host dict; returns (O fp64 [rows][hq][d], lse fp64 [rows][hq])."""
    from paper_2502_12085_b200 import apb
    d = dims_of(cfg, host)
    q, k, v = dev(x["q"]), dev(x["k"]), dev(x["v"])
    out = torch.full_like(q, float("nan"))
    lse = torch.full((cfg.hq, d.rows), float("nan"), device="cuda")
    g = dev(gathered_bits) if gathered_bits is not None else None
    n_ws = apb.workspace_size(d, apb.WS_ATTENTION)
    ws = torch.empty(max(n_ws, 16), dtype=torch.uint8, device="cuda")
    if phase == "split":
        apb.attention_fwd(d, q, k, v, None, out, lse, phase=apb.PHASE_LOCAL, ws=ws)
        apb.attention_fwd(d, q, k, v, g, out, lse, phase=apb.PHASE_PASSING, ws=ws)
    else:
        apb.attention_fwd(d, q, k, v, g, out, lse, phase=apb.PHASE_ALL, ws=ws)
    torch.cuda.synchronize()
    return out.float().cpu().double().numpy(), lse.cpu().double().numpy().T


def oracle_layer(cfg):
    hosts = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    return hosts, oracle.prefill_layer(hosts, synth.retain_weights(cfg, 0), cfg.l_p)


# ----------------------------------------------------------------------------- attention

CASES = {
    "toy": synth.CONFIGS["toy"],
    "d128-ragged": synth.Config("d128-ragged", 11, n=1536, H=3, l_a=200, l_p=100, hq=8, hk=2, d=128, d_hidden=256),
    "gqa3": synth.Config("gqa3", 12, n=1024, H=4, l_a=64, l_p=48, hq=6, hk=2, d=128, d_hidden=256),
    "d64-peaky": synth.Config("d64-peaky", 13, n=1280, H=5, l_a=40, l_p=30, hq=4, hk=1, d=64, d_hidden=256,
                              dist="D2"),
    "d128-sink": synth.Config("d128-sink", 14, n=2048, H=4, l_a=256, l_p=128, hq=4, hk=2, d=128, d_hidden=256,
                              dist="D3"),
    "lq": synth.Config("lq", 15, n=1024, H=2, l_a=100, l_p=64, hq=4, hk=2, d=64, d_hidden=256, l_q=37),
    # MHA (g = 1: one query head per KV head, odd unit count per KV head) and g = 8 (Llama-70B ratio)
    "mha": synth.Config("mha", 16, n=1152, H=3, l_a=70, l_p=40, hq=3, hk=3, d=128, d_hidden=256),
    "gqa8": synth.Config("gqa8", 17, n=768, H=2, l_a=130, l_p=96, hq=16, hk=2, d=64, d_hidden=256),
    # d = 128 with g % 4 == 0 runs the paired (2-CTA cluster, multicast K/V) kernel; g = 8 pairs
    # two items of one row tile, ragged anchor / local tails
    "gqa8-d128": synth.Config("gqa8-d128", 18, n=1656, H=3, l_a=150, l_p=70, hq=16, hk=2, d=128, d_hidden=256),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("phase", ["all", "split"])
def test_attention_parity(name, phase):
    cfg = CASES[name]
    hosts, ref = oracle_layer(cfg)
    for h in range(cfg.H):
        O, lse = run_attention(cfg, h, hosts[h], ref["gathered"], phase)
        check_attention(O, lse, ref["O"][h], ref["lse"][h], f"{name} host {h} {phase}")


def test_attention_single_host_causal():
    """H = 1: plain causal attention, no anchor, no passing."""
    cfg = synth.Config("h1", 16, n=700, H=1, l_a=64, l_p=32, hq=4, hk=2, d=128, d_hidden=256)
    hosts, ref = oracle_layer(cfg)
    O, lse = run_attention(cfg, 0, hosts[0], None, "all")
    check_attention(O, lse, ref["O"][0], ref["lse"][0], "H=1")


def test_attention_lp_zero():
    """l_p = 0: StarAttn-style, gathered may be NULL."""
    cfg = synth.CONFIGS["toy"].replace(l_p=0)
    hosts, ref = oracle_layer(cfg)
    for h in range(cfg.H):
        O, lse = run_attention(cfg, h, hosts[h], None, "split")
        check_attention(O, lse, ref["O"][h], ref["lse"][h], f"lp0 host {h}")


def test_attention_uniform_closed_form():
    """Q = 0 => lse = ln|vis(r)| and O = mean of visible V (pin P16 on the GPU path).  One pass
    (ALL): every weight is 2^0 = 1, exact.  LOCAL + PASSING: the passing weights are
    2^-log2(count_local), rounded to bf16 for the PV MMA, and the normaliser sums those rounded
    weights (reading G21), so |d lse| <= ln(1 + 2^-8) (one bf16 ulp of relative weight
    error) while O, an average with equal weights, stays exact to fp32 rounding."""
    from paper_2502_12085_b200 import apb
    cfg = CASES["d128-ragged"]
    h = 2
    x = dict(synth.host_qkv(cfg, 0, h))
    x["q"] = np.zeros_like(x["q"])
    hosts, ref = oracle_layer(cfg)
    L_A, P = cfg.L_A(h), cfg.P(h)
    counts = np.array([r + 1 for r in range(L_A)] + [L_A + P + i + 1 for i in range(cfg.l_b)], np.float64)
    for phase, tol in (("all", 1e-5), ("split", math.log1p(2.0 ** -8))):
        O, lse = run_attention(cfg, h, x, ref["gathered"], phase)
        assert np.abs(lse - np.log(counts)[:, None]).max() < tol, phase


# ----------------------------------------------------------------------------- scoring / selection

@pytest.mark.parametrize("name", ["toy", "d128-ragged", "gqa3", "yi-heads"])
@pytest.mark.parametrize("n_out", ["hq", "hk"])
def test_retain_score_parity(name, n_out):
    from paper_2502_12085_b200 import apb
    # yi-heads: 56 query heads (n_out = 56 > 32: two 32-output passes of the pair-GEMM epilogue),
    # l_b = 700 (a ragged last 256-row pair tile)
    cfg = (CASES[name] if name in CASES else
           synth.Config("yi-heads", 20, n=1400, H=2, l_a=64, l_p=100, hq=56, hk=8, d=64)).replace(d_hidden=1024)
    w = synth.retain_weights(cfg, 0, n_out=cfg.hq if n_out == "hq" else cfg.hk)
    for h in range(cfg.H):
        x = synth.host_qkv(cfg, 0, h)
        s = torch.empty((cfg.hk, cfg.l_b), dtype=torch.float32, device="cuda")
        apb.retain_score(dims_of(cfg, h), weights_dev(w), dev(x["q"]), dev(x["k"]), dev(x["v"]), s)
        torch.cuda.synchronize()
        s = s.cpu().double().numpy()
        s_or = oracle.retain_score(x["q"], x["k"], x["v"], x["L_A"], w["w1"], w["b1"], w["w2"], w["b2"], cfg.hk)
        floor = np.sqrt((s_or ** 2).mean(axis=1, keepdims=True))
        rel = np.abs(s - s_or) / np.maximum(np.abs(s_or), floor)
        print(f"{name} h{h} n_out={n_out}: max rel {rel.max():.3e} max abs {np.abs(s - s_or).max():.3e}")
        assert rel.max() <= 1e-2
        # determinism (pin P15): bit-identical on a second run
        s2 = torch.empty((cfg.hk, cfg.l_b), dtype=torch.float32, device="cuda")
        apb.retain_score(dims_of(cfg, h), weights_dev(w), dev(x["q"]), dev(x["k"]), dev(x["v"]), s2)
        assert np.array_equal(s2.cpu().double().numpy(), s)


@pytest.mark.parametrize("plan", ["s3", "p2"])
def test_retain_score_plans_bit_identical(plan, monkeypatch):
    """The single-CTA scoring kernel's pipeline plans (APB_SCORE_PLAN: 3- or 4-stage ring, one or
    two hidden chunks per pass over the A rows) run the same MMAs in the same K order and the same
    epilogue: bit-identical.  (The default CTA-pair GEMM sums in its own fixed order: checked
    against the oracle and for run-to-run determinism in test_retain_score_parity.)"""
    from paper_2502_12085_b200 import apb
    cfg = CASES["d128-ragged"].replace(d_hidden=1024)
    w = synth.retain_weights(cfg, 0, n_out=cfg.hq)
    x = synth.host_qkv(cfg, 0, 1)
    out = []
    for env in ("legacy", plan):
        monkeypatch.setenv("APB_SCORE_PLAN", env)
        s = torch.empty((cfg.hk, cfg.l_b), dtype=torch.float32, device="cuda")
        apb.retain_score(dims_of(cfg, 1), weights_dev(w), dev(x["q"]), dev(x["k"]), dev(x["v"]), s)
        torch.cuda.synchronize()
        out.append(s.cpu().numpy())
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("name", ["toy", "d128-ragged", "gqa3", "yi-heads"])
@pytest.mark.parametrize("tail", ["", "0"])
def test_retain_score_hosts_equals_per_host(name, tail, monkeypatch):
    """apb_retain_score_hosts (every host's tiles in one CTA-pair GEMM launch: tile T of host
    T / tiles_per_host, the partial last wave split into half tiles across hosts; one finalize
    launch) gives the per-host apb_retain_score scores bit for bit — each tile and each partial
    slot is computed in the same fixed order whichever launch it belongs to."""
    from paper_2502_12085_b200 import apb
    monkeypatch.setenv("APB_GEMM_TAIL_SPLIT", tail)
    cfg = (CASES[name] if name in CASES else
           synth.Config("yi-heads", 20, n=1400, H=2, l_a=64, l_p=100, hq=56, hk=8, d=64)).replace(d_hidden=1024)
    w = weights_dev(synth.retain_weights(cfg, 0, n_out=cfg.hq))
    xs = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    for hs in (list(range(cfg.H)), list(range(cfg.H - 1, -1, -2))):
        ds = [dims_of(cfg, h) for h in hs]
        q = [dev(xs[h]["q"]) for h in hs]
        k = [dev(xs[h]["k"]) for h in hs]
        v = [dev(xs[h]["v"]) for h in hs]
        sc = [torch.full((cfg.hk, cfg.l_b), float("nan"), device="cuda") for _ in hs]
        ws = torch.empty(apb.retain_workspace_size(ds[0], w) * len(hs), dtype=torch.uint8, device="cuda")
        apb.retain_score_hosts(ds, w, q, k, v, sc, ws)
        for i, h in enumerate(hs):
            ref = torch.empty((cfg.hk, cfg.l_b), device="cuda")
            apb.retain_score(ds[i], w, q[i], k[i], v[i], ref)
            torch.cuda.synchronize()
            assert torch.equal(sc[i], ref), (hs, h)


@pytest.mark.parametrize("name", ["toy", "d128-ragged", "gqa3", "big"])
def test_select_topk_hosts_equals_per_host(name):
    """apb_select_topk_hosts (one select launch over every host's KV heads, one gather launch;
    "big": l_b = 40000 > 32K, where each host runs the 8-CTA cluster kernel) gives the oracle's
    indices and send slots bit for bit."""
    from paper_2502_12085_b200 import apb
    cfg = CASES[name] if name in CASES else synth.Config("big", 24, n=3 * 40000, H=3, l_a=64, l_p=2048, hq=8,
                                                        hk=4, d=128, d_hidden=256)
    xs = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    sc = [torch.from_numpy(np.ascontiguousarray(synth.random_scores(cfg, 0, h, ties=True), dtype=np.float32)).cuda()
          for h in range(cfg.H)]
    hs = list(range(cfg.H))
    ds = [dims_of(cfg, h) for h in hs]
    k = [dev(xs[h]["k"]) for h in hs]
    v = [dev(xs[h]["v"]) for h in hs]
    idx = [torch.full((cfg.hk, cfg.l_pp), -1, dtype=torch.int32, device="cuda") for _ in hs]
    send = [torch.zeros((2, cfg.hk, cfg.l_pp, cfg.d), dtype=torch.bfloat16, device="cuda") for _ in hs]
    apb.select_topk_hosts(ds, sc, k, v, idx, send)
    torch.cuda.synchronize()
    for h in hs:
        idx_or = oracle.select_all_heads(sc[h].cpu().double().numpy(), cfg.l_p)
        assert np.array_equal(idx[h].cpu().numpy(), idx_or), h
        assert np.array_equal(to_bits(send[h]), oracle.compact(xs[h]["k"], xs[h]["v"], xs[h]["L_A"], idx_or)), h


def _select_gpu(cfg, h, x, scores_np):
    from paper_2502_12085_b200 import apb
    s = torch.from_numpy(np.ascontiguousarray(scores_np, dtype=np.float32)).cuda()
    idx = torch.full((cfg.hk, cfg.l_pp), -1, dtype=torch.int32, device="cuda")
    send = torch.zeros((2, cfg.hk, cfg.l_pp, cfg.d), dtype=torch.bfloat16, device="cuda")
    apb.select_topk(dims_of(cfg, h), s, dev(x["k"]), dev(x["v"]), idx, send)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), to_bits(send)


@pytest.mark.parametrize("ties", [False, True])
@pytest.mark.parametrize("name", ["toy", "d128-ragged", "gqa3"])
def test_select_compact_bit_exact(name, ties):
    cfg = CASES[name]
    for h in range(cfg.H):
        x = synth.host_qkv(cfg, 0, h)
        sc = synth.random_scores(cfg, 0, h, ties=ties)
        if h == 1:
            sc[:, ::7] = -0.0  # -0.0 and +0.0 must tie
            sc[:, 3::7] = 0.0
            sc[0, 5] = np.inf
            sc[-1, 9] = -np.inf
        idx, send = _select_gpu(cfg, h, x, sc)
        idx_or = oracle.select_all_heads(sc.astype(np.float64), cfg.l_p)
        assert np.array_equal(idx, idx_or), f"host {h}"
        assert np.array_equal(send, oracle.compact(x["k"], x["v"], x["L_A"], idx_or))


@pytest.mark.parametrize("lp,l_b", [(1, 300), (300, 300), (500, 300), (129, 1000), (4096, 70000), (8192, 65536),
                                    (2048, 131072), (3, 5), (7, 7), (3000, 400000), (1, 200000)])
def test_select_sizes(lp, l_b):
    cfg = synth.Config("sel", 17, n=l_b * 2, H=2, l_a=8, l_p=lp, hq=2, hk=2, d=64, d_hidden=256)
    x = synth.host_qkv(cfg, 0, 1)
    sc = synth.random_scores(cfg, 0, 1, ties=True)
    idx, send = _select_gpu(cfg, 1, x, sc)
    idx_or = oracle.select_all_heads(sc.astype(np.float64), cfg.l_p)
    assert np.array_equal(idx, idx_or)
    assert np.array_equal(send, oracle.compact(x["k"], x["v"], x["L_A"], idx_or))


@pytest.mark.parametrize("lp,l_b,ties", [(2048, 16384, False), (2048, 16384, True), (64, 512, True), (3000, 400000, True),
                                         (2048, 131072, True), (4096, 131076, False), (129, 1001, True),
                                         (1000, 1000, True), (25, 26, False), (8192, 65536, True),
                                         (2048, 40001, False), (40000, 40000, True)])
def test_select_cluster_equals_legacy(lp, l_b, ties, monkeypatch):
    """The default path (l_b <= 32K: single-CTA register select + PDL gather; up to 128K: one-launch
    8-CTA cluster select + gather; beyond: staged select), the single-CTA paths (APB_SELECT=reg)
    and the round-1 two-kernel path (APB_SELECT=legacy) produce identical indices and send payloads
    (all bit-exact integer logic)."""
    cfg = synth.Config("sel", 19, n=l_b * 2, H=2, l_a=8, l_p=lp, hq=8, hk=4, d=128, d_hidden=256)
    x = synth.host_qkv(cfg, 0, 1)
    sc = synth.random_scores(cfg, 0, 1, ties=ties)
    res = []
    for env in ("", "reg", "legacy"):
        monkeypatch.setenv("APB_SELECT", env)
        res.append(_select_gpu(cfg, 1, x, sc))
    for r in res[1:]:
        assert np.array_equal(res[0][0], r[0]) and np.array_equal(res[0][1], r[1])


# ----------------------------------------------------------------------------- whole layer

def _index_sets_ok(idx_gpu, s_or, lp):
    for j in range(s_or.shape[0]):
        tau = np.sort(s_or[j])[::-1][lp - 1]
        diff = set(idx_gpu[j].tolist()) ^ set(oracle.select_topk(s_or[j], lp).tolist())
        for i in diff:
            assert abs(s_or[j][i] - tau) < 1e-3, (j, i, s_or[j][i], tau)


@pytest.mark.parametrize("name", ["toy", "d128-sink"])
@pytest.mark.parametrize("mode", ["ordered", "split", "serial", "batched", "split-batched"])
def test_prefill_layer_end_to_end(name, mode):
    """All four steps through PrefillRank, every host of the layer emulated on one GPU, in the
    three schedules: ordered one-pass (single rank), LOCAL/PASSING split around the exchange
    (the multi-rank schedule), and fully serial."""
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.prefill import HostIO, PrefillRank
    cfg = CASES[name].replace(d_hidden=1024)
    hosts = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    w = synth.retain_weights(cfg, 0)
    rank = PrefillRank(dims_of(cfg, 0), list(range(cfg.H)), split_phases=mode.startswith("split"),
                       batched=mode.endswith("batched"))
    io = {}
    for h in range(cfg.H):
        q = dev(hosts[h]["q"])
        io[h] = HostIO(q=q, k=dev(hosts[h]["k"]), v=dev(hosts[h]["v"]), out=torch.empty_like(q),
                       lse=torch.empty((cfg.hq, q.shape[0]), device="cuda"))
    rank.layer(io, weights_dev(w), overlap=(mode != "serial"))
    torch.cuda.synchronize()
    gathered = to_bits(rank.gathered)
    for h in range(cfg.H):
        x = hosts[h]
        s_or = oracle.retain_score(x["q"], x["k"], x["v"], x["L_A"], w["w1"], w["b1"], w["w2"], w["b2"], cfg.hk)
        idx = rank.indices[h].cpu().numpy()
        _index_sets_ok(idx, s_or, cfg.l_pp)
        # selection is bit-exact on the GPU's own scores; compaction is verbatim
        s_gpu = rank.scores[h].cpu().double().numpy()
        assert np.array_equal(idx, oracle.select_all_heads(s_gpu, cfg.l_p))
        assert np.array_equal(gathered[h], oracle.compact(x["k"], x["v"], x["L_A"], idx))
    for h in range(cfg.H):
        x = hosts[h]
        pk, pv = oracle.passing(gathered, h)
        O_or, lse_or = oracle.attention(x["q"], x["k"], x["v"], x["L_A"], pk, pv)
        O = io[h].out.float().cpu().double().numpy()
        lse = io[h].lse.cpu().double().numpy().T
        check_attention(O, lse, O_or, lse_or, f"{name} e2e host {h}")


def test_attention_determinism():
    cfg = CASES["toy"]
    hosts, ref = oracle_layer(cfg)
    a = run_attention(cfg, 3, hosts[3], ref["gathered"], "split")
    b = run_attention(cfg, 3, hosts[3], ref["gathered"], "split")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("name", ["d128-ragged", "gqa8-d128", "gqa3", "mha", "d128-sink"])
@pytest.mark.parametrize("phase", ["all", "split"])
def test_attention_paired_matches_single_cta(name, phase, monkeypatch):
    """The paired kernel (2-CTA cluster, each CTA multicasting half of every K/V tile of the walk
    prefix it shares with its partner) feeds the MMAs the same tiles in the same order as the
    single-CTA kernel: bit-identical O and lse.  g = 4, 8 (equal walks) and g = 1, 2, 3 (partner
    walks one diagonal tile shorter; paired wherever each KV head holds an even item count)."""
    cfg = CASES[name]
    assert cfg.d == 128
    hosts, ref = oracle_layer(cfg)
    for h in range(cfg.H):
        monkeypatch.setenv("APB_ATTN_PAIR", "1")
        a = run_attention(cfg, h, hosts[h], ref["gathered"], phase)
        monkeypatch.setenv("APB_ATTN_PAIR", "")
        b = run_attention(cfg, h, hosts[h], ref["gathered"], phase)
        assert np.array_equal(a[0], b[0], equal_nan=True) and np.array_equal(a[1], b[1], equal_nan=True), f"host {h}"


def run_attention_hosts(cfg, hs, xs, gathered_bits, phase):
    """apb_attention_fwd_hosts over hosts hs (one launch per phase); returns {h: (O, lse)}."""
    from paper_2502_12085_b200 import apb
    ds = [dims_of(cfg, h) for h in hs]
    q = [dev(xs[h]["q"]) for h in hs]
    k = [dev(xs[h]["k"]) for h in hs]
    v = [dev(xs[h]["v"]) for h in hs]
    out = [torch.full_like(x, float("nan")) for x in q]
    lse = [torch.full((cfg.hq, d.rows), float("nan"), device="cuda") for d in ds]
    ws = [torch.empty(max(apb.workspace_size(d, apb.WS_ATTENTION), 16), dtype=torch.uint8, device="cuda") for d in ds]
    g = dev(gathered_bits) if gathered_bits is not None else None
    if phase == "split":
        apb.attention_fwd_hosts(ds, q, k, v, None, out, lse, phase=apb.PHASE_LOCAL, ws=ws)
        apb.attention_fwd_hosts(ds, q, k, v, g, out, lse, phase=apb.PHASE_PASSING, ws=ws)
    else:
        apb.attention_fwd_hosts(ds, q, k, v, g, out, lse, phase=apb.PHASE_ALL, ws=ws)
    torch.cuda.synchronize()
    return {h: (out[i].float().cpu().double().numpy(), lse[i].cpu().double().numpy().T) for i, h in enumerate(hs)}


@pytest.mark.parametrize("name", ["toy", "d128-ragged", "gqa8-d128", "mha", "d128-sink", "lq"])
@pytest.mark.parametrize("phase", ["all", "split"])
@pytest.mark.parametrize("pair", ["", "1"])
def test_attention_hosts_equals_per_host(name, phase, pair, monkeypatch):
    """apb_attention_fwd_hosts (one launch over several hosts' items, heaviest host first) is
    bit-identical to one apb_attention_fwd call per host — every host, a strict subset in a
    scrambled order (a rank owning cyclic hosts), with and without the paired kernel."""
    monkeypatch.setenv("APB_ATTN_PAIR", pair)
    cfg = CASES[name]
    hosts, ref = oracle_layer(cfg)
    subsets = [list(range(cfg.H)), list(range(cfg.H - 1, -1, -2))]
    for hs in subsets:
        got = run_attention_hosts(cfg, hs, hosts, ref["gathered"], phase)
        for h in hs:
            a = run_attention(cfg, h, hosts[h], ref["gathered"], phase)
            b = got[h]
            assert np.array_equal(a[0], b[0], equal_nan=True) and np.array_equal(a[1], b[1], equal_nan=True), (hs, h)


def test_attention_hosts_contract():
    """Mismatched dims across the hosts of one launch and a repeated host are APB_ERR_CONFIG."""
    from paper_2502_12085_b200 import apb
    cfg = CASES["toy"]
    hosts, ref = oracle_layer(cfg)
    ds = [dims_of(cfg, 1), dims_of(cfg, 1)]
    q = [dev(hosts[1]["q"])] * 2
    k = [dev(hosts[1]["k"])] * 2
    v = [dev(hosts[1]["v"])] * 2
    out = [torch.empty_like(q[0])] * 2
    with pytest.raises(apb.ApbError) as e:
        apb.attention_fwd_hosts(ds, q, k, v, dev(ref["gathered"]), out)
    assert e.value.status == apb.ERR_CONFIG
    import dataclasses
    ds = [dims_of(cfg, 1), dataclasses.replace(dims_of(cfg, 2), l_p=cfg.l_p + 1)]
    with pytest.raises(apb.ApbError) as e:
        apb.attention_fwd_hosts(ds, q, k, v, dev(ref["gathered"]), out)
    assert e.value.status == apb.ERR_CONFIG


@pytest.mark.parametrize("phase", ["all", "split"])
def test_attention_persistent_steals_matches_paired(phase, monkeypatch):
    """More work items than persistent CTAs (host 1: 544 items, host 3: 576 over 148 SMs), so the
    persistent kernel's CTAs take items from the launch's work counter and run several items each, with Q reloads, O hand-offs and barrier phases carried across items.  The
    paired kernel runs one item per cluster; both feed the same tiles to the same MMAs in the same
    order per item: bit-identical O and lse, in one launch per host and in one launch over hosts."""
    cfg = synth.Config("steal", 21, n=4 * 8192, H=4, l_a=512, l_p=256, hq=16, hk=4, d=128, d_hidden=256)
    hosts = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    rng = np.random.default_rng(5)
    g = rng.standard_normal((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d)).astype(np.float32)
    gathered = synth.f32_to_bf16_bits(g)
    monkeypatch.setenv("APB_ATTN_PAIR", "1")
    ref = {h: run_attention(cfg, h, hosts[h], gathered, phase) for h in (1, 3)}
    monkeypatch.setenv("APB_ATTN_PAIR", "")
    monkeypatch.setenv("APB_ATTN_PERSIST", "")
    for h in (1, 3):
        a = run_attention(cfg, h, hosts[h], gathered, phase)
        assert np.array_equal(a[0], ref[h][0], equal_nan=True) and np.array_equal(a[1], ref[h][1], equal_nan=True), h
    got = run_attention_hosts(cfg, [0, 1, 2, 3], hosts, gathered, phase)
    for h in (1, 3):
        assert np.array_equal(got[h][0], ref[h][0], equal_nan=True) and np.array_equal(got[h][1], ref[h][1],
                                                                                         equal_nan=True), h
    assert np.isfinite(got[0][0]).all() and np.isfinite(got[2][0]).all()


@pytest.mark.parametrize("phase", ["all", "split"])
def test_attention_persistent_d64_steals_vs_oracle(phase, monkeypatch):
    """d = 64 (never paired) with more items than resident CTAs (host 2: 272 items): the
    persistent kernel against the fp64 oracle on 640 sampled rows (every 128-row tile boundary of
    both segments +-1 included), per-host launch and one launch over every host."""
    monkeypatch.setenv("APB_ATTN_PERSIST", "")
    cfg = synth.Config("steal64", 22, n=4 * 4096, H=4, l_a=500, l_p=300, hq=16, hk=4, d=64, d_hidden=256)
    hosts = [synth.host_qkv(cfg, 0, hh) for hh in range(cfg.H)]
    g = np.random.default_rng(6).standard_normal((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d)).astype(np.float32)
    ref = {"gathered": synth.f32_to_bf16_bits(g)}
    h = 2
    x = hosts[h]
    rng = np.random.default_rng(9)
    rows = set()
    for seg0, n in ((0, x["L_A"]), (x["L_A"], cfg.l_b)):
        for b in range(0, n, 128):
            rows.update(r for r in (seg0 + b - 1, seg0 + b, seg0 + b + 127) if seg0 <= r < seg0 + n)
    rows = np.array(sorted(rows | set(rng.integers(0, x["L_A"] + cfg.l_b, 640 - len(rows)).tolist())))
    pk, pv = oracle.passing(ref["gathered"], h)
    O_or, lse_or = oracle.attention_blas(x["q"], x["k"], x["v"], x["L_A"], pk, pv, rows)
    a = run_attention(cfg, h, x, ref["gathered"], phase)
    b = run_attention_hosts(cfg, list(range(cfg.H)), hosts, ref["gathered"], phase)[h]
    assert np.array_equal(a[0], b[0], equal_nan=True) and np.array_equal(a[1], b[1], equal_nan=True)
    check_attention(a[0][rows], a[1][rows], O_or, lse_or, f"steal64 host {h} {phase}")


def test_attention_persistent_stress_back_to_back():
    """300 back-to-back persistent launches (576 items each over 148 CTAs, no host sync between
    them, every launch reusing the work-counter ring) finish, and the last output equals the first
    bit for bit.  A hang is detected by polling an event (30 s limit) and ends the process, so a
    regression fails the suite instead of stalling it (this is how the barrier-area overlap of the
    first persistent version showed up: ~1 % of L8 launches hung)."""
    import os as _os
    import time as _time
    from paper_2502_12085_b200 import apb
    cfg = synth.Config("steal", 21, n=4 * 8192, H=4, l_a=512, l_p=256, hq=16, hk=4, d=128, d_hidden=256)
    x = synth.host_qkv(cfg, 0, 3)
    g = np.random.default_rng(5).standard_normal((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d)).astype(np.float32)
    d = dims_of(cfg, 3)
    q, k, v, gd = dev(x["q"]), dev(x["k"]), dev(x["v"]), dev(synth.f32_to_bf16_bits(g))
    outs = [torch.empty_like(q), torch.empty_like(q)]
    lse = torch.empty((cfg.hq, d.rows), device="cuda")
    apb.attention_fwd(d, q, k, v, gd, outs[0], lse)
    for i in range(300):
        apb.attention_fwd(d, q, k, v, gd, outs[1], lse)
    ev = torch.cuda.Event()
    ev.record()
    t0 = _time.time()
    while not ev.query():
        if _time.time() - t0 > 30:
            print("persistent attention stress: launches did not finish within 30 s (hang)", flush=True)
            _os._exit(3)
        _time.sleep(0.05)
    assert torch.equal(outs[0], outs[1])


# ----------------------------------------------------------------------------- full size

def _sample_rows(L_A, l_b, extra, rng):
    rows = {0, max(L_A - 1, 0), L_A, L_A + 1, L_A + l_b - 1}
    for t in range(128, L_A + l_b, 128 * 16):
        rows.update({t - 1, t, t + 1})
    rows.update(rng.choice(L_A + l_b, extra, replace=False).tolist())
    return sorted(r for r in rows if 0 <= r < L_A + l_b)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["llama8b-512k", "llama8b-1m"])
def test_full_size_max_sampled(name):
    """Maximum sizes (512K with l_a = l_p = 8K, and 1M tokens; H = 8): the
    critical host's attention (135K-rows Q, 150K-key sequences, 64-bit offsets) in the ordered
    one-launch form and as the LOCAL / PASSING pair, on sampled rows (boundaries of every
    segment + random) against the oracle.  Inputs: seeded N(0,1) on the device; the passing
    buffer is random too (attention is exact for any passing keys)."""
    from paper_2502_12085_b200 import apb
    cfg = synth.CONFIGS[name]
    h = cfg.H - 1
    d = dims_of(cfg, h)
    n = d.rows
    g = torch.Generator(device="cuda")
    g.manual_seed(1 + cfg.cfg_id)
    rnd = lambda *shape: torch.randn(*shape, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    q, k, v = rnd(n, cfg.hq, cfg.d), rnd(n, cfg.hk, cfg.d), rnd(n, cfg.hk, cfg.d)
    gathered = rnd(cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d)
    ws = torch.empty(max(apb.workspace_size(d, apb.WS_ATTENTION), 16), dtype=torch.uint8, device="cuda")
    L_A, l_b = d.L_A, cfg.l_b
    rng = np.random.default_rng(cfg.cfg_id)
    rows = sorted({0, L_A - 1, L_A, L_A + 1, L_A + 127, L_A + 128, n - 129, n - 1}
                  | set(rng.choice(n, 8, replace=False).tolist()))
    kb, vb, gb = to_bits(k), to_bits(v), to_bits(gathered)
    pk, pv = oracle.passing(gb, h)
    O_or, lse_or = oracle.attention(to_bits(q[rows]), kb, vb, L_A, pk, pv, rows=rows, q_subset=True)
    for split in (False, True):
        out = torch.full_like(q, float("nan"))
        lse = torch.full((cfg.hq, n), float("nan"), device="cuda")
        if split:
            apb.attention_fwd(d, q, k, v, gathered, out, lse, phase=apb.PHASE_LOCAL, ws=ws)
            apb.attention_fwd(d, q, k, v, gathered, out, lse, phase=apb.PHASE_PASSING, ws=ws)
        else:
            apb.attention_fwd(d, q, k, v, gathered, out, lse, phase=apb.PHASE_ALL, ws=ws)
        torch.cuda.synchronize()
        O = out[rows].float().cpu().double().numpy()
        L = lse[:, rows].cpu().double().numpy().T
        check_attention(O, L, O_or, lse_or, f"{name} host {h} {'split' if split else 'ordered'} ({len(rows)} rows)")
        assert torch.isfinite(out.float()).all()


def test_nccl_unique_id_and_single_rank_comm():
    """libapb's NCCL plumbing on a GPU box: a 128-byte id, a 1-rank communicator (exchange is a
    no-op), and a clean destroy."""
    from paper_2502_12085_b200 import apb
    uid = apb.Comm.unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)
    c = apb.Comm(uid, 1, 0)
    cfg = CASES["toy"]
    g = torch.zeros((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d), dtype=torch.bfloat16, device="cuda")
    apb.exchange_passing(c, dims_of(cfg, 0), g)
    c.close()


@pytest.mark.parametrize("name", ["qwen14b-128k", "yi34b-200k"])
def test_full_size_odd_gqa_sampled(name):
    """BASELINE configs[2] / [3] (Qwen-2.5-14B: 40 Q / 8 KV heads, g = 5; Yi-34B: 56 / 8, g = 7,
    n = 200K): the critical host's one-pass attention at full size (query-tile pairs spanning two
    row tiles), sampled rows vs the oracle."""
    cfg = synth.CONFIGS[name]
    h = cfg.H - 1
    x = synth.host_qkv(cfg, 0, h)
    rng = np.random.default_rng(1)
    gathered = synth.f32_to_bf16_bits(rng.standard_normal((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d)).astype(np.float32))
    O, lse = run_attention(cfg, h, x, gathered, "all")
    rows = _sample_rows(x["L_A"], cfg.l_b, 16, rng)
    pk, pv = oracle.passing(gathered, h)
    O_or, lse_or = oracle.attention(x["q"], x["k"], x["v"], x["L_A"], pk, pv, rows=rows)
    check_attention(O[rows], lse[rows], O_or, lse_or, f"{name} host {h} sampled ({len(rows)} rows)")
