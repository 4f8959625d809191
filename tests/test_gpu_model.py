"""GPU parity for the APB prefill layer around the hot path, through
the C ABI, against oracle/layer.py (fp64, pinned against transformers' LlamaDecoderLayer).

Tolerances (each GPU output is bf16, rounded once from fp32 math; reading G9):
  rmsnorm / rope / swiglu   |gpu - ref| <= 2^-8 |ref| + 1e-6           (<= 1 bf16 ulp)
  gemm                      |gpu - ref| <= 2^-8 |ref| + 2^-20 * sum_k |a_k w_k|
                            (+ 2^-8 |A W^T| with beta = 1: the product is rounded first, G20)
  layer, step-wise          each step from the GPU's own previous output, same bounds x4
                            (a bf16 input feeding a reduction can move the output by ~1 ulp)
  hot path inside the layer: the test_gpu.py rules (selection bit-exact on the GPU's scores,
                            attention vs the oracle over the GPU's gathered buffer)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import layer as OL

pytestmark = pytest.mark.gpu

ULP = 2.0 ** -8


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_12085_b200 import apb, build
    build.build()
    apb.load()


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def f64(t):
    return t.float().cpu().double().numpy()


def bits_of(x):
    return synth.f32_to_bf16_bits(np.asarray(x, np.float32))


def check(got, ref, what, rel=ULP, abs_=1e-6, scale=None):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    tol = rel * np.abs(ref) + abs_ + (0.0 if scale is None else scale)
    bad = np.abs(got - ref) > tol
    print(f"{what}: max err {np.abs(got - ref).max():.3e}, violations {bad.sum()} / {bad.size}")
    assert not bad.any(), what


@pytest.mark.parametrize("rows,dim", [(1, 8), (37, 256), (300, 4096), (5, 5120)])
def test_rmsnorm(rows, dim):
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(rows + dim)
    x = bits_of(rng.standard_normal((rows, dim)) * 3)
    w = bits_of(1 + 0.1 * rng.standard_normal(dim))
    out = torch.empty((rows, dim), dtype=torch.bfloat16, device="cuda")
    apb.rmsnorm(dev(x), dev(w), 1e-5, out)
    torch.cuda.synchronize()
    check(f64(out), OL.rmsnorm(synth.bf16_bits_to_f64(x), synth.bf16_bits_to_f64(w), 1e-5), "rmsnorm")
    # in place
    xt = dev(x)
    apb.rmsnorm(xt, dev(w), 1e-5, xt)
    torch.cuda.synchronize()
    assert torch.equal(xt, out)


@pytest.mark.parametrize("rows,heads,d,theta,pos_offset", [(7, 3, 64, 10000.0, 0), (300, 40, 128, 500000.0, 0),
                                                          (33, 5, 128, 500000.0, 1_000_000), (4, 2, 16, 1e4, 12345)])
def test_rope(rows, heads, d, theta, pos_offset):
    """In place on the first `heads` heads of a wider row (the Q|K part of a qkv row); the
    V heads after them stay untouched; explicit positions equal the offset rule."""
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(heads * d)
    extra = 2
    x = bits_of(rng.standard_normal((rows, heads + extra, d)))
    t = dev(x)
    apb.rope(t.view(rows, -1), heads, d, theta, pos_offset=pos_offset)
    torch.cuda.synchronize()
    pos = pos_offset + np.arange(rows)
    got = f64(t)
    check(got[:, :heads], OL.rope(synth.bf16_bits_to_f64(x[:, :heads]), pos, theta), "rope")
    assert np.array_equal(t.view(torch.int16).cpu().numpy()[:, heads:].view(np.uint16), x[:, heads:])
    t2 = dev(x)
    apb.rope(t2.view(rows, -1), heads, d, theta, positions=torch.from_numpy(pos.astype(np.int32)).cuda())
    torch.cuda.synchronize()
    assert torch.equal(t2, t)


@pytest.mark.parametrize("rows,inter", [(1, 8), (129, 512), (64, 14336)])
def test_swiglu(rows, inter):
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(inter)
    gu = bits_of(rng.standard_normal((rows, 2 * inter)) * 3)
    out = torch.empty((rows, inter), dtype=torch.bfloat16, device="cuda")
    apb.swiglu(dev(gu), out)
    torch.cuda.synchronize()
    check(f64(out), OL.swiglu(synth.bf16_bits_to_f64(gu), inter), "swiglu", abs_=1e-5)


@pytest.mark.parametrize("M,N,K,beta", [(1, 8, 8, 0.0), (257, 384, 256, 0.0), (300, 512, 4096, 1.0),
                                        (128, 14336, 4096, 0.0), (1000, 6144, 4096, 0.0), (513, 264, 72, 1.0),
                                        (700, 4096, 14336, 1.0), (90, 136, 200, 0.5)])
def test_gemm(M, N, K, beta):
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(M + N + K)
    a = bits_of(rng.standard_normal((M, K)))
    w = bits_of(rng.standard_normal((N, K)) / np.sqrt(K))
    c0 = bits_of(rng.standard_normal((M, N)))
    c = dev(c0)
    apb.gemm_bf16(dev(a), dev(w), c, beta=beta)
    torch.cuda.synchronize()
    A, W = synth.bf16_bits_to_f64(a), synth.bf16_bits_to_f64(w)
    ref = A @ W.T + beta * synth.bf16_bits_to_f64(c0)
    mag = np.abs(A) @ np.abs(W).T
    # with beta != 0 the product is rounded to bf16 before adding C (two roundings, reading
    # G20): allow one more ulp of the product term
    extra = ULP * np.abs(A @ W.T) if beta else 0.0
    check(f64(c), ref, f"gemm {M}x{N}x{K}", abs_=1e-6, scale=2.0 ** -20 * mag + extra)


def _model(cfg, hidden, inter, compressor="retain"):
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.model import ApbModelRank, LayerWeights, ModelShape
    shape = ModelShape(hidden=hidden, inter=inter, n_heads=cfg.hq, n_kv_heads=cfg.hk, head_dim=cfg.d,
                       eps=1e-5, theta=500000.0)
    base = apb.Dims(n=cfg.n, H=cfg.H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d, l_q=cfg.l_q)
    rank = ApbModelRank(base, shape, list(range(cfg.H)), compressor=compressor, seed=5)
    mw = synth.model_weights(cfg, 0, hidden, inter)
    rw = synth.retain_weights(cfg.replace(d_hidden=1024), 0)
    retain = apb.RetainWeights(w1=dev(rw["w1"]), w2=torch.from_numpy(rw["w2"]).cuda(),
                               b1=torch.from_numpy(rw["b1"]).cuda(), b2=torch.from_numpy(rw["b2"]).cuda())
    lw = LayerWeights(**{k: dev(v) for k, v in mw.items()}, retain=retain if compressor == "retain" else None)
    lw_np = {k: synth.bf16_bits_to_f64(v) for k, v in mw.items()}
    lw_np.update(eps=1e-5, theta=500000.0)
    return rank, lw, lw_np, rw


@pytest.mark.parametrize("name", ["toy", "lq-gqa3"])
def test_apb_layer_stepwise(name):
    """One full APB layer (all hosts on one GPU) — every step of Alg. apb_prefill checked
    against the oracle fed with the GPU's previous step."""
    cfg = {"toy": synth.CONFIGS["toy"],
           "lq-gqa3": synth.Config("lq-gqa3", 31, n=1536, H=3, l_a=96, l_p=64, hq=6, hk=2, d=128, l_q=20)}[name]
    hidden, inter = 256, 512
    rank, lw, lw_np, rw = _model(cfg, hidden, inter)
    x_bits = [synth.host_hidden(cfg, h, hidden) for h in range(cfg.H)]
    xs = {h: dev(x_bits[h]) for h in range(cfg.H)}
    # step 1: pre-attention (one host at a time so the intermediate is observable)
    qkv_gpu = {}
    for h in range(cfg.H):
        rank.attn_in(h, xs[h], lw)
        torch.cuda.synchronize()
        qkv_gpu[h] = f64(rank.qkv[h])
        x = synth.bf16_bits_to_f64(x_bits[h])
        hb = f64(rank.hbuf[:x.shape[0]])
        check(hb, OL.rmsnorm(x, lw_np["attn_norm"], 1e-5), f"host {h} rmsnorm")
        qkv_lin = hb @ lw_np["w_qkv"].T
        pos = np.arange(x.shape[0])
        ref = np.concatenate([OL.rope(OL.bf16(qkv_lin).reshape(len(x), -1, cfg.d)[:, :cfg.hq + cfg.hk], pos, 500000.0),
                              qkv_lin.reshape(len(x), -1, cfg.d)[:, cfg.hq + cfg.hk:]], axis=1)
        # two roundings on the Q/K path (GEMM output, then RoPE): a 1-ulp difference in an input
        # pair moves the rotated value by ~1 ulp of the PAIR magnitude (the output itself can
        # be small by cancellation), plus the GEMM's fp32 accumulation
        lin = qkv_lin.reshape(ref.shape)
        half = cfg.d // 2
        pm = np.zeros_like(lin)
        nqk = cfg.hq + cfg.hk
        r2 = np.sqrt(lin[:, :nqk, :half] ** 2 + lin[:, :nqk, half:] ** 2)
        pm[:, :nqk] = np.concatenate([r2, r2], axis=-1)
        mag = (np.abs(hb) @ np.abs(lw_np["w_qkv"]).T).reshape(ref.shape)
        check(qkv_gpu[h], ref, f"host {h} qkv", rel=ULP, scale=2 * ULP * pm + 2.0 ** -20 * 2 * mag)
    # step 2: the hot path, as PrefillRank runs it
    rank.hot.layer(rank.io, lw.retain)
    torch.cuda.synchronize()
    gathered = rank.hot.gathered.view(torch.int16).cpu().numpy().view(np.uint16)
    for h in range(cfg.H):
        qkv = qkv_gpu[h]
        L_A = cfg.L_A(h)
        q, k, v = qkv[:, :cfg.hq], qkv[:, cfg.hq:cfg.hq + cfg.hk], qkv[:, cfg.hq + cfg.hk:]
        if cfg.l_pp and h < cfg.H - 1:
            idx = rank.hot.indices[h].cpu().numpy()
            assert np.array_equal(idx, oracle.select_all_heads(rank.hot.scores[h].cpu().double().numpy(), cfg.l_p))
            s_or = oracle.retain_score(q, k, v, L_A, rw["w1"], rw["b1"], rw["w2"], rw["b2"], cfg.hk)
            for j in range(cfg.hk):
                tau = np.sort(s_or[j])[::-1][cfg.l_pp - 1]
                for i in set(idx[j].tolist()) ^ set(oracle.select_topk(s_or[j], cfg.l_p).tolist()):
                    assert abs(s_or[j][i] - tau) < 1e-3
        pk, pv = oracle.passing(gathered, h)
        O_or, _ = oracle.attention(q, k, v, L_A, pk, pv)
        err = np.abs(f64(rank.attn[h]) - O_or)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3, (h, err.max(), err.mean())
    # step 3: O projection + residual, FFN + residual
    for h in range(cfg.H):
        x = synth.bf16_bits_to_f64(x_bits[h])
        attn = f64(rank.attn[h])
        rank.attn_out_ffn(h, xs[h], lw)
        torch.cuda.synchronize()
        ref = OL.attn_out_ffn(x, attn, lw_np, rnd=True)
        # the oracle rounds where the GPU does (G20), so differences come from fp32-vs-fp64
        # accumulation flipping an intermediate by 1 ulp (<= 2^-7 |v|): bound by 4 * 2^-8 of every term
        x1 = OL.bf16(x + OL.bf16(attn.reshape(len(x), -1) @ lw_np["w_o"].T))
        terms = np.abs(x) + np.abs(x1 - x) + np.abs(ref - x1)
        # ... and a flip in h2 / gu / act reaches the output through W_down: allow every act
        # element 2 ulp, i.e. 4 * 2^-8 of sum_k |act_k| |W_down[., k]|
        h2 = OL.bf16(OL.rmsnorm(x1, lw_np["ffn_norm"], 1e-5))
        act = OL.bf16(OL.swiglu(OL.bf16(h2 @ lw_np["w_gu"].T), inter))
        mag_f = np.abs(act) @ np.abs(lw_np["w_down"]).T
        check(f64(xs[h]), ref, f"host {h} layer out", rel=2 * ULP, scale=4 * ULP * (terms + mag_f))


def test_apb_layer_whole_and_anchor_consistency():
    """ApbModelRank.layer end to end (ordered schedule): outputs finite, the anchor rows of every
    host equal host 0's first rows (consistent anchor: anchor rows see only the anchor
    at the same positions, so every host computes the same anchor outputs), and every host's
    rows match the oracle's whole layer within the end-to-end tolerance."""
    cfg = synth.CONFIGS["toy"]
    hidden, inter = 256, 512
    rank, lw, lw_np, rw = _model(cfg, hidden, inter)
    x_bits = [synth.host_hidden(cfg, h, hidden) for h in range(cfg.H)]
    xs = {h: dev(x_bits[h]) for h in range(cfg.H)}
    rank.layer(xs, lw)
    torch.cuda.synchronize()
    out = {h: f64(xs[h]) for h in range(cfg.H)}
    assert all(np.isfinite(o).all() for o in out.values())
    for h in range(1, cfg.H):
        # same math on the same bits, row-local everywhere except attention, whose anchor rows see
        # only the anchor: libapb's GEMM accumulates a row in the same K order whatever M is, so
        # the anchor rows of every host are bit-identical to host 0's first rows
        assert np.array_equal(out[h][:cfg.l_a], out[0][:cfg.l_a]), f"anchor rows host {h}"
    xs64 = [synth.bf16_bits_to_f64(b) for b in x_bits]
    L_As = [cfg.L_A(h) for h in range(cfg.H)]
    rwd = {k: rw[k] for k in ("w1", "b1", "w2", "b2")}
    # (a) the oracle's own pipeline (its own scores and Top-l_p): near-tie swaps of the passing set
    # are legitimate (rule (ii)), so only a loose bound holds element-wise
    res = OL.apb_layer(xs64, L_As, lw_np, rwd, cfg.l_p, cfg.hq, cfg.hk, cfg.d)
    for h in range(cfg.H):
        err = np.abs(out[h] - res["out"][h])
        scale = np.abs(res["out"][h]).mean()
        print(f"oracle selection, host {h}: max {err.max():.3e} mean {err.mean():.3e} (|out| mean {scale:.3f})")
        assert err.mean() <= 2e-2 * scale and err.max() <= 0.25 * scale + 0.1
    # (b) the oracle fed the GPU's scores (its Top-l_p on them is the GPU's set bit for bit, rule
    # (i)): the same passing keys, so what remains is rounding — bf16 flips of single elements
    # (<= 1 ulp) at the G20 points and the attention tolerance (2e-2 max / 2e-3 mean), carried
    # through W_o and the FFN.  Bound: mean <= 3e-3 |out|, max <= 2 bf16 ulp of max |out| + 1e-2
    # (B200, toy: max 3.1e-2 = one ulp at |out| in [4, 8), mean 1.7e-3 at |out| mean 0.94)
    gpu_scores = [rank.hot.scores[h].cpu().double().numpy() for h in range(cfg.H)]
    res2 = OL.apb_layer(xs64, L_As, lw_np, rwd, cfg.l_p, cfg.hq, cfg.hk, cfg.d, compressor_scores=gpu_scores)
    for h in range(cfg.H):
        err = np.abs(out[h] - res2["out"][h])
        scale = np.abs(res2["out"][h]).mean()
        mx = np.abs(res2["out"][h]).max()
        print(f"GPU selection, host {h}: max {err.max():.3e} mean {err.mean():.3e} (|out| mean {scale:.3f}, max {mx:.2f})")
        assert err.mean() <= 3e-3 * scale and err.max() <= 2 * ULP * mx + 1e-2


def test_apb_layer_random_compressor_runs():
    """The Rd. compressor inside the full layer (Table 4 rows 2-5): no retaining-head weights."""
    cfg = synth.CONFIGS["toy"]
    rank, lw, _, _ = _model(cfg, 256, 512, compressor="random")
    xs = {h: dev(synth.host_hidden(cfg, h, 256)) for h in range(cfg.H)}
    rank.layer(xs, lw, layer_idx=2)
    torch.cuda.synchronize()
    idx = rank.hot.indices[1].cpu().numpy()
    s = oracle.random_scores(5, 2, cfg.H, 1, cfg.hk, cfg.l_b)
    assert np.array_equal(idx, oracle.select_all_heads(s, cfg.l_p))
    assert all(torch.isfinite(x.float()).all() for x in xs.values())


@pytest.mark.slow
def test_full_size_llama8b_layer_sampled():
    """NEXT #2 at the bench's size and launch configuration (bench_model.py: Llama-3.1-8B shape,
    hidden 4096 / FFN 14336, n = 128K, H = 8 hosts on one GPU, ordered schedule): one layer,
    every step checked on sampled rows of the critical host (and host 1) — the row-local steps
    (RMSNorm, QKV projection, RoPE; O projection + FFN) against the oracle fed the GPU's inputs of
    that step, attention against the oracle over the GPU's own Q/K/V and gathered buffer."""
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.model import ApbModelRank, LayerWeights, ModelShape
    cfg = synth.CONFIGS["llama8b-128k"]
    hidden, inter = 4096, 14336
    shape = ModelShape(hidden=hidden, inter=inter, n_heads=cfg.hq, n_kv_heads=cfg.hk, head_dim=cfg.d)
    base = apb.Dims(n=cfg.n, H=cfg.H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d)
    rank = ApbModelRank(base, shape, list(range(cfg.H)))
    g = torch.Generator(device="cuda")
    g.manual_seed(12085)
    rnd = lambda *s, scale=1.0, mean=0.0: (torch.randn(*s, generator=g, device="cuda") * scale + mean).to(torch.bfloat16)
    lw = LayerWeights(attn_norm=rnd(hidden, scale=0.1, mean=1.0),
                      w_qkv=rnd((cfg.hq + 2 * cfg.hk) * cfg.d, hidden, scale=hidden ** -0.5),
                      w_o=rnd(hidden, cfg.hq * cfg.d, scale=(cfg.hq * cfg.d) ** -0.5),
                      ffn_norm=rnd(hidden, scale=0.1, mean=1.0), w_gu=rnd(2 * inter, hidden, scale=hidden ** -0.5),
                      w_down=rnd(hidden, inter, scale=inter ** -0.5),
                      retain=apb.RetainWeights(w1=rnd(cfg.d_hidden, cfg.d_in, scale=cfg.d_in ** -0.5),
                                               w2=torch.randn(cfg.hq, cfg.d_hidden, generator=g, device="cuda")
                                               * cfg.d_hidden ** -0.5,
                                               b1=torch.zeros(cfg.d_hidden, device="cuda"),
                                               b2=torch.zeros(cfg.hq, device="cuda")))
    xs = {h: rnd(rank.rows[h], hidden) for h in range(cfg.H)}
    x_in = {h: xs[h].clone() for h in (1, cfg.H - 1)}
    rank.layer(xs, lw)
    torch.cuda.synchronize()
    W = {k: f64(getattr(lw, k)) for k in ("attn_norm", "w_qkv", "w_o", "ffn_norm", "w_gu", "w_down")}
    W.update(eps=shape.eps, theta=shape.theta)
    gathered = rank.hot.gathered.view(torch.int16).cpu().numpy().view(np.uint16)
    rng = np.random.default_rng(3)
    for h in (1, cfg.H - 1):
        L_A = rank.hot.dims(h).L_A
        n = rank.rows[h]
        rows = sorted({0, L_A - 1, L_A, n - 1} | set(rng.choice(n, 6, replace=False).tolist()))
        x = f64(x_in[h][rows])
        # pre-attention, row-local: RMSNorm -> QKV -> RoPE at the row's position (G19)
        hb = OL.bf16(OL.rmsnorm(x, W["attn_norm"], shape.eps))
        qkv_lin = hb @ W["w_qkv"].T
        ref = np.concatenate([OL.rope(OL.bf16(qkv_lin).reshape(len(rows), -1, cfg.d)[:, :cfg.hq + cfg.hk],
                                      np.array(rows), shape.theta),
                              qkv_lin.reshape(len(rows), -1, cfg.d)[:, cfg.hq + cfg.hk:]], axis=1)
        got = f64(rank.qkv[h][rows])
        err = np.abs(got - ref)
        assert err.max() <= 4 * ULP * np.abs(ref).max() + 1e-2, (h, err.max())
        # attention over the GPU's Q/K/V and gathered buffer
        qkv_bits = rank.qkv[h].view(torch.int16).cpu().numpy().view(np.uint16)
        q, k, v = qkv_bits[:, :cfg.hq], qkv_bits[:, cfg.hq:cfg.hq + cfg.hk], qkv_bits[:, cfg.hq + cfg.hk:]
        pk, pv = oracle.passing(gathered, h)
        O_or, _ = oracle.attention(q[rows], k, v, L_A, pk, pv, rows=rows, q_subset=True)
        e2 = np.abs(f64(rank.attn[h][rows]) - O_or)
        assert e2.max() <= 2e-2 and e2.mean() <= 2e-3, (h, e2.max(), e2.mean())
        # O projection + FFN, row-local, from the GPU's attention output
        ref_out = OL.attn_out_ffn(x, f64(rank.attn[h][rows]), W, rnd=True)
        x1 = OL.bf16(x + OL.bf16(f64(rank.attn[h][rows]).reshape(len(rows), -1) @ W["w_o"].T))
        h2 = OL.bf16(OL.rmsnorm(x1, W["ffn_norm"], shape.eps))
        act = OL.bf16(OL.swiglu(OL.bf16(h2 @ W["w_gu"].T), inter))
        terms = np.abs(x) + np.abs(x1 - x) + np.abs(ref_out - x1) + np.abs(act) @ np.abs(W["w_down"]).T
        check(f64(xs[h][rows]), ref_out, f"L8 layer host {h} out ({len(rows)} rows)", rel=2 * ULP, scale=4 * ULP * terms)
