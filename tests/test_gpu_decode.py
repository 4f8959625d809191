"""GPU parity of the APB decode step (Alg. apb_decode) against
the fp64 oracle: per-host partials, MergeScore, and the whole step through DecodeRank.
Tolerances as the prefill attention (north star): max|dO| <= 2e-2, mean <= 2e-3, |dlse| <= 1e-2."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_12085_b200 import apb, build
    build.build()
    apb.load()


def _bits(shape, rng, scale=1.0):
    return synth.f32_to_bf16_bits(rng.standard_normal(shape).astype(np.float32) * scale)


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _check(O, lse, O_or, lse_or, what):
    err = np.abs(O - O_or)
    fin = np.isfinite(lse_or)
    lerr = np.abs(lse[fin] - lse_or[fin]).max() if fin.any() else 0.0
    print(f"{what}: max {err.max():.3e} mean {err.mean():.3e} lse {lerr:.3e}")
    assert err.max() <= 2e-2 and err.mean() <= 2e-3 and lerr <= 1e-2, what
    assert np.array_equal(np.isneginf(lse), np.isneginf(lse_or)), what


@pytest.mark.parametrize("c", [0, 1, 255, 256, 257, 1000])
@pytest.mark.parametrize("t", [1, 4])
@pytest.mark.parametrize("last", [False, True])
@pytest.mark.parametrize("d,hq,hk", [(128, 8, 2), (64, 6, 2)])
def test_decode_partial_parity(c, t, last, d, hq, hk):
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(c * 10 + t)
    q = _bits((t, hq, d), rng, 1.5)
    kc, vc = _bits((c, hk, d), rng, 1.5), _bits((c, hk, d), rng)
    kn, vn = _bits((t, hk, d), rng, 1.5), _bits((t, hk, d), rng)
    H, host = 3, (2 if last else 1)
    dims = apb.DecodeDims(H, host, t, c, hq, hk, d)
    po = torch.full((t, hq, d), float("nan"), device="cuda")
    pl = torch.full((t, hq), float("nan"), device="cuda")
    ws = torch.zeros(max(apb.decode_workspace_size(dims), 16), dtype=torch.uint8, device="cuda")
    kct = dev(kc) if c else torch.empty((0, hk, d), dtype=torch.bfloat16, device="cuda")
    vct = dev(vc) if c else torch.empty((0, hk, d), dtype=torch.bfloat16, device="cuda")
    apb.decode_attention(dims, dev(q), kct, vct, dev(kn) if last else None, dev(vn) if last else None, po, pl, ws)
    torch.cuda.synchronize()
    O_or, l_or = oracle.decode_partial(q, kc, vc, kn if last else None, vn if last else None)
    _check(po.cpu().double().numpy(), pl.cpu().double().numpy(), O_or, l_or, f"partial c={c} t={t} last={last}")


@pytest.mark.parametrize("lens,host0,H", [([0, 1, 255, 257, 1000], 0, 5), ([64, 0, 130], 2, 5), ([300], 3, 4),
                                           ([513, 70, 0, 2000, 5, 128, 64, 9], 0, 8)])
@pytest.mark.parametrize("t", [1, 4])
@pytest.mark.parametrize("d,hq,hk", [(128, 8, 2), (64, 6, 2)])
def test_decode_hosts_partials_parity(lens, host0, H, t, d, hq, hk):
    """apb_decode_attention_hosts (one launch for the hosts a rank owns): every host's partial vs
    the oracle, ragged cache lengths (empty, chunk boundaries), with and without the last host."""
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(sum(lens) + 7 * t + d)
    q = _bits((t, hq, d), rng, 1.5)
    kn, vn = _bits((t, hk, d), rng, 1.5), _bits((t, hk, d), rng)
    caches = [(_bits((c, hk, d), rng, 1.5), _bits((c, hk, d), rng)) for c in lens]
    n, rows = len(lens), t * hq
    stride = (rows * d + rows + 3) // 4 * 4 + 4  # a padded part stride: exercises part_stride != rows*(d+1)
    parts = torch.full((n, stride), float("nan"), device="cuda")
    dims = apb.DecodeDims(H, host0, t, 0, hq, hk, d)
    ws = torch.zeros(max(apb.decode_hosts_workspace_size(dims, lens), 16), dtype=torch.uint8, device="cuda")
    kcs = [dev(k) if c else torch.empty((0, hk, d), dtype=torch.bfloat16, device="cuda") for (k, _), c in zip(caches, lens)]
    vcs = [dev(v) if c else torch.empty((0, hk, d), dtype=torch.bfloat16, device="cuda") for (_, v), c in zip(caches, lens)]
    last = host0 + n == H
    apb.decode_attention_hosts(dims, dev(q), kcs, vcs, dev(kn) if last else None, dev(vn) if last else None,
                               parts, rows * d, ws)
    torch.cuda.synchronize()
    P = parts.cpu().double().numpy()
    for i in range(n):
        is_last = host0 + i == H - 1
        O_or, l_or = oracle.decode_partial(q, caches[i][0], caches[i][1], kn if is_last else None,
                                           vn if is_last else None)
        _check(P[i, : rows * d].reshape(t, hq, d), P[i, rows * d: rows * d + rows].reshape(t, hq), O_or, l_or,
               f"hosts partial {host0 + i} c={lens[i]} t={t}")


def test_merge_partials_parity():
    from paper_2502_12085_b200 import apb
    rng = np.random.default_rng(3)
    n, rows, d = 5, 37, 128
    po = rng.standard_normal((n, rows, d)).astype(np.float32)
    pl = (rng.standard_normal((n, rows)) * 3).astype(np.float32)
    pl[1, 3] = -np.inf  # a host that saw no key for this row
    pl[:, 7] = -np.inf  # a row nobody saw
    out = torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
    ol = torch.empty(rows, device="cuda")
    apb.merge_partials(n, rows, d, torch.from_numpy(po).cuda(), rows * d, torch.from_numpy(pl).cuda(), rows, out, ol)
    torch.cuda.synchronize()
    A, L = oracle.merge_score(po.astype(np.float64), pl.astype(np.float64))
    A[7] = 0.0
    err = np.abs(out.float().cpu().double().numpy() - A)
    assert err.max() <= 2e-2
    fin = np.isfinite(L)
    assert np.abs(ol.cpu().double().numpy()[fin] - L[fin]).max() <= 1e-5
    assert np.isneginf(ol.cpu().numpy()[7])


@pytest.mark.parametrize("mode", ["fused", "hosts", "per-host"])
@pytest.mark.parametrize("name,t", [("toy", 1), ("toy", 3), ("gqa3", 2)])
def test_decode_step_end_to_end(name, t, mode):
    """All hosts on one GPU through DecodeRank: partials -> (in-place) gather -> MergeScore, vs the
    oracle's decode step AND vs exact attention over [B_1 .. B_H | new] (the step is exact)."""
    from paper_2502_12085_b200.decode import DecodeRank
    cfg = {"toy": synth.CONFIGS["toy"],
           "gqa3": synth.Config("gqa3", 12, n=1024, H=4, l_a=64, l_p=48, hq=6, hk=2, d=128)}[name]
    rng = np.random.default_rng(5)
    hosts = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    caches = [(x["k"][x["L_A"]:], x["v"][x["L_A"]:]) for x in hosts]  # block KV cache
    q = _bits((t, cfg.hq, cfg.d), rng)
    kn, vn = _bits((t, cfg.hk, cfg.d), rng), _bits((t, cfg.hk, cfg.d), rng)
    dr = DecodeRank(cfg.H, list(range(cfg.H)), t, cfg.hq, cfg.hk, cfg.d, batch_hosts=mode != "per-host",
                    fuse_merge=mode == "fused")
    out = torch.empty((t, cfg.hq, cfg.d), dtype=torch.bfloat16, device="cuda")
    ol = torch.empty((t, cfg.hq), device="cuda")
    dr.step(dev(q), {h: (dev(kc), dev(vc)) for h, (kc, vc) in enumerate(caches)}, dev(kn), dev(vn), out, ol)
    torch.cuda.synchronize()
    A, L, _ = oracle.decode_step(q, caches, kn, vn)
    _check(out.float().cpu().double().numpy(), ol.cpu().double().numpy(), A, L, f"decode step {name} t={t}")
    # exactness: one-shot attention over [all caches | new] with the prefill oracle (L_A = 0,
    # the caches as the "passing" segment, the new tokens as the local block)
    pk = np.concatenate([c[0] for c in caches]); pv = np.concatenate([c[1] for c in caches])
    O1, l1 = oracle.attention(q, kn, vn, 0, pk, pv)
    assert np.allclose(A, O1, atol=1e-10) and np.allclose(L, l1, atol=1e-10)


def test_decode_full_size_llama8b():
    """Llama-3.1-8B-shaped decode after a 128K prefill on H = 8 hosts (cache 16K rows per host),
    one new token: every head of the merged output vs the oracle."""
    from paper_2502_12085_b200.decode import DecodeRank
    cfg = synth.CONFIGS["llama8b-128k"]
    rng = np.random.default_rng(9)
    caches = []
    for h in range(cfg.H):
        caches.append((_bits((cfg.l_b, cfg.hk, cfg.d), rng), _bits((cfg.l_b, cfg.hk, cfg.d), rng)))
    q = _bits((1, cfg.hq, cfg.d), rng)
    kn, vn = _bits((1, cfg.hk, cfg.d), rng), _bits((1, cfg.hk, cfg.d), rng)
    dr = DecodeRank(cfg.H, list(range(cfg.H)), 1, cfg.hq, cfg.hk, cfg.d)
    out = torch.empty((1, cfg.hq, cfg.d), dtype=torch.bfloat16, device="cuda")
    ol = torch.empty((1, cfg.hq), device="cuda")
    dr.step(dev(q), {h: (dev(kc), dev(vc)) for h, (kc, vc) in enumerate(caches)}, dev(kn), dev(vn), out, ol)
    torch.cuda.synchronize()
    A, L, _ = oracle.decode_step(q, caches, kn, vn)
    _check(out.float().cpu().double().numpy(), ol.cpu().double().numpy(), A, L, "decode L8-128K H=8")
