"""A real multi-rank exchange through libapb on one GPU: the peer-memory exchange (apb_peers_*,
CUDA IPC) between two processes.

Two processes share cuda:0 (CUDA IPC maps one process's allocation into the other; on an 8-GPU
box the same mappings run over NVLink / NVSwitch).  Each rank owns half of the toy config's hosts
(block or cyclic), runs three layers of the hot path through PrefillRank(peers=...) — scoring,
select with the compaction pushing every selected row into BOTH ranks' buffers (the AllGather
fused into the gather), the device-side slot wait, LOCAL / PASSING attention, the buffer release —
and ships its gathered buffer and outputs back.  Three layers exercise both parity buffers and the
wait for the peers' release of epoch e - 2.  Checked against the fp64 oracle's Alg. apb_prefill
(P:700-733): selection bit-exact on the GPU's scores; every slot a rank reads (slots below its
largest host, pushed by whichever rank owns that host) equal to the oracle's compaction of those
indices; attention within the north-star tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu

LAYERS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    return synth.CONFIGS["toy"].replace(d_hidden=1024)


def _dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _worker(rank, world, port, layout, q, batched=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.prefill import HostIO, PrefillRank, hosts_of_rank
    cfg = _cfg()
    base = apb.Dims(n=cfg.n, H=cfg.H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d)
    peers = apb.Peers(base, world, rank)
    handles = [None] * world
    dist.all_gather_object(handles, peers.handle)
    peers.open(handles)
    mine = hosts_of_rank(cfg.H, world, rank, layout)
    pr = PrefillRank(base, mine, peers=peers, batched=batched)
    results = []
    for layer in range(LAYERS):
        io = {}
        for h in mine:
            x = synth.host_qkv(cfg, layer, h)
            qd = _dev(x["q"])
            io[h] = HostIO(q=qd, k=_dev(x["k"]), v=_dev(x["v"]), out=torch.full_like(qd, float("nan")),
                           lse=torch.empty((cfg.hq, qd.shape[0]), device="cuda"))
        w = synth.retain_weights(cfg, layer)
        wd = apb.RetainWeights(w1=_dev(w["w1"]), w2=torch.from_numpy(w["w2"]).cuda(),
                               b1=torch.from_numpy(w["b1"]).cuda(), b2=torch.from_numpy(w["b2"]).cuda())
        pr.layer(io, wd, layer_idx=layer)
        torch.cuda.synchronize()
        gathered = pr.gathered.view(torch.int16).cpu().numpy().view(np.uint16).copy()
        outs = {h: (io[h].out.float().cpu().double().numpy(), pr.scores[h].cpu().double().numpy(),
                    pr.indices[h].cpu().numpy()) for h in mine}
        results.append((gathered, outs))
    q.put((rank, results))
    dist.barrier()  # no rank may still push into a buffer that is freed
    peers.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("layout,batched", [("block", False), ("cyclic", False), ("cyclic", True)])
def test_peer_exchange_two_ranks_one_gpu(layout, batched):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, q, batched)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = _cfg()
    from paper_2502_12085_b200.prefill import hosts_of_rank
    owner = {h: r for r in range(world) for h in hosts_of_rank(cfg.H, world, r, layout)}
    for layer in range(LAYERS):
        hosts = [synth.host_qkv(cfg, layer, h) for h in range(cfg.H)]
        outs = {**res[0][layer][1], **res[1][layer][1]}
        comp = {}
        for h in range(cfg.H):
            _, s_gpu, idx = outs[h]
            assert np.array_equal(idx, oracle.select_all_heads(s_gpu, cfg.l_p)), (layer, h)  # rule (i)
            comp[h] = oracle.compact(hosts[h]["k"], hosts[h]["v"], hosts[h]["L_A"], idx)
        # each rank's buffer holds, bit for bit, every slot its hosts read (slots < its largest host),
        # whichever rank pushed it
        for r in range(world):
            g = res[r][layer][0]
            for s_ in range(max(hosts_of_rank(cfg.H, world, r, layout))):
                assert np.array_equal(g[s_], comp[s_]), (layer, r, s_)
        for h in range(cfg.H):
            x = hosts[h]
            pk, pv = oracle.passing(res[owner[h]][layer][0], h)
            O_or, _ = oracle.attention(x["q"], x["k"], x["v"], x["L_A"], pk, pv)
            err = np.abs(outs[h][0] - O_or)
            assert err.max() <= 2e-2 and err.mean() <= 2e-3, (layer, h, err.max(), err.mean())


@pytest.mark.parametrize("l_b,lp", [(2048, 256), (40000, 2048), (131072, 2048)])
def test_peer_push_single_rank_matches_oracle(l_b, lp):
    """The compaction's peer push (apb_select_topk_peers) at l_b in both select regimes (single-CTA
    register select + PDL gather up to 32K; the 8-CTA cluster kernel beyond): a one-rank Peers
    (its own buffer is its only destination); indices bit-exact against the
    oracle's stable sort, the pushed slot bit-exact against oracle.compact."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_12085_b200 import apb
    cfg = synth.Config("push", 23, n=2 * l_b, H=2, l_a=8, l_p=lp, hq=8, hk=4, d=128, d_hidden=256)
    x = synth.host_qkv(cfg, 0, 1)
    sc = synth.random_scores(cfg, 0, 1, ties=True)
    base = apb.Dims(n=cfg.n, H=cfg.H, host=1, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d)
    peers = apb.Peers(base, 1, 0)
    peers.open([peers.handle])
    try:
        s = torch.from_numpy(np.ascontiguousarray(sc, dtype=np.float32)).cuda()
        idx = torch.full((cfg.hk, cfg.l_pp), -1, dtype=torch.int32, device="cuda")
        peers.select_topk(base, s, _dev(x["k"]), _dev(x["v"]), idx, 1)
        torch.cuda.synchronize()
    except Exception:
        peers.close()
        raise
    idx_or = oracle.select_all_heads(sc.astype(np.float64), cfg.l_p)
    assert np.array_equal(idx.cpu().numpy(), idx_or)
    g = peers.gathered(1).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(g[1], oracle.compact(x["k"], x["v"], x["L_A"], idx_or))
    peers.close()
