"""N > 1 host logic on CPU (gloo, world size 2): host ownership, the in-place slot layout the
exchange uses (rank r owns slots [r*H/N, (r+1)*H/N) of gathered [H][2][hk][l_p'][d]), the
128-byte communicator-id broadcast, and that a 2-rank run reproduces the single-process APB
layer.  The arithmetic here is the oracle's (CPU); the exchange rounds are libapb's own
(apb_exchange_plan, the plan apb_exchange_passing{,_cyclic} hand to NCCL) run over gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2502_12085_b200 import apb
from paper_2502_12085_b200.prefill import hosts_of_rank


def test_hosts_of_rank():
    assert hosts_of_rank(8, 1, 0) == list(range(8))
    assert hosts_of_rank(8, 2, 1) == [4, 5, 6, 7]
    assert hosts_of_rank(8, 8, 3) == [3]
    assert hosts_of_rank(8, 2, 1, "cyclic") == [1, 3, 5, 7]
    assert hosts_of_rank(8, 4, 2, "cyclic") == [2, 6]
    assert hosts_of_rank(8, 8, 3, "cyclic") == [3]
    assert hosts_of_rank(8, 1, 0, "cyclic") == list(range(8))
    with pytest.raises(ValueError):
        hosts_of_rank(8, 3, 0)
    with pytest.raises(ValueError):
        hosts_of_rank(8, 2, 0, "snake")


def test_cyclic_layout_balances_work():
    """The per-rank attention work (mask-counted FLOPs, Appendix A) of the busiest rank is lower
    with cyclic ownership than with contiguous blocks, and every host is owned exactly once."""
    from paper_2502_12085_b200 import workload
    c = synth.CONFIGS["llama8b-128k"]
    f = [workload.attention_flops(c.n, c.H, h, c.l_a, c.l_p, c.hq, c.d, c.l_q) for h in range(c.H)]
    for world in (2, 4):
        for layout in ("block", "cyclic"):
            owned = sorted(h for r in range(world) for h in hosts_of_rank(c.H, world, r, layout))
            assert owned == list(range(c.H))
        busiest = {lay: max(sum(f[h] for h in hosts_of_rank(c.H, world, r, lay)) for r in range(world))
                   for lay in ("block", "cyclic")}
        assert busiest["cyclic"] < 0.9 * busiest["block"], (world, busiest)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    return synth.CONFIGS["toy"].replace(n=512, H=4, l_a=32, l_p=16, d_hidden=32)


def _worker(rank, world, port, q, layout="block"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg()
    # communicator id: rank 0 draws 128 bytes, everyone receives the same
    uid = [os.urandom(128) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ids = [None] * world
    dist.all_gather_object(ids, uid[0])
    w = synth.retain_weights(cfg, 0)
    mine = hosts_of_rank(cfg.H, world, rank, layout)
    hosts = {h: synth.host_qkv(cfg, 0, h) for h in mine}
    # steps 1-2 for owned hosts, written into their own slots of a full-size buffer
    gathered = np.zeros((cfg.H, 2, cfg.hk, cfg.l_pp, cfg.d), np.uint16)
    for h in mine:
        x = hosts[h]
        s = oracle.retain_score(x["q"], x["k"], x["v"], x["L_A"], w["w1"], w["b1"], w["w2"], w["b2"], cfg.hk)
        gathered[h] = oracle.compact(x["k"], x["v"], x["L_A"], oracle.select_all_heads(s, cfg.l_p))
    # step 3: the in-place all-gather rounds libapb's apb_exchange_passing{,_cyclic} enqueue, as
    # apb_exchange_plan states them (send / recv offsets and counts in bf16 elements), run on gloo
    dims = apb.Dims(n=cfg.n, H=cfg.H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d)
    plan = apb.exchange_plan(dims, world, rank, apb.LAYOUT_CYCLIC if layout == "cyclic" else apb.LAYOUT_BLOCK)
    assert len(plan) == (1 if layout == "block" else cfg.H // world)
    flat = torch.from_numpy(gathered.reshape(-1).view(np.int32))  # bf16 pairs as int32 (gloo)
    for send, recv, count in plan:
        assert send % 2 == 0 and recv % 2 == 0 and count % 2 == 0
        parts = [torch.empty(count // 2, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, flat[send // 2: (send + count) // 2].clone())
        flat[recv // 2: (recv + world * count) // 2] = torch.cat(parts)
    gathered = flat.numpy().view(np.uint16).reshape(gathered.shape)
    # step 4
    outs = {}
    for h in mine:
        x = hosts[h]
        pk, pv = oracle.passing(gathered, h)
        outs[h] = oracle.attention(x["q"], x["k"], x["v"], x["L_A"], pk, pv)[0]
    q.put((rank, ids[0] == ids[-1], gathered, outs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["block", "cyclic"])
def test_two_rank_layer_matches_single_process(layout):
    cfg = _cfg()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, layout)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        try:
            res.append(q.get(timeout=120))
        except Exception:
            break
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res) == world
    ref = oracle.prefill_layer([synth.host_qkv(cfg, 0, h) for h in range(cfg.H)], synth.retain_weights(cfg, 0),
                               cfg.l_p)
    for rank, same_id, gathered, outs in res:
        assert same_id
        assert np.array_equal(gathered, ref["gathered"])  # every rank holds [C_1..C_H]
        for h, O in outs.items():
            assert np.array_equal(O, ref["O"][h])
