"""The NCCL exchange through libapb with real ranks (needs >= 2 GPUs; skipped on a 1-GPU box).

Two processes, one GPU each, a libapb communicator (apb_comm_init over NCCL): every rank writes
its own hosts' slots of `gathered` [H][2][hk][l_p'][d] with a rank-dependent bit pattern, runs
apb_exchange_passing (block ownership) or apb_exchange_passing_cyclic (cyclic ownership), and
must end with the full buffer bit for bit.  Then
apb_comm_check reports no asynchronous error.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, HK, LP, D = 8, 2, 48, 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slot_bits(h):
    rng = np.random.default_rng(100 + h)
    return rng.integers(0, 1 << 16, size=(2, HK, LP, D), dtype=np.uint16)


def _worker(rank, world, port, layout, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # only to broadcast the NCCL id
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.prefill import hosts_of_rank
    uid = [apb.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = apb.Comm(uid[0], world, rank)
    dims = apb.Dims(n=H * 512, H=H, host=0, l_a=64, l_p=LP, n_heads=4, n_kv_heads=HK, head_dim=D)
    g = torch.zeros((H, 2, HK, LP, D), dtype=torch.int16, device="cuda")
    for h in hosts_of_rank(H, world, rank, layout):
        g[h] = torch.from_numpy(_slot_bits(h).view(np.int16)).cuda()
    gb = g.view(torch.bfloat16)
    apb.exchange_passing(comm, dims, gb, cyclic=(layout == "cyclic"))
    torch.cuda.synchronize()
    comm.check()
    q.put((rank, g.cpu().numpy().view(np.uint16)))
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["block", "cyclic"])
def test_nccl_exchange_two_ranks(layout):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (NCCL refuses two ranks on one device)")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.stack([_slot_bits(h) for h in range(H)])
    for rank, got in res:
        assert np.array_equal(got, want), rank
