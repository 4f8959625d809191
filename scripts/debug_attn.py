#!/usr/bin/env python
"""Debug helper: per-launch synchronised runs of the attention kernel with error patterns.

    python scripts/debug_attn.py parity <case> <host> [phase]
    python scripts/debug_attn.py layer <config> [--layers L]      # PrefillRank launches one by one
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def parity(case, host, phase="all"):
    import test_gpu as T
    cfg = T.CASES[case]
    hosts, ref = T.oracle_layer(cfg)
    for rep in range(2):
        O, lse = T.run_attention(cfg, host, hosts[host], ref["gathered"], phase)
        err = np.abs(O - ref["O"][host])
        bad = np.argwhere(err.max(axis=2) > 2e-2)
        print(f"rep {rep}: max {err.max():.3e}; bad (row, head) count {len(bad)}")
        rows = sorted(set(bad[:, 0].tolist()))
        print("  bad rows:", rows[:40], "..." if len(rows) > 40 else "")
        print("  bad heads:", sorted(set(bad[:, 1].tolist())))


def hang(config, host, phase):
    """Run one launch with the trace build; while it runs, poll host-mapped progress words."""
    import ctypes
    import time
    from paper_2502_12085_b200 import apb
    lib = apb.load(apb.LIB_PATH.replace("libapb.so", "libapb_trace.so"))
    cfg = synth.CONFIGS[config]
    d = apb.Dims(n=cfg.n, H=cfg.H, host=host, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                 head_dim=cfg.d)
    dev = torch.device("cuda")
    prog_h = torch.zeros(8192 * 8, dtype=torch.int32).pin_memory()
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
    ptr = ctypes.c_void_p()
    # device pointer of the pinned (mapped) host buffer
    torch.cuda.init()
    rt = ctypes.CDLL([p for p in __import__("glob").glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*"))][0]) \
        if __import__("glob").glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*")) else None
    if rt is None:
        import nvidia.cuda_runtime as ncr
        rt = ctypes.CDLL(__import__("glob").glob(os.path.join(os.path.dirname(ncr.__file__), "lib", "libcudart.so*"))[0])
    rc = rt.cudaHostGetDevicePointer(ctypes.byref(ptr), ctypes.c_void_p(prog_h.data_ptr()), 0)
    print("hostGetDevicePointer rc", rc, flush=True)
    lib.apb_debug_prog.argtypes = [ctypes.c_void_p]
    lib.apb_debug_prog(None)
    q = torch.randn((d.rows, cfg.hq, cfg.d), device=dev).bfloat16()
    k = torch.randn((d.rows, cfg.hk, cfg.d), device=dev).bfloat16()
    v = torch.randn((d.rows, cfg.hk, cfg.d), device=dev).bfloat16()
    out = torch.empty_like(q)
    lse = torch.empty((cfg.hq, d.rows), device=dev)
    g = torch.zeros((cfg.H, 2, cfg.hk, d.l_pp, cfg.d), device=dev, dtype=torch.bfloat16)
    ws = torch.empty(max(apb.workspace_size(d, apb.WS_ATTENTION), 16), dtype=torch.uint8, device=dev)
    ws.zero_()
    lib.apb_debug_prog(ptr)
    torch.cuda.synchronize()
    print("launching", flush=True)
    apb.attention_fwd(d, q, k, v, g, out, lse, phase, ws)
    time.sleep(5)
    snap1 = prog_h.numpy().reshape(8192, 8).copy()
    time.sleep(5)
    pr = prog_h.numpy().reshape(8192, 8)
    print("progress changed between snapshots:", int((snap1 != pr).sum()), flush=True)
    started = np.nonzero(pr[:, 4])[0]
    done = [c for c in started if pr[c, 2] == 1000000 and pr[c, 3] in (0, 1000000)]
    stuck = [c for c in started if c not in set(done)]
    print(f"started {len(started)} done {len(done)} stuck {len(stuck)}", flush=True)
    for c in stuck[:20]:
        print(f"cta {c}: nkv {pr[c, 4] - 1} loader {pr[c, 0]} mma {pr[c, 1]} sm0 {pr[c, 2]} sm1 {pr[c, 3]}", flush=True)
    os._exit(0)


def layer(config, layers=1):
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.prefill import HostIO, PrefillRank
    cfg = synth.CONFIGS[config]
    base = apb.Dims(n=cfg.n, H=cfg.H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d)
    pr = PrefillRank(base, list(range(cfg.H)))
    dev = torch.device("cuda")
    io = {}
    for h in range(cfg.H):
        r = pr.dims(h).rows
        io[h] = HostIO(q=torch.randn((r, cfg.hq, cfg.d), device=dev).bfloat16(),
                       k=torch.randn((r, cfg.hk, cfg.d), device=dev).bfloat16(),
                       v=torch.randn((r, cfg.hk, cfg.d), device=dev).bfloat16(),
                       out=torch.empty((r, cfg.hq, cfg.d), device=dev, dtype=torch.bfloat16),
                       lse=torch.empty((cfg.hq, r), device=dev))
    for h in range(cfg.H):
        for ph in (apb.PHASE_LOCAL, apb.PHASE_PASSING):
            print(f"host {h} phase {ph} ...", end=" ", flush=True)
            x = io[h]
            apb.attention_fwd(pr.dims(h), x.q, x.k, x.v, pr.gathered, x.out, x.lse, phase=ph, ws=pr.ws[h])
            torch.cuda.synchronize()
            print("ok", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "parity":
        parity(sys.argv[2], int(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else "all")
    elif sys.argv[1] == "hang":
        hang(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        layer(sys.argv[2])
