#!/usr/bin/env python
"""Launch the attention kernel of one host of the L8-128K workload a few times (for ncu / timing).

    python scripts/attn_profile.py [--host 7] [--phase local|passing|all] [--iters 3] [--config llama8b-128k]
Prints the CUDA-event time per launch and the useful TFLOP/s.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_12085_b200 import apb, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--host", type=int, default=7)
    ap.add_argument("--phase", default="local")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--config", default="llama8b-128k")
    ap.add_argument("--score", action="store_true", help="profile apb_retain_score instead")
    ap.add_argument("--trace", type=int, default=None, help="CTA index to trace (uses libapb_trace.so)")
    a = ap.parse_args()
    if a.trace is not None:
        import ctypes
        lib = apb.load(apb.LIB_PATH.replace("libapb.so", "libapb_trace.so"))
        lib.apb_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.apb_debug_trace(None, 0, a.trace)
    cfg = synth.CONFIGS[a.config]
    d = apb.Dims(n=cfg.n, H=cfg.H, host=a.host, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                 head_dim=cfg.d)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = torch.randn((d.rows, cfg.hq, cfg.d), generator=g, device=dev).bfloat16()
    k = torch.randn((d.rows, cfg.hk, cfg.d), generator=g, device=dev).bfloat16()
    v = torch.randn((d.rows, cfg.hk, cfg.d), generator=g, device=dev).bfloat16()
    out = torch.empty_like(q)
    lse = torch.empty((cfg.hq, d.rows), device=dev)
    gathered = torch.randn((cfg.H, 2, cfg.hk, d.l_pp, cfg.d), generator=g, device=dev).bfloat16()
    ws = torch.empty(max(apb.workspace_size(d, apb.WS_ATTENTION), 16), dtype=torch.uint8, device=dev)
    loc, pas = workload.attention_flops_split(cfg.n, cfg.H, a.host, cfg.l_a, cfg.l_p, cfg.hq, cfg.d)
    if a.score:
        w = apb.RetainWeights(w1=(torch.randn((cfg.d_hidden, cfg.d_in), generator=g, device=dev) * cfg.d_in ** -0.5).bfloat16(),
                              w2=torch.randn((cfg.hq, cfg.d_hidden), generator=g, device=dev) * cfg.d_hidden ** -0.5)
        s = torch.empty((cfg.hk, d.l_b), device=dev)
        fn = lambda: apb.retain_score(d, w, q, k, v, s)  # noqa: E731
        flops = workload.score_flops(d.l_b, cfg.d_in, cfg.d_hidden, cfg.hq)
    else:
        phase = {"local": apb.PHASE_LOCAL, "passing": apb.PHASE_PASSING, "all": apb.PHASE_ALL}[a.phase]
        if phase == apb.PHASE_PASSING:
            apb.attention_fwd(d, q, k, v, gathered, out, lse, apb.PHASE_LOCAL, ws)
        flops = {"local": loc, "passing": pas, "all": loc + pas}[a.phase]
        fn = lambda: apb.attention_fwd(d, q, k, v, gathered, out, lse, phase, ws)  # noqa: E731
    for i in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"iter {i}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
    if a.trace is not None:
        import numpy as np
        buf = (ctypes.c_ulonglong * 2048)()
        lib.apb_debug_trace(buf, 2048, -1)
        t = np.array(list(buf), dtype=np.int64).reshape(64, 32)
        t0 = t[0, 0]
        names = ["S0iss", "S1iss", "P0h0w", "P0h1w", "P1h0w", "P1h1w", "S0rdy", "S1rdy", "P0h0", "P0h1", "P1h0", "P1h1",
                 "Vrdy", "Krdy", "-", "-", "ld0", "max0", "exp0", "st0", "ld1", "max1", "exp1", "st1",
                 "t0w0", "t0w1", "t0w2", "t0w3", "t1w0", "t1w1", "t1w2", "t1w3"]
        print("step " + " ".join(f"{n:>7s}" for n in names) + "   (clk since S0(0) issue)")
        for i in range(64):
            if t[i, 0] == 0 and i > 0:
                break
            print(f"{i:4d} " + " ".join(f"{(x - t0) if x else -1:7d}" for x in t[i, :32]))


if __name__ == "__main__":
    main()
