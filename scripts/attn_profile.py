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
    ap.add_argument("--select", action="store_true", help="profile apb_select_topk (select + compaction) instead")
    ap.add_argument("--queued", type=int, default=0,
                    help="N launches queued behind a ~1 ms GPU spin between the events (device time per launch, "
                         "no host launch overhead)")
    ap.add_argument("--trace", type=int, default=None, help="CTA index to trace (uses libapb_trace.so)")
    ap.add_argument("--ctatimes", action="store_true", help="per-CTA timeline of the last launch (libapb_trace.so): "
                    "SM utilisation, tail, gaps between CTAs on one SM")
    ap.add_argument("--clock", type=int, default=0, help="N extra launches with NVML SM-clock sampling: "
                    "prints the median clock and the fraction of the tensor peak at that clock")
    a = ap.parse_args()
    if a.ctatimes and a.trace is None:
        a.trace = 0
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
    if a.select:
        s = torch.randn((cfg.hk, d.l_b), generator=g, device=dev)
        idx = torch.empty((cfg.hk, d.l_pp), dtype=torch.int32, device=dev)
        send = torch.empty((2, cfg.hk, d.l_pp, cfg.d), dtype=torch.bfloat16, device=dev)
        fn = lambda: apb.select_topk(d, s, k, v, idx, send)  # noqa: E731
        flops = 1e6  # report ms; "TFLOP/s" column is meaningless here
    elif a.score:
        w = apb.RetainWeights(w1=(torch.randn((cfg.d_hidden, cfg.d_in), generator=g, device=dev) * cfg.d_in ** -0.5).bfloat16(),
                              w2=torch.randn((cfg.hq, cfg.d_hidden), generator=g, device=dev) * cfg.d_hidden ** -0.5)
        s = torch.empty((cfg.hk, d.l_b), device=dev)
        sws = torch.empty(apb.retain_workspace_size(d, w), dtype=torch.uint8, device=dev)
        fn = lambda: apb.retain_score(d, w, q, k, v, s, ws=sws)  # noqa: E731
        flops = workload.score_flops(d.l_b, cfg.d_in, cfg.d_hidden, cfg.hq)
    else:
        phase = {"local": apb.PHASE_LOCAL, "passing": apb.PHASE_PASSING, "all": apb.PHASE_ALL}[a.phase]
        if phase == apb.PHASE_PASSING:
            apb.attention_fwd(d, q, k, v, gathered, out, lse, apb.PHASE_LOCAL, ws)
        flops = {"local": loc, "passing": pas, "all": loc + pas}[a.phase]
        fn = lambda: apb.attention_fwd(d, q, k, v, gathered, out, lse, phase, ws)  # noqa: E731
    for i in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nq = max(a.queued, 1)
        if a.queued:
            torch.cuda._sleep(2_000_000)
        e0.record()
        for _ in range(nq):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nq
        print(f"iter {i}: {ms:.4f} ms  {flops / ms / 1e9:.1f} TFLOP/s" + (f" ({nq} queued launches)" if a.queued else ""))
    if a.clock:
        import threading
        import pynvml
        pynvml.nvmlInit()
        hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        mhz, watts, stop = [], [], threading.Event()

        def sample():
            while not stop.is_set():
                mhz.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
                watts.append(pynvml.nvmlDeviceGetPowerUsage(hdl) / 1e3)
                stop.wait(0.005)
        th = threading.Thread(target=sample)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th.start()
        e0.record()
        for _ in range(a.clock):
            fn()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / a.clock
        f = sorted(mhz)[len(mhz) // 2]
        tf = flops / ms / 1e9
        # dense bf16 tcgen05 rate: 8192 FLOP/clk/SM (M=128, N=128, K=16 in 64 cycles) x 148 SMs
        peak = 148 * 8192 * f * 1e6 / 1e12
        late = mhz[len(mhz) // 2:]  # second half of the run: steady state
        w_late = sorted(watts[len(watts) // 2:])
        print(f"clock: {ms:.3f} ms/launch  {tf:.1f} TFLOP/s  SM {f} MHz ({len(mhz)} samples)  "
              f"tensor peak at that clock {peak:.0f} TF/s -> {tf / peak:.3f}; second half: SM "
              f"{sorted(late)[len(late) // 2]} MHz, board {w_late[len(w_late) // 2]:.0f} W "
              f"(max {w_late[-1]:.0f} W)")
    if a.ctatimes:
        import numpy as np
        g_ = cfg.hq // cfg.hk
        nB, nA = -(-d.l_b // 128), -(-(d.rows - d.l_b) // 128)
        n_loc = (nB * g_ + 1) // 2 * cfg.hk
        n_anc = 0 if a.phase == "passing" else (nA * g_ + 1) // 2 * cfg.hk
        n = n_loc + n_anc
        if os.environ.get("APB_ATTN_PERSIST", "")[:1] != "0" and os.environ.get("APB_ATTN_PAIR", "")[:1] != "1":
            n = min(n, torch.cuda.get_device_properties(0).multi_processor_count)  # persistent CTAs
            n_loc = min(n_loc, n)
        buf = (ctypes.c_ulonglong * (5 * n))()
        lib.apb_debug_cta_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.apb_debug_cta_times(buf, n)
        t = np.array(list(buf), dtype=np.int64).reshape(n, 5)
        pro = (t[:, 3] - t[:, 0]).astype(np.float64)
        epi = (t[:, 1] - t[:, 4]).astype(np.float64)
        tot = (t[:, 1] - t[:, 0]).astype(np.float64)
        print(f"per CTA: prologue (start -> first S issued) mean {pro.mean():.0f} ns, epilogue (O final -> end) "
              f"mean {epi.mean():.0f} ns, CTA mean {tot.mean():.0f} ns; (prologue + epilogue) / CTA time "
              f"{(pro.sum() + epi.sum()) / tot.sum():.4f}")
        t0 = t[:, 0].min()
        st, en, sm = t[:, 0] - t0, t[:, 1] - t0, t[:, 2]
        span = en.max()
        busy = (en - st).sum()
        nsm = 148
        last = np.array([en[sm == s_].max() for s_ in range(nsm) if (sm == s_).any()])
        gaps = []
        for s_ in range(nsm):
            idx = np.where(sm == s_)[0]
            o = idx[np.argsort(st[idx])]
            gaps += list(st[o][1:] - en[o][:-1])
        gaps = np.array(gaps if gaps else [0])
        dur = en - st
        print(f"ctas {n} (local {n_loc}, anchor {n_anc}); span {span / 1e3:.1f} us; SM util {busy / (nsm * span):.3f}; "
              f"SM last-finish p10/p50/p90 {np.percentile(last, 10) / span:.3f}/{np.percentile(last, 50) / span:.3f}/"
              f"{np.percentile(last, 90) / span:.3f}; gap between CTAs on an SM mean {gaps.mean():.0f} ns "
              f"p90 {np.percentile(gaps, 90):.0f} ns; CTA us local mean {dur[:n_loc].mean() / 1e3:.1f} max "
              f"{dur[:n_loc].max() / 1e3:.1f} min {dur[:n_loc].min() / 1e3:.1f}"
              + (f"; anchor mean {dur[n_loc:].mean() / 1e3:.1f}" if n_anc and n > n_loc else ""))
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
