#!/usr/bin/env python
"""Time the APB decode step (Alg. apb_decode) for one layer of the L8-128K workload: H hosts'
block caches (l_b rows each) on one GPU, t new tokens.  Reports per-host partial time, the whole
step (partials + merge) and the achieved HBM bandwidth on the algorithmic bytes (cache K+V read)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_12085_b200 import apb  # noqa: E402
from paper_2502_12085_b200.decode import DecodeRank  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b-128k")
    ap.add_argument("--t", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--hq", type=int, default=None, help="override query heads (layout experiments)")
    ap.add_argument("--hk", type=int, default=None, help="override KV heads")
    ap.add_argument("--lb", type=int, default=None, help="override cache rows per host")
    ap.add_argument("--per-host", action="store_true", help="one apb_decode_attention per host (no batched launch)")
    ap.add_argument("--queued", action="store_true",
                    help="spin the GPU ~1 ms before the start event so the step's launches are queued (device time only)")
    ap.add_argument("--no-fuse", action="store_true", help="batched partials + MergeScore (not apb_decode_step_hosts)")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    over = {k: v for k, v in (("hq", a.hq), ("hk", a.hk)) if v is not None}
    if a.lb is not None:
        over["n"] = a.lb * cfg.H
    if over:
        cfg = cfg.replace(**over)
    dev = torch.device("cuda")
    caches = {h: (torch.randn((cfg.l_b, cfg.hk, cfg.d), device=dev).bfloat16(),
                  torch.randn((cfg.l_b, cfg.hk, cfg.d), device=dev).bfloat16()) for h in range(cfg.H)}
    q = torch.randn((a.t, cfg.hq, cfg.d), device=dev).bfloat16()
    kn = torch.randn((a.t, cfg.hk, cfg.d), device=dev).bfloat16()
    vn = torch.randn((a.t, cfg.hk, cfg.d), device=dev).bfloat16()
    dr = DecodeRank(cfg.H, list(range(cfg.H)), a.t, cfg.hq, cfg.hk, cfg.d, batch_hosts=not a.per_host,
                    fuse_merge=not a.no_fuse)
    out = torch.empty((a.t, cfg.hq, cfg.d), dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2: cold caches each iteration
    times = []
    for i in range(a.iters + 3):
        flush.zero_()
        if a.queued:
            torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dr.step(q, caches, kn, vn, out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            times.append(e0.elapsed_time(e1))
    ms = sorted(times)[len(times) // 2]
    cache_bytes = cfg.H * 2 * cfg.l_b * cfg.hk * cfg.d * 2
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    gbs = cache_bytes / (ms / 1e3) / 1e9
    print(json.dumps({"config": a.config, "launch": "per-host" if a.per_host else ("batched partials (apb_decode_attention_hosts)" if a.no_fuse
                                                                    else "fused step (apb_decode_step_hosts)"), "hq": cfg.hq, "hk": cfg.hk, "t_new": a.t, "hosts": cfg.H, "cache_rows_per_host": cfg.l_b,
                      "queued": a.queued, "ms_per_layer_step": round(ms, 4), "cache_bytes": cache_bytes, "achieved_gbs": round(gbs, 1),
                      "hbm_peak_gbs": peaks["hbm_gbs"], "frac": round(gbs / peaks["hbm_gbs"], 3)}))


if __name__ == "__main__":
    main()
