#!/usr/bin/env python
"""Same-box comparison of APB with the paper's comparison systems, all on libapb's attention
kernel (the paper's per-block breakdown `tab:breakdown-tb`,
PAPER.md:1274-1280, Llama-3.1-8B, 128K, 8 hosts).

Each method's critical-path attention per layer is one APB-kernel launch with the method's
key set (the kernel's mask is "anchor | passing | local causal", reading G1):

  apb        l_a = 4K, l_p = 2K; critical host H
  star       StarAttn: l_a = l_b, l_p = 0; critical host H
  ring       RingAttn: every earlier block passes whole (l_a = 0, l_p = l_b) — host H computes
             exact causal attention of its block over the whole prefix, as the ring does
  ulysses    Ulysses: all-to-all over heads, each GPU runs full causal attention over all n
             tokens for hq/H query heads (hk/H KV heads)
  full       FlashAttn on 1 GPU: full causal attention, all heads

Per-layer exchange volume received by the critical GPU is reported beside it (bf16):
apb (H-1) compressed blocks; ring (H-1) whole KV blocks; ulysses the all-to-all of Q, K, V
and O ((H-1)/H of each GPU's share); star and full none.

    python scripts/method_table.py [--config llama8b-128k] [--iters 5] > profiles/rNN_method_table.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_12085_b200 import apb, workload  # noqa: E402

PAPER_MS = {"apb": 34.07, "star": 41.84, "ring": 152.12, "ulysses": 84.53, "full": 664.01}


def method_dims(m: str, cfg) -> tuple[apb.Dims, int]:
    """(dims of the critical launch, number of GPUs the method uses)."""
    H, l_b = cfg.H, cfg.l_b
    if m == "apb":
        return apb.Dims(n=cfg.n, H=H, host=H - 1, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                        head_dim=cfg.d), H
    if m == "star":
        return apb.Dims(n=cfg.n, H=H, host=H - 1, l_a=l_b, l_p=0, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                        head_dim=cfg.d), H
    if m == "ring":
        return apb.Dims(n=cfg.n, H=H, host=H - 1, l_a=0, l_p=l_b, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                        head_dim=cfg.d), H
    if m == "ulysses":
        return apb.Dims(n=cfg.n, H=1, host=0, l_a=0, l_p=0, n_heads=cfg.hq // H, n_kv_heads=max(cfg.hk // H, 1),
                        head_dim=cfg.d), H
    if m == "full":
        return apb.Dims(n=cfg.n, H=1, host=0, l_a=0, l_p=0, n_heads=cfg.hq, n_kv_heads=cfg.hk, head_dim=cfg.d), 1
    raise ValueError(m)


def recv_bytes(m: str, cfg) -> int:
    H, l_b, hk, hq, d = cfg.H, cfg.l_b, cfg.hk, cfg.hq, cfg.d
    if m == "apb":
        return (H - 1) * 2 * hk * cfg.l_pp * d * 2
    if m == "ring":
        return (H - 1) * 2 * hk * l_b * d * 2
    if m == "ulysses":
        per_gpu = l_b * ((hq + 2 * hk) * d + hq * d) * 2  # Q, K, V in and O back
        return per_gpu * (H - 1) // H
    return 0


def useful_flops(dims: apb.Dims) -> int:
    L_A, P = dims.L_A, dims.P
    return workload.visible_pairs(L_A, P, dims.l_b) * 4 * dims.head_dim * dims.n_heads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b-128k")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    out = {"config": a.config, "n": cfg.n, "H": cfg.H, "what": "critical-path attention per layer, one B200, "
           "libapb attention kernel, bf16, synthetic N(0,1) Q/K/V", "methods": {}}
    for m in ("apb", "star", "ring", "ulysses", "full"):
        dims, gpus = method_dims(m, cfg)
        rows = dims.rows
        rnd = lambda *s: torch.randn(*s, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
        q, k, v = rnd(rows, dims.n_heads, dims.head_dim), rnd(rows, dims.n_kv_heads, dims.head_dim), \
            rnd(rows, dims.n_kv_heads, dims.head_dim)
        gathered = rnd(dims.H, 2, dims.n_kv_heads, dims.l_pp, dims.head_dim) if dims.P else None
        o = torch.empty_like(q)
        nws = apb.workspace_size(dims, apb.WS_ATTENTION)
        ws = torch.empty(max(nws, 16), dtype=torch.uint8, device=dev)
        fn = lambda: apb.attention_fwd(dims, q, k, v, gathered, o, None, phase=apb.PHASE_ALL, ws=ws)
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        fl = useful_flops(dims)
        rb = recv_bytes(m, cfg)
        out["methods"][m] = {"attn_ms": round(ms, 3), "useful_tflop": round(fl / 1e12, 3),
                             "tflops": round(fl / ms / 1e9, 1), "gpus": gpus, "recv_mib": round(rb / 2 ** 20, 1),
                             "recv_ms_at_900GBs": round(rb / 900e9 * 1e3, 3), "paper_a800_ms": PAPER_MS[m],
                             "dims": {"n": dims.n, "H": dims.H, "host": dims.host, "l_a": dims.l_a, "l_p": dims.l_p,
                                      "hq": dims.n_heads, "hk": dims.n_kv_heads}}
        del q, k, v, gathered, o, ws
        torch.cuda.empty_cache()
    base = out["methods"]["apb"]["attn_ms"]
    for m, r in out["methods"].items():
        r["apb_speedup"] = round(r["attn_ms"] / base, 2)
        r["paper_apb_speedup"] = round(PAPER_MS[m] / PAPER_MS["apb"], 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
