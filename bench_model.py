#!/usr/bin/env python
"""APB prefill of a whole decoder stack: end-to-end prefill tokens/s
of a Llama-3.1-8B-shaped model (hidden 4096, FFN 14336, 32 heads / 8 KV heads, head_dim 128,
32 layers; public model card) around the APB hot path, for one 128K-token input, H = 8 hosts
(the paper's `tab:pt` setting).  Embedding and LM head are out of scope
(the input is synthetic hidden states; the paper's FLOP table P:933 also excludes them).

    python bench.py --workload model [--gpus N] [--steps K] [--warmup W] [--layers L]
    python bench_model.py ...                      (same)

One step = Alg. apb_prefill for every layer and host: RMSNorm -> QKV projection ->
RoPE -> retaining-head scoring -> top-l_p + compaction -> exchange -> masked attention -> O
projection + residual -> RMSNorm -> SwiGLU FFN + residual.  Timing rules as bench.py (W warm-up
steps, K timed steps between barrier + synchronize, CUDA events, max over ranks).  Every layer
has its own random-init weights (14 GB), and the residual stream (1.3 GB at N = 1) is larger
than L2.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_12085_b200 import workload  # noqa: E402

METRIC = "APB full-model prefill tokens/s (128K, Llama-3.1-8B shape, 32 layers)"
UNIT = "tokens/s"
HIDDEN, INTER = 4096, 14336


def gemm_flops_per_row(cfg, hidden=HIDDEN, inter=INTER) -> int:
    """2 * (QKV + O + gate/up + down) multiply-adds per row of one layer."""
    return 2 * hidden * ((cfg.hq + 2 * cfg.hk) * cfg.d + cfg.hq * cfg.d + 3 * inter)


def cpu_sample(cfg, H, layers, rows=32):
    """The fp64 oracle (as it stands) on a bounded sample: the dense part of one layer on `rows`
    rows with full-size weights, plus bench.py's hot-path sample; extrapolated per step."""
    import numpy as np

    import bench
    from oracle import layer as OL
    rng = np.random.default_rng(0)
    lw = {"attn_norm": np.ones(HIDDEN), "ffn_norm": np.ones(HIDDEN), "eps": 1e-5, "theta": 5e5,
          "w_qkv": rng.standard_normal(((cfg.hq + 2 * cfg.hk) * cfg.d, HIDDEN)) / 64,
          "w_o": rng.standard_normal((HIDDEN, cfg.hq * cfg.d)) / 64,
          "w_gu": rng.standard_normal((2 * INTER, HIDDEN)) / 64, "w_down": rng.standard_normal((HIDDEN, INTER)) / 120}
    x = rng.standard_normal((rows, HIDDEN))
    t0 = time.perf_counter()
    qkv = OL.attn_in(x, lw, cfg.hq, cfg.hk, cfg.d, np.arange(rows))
    OL.attn_out_ffn(x, qkv[:, :cfg.hq], lw)
    t_dense = (time.perf_counter() - t0) / rows
    total_rows = cfg.n + (H - 1) * (cfg.l_q + cfg.l_a)
    hot_v, hot_secs, hot_sample = bench.oracle_sample(cfg, H, layers)
    secs = t_dense * total_rows * layers + cfg.n / hot_v
    return cfg.n / secs, (f"dense layer part: {rows} rows x 1 layer, full-size weights ({t_dense * rows:.1f} s), "
                          f"extrapolated to {total_rows} rows x {layers} layers; hot path: {hot_sample}")


def main(args=None):
    if args is None:
        import bench
        args = bench.parse()
    import torch.distributed as dist

    import bench
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.model import ApbModelRank, LayerWeights, ModelShape
    from paper_2502_12085_b200.prefill import hosts_of_rank

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if rank != 0 and args.impl == "reference":
        return
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[args.config]
    H = args.hosts or cfg.H
    layers = args.layers or cfg.layers
    base = apb.Dims(n=cfg.n, H=H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d, l_q=cfg.l_q)
    hosts = hosts_of_rank(H, world, rank, args.host_layout)
    comm = None
    if world > 1:
        uid = [apb.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = apb.Comm(uid[0], world, rank)
    shape = ModelShape(hidden=HIDDEN, inter=INTER, n_heads=cfg.hq, n_kv_heads=cfg.hk, head_dim=cfg.d)
    model = ApbModelRank(base, shape, hosts, comm, dev, skip_unused_last=True,
                         batched=getattr(args, "attn_launch", "batched") == "batched")

    gen = torch.Generator(device=dev)
    gen.manual_seed(2502 * 12085 + 7 + rank)

    def rnd(*shp, dtype=torch.bfloat16, scale=1.0, mean=0.0):
        t = torch.empty(shp, dtype=torch.float32, device=dev)
        t.normal_(mean, scale, generator=gen)
        return t.to(dtype)

    lws = []
    for _ in range(layers):
        retain = apb.RetainWeights(w1=rnd(cfg.d_hidden, cfg.d_in, scale=cfg.d_in ** -0.5),
                                   w2=rnd(cfg.hq, cfg.d_hidden, dtype=torch.float32, scale=cfg.d_hidden ** -0.5),
                                   b1=rnd(cfg.d_hidden, dtype=torch.float32, scale=0.02),
                                   b2=torch.zeros(cfg.hq, dtype=torch.float32, device=dev))
        lws.append(LayerWeights(attn_norm=rnd(HIDDEN, scale=0.1, mean=1.0),
                                w_qkv=rnd((cfg.hq + 2 * cfg.hk) * cfg.d, HIDDEN, scale=HIDDEN ** -0.5),
                                w_o=rnd(HIDDEN, cfg.hq * cfg.d, scale=(cfg.hq * cfg.d) ** -0.5),
                                ffn_norm=rnd(HIDDEN, scale=0.1, mean=1.0),
                                w_gu=rnd(2 * INTER, HIDDEN, scale=HIDDEN ** -0.5),
                                w_down=rnd(HIDDEN, INTER, scale=INTER ** -0.5), retain=retain))
    # input hidden states [A; B_h] per host (consistent anchor = the document's first rows)
    doc = None
    x_in, xs = {}, {}
    for h in hosts:
        rows = model.rows[h]
        x_in[h] = rnd(rows, HIDDEN)
        xs[h] = torch.empty_like(x_in[h])
    if hosts[0] > 0 or len(hosts) > 1:
        doc = rnd(cfg.l_q + cfg.l_a, HIDDEN)
        for h in hosts:
            if h > 0:
                x_in[h][:cfg.l_q + cfg.l_a].copy_(doc)
    torch.cuda.synchronize()
    main_stream = torch.cuda.current_stream(dev)

    def step():
        for h in hosts:
            xs[h].copy_(x_in[h])
        for l in range(layers):
            model.layer(xs, lws[l], layer_idx=l)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    n_launch0 = apb.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(main_stream)
        for _ in range(args.steps):
            step()
        ev1.record(main_stream)
        barrier()
    launches = apb.launch_count() - n_launch0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_per_step = ms / args.steps
    value = cfg.n * args.steps / (ms / 1e3)
    ok = all(bool(torch.isfinite(xs[h].float()).all()) for h in hosts)

    # ---- useful FLOPs of the step on this rank: projections + FFN on every row it holds,
    # retaining heads on the scored blocks, masked attention (visible pairs)
    rows_rank = sum(model.rows[h] for h in hosts)
    scored = [h for h in hosts if h < H - 1]
    f_gemm = gemm_flops_per_row(cfg) * rows_rank * layers
    f_score = sum(workload.score_flops(cfg.l_b, cfg.d_in, cfg.d_hidden, cfg.hq) for _ in scored) * layers
    f_attn = sum(workload.attention_flops(cfg.n, H, h, cfg.l_a, cfg.l_p, cfg.hq, cfg.d, cfg.l_q) for h in hosts) * layers
    flops = f_gemm + f_score + f_attn
    peaks, peak_src = bench.load_peaks()
    peak_tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    achieved = flops / (ms_per_step / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak_tf, "unit": "TFLOP/s",
                "frac": round(achieved / peak_tf, 4), "traffic": None,
                "kernel": "whole step (libapb tcgen05 GEMMs with fused epilogues + apb attention + apb scoring), useful FLOPs",
                "peak_source": f"bf16_tflops_sustained, {peak_src}",
                "flops_per_step": flops, "flops_split": {"gemm": f_gemm, "retain_score": f_score, "attention": f_attn}}

    # ---- end to end: pinned host hidden states -> H2D -> all layers -> D2H of the block rows
    e2e = None
    if not args.no_e2e:
        pin_in = {h: x_in[h].cpu().pin_memory() for h in hosts}
        pin_out = {h: torch.empty((cfg.l_b, HIDDEN), dtype=torch.bfloat16).pin_memory() for h in hosts}

        def e2e_step():
            for h in hosts:
                xs[h].copy_(pin_in[h], non_blocking=True)
            for l in range(layers):
                model.layer(xs, lws[l], layer_idx=l)
            for h in hosts:
                pin_out[h].copy_(xs[h][model.rows[h] - cfg.l_b:], non_blocking=True)

        e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main_stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(main_stream)
        barrier()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": cfg.n * args.e2e_steps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": sum(p.numel() * 2 for p in pin_in.values()),
               "d2h_bytes_per_step": sum(p.numel() * 2 for p in pin_out.values()), "steps": args.e2e_steps,
               "how": "pinned host hidden states -> H2D -> every layer -> D2H of the block rows' final hidden "
                      "states, inside the timed region (per-rank volumes)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        v, sample = cpu_sample(cfg, H, layers)
        cpu = {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": sample}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "finite": ok,
                "data": "synthetic (seeded N(0,1) hidden states, random-init Llama-3.1-8B-shaped weights and "
                        "retaining heads)",
                "config": {"workload": f"{cfg.name}: APB prefill of a Llama-3.1-8B-shaped decoder stack "
                                       f"(hidden {HIDDEN}, FFN {INTER}, hq={cfg.hq}, hk={cfg.hk}, d={cfg.d}), "
                                       f"n={cfg.n}, H={H} hosts over {world} GPU(s), l_a={cfg.l_a}, "
                                       f"l_p={cfg.l_p}, {layers} layers",
                           "n": cfg.n, "H": H, "layers": layers, "parallelism": f"apb-sp{H}/{world}gpu",
                           "host_layout": ("all hosts on one GPU" if world == 1 else
                                           args.host_layout if world < H else "one host per GPU"),
                           "l2": "residual stream 1.3 GB and 14 GB of per-layer weights, far larger than L2"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
