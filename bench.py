#!/usr/bin/env python
"""APB prefill hot-path benchmark (BASELINE.json metric: APB prefill tokens/s, 128K tokens,
Llama-3.1-8B shape, at 1/2/4/8 B200; % attention FLOP peak).

One step = one pass of the whole hot path (retaining-head scoring, top-l_p
selection + compaction, the passing-block exchange, masked attention) over every layer of a
synthetic Llama-3.1-8B-shaped layer stack for one 128K-token input: the paper's
configuration (n = 131072, H = 8 hosts, l_a = 4K, l_p = 2K, 32 layers).
The H hosts are spread over the N GPUs (N = 8: one host per GPU, the paper's deployment;
N < 8: several hosts emulated per GPU, same total work), so `scaling` is "strong".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b-128k] [--impl apb|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: W warm-up steps, then exactly K steps between barrier + synchronize on both sides,
CUDA events on the launching stream, max over ranks.  Inputs per layer (~2 GiB at N = 1) are
far larger than L2 and alternate between two buffer sets, so nothing survives in L2 from one
layer to the next.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_12085_b200 import workload  # noqa: E402

METRIC = "APB prefill tokens/s (128K, 8B-shape) at 1/2/4/8 B200; % attention FLOP peak"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["apb", "reference"], default="apb")
    ap.add_argument("--compressor", choices=["retain", "random"], default="retain",
                    help="Table 4 compressor: retaining heads R (default) or the random selector Rd.")
    ap.add_argument("--shared-set", action="store_true", help="one index set per host (SPEC S:294 reading)")
    ap.add_argument("--workload", choices=["hotpath", "model"], default="hotpath",
                    help="model: the full decoder stack around the hot path (bench_model.py, NEXT #2)")
    ap.add_argument("--config", default="llama8b-128k")
    ap.add_argument("--layers", type=int, default=None, help="override the layer count (default: the model's)")
    ap.add_argument("--hosts", type=int, default=None, help="override H (default: the paper's 8)")
    ap.add_argument("--host-layout", choices=["cyclic", "block"], default="cyclic",
                    help="host ownership when N < H ranks: cyclic r, r+N, ... (work-balanced) or contiguous blocks")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--attn-launch", choices=["batched", "per-host"], default="batched",
                    help="batched: one attention launch per phase over every owned host (apb_attention_fwd_hosts; "
                         "single rank: compress every host first, then the layer's attention as one launch); "
                         "per-host: one launch per host (single rank: ordered, compression on a side stream)")
    ap.add_argument("--schedule", choices=["auto", "split", "ordered"], default="auto",
                    help="auto: LOCAL/PASSING split around the exchange only when N > 1")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank uses cuda:0 (the multi-rank schedule on a single GPU; with the default peer "
                         "exchange the ranks really exchange their compressed blocks through CUDA IPC)")
    ap.add_argument("--exchange", choices=["auto", "nccl", "peer"], default="auto",
                    help="N > 1 exchange: NCCL AllGather, or peer memory (CUDA IPC: the AllGather fused into the "
                         "compaction, apb_peers_*); auto = peer with --same-device, else nccl")
    ap.add_argument("--dist", choices=["D1", "D2"], default="D1",
                    help="Q/K/V distribution: D1 N(0,1) (the paper's synthetic timing input) or D2 'peaky' "
                         "(Q, K ~ N(0, 2^2): logit std 4, more online-softmax rescales)")
    ap.add_argument("--no-breakdown", action="store_true", help="skip the per-op breakdown pass")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks + throttle reasons every 200 ms."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
               0x1: "gpu_idle", 0x10: "sync_boost"}

    def __init__(self, index: int):
        self.index, self.samples, self.reasons = index, [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle

def oracle_sample(cfg, H, layers, rows_per_host=64, tokens=16, hosts_sample=None):
    """Time the fp64 oracle (as it stands) on a bounded sample of ONE layer and extrapolate
    linearly to the whole step (all hosts, all layers).  Returns (tokens/s, seconds, sample text)."""
    import numpy as np
    import oracle
    oracle.build()
    l_b, lpp = cfg.n // H, min(cfg.l_p, cfg.n // H)
    hosts_sample = hosts_sample or sorted({1 % H, H - 1})
    rng = np.random.default_rng(0)
    t_attn, pairs_done = 0.0, 0
    for h in hosts_sample:
        x = synth.host_qkv(cfg.replace(H=H), 0, h)
        L_A = x["L_A"]
        gathered = rng.integers(0, 1 << 16, size=(H, 2, cfg.hk, lpp, cfg.d), dtype=np.uint16) & 0x3FFF
        pk, pv = oracle.passing(gathered, h)
        rows = np.unique(rng.integers(0, L_A + l_b, size=rows_per_host))
        t0 = time.perf_counter()
        oracle.attention(x["q"], x["k"], x["v"], L_A, pk, pv, rows=rows)
        t_attn += time.perf_counter() - t0
        P = h * lpp
        pairs_done += sum((r + 1) if r < L_A else (L_A + P + (r - L_A) + 1) for r in rows)
    x = synth.host_qkv(cfg.replace(H=H), 0, 1 % H)
    w = synth.retain_weights(cfg, 0)
    L_A = x["L_A"]
    sub = {k: x[k][L_A:L_A + tokens] for k in ("q", "k", "v")}
    t0 = time.perf_counter()
    s = oracle.retain_score(sub["q"], sub["k"], sub["v"], 0, w["w1"], w["b1"], w["w2"], w["b2"], cfg.hk)
    t_score = time.perf_counter() - t0
    srow = rng.standard_normal(l_b)
    t0 = time.perf_counter()
    idx = oracle.select_topk(srow, cfg.l_p)
    t_sel = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.compact(x["k"], x["v"], L_A, np.stack([idx] * cfg.hk))
    t_cmp = time.perf_counter() - t0
    total_pairs = sum(workload.visible_pairs(workload.host_L_A(h, cfg.l_q, cfg.l_a), h * lpp, l_b) for h in range(H))
    layer_s = (t_attn / pairs_done * total_pairs) + t_score / tokens * l_b * (H - 1) + t_sel * cfg.hk * (H - 1) \
        + t_cmp * (H - 1)
    step_s = layer_s * layers
    measured = t_attn + t_score + t_sel + t_cmp
    sample = (f"1 layer: attention for {rows_per_host} sampled query rows x {cfg.hq} heads on hosts "
              f"{[h + 1 for h in hosts_sample]}, retaining head on {tokens} tokens, top-l_p on 1 KV head, "
              f"compaction of 1 host ({measured:.1f} s measured); extrapolated linearly in visible pairs, "
              f"tokens, KV heads, hosts and layers to the {layers}-layer, {H}-host step")
    return cfg.n / step_s, measured, sample


def host_cores():
    """(physical cores, cores this process may run on) of the host."""
    phys = None
    try:
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        phys = len({ln for ln in out.splitlines() if ln and not ln.startswith("#")})
    except Exception:
        pass
    return phys, len(os.sched_getaffinity(0))


def oracle_toy_full():
    """The toy config (BASELINE configs[0]) through the whole oracle layer (Alg. apb_prefill,
    every host, every row: no sampling), with all threads and with one: (tokens/s, s) each."""
    import oracle
    cfg = synth.CONFIGS["toy"]
    hosts = [synth.host_qkv(cfg, 0, h) for h in range(cfg.H)]
    w = synth.retain_weights(cfg, 0)
    res = {}
    threads = oracle.num_threads()
    for label, nt in (("all_threads", threads), ("single_thread", 1)):
        oracle.set_num_threads(nt)
        t0 = time.perf_counter()
        oracle.prefill_layer(hosts, w, cfg.l_p)
        dt = time.perf_counter() - t0
        res[label] = {"tokens_per_s": round(cfg.n / dt, 1), "seconds": round(dt, 3), "threads": nt}
    oracle.set_num_threads(threads)
    return res


def cpu_baseline_line(cfg, H, layers, value=None, sample=None):
    """The cpu_baseline object: the oracle's extrapolated tokens/s on this workload, plus the
    toy full run, the single-thread rate and the host's core counts."""
    import oracle
    if value is None:
        value, _, sample = oracle_sample(cfg, H, layers)
    phys, avail = host_cores()
    toy = oracle_toy_full()
    return {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": sample,
            "physical_cores": phys, "affinity_cores": avail,
            "toy_full_oracle": dict(toy, config="toy: n=2048, H=4, l_a=128, l_p=64, hq=4, hk=2, d=64, 1 layer, "
                                                "every row of every host (no extrapolation)"),
            "single_thread_extrapolated": round(value * toy["all_threads"]["seconds"]
                                                / toy["single_thread"]["seconds"], 4)}


def host_layout_desc(world, H, layout):
    return "all hosts on one GPU" if world == 1 else layout if world < H else "one host per GPU"


def run_reference(args, rank):
    """--impl reference: the oracle (as it stands) on the host cores, bounded sample per step."""
    if rank != 0:
        return
    import oracle
    cfg = synth.CONFIGS[args.config]
    H = args.hosts or cfg.H
    layers = args.layers or cfg.layers
    # Same bounded sample as the GPU arm's cpu_baseline leg (64 rows/host, 16 tokens: ~4 s per step
    # on 16 cores), so both report one oracle throughput; a smaller sample is dominated by the
    # oracle's fixed per-call cost and extrapolates to a ~4x lower number.
    for _ in range(args.warmup):
        oracle_sample(cfg, H, layers)
    vals, secs = [], []
    for _ in range(args.steps):
        v, s, sample = oracle_sample(cfg, H, layers)
        vals.append(v)
        secs.append(s)
    value = statistics.median(vals)
    world = args.gpus or 1
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg.n / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(cfg, H, layers, world),
                           host_layout=host_layout_desc(world, H, args.host_layout)),
            "cpu_baseline": cpu_baseline_line(cfg, H, layers, value, sample),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


MODEL_SHAPES = {"llama8b-128k": "Llama-3.1-8B", "llama8b-32k": "Llama-3.1-8B", "qwen14b-128k": "Qwen-2.5-14B",
                "yi34b-200k": "Yi-34B-200K", "llama8b-512k": "Llama-3-8B-1M", "llama8b-1m": "Llama-3-8B-1M"}


def workload_config(cfg, H, layers, n_gpus, variant=""):
    shape = MODEL_SHAPES.get(cfg.name, cfg.name)
    l_b = cfg.n // H
    rows = sum(l_b + (0 if h == 0 else cfg.l_q + cfg.l_a) for h in range(H))
    qkv_gib = rows * (cfg.hq + 2 * cfg.hk) * cfg.d * 2 / 2 ** 30
    return {"workload": f"{cfg.name}{variant}: APB prefill hot path, {shape}-shaped layer stack "
                        f"(hq={cfg.hq}, hk={cfg.hk}, d={cfg.d}), n={cfg.n}, H={H} hosts over {n_gpus} GPU(s), "
                        f"l_a={cfg.l_a}, l_p={cfg.l_p}, {layers} layers, retaining head d_R={cfg.d_hidden}",
            "n": cfg.n, "H": H, "l_a": cfg.l_a, "l_p": cfg.l_p, "layers": layers, "hq": cfg.hq, "hk": cfg.hk,
            "d": cfg.d, "parallelism": f"apb-sp{H}/{n_gpus}gpu",
            "l2": f"inputs larger than L2: {qkv_gib:.1f} GiB of Q/K/V per layer over all hosts (126 MB L2), "
                  "two alternating layer buffer sets"}


# ----------------------------------------------------------------------------- GPU arm

_T0 = time.time()


def progress(msg):
    """Phase marker on stderr (the JSON line stays the only stdout output)."""
    print(f"bench [{time.time() - _T0:7.1f} s] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    if args.workload == "model":
        import bench_model
        bench_model.main(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus is None:
        args.gpus = world
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch.distributed as dist
    from paper_2502_12085_b200 import apb
    from paper_2502_12085_b200.prefill import HostIO, PrefillRank, hosts_of_rank

    if args.same_device:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL init logging (ranks, channels, NVLS) so the N-rank run is visible in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.same_device:  # NCCL refuses two ranks on one GPU: plumbing-only test mode
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[args.config]
    H = args.hosts or cfg.H
    layers = args.layers or cfg.layers
    base = apb.Dims(n=cfg.n, H=H, host=0, l_a=cfg.l_a, l_p=cfg.l_p, n_heads=cfg.hq, n_kv_heads=cfg.hk,
                    head_dim=cfg.d, l_q=cfg.l_q)
    hosts = hosts_of_rank(H, world, rank, args.host_layout)
    comm = peers = None
    exchange = args.exchange if args.exchange != "auto" else ("peer" if args.same_device else "nccl")
    if world > 1 and exchange == "peer":
        peers = apb.Peers(base, world, rank)
        handles = [None] * world
        dist.all_gather_object(handles, peers.handle)
        peers.open(handles)
    elif world > 1 and not args.same_device:
        uid = [apb.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = apb.Comm(uid[0], world, rank)
    split = None if args.schedule == "auto" else (args.schedule == "split")
    if args.same_device and world > 1 and split is None:
        split = True  # the multi-rank schedule (a real exchange with --exchange peer, the default here)
    pr = PrefillRank(base, hosts, comm, dev, skip_unused_last=True, split_phases=split,
                     compressor=args.compressor, shared_set=args.shared_set, seed=2502,
                     same_device=args.same_device and peers is None, peers=peers, batched=args.attn_launch == "batched")

    # ---- synthetic inputs: D1 N(0,1) Q/K/V (the paper's timing input is synthetic random
    # input), two alternating layer buffer sets, random-init retaining heads.
    gen = torch.Generator(device=dev)
    gen.manual_seed(2502 * 12085 + rank)

    def rnd(*shape, dtype=torch.bfloat16, scale=1.0):
        t = torch.empty(shape, dtype=torch.float32, device=dev)
        t.normal_(0.0, scale, generator=gen)
        return t.to(dtype)

    sets = []
    outs = {h: None for h in hosts}
    for s in range(2):
        io = {}
        for h in hosts:
            rows = pr.dims(h).rows
            if outs[h] is None:
                outs[h] = (torch.empty((rows, cfg.hq, cfg.d), dtype=torch.bfloat16, device=dev),
                           torch.empty((cfg.hq, rows), dtype=torch.float32, device=dev))
            qk_scale = 2.0 if args.dist == "D2" else 1.0
            io[h] = HostIO(q=rnd(rows, cfg.hq, cfg.d, scale=qk_scale), k=rnd(rows, cfg.hk, cfg.d, scale=qk_scale),
                           v=rnd(rows, cfg.hk, cfg.d), out=outs[h][0], lse=outs[h][1])
        if 0 in io and cfg.l_q == 0:
            # consistent anchors: hosts >= 1 see the document's first l_a rows, which are
            # host 0's first rows — the same bytes on every host (the e2e leg uploads them once)
            for h in hosts:
                if h > 0 and cfg.l_a <= io[0].q.shape[0]:
                    for a, b in ((io[h].q, io[0].q), (io[h].k, io[0].k), (io[h].v, io[0].v)):
                        a[:cfg.l_a].copy_(b[:cfg.l_a])
        sets.append(io)
    weights = [apb.RetainWeights(w1=rnd(cfg.d_hidden, cfg.d_in, scale=cfg.d_in ** -0.5),
                                 w2=rnd(cfg.hq, cfg.d_hidden, dtype=torch.float32, scale=cfg.d_hidden ** -0.5),
                                 b1=rnd(cfg.d_hidden, dtype=torch.float32, scale=0.02),
                                 b2=torch.zeros(cfg.hq, dtype=torch.float32, device=dev)) for _ in range(layers)]
    torch.cuda.synchronize()

    main_stream = torch.cuda.current_stream(dev)
    attn_events = []

    def step(timed=False):
        for l in range(layers):
            pr.layer(sets[l % 2], weights[l], overlap=not args.no_overlap,
                     events=attn_events if timed else None, layer_idx=l)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier() if args.same_device else dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    progress("inputs ready")
    for _ in range(args.warmup):
        step()
    barrier()
    progress("warmup done")

    # ---- timed region
    n_launch0 = apb.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(main_stream)
        for _ in range(args.steps):
            step(timed=True)
        ev1.record(main_stream)
        barrier()
    launches = apb.launch_count() - n_launch0
    ms = ev0.elapsed_time(ev1)
    attn_ms = sum(a.elapsed_time(b) for a, b in attn_events)
    if world > 1:
        t = torch.tensor([ms], device="cpu" if args.same_device else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the step time is the slowest rank's
        ms = t.item()
    ms_per_step = ms / args.steps
    value = cfg.n * args.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (attention): useful FLOPs / in-situ kernel time
    flops_rank = sum(workload.attention_flops(cfg.n, H, h, cfg.l_a, cfg.l_p, cfg.hq, cfg.d, cfg.l_q) for h in hosts)
    flops_all = sum(workload.attention_flops(cfg.n, H, h, cfg.l_a, cfg.l_p, cfg.hq, cfg.d, cfg.l_q) for h in range(H))
    crit = workload.attention_flops(cfg.n, H, H - 1, cfg.l_a, cfg.l_p, cfg.hq, cfg.d, cfg.l_q)
    executed_rank = sum(workload.attention_executed_flops(cfg.n, H, h, cfg.l_a, cfg.l_p, cfg.hq, cfg.d, cfg.l_q)
                        for h in hosts)
    peaks, peak_src = load_peaks()
    peak_tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    achieved = flops_rank * layers * args.steps / (attn_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "attention_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.config, {}).get("dram_bytes_per_launch")
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak_tf, "unit": "TFLOP/s",
                "frac": round(achieved / peak_tf, 4), "traffic": traffic,
                "kernel": "apb_attention_kernel<128" + (
                    ", paired: 2-CTA clusters multicasting K/V"
                    if cfg.d == 128 and (os.environ.get("APB_ATTN_PAIR", "")[:1] == "1"
                                         or (os.environ.get("APB_ATTN_PAIR", "")[:1] == "a" and not pr.split_phases))
                    else ", persistent: one CTA per SM taking items from a work counter"
                    + (" (LOCAL one item per CTA)" if pr.split_phases else "")
                    if os.environ.get("APB_ATTN_PERSIST", "")[:1] != "0" else "") + "> ("
                + (("one LOCAL + one PASSING launch over the rank's hosts" if pr.batched
                    else "LOCAL + PASSING launches") if pr.split_phases
                   else ("one PHASE_ALL launch per layer over every host" if pr.batched
                         else "one ordered PHASE_ALL launch per host")) + ")",
                "peak_source": f"bf16_tflops_sustained, {peak_src}",
                "flops_per_step": flops_rank * layers,
                "executed_mma_flops_per_step": executed_rank * layers,
                "tile_efficiency": round(flops_rank / executed_rank, 4),
                "attn_ms_per_step": round(attn_ms / args.steps, 3)}

    progress("timed region done")
    # ---- per-op breakdown (one extra, untimed step with events around every libapb call)
    breakdown = None
    if not args.no_breakdown:
        breakdown = op_breakdown(pr, step, cfg, H, hosts, layers, world, peaks, barrier)
        progress("breakdown done")

    # ---- end to end through the public API: pinned host inputs -> H2D every layer -> ... -> D2H
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, pr, sets, weights, layers, hosts, dev, world, local_rank, barrier)
        progress("e2e done")

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:  # rank 0 only, at any N (the others wait below)
        cpu = cpu_baseline_line(cfg, H, layers)
        progress("cpu baseline done")

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) Q/K/V, random-init retaining heads)",
                "config": dict(workload_config(cfg, H, layers, world,
                                               ("" if args.compressor == "retain" else " [compressor Rd.]")
                                               + (" [shared index set]" if args.shared_set else "")
                                               + (" [D2 peaky Q/K]" if args.dist == "D2" else "")),
                               host_layout=host_layout_desc(world, H, args.host_layout),
                               **({"exchange": exchange} if world > 1 else {}),
                               **({"same_device": True} if args.same_device else {})),
                "attn_peak_frac": {"critical_host": round(crit * layers / (ms_per_step / 1e3) / 1e12 / peak_tf, 4)
                                   if world == H else None,
                                   "aggregate": round(flops_all * layers / (ms_per_step / 1e3) / 1e12 / (peak_tf * world), 4)},
                "roofline": roofline, "breakdown": breakdown, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        barrier()  # ranks > 0 wait here while rank 0 times the CPU oracle
    if comm is not None:
        comm.check()
        comm.close()
    if peers is not None:
        peers.close()  # after the barrier above: no rank still pushes into this buffer
    if world > 1:
        dist.destroy_process_group()


NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (hardware fact; no measured figure on this pool)


def op_breakdown(pr, step, cfg, H, hosts, layers, world, peaks, barrier):
    """Per-step device time of every libapb op of this rank (CUDA events around each call on the
    stream it runs on; one extra untimed step), beside its roofline lower bound.  With a side
    stream (N > 1, or --attn-launch per-host) score / select_compact / exchange overlap the
    attention: these are op times, not a partition of ms_per_step (at N = 1 batched they run
    serially on the main stream, before the layer's attention launch)."""
    pr.trace = []
    barrier()
    step()
    barrier()
    tr, pr.trace = pr.trace, None
    lpp = min(cfg.l_p, cfg.n // H)
    l_b = cfg.n // H
    hbm = peaks["hbm_gbs"] * 1e9
    tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 1e12
    slot = 2 * cfg.hk * lpp * cfg.d * 2
    score_flops = l_b * (2 * cfg.d_in * cfg.d_hidden + 2 * cfg.d_hidden * cfg.hq)
    sel_bytes = 4 * cfg.hk * l_b + 4 * cfg.hk * lpp + 2 * slot
    recv = (H - len(hosts)) * slot if world > 1 else 0
    out = {}
    for name, h, a, b in tr:
        e = out.setdefault(name, {"ms_per_step": 0.0, "launches": 0, "lower_bound_ms": 0.0})
        e["ms_per_step"] += a.elapsed_time(b)
        e["launches"] += 1
        hs = h if isinstance(h, list) else [h]  # a list: one batched launch over those hosts
        if name == "score":
            e["lower_bound_ms"] += len(hs) * score_flops / tf * 1e3
        elif name == "select_compact":
            e["lower_bound_ms"] += len(hs) * sel_bytes / hbm * 1e3
        elif name == "exchange":
            e["lower_bound_ms"] += recv / (NVLINK_GBS * 1e9) * 1e3
        else:
            for hh in hs:
                f_all = workload.attention_flops(cfg.n, H, hh, cfg.l_a, cfg.l_p, cfg.hq, cfg.d, cfg.l_q)
                f_pass = 4 * cfg.d * cfg.hq * l_b * hh * lpp
                f = {"attn_all": f_all, "attn_local": f_all - f_pass, "attn_passing": f_pass}[name]
                e["lower_bound_ms"] += f / tf * 1e3
    for name, e in out.items():
        e["us_per_launch"] = round(1e3 * e["ms_per_step"] / max(e["launches"], 1), 2)
        e["frac_of_bound"] = round(e["lower_bound_ms"] / e["ms_per_step"], 4) if e["ms_per_step"] > 0 else None
        e["ms_per_step"] = round(e["ms_per_step"], 3)
        e["lower_bound_ms"] = round(e["lower_bound_ms"], 4)
    out["bounds"] = {"score": "tensor (sustained bf16)", "select_compact": "HBM (scores + indices + 2x payload)",
                     "exchange": f"NVLink {NVLINK_GBS:.0f} GB/s per direction, received bytes"
                                 + ("" if world > 1 else " (N = 1: no exchange, the slots are written in place)"),
                     "attn_*": "tensor (sustained bf16), useful mask-counted FLOPs"}
    if world > 1 and "exchange" in out and out["exchange"]["ms_per_step"] > 0:
        out["exchange"]["nvlink_frac"] = round(recv * layers / (out["exchange"]["ms_per_step"] / 1e3)
                                               / (NVLINK_GBS * 1e9), 4)
    return out


def run_e2e(args, cfg, pr, sets, weights, layers, hosts, dev, world, local_rank, barrier):
    """Same hot path, inputs streamed from pinned host memory every layer (prefetched on a copy
    stream one layer ahead, continuing across steps) and every step's last-layer outputs read back
    to the host on their own stream."""
    import torch.distributed as dist
    # Each document row crosses PCIe once per layer.  Hosts >= 1 share the anchor (the document's
    # first l_a rows; l_q = 0): it is uploaded once per rank (with host 0's block when
    # this rank owns host 0, else into the first anchored host) and duplicated on the device.
    L_A = cfg.l_q + cfg.l_a
    share_anchor = cfg.l_q == 0 and 0 < L_A <= cfg.n // pr.base.H
    anchored = [h for h in hosts if h > 0]
    carrier = None
    if share_anchor and anchored:
        carrier = 0 if 0 in hosts else anchored[0]
    pinned = {}
    for h in hosts:
        x = sets[0][h]
        r0 = L_A if (share_anchor and h > 0 and h != carrier) else 0
        pinned[h] = tuple(t[r0:].cpu().pin_memory() for t in (x.q, x.k, x.v))
    out_host = {h: torch.empty(sets[0][h].out.shape, dtype=torch.bfloat16).pin_memory() for h in hosts}
    h2d_layer = sum(t.numel() * t.element_size() for h in hosts for t in pinned[h])
    d2h = sum(t.numel() * t.element_size() for t in out_host.values())
    copy = torch.cuda.Stream(device=dev)
    d2h_stream = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    read = [torch.cuda.Event(), torch.cuda.Event()]
    for e in done + read:
        e.record(main)
    # own output buffers per buffer set, so a step's D2H (on its own stream) overlaps the next
    # step's first layers instead of serialising with them
    from paper_2502_12085_b200.prefill import HostIO
    sets = [{h: HostIO(q=x.q, k=x.k, v=x.v, out=torch.empty_like(x.out), lse=x.lse) for h, x in st.items()}
            for st in sets]

    def upload(s):
        copy.wait_event(done[s])
        with torch.cuda.stream(copy):
            for h in hosts:
                x = sets[s][h]
                for dst, src in zip((x.q, x.k, x.v), pinned[h]):
                    dst[dst.shape[0] - src.shape[0]:].copy_(src, non_blocking=True)
            if carrier is not None:  # the anchor rows of the other hosts, device to device
                src = sets[s][carrier]
                for h in anchored:
                    if h != carrier:
                        for dst_t, src_t in ((sets[s][h].q, src.q), (sets[s][h].k, src.k), (sets[s][h].v, src.v)):
                            dst_t[:L_A].copy_(src_t[:L_A], non_blocking=True)
        copied[s].record(copy)

    def run(n_steps):
        # layers of consecutive steps form one stream of uploads: layer l+1's inputs (the next
        # step's layer 0 after the last layer) are copied while layer l computes
        total = n_steps * layers
        upload(0)
        for g in range(total):
            l, s = g % layers, g % 2
            if g + 1 < total:
                upload((g + 1) % 2)
            main.wait_event(copied[s])
            main.wait_event(read[s])  # set s's outputs of an earlier step are on the host
            pr.layer(sets[s], weights[l], overlap=not args.no_overlap, layer_idx=l)
            done[s].record(main)
            if l == layers - 1:  # this step's result back to the host, off the compute stream
                d2h_stream.wait_event(done[s])
                with torch.cuda.stream(d2h_stream):
                    for h in hosts:
                        out_host[h].copy_(sets[s][h].out, non_blocking=True)
                read[s].record(d2h_stream)

    run(1)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(main)
    run(args.e2e_steps)
    main.wait_stream(d2h_stream)  # the last step's result is on the host inside the timed region
    ev1.record(main)
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cpu" if args.same_device else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    return {"value": cfg.n * args.e2e_steps / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d_layer * layers,
            "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "how": "pinned host Q/K/V -> H2D every layer on a copy stream (one layer ahead, continuing across "
                   "steps; each document row once, the shared anchor rows duplicated device to device) -> libapb "
                   "hot path -> D2H of every step's last-layer attention output, all inside the timed region "
                   "(per-rank volumes)"}


if __name__ == "__main__":
    main()
