"""APB prefill hot path for the hosts one rank owns — stream/event orchestration over libapb.

Alg. apb_prefill per layer, for every host h this rank owns:

    side stream:  apb_retain_score(h) -> apb_select_topk(h) (writes gathered[h] in place)
                  -> apb_exchange_passing (one NCCL AllGather of all slots)  -> event E
    main stream:  apb_attention_fwd(h, LOCAL)   (anchor rows + local rows over anchor/local
                                                 keys: overlaps the side stream)
                  wait E -> apb_attention_fwd(h, PASSING)  (local rows over the passing keys,
                                                 merged with the LOCAL partial by LSE)

With a single rank (all hosts on this GPU) the exchange is just the slot layout, so each host
runs one APB_PHASE_ALL launch as soon as the side stream has compressed hosts < h.

With H hosts over N ranks (N = H is the paper's deployment, one host per GPU; N < H emulates
several hosts per GPU) rank r owns either the contiguous block [r*H/N, (r+1)*H/N) or, work-balanced,
the cyclic set r, r+N, r+2N, ... (hosts_of_rank); the exchange follows the ownership.  Everything numeric runs
in libapb; this module only allocates buffers and orders launches.
"""
from __future__ import annotations

import dataclasses

import torch

from . import apb


@dataclasses.dataclass
class HostIO:
    """One host's per-layer tensors (device): q [L_A+l_b][hq][d], k/v [L_A+l_b][hk][d] bf16;
    out like q; lse fp32 [hq][L_A+l_b] or None."""
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    out: torch.Tensor
    lse: torch.Tensor | None = None


class PrefillRank:
    def __init__(self, base: apb.Dims, hosts: list[int], comm: apb.Comm | None = None,
                 device: torch.device | str = "cuda", skip_unused_last: bool = False,
                 split_phases: bool | None = None, compressor: str = "retain", shared_set: bool = False,
                 seed: int = 0, same_device: bool = False, peers: "apb.Peers | None" = None,
                 batched: bool = False):
        """base: problem dims (its `host` field is ignored); hosts: host indices this rank owns
        (contiguous, in order).  skip_unused_last: do not score/select host H-1 — its
        compressed block is ignored by every host, so outputs are unchanged.
        split_phases: LOCAL/PASSING launches around the exchange (default: only when a multi-rank
        communicator is given; a single rank uses one ordered APB_PHASE_ALL launch per host).
        compressor: "retain" (retaining heads R) or "random" (the "Rd." selector of
        Table 4, seeded by `seed` and the layer index); shared_set: one index set per host, the
        max over KV heads instead of per-KV-head sets (reading G3).
        same_device: debug only — allow owning a strict subset of the hosts WITHOUT a multi-rank
        communicator (the passing slots of hosts owned elsewhere are then never filled, so the
        outputs are not APB's; used to exercise the N > 1 schedule on one GPU).
        peers: an opened apb.Peers — the exchange over peer memory (CUDA IPC) instead of NCCL: the
        compaction pushes every selected row into every rank's buffer (apb_select_topk_peers), the
        PASSING launch waits for its slots on the device, then releases the buffer (two buffers
        alternate by layer).  Implies the LOCAL / PASSING split.
        batched: every attention phase of the owned hosts is ONE launch (apb_attention_fwd_hosts,
        heaviest host first) instead of one launch per host, and so are their scoring
        (apb_retain_score_hosts) and selection (apb_select_topk_hosts).  The single-rank schedule then
        compresses every host first (scoring + selection on the main stream) and runs the whole
        layer's attention as one launch with the GPU to itself; the split schedule runs one LOCAL
        and one PASSING launch."""
        if compressor not in ("retain", "random"):
            raise ValueError(f"compressor must be 'retain' or 'random', not {compressor!r}")
        self.compressor, self.shared_set, self.seed = compressor, shared_set, seed
        self.base, self.hosts, self.comm = base, list(hosts), comm
        self.device = torch.device(device)
        self.skip_unused_last = skip_unused_last
        self.peers, self.epoch = peers, 0
        if peers is not None and comm is not None:
            raise ValueError("pass either a NCCL communicator or peers, not both")
        if split_phases is None:
            split_phases = peers is not None or (comm is not None and comm.nranks > 1)
        self.split_phases = split_phases
        nr = comm.nranks if comm is not None else (peers.nranks if peers is not None else 1)
        if nr > 1 and not self.split_phases:
            # the ordered one-pass schedule waits only on this rank's own slot events, never on
            # the AllGather that fills the other ranks' slots: it is a single-rank schedule
            raise ValueError("split_phases=False (the ordered schedule) needs a single rank; "
                             "a multi-rank communicator requires the LOCAL/PASSING split")
        if nr == 1 and sorted(self.hosts) != list(range(base.H)) and not same_device:
            raise ValueError(f"hosts {self.hosts} are a strict subset of range(H={base.H}) but there is no "
                             "multi-rank communicator to fill the other hosts' passing slots")
        self.same_device = same_device
        self.batched = batched
        self.cyclic = nr > 1 and nr < base.H and self.hosts == list(range(self.hosts[0], base.H, nr))
        if nr > 1 and not self.cyclic and self.hosts != list(range(self.hosts[0], self.hosts[0] + len(self.hosts))):
            raise ValueError("owned hosts must be a contiguous block or the cyclic set r, r+N, ...")
        b = base
        lpp, hk, hq, d = b.l_pp, b.n_kv_heads, b.n_heads, b.head_dim
        if peers is not None:  # two library-owned buffers, alternated by layer parity
            self.peer_gathered = [peers.gathered(0), peers.gathered(1)]
            self.gathered = self.peer_gathered[0]
        else:
            self.gathered = torch.zeros((b.H, 2, hk, lpp, d), dtype=torch.bfloat16, device=self.device)
        self.scores = {h: torch.empty((hk, b.l_b), dtype=torch.float32, device=self.device) for h in hosts}
        self.indices = {h: torch.empty((hk, max(lpp, 1)), dtype=torch.int32, device=self.device) for h in hosts}
        self.ws = {}
        self.score_ws = {}  # retaining-head partial sums, sized by the weights on first use
        for h in hosts:
            n = apb.workspace_size(b.with_host(h), apb.WS_ATTENTION)
            self.ws[h] = torch.empty(max(n, 16), dtype=torch.uint8, device=self.device) if n else None
        # high priority: the side stream's scoring / selection / NCCL CTAs are scheduled ahead of
        # the main stream's queued attention CTAs, so the exchange completes while LOCAL runs
        self.side = torch.cuda.Stream(device=self.device, priority=-1)
        # per-op timing (bench breakdown): a list receives (op, host, start, end) CUDA-event
        # tuples recorded on the stream each op is launched on; None = no events
        self.trace: list | None = None
        self.ev_exchanged = torch.cuda.Event()
        self.ev_slot = {h: torch.cuda.Event() for h in hosts}

    def dims(self, h: int) -> apb.Dims:
        return self.base.with_host(h)

    def _op(self, name: str, h, stream, fn) -> None:
        """h: the host of the op, a list of hosts (one batched launch) or -1 (all / none)."""
        if self.trace is None:
            return fn()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        self.trace.append((name, h, a, b))

    def _compress_host(self, h: int, io: dict[int, HostIO], weights, layer_idx: int, stream) -> None:
        """Steps 1-2 for host h: scores (compressor) -> top-l_p indices -> gathered[h] (in place)."""
        d, x = self.dims(h), io[h]
        if self.compressor == "random":
            self._op("score", h, stream, lambda: apb.random_scores(d, self.seed, layer_idx, self.scores[h],
                                                                   stream=stream))
        else:
            n = apb.retain_workspace_size(d, weights)
            if self.score_ws.get(h) is None or self.score_ws[h].numel() < n:
                self.score_ws[h] = torch.empty(max(n, 16), dtype=torch.uint8, device=self.device)
            self._op("score", h, stream, lambda: apb.retain_score(d, weights, x.q, x.k, x.v, self.scores[h],
                                                                  stream=stream, ws=self.score_ws[h]))
        if self.shared_set:
            apb.share_scores(d, self.scores[h], stream=stream)
        if self.peers is not None:  # select + compaction pushed into every rank's buffer
            self._op("select_compact", h, stream, lambda: self.peers.select_topk(d, self.scores[h], x.k, x.v,
                                                                                 self.indices[h], self.epoch,
                                                                                 stream=stream))
            return
        self._op("select_compact", h, stream, lambda: apb.select_topk(d, self.scores[h], x.k, x.v, self.indices[h],
                                                                      self.gathered[h], stream=stream))

    def _compresses(self, h: int) -> bool:
        return self.base.l_pp > 0 and not (self.skip_unused_last and h == self.base.H - 1)

    def compress(self, io: dict[int, HostIO], weights: apb.RetainWeights | None, stream=None,
                 layer_idx: int = 0) -> None:
        """Steps 1-2 for every owned host (batched: one scoring launch and one select launch pair
        for up to 8 hosts at a time)."""
        hs_all = [h for h in self.hosts if self._compresses(h)]
        if not self.batched or self.peers is not None or self.compressor != "retain" or self.shared_set:
            for h in hs_all:
                self._compress_host(h, io, weights, layer_idx, stream)
            return
        for c in range(0, len(hs_all), 8):
            hs = hs_all[c:c + 8]
            ds = [self.dims(h) for h in hs]
            n = apb.retain_workspace_size(ds[0], weights) * len(hs)
            if self.score_ws.get("batch") is None or self.score_ws["batch"].numel() < n:
                self.score_ws["batch"] = torch.empty(max(n, 16), dtype=torch.uint8, device=self.device)
            self._op("score", hs, stream, lambda: apb.retain_score_hosts(
                ds, weights, [io[h].q for h in hs], [io[h].k for h in hs], [io[h].v for h in hs],
                [self.scores[h] for h in hs], self.score_ws["batch"], stream=stream))
            self._op("select_compact", hs, stream, lambda: apb.select_topk_hosts(
                ds, [self.scores[h] for h in hs], [io[h].k for h in hs], [io[h].v for h in hs],
                [self.indices[h] for h in hs], [self.gathered[h] for h in hs], stream=stream))

    def exchange(self, stream=None) -> None:
        """Step 3: in-place AllGather(s) of the packed [2][hk][l_p'][d] slots (with peers the
        exchange already happened inside the compaction)."""
        if self.peers is not None:
            return
        self._op("exchange", -1, stream, lambda: apb.exchange_passing(self.comm, self.base, self.gathered,
                                                                      stream=stream, cyclic=self.cyclic))

    def attention(self, io: dict[int, HostIO], phase: int, stream=None) -> None:
        name = {apb.PHASE_ALL: "attn_all", apb.PHASE_LOCAL: "attn_local", apb.PHASE_PASSING: "attn_passing"}[phase]
        if self.batched:
            for c in range(0, len(self.hosts), 8):  # at most 8 hosts per launch
                hs = self.hosts[c:c + 8]
                self._op(name, hs, stream, lambda: apb.attention_fwd_hosts(
                    [self.dims(h) for h in hs], [io[h].q for h in hs], [io[h].k for h in hs], [io[h].v for h in hs],
                    self.gathered, [io[h].out for h in hs], [io[h].lse for h in hs], phase=phase,
                    ws=[self.ws[h] for h in hs], stream=stream))
            return
        for h in self.hosts:
            x = io[h]
            self._op(name, h, stream, lambda: apb.attention_fwd(self.dims(h), x.q, x.k, x.v, self.gathered, x.out,
                                                                x.lse, phase=phase, ws=self.ws[h], stream=stream))

    def layer(self, io: dict[int, HostIO], weights: apb.RetainWeights | None, overlap: bool = True,
              events: list | None = None, layer_idx: int = 0) -> None:
        """One layer of the hot path for all owned hosts, enqueued on the current stream.
        events: if a list is given, (start, end) timing-event pairs bracketing the attention
        launches on the main stream are appended to it (the bench's in-situ kernel time)."""
        main = torch.cuda.current_stream(self.device)

        def timed(fn):
            if events is None:
                return fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main)
            fn()
            b.record(main)
            events.append((a, b))

        if not overlap or (self.batched and not self.split_phases):
            self.compress(io, weights, main, layer_idx)
            self.exchange(main)
            timed(lambda: self.attention(io, apb.PHASE_ALL, main))
            return
        if not self.split_phases:
            # Every host lives on this GPU: the "exchange" is the in-place slot layout itself, so
            # host h's one-pass attention only has to wait for the compressed blocks of hosts
            # < h (side stream, one event per host) — no LOCAL/PASSING split, no fp32 partial.
            self.side.wait_stream(main)
            for h in self.hosts:
                if self._compresses(h):
                    self._compress_host(h, io, weights, layer_idx, self.side)
                self.ev_slot[h].record(self.side)
            self.exchange(self.side)  # no-op without a communicator
            for h in self.hosts:
                if h > self.hosts[0]:
                    main.wait_event(self.ev_slot[h - 1])
                x = io[h]
                timed(lambda: self._op("attn_all", h, main, lambda: apb.attention_fwd(
                    self.dims(h), x.q, x.k, x.v, self.gathered, x.out, x.lse, phase=apb.PHASE_ALL, ws=self.ws[h],
                    stream=main)))
            main.wait_stream(self.side)  # the last host's compression still reads io[h].k/v
            return
        if self.peers is not None:
            self.epoch += 1
            self.gathered = self.peer_gathered[self.epoch & 1]
        self.side.wait_stream(main)  # this layer's inputs are produced on the main stream
        self.compress(io, weights, self.side, layer_idx)
        self.exchange(self.side)
        self.ev_exchanged.record(self.side)
        timed(lambda: self.attention(io, apb.PHASE_LOCAL, main))
        if self.peers is not None:
            # device-side wait for the slots this rank's hosts read (hosts < max owned host)
            self.peers.wait(max(self.hosts), self.epoch, stream=main)
        else:
            main.wait_event(self.ev_exchanged)
        timed(lambda: self.attention(io, apb.PHASE_PASSING, main))
        if self.peers is not None:
            self.peers.release(self.epoch, stream=main)
        # the side stream's buffers (scores, gathered) are reused next layer only after main
        # has consumed them: next layer's side.wait_stream(main) orders that.  Conversely the
        # caller may overwrite io's Q/K/V once main is past this point.
        main.wait_stream(self.side)


def hosts_of_rank(H: int, world: int, rank: int, layout: str = "block") -> list[int]:
    """Hosts rank `rank` of `world` owns: "block" = [rank*H/world, (rank+1)*H/world); "cyclic" =
    rank, rank+world, ... — balances the per-rank attention work, which grows with the host index
    (host h attends to h*l_p' passing keys), e.g. L8-128K, N = 2: 22.5 vs 25.8 TFLOP per layer on
    the busiest rank; N = 4: 12.4 vs 14.0."""
    if H % world:
        raise ValueError(f"world size {world} must divide H={H}")
    if layout == "cyclic":
        return list(range(rank, H, world))
    if layout != "block":
        raise ValueError(f"layout must be 'block' or 'cyclic', not {layout!r}")
    per = H // world
    return list(range(rank * per, (rank + 1) * per))
