"""APB decode step (Alg. apb_decode) for the hosts one rank owns.

Per layer:  every owned host h -> apb_decode_attention (partial A_h, lse_h over its block KV cache;
the last host also over the new tokens' own keys) written into its slot of a packed
partials buffer [H][t*hq*d + t*hq] (fp32) -> apb_exchange_partials (Gather; one in-place
AllGather) -> apb_merge_partials (MergeScore) -> the same bf16 A [t][hq][d] on every rank.
Appending the new K/V to the last host's cache (Alg. apb_infer) is the caller's job.
"""
from __future__ import annotations

import torch

from . import apb


class DecodeRank:
    def __init__(self, H: int, hosts: list[int], t_new: int, n_heads: int, n_kv_heads: int, head_dim: int,
                 comm: apb.Comm | None = None, device="cuda", softmax_scale: float = 0.0,
                 batch_hosts: bool = True, fuse_merge: bool = True):
        """batch_hosts: with several owned hosts, one apb_decode_attention_hosts call (one
        streaming launch + one fold) instead of one apb_decode_attention per host.  fuse_merge:
        when this single rank holds every host, apb_decode_step_hosts (the streaming launch and
        MergeScore over all hosts' splits, no per-host partials): 0.122 ms per L8 step against
        0.124 ms for the per-host fold + MergeScore."""
        self.H, self.hosts, self.t = H, list(hosts), t_new
        self.hq, self.hk, self.d = n_heads, n_kv_heads, head_dim
        self.comm, self.scale, self.batch_hosts, self.fuse_merge = comm, softmax_scale, batch_hosts, fuse_merge
        nr = comm.nranks if comm is not None else 1
        self.contiguous = self.hosts == list(range(self.hosts[0], self.hosts[0] + len(self.hosts)))
        self.cyclic = nr > 1 and not self.contiguous
        if self.cyclic and self.hosts != list(range(self.hosts[0], H, nr)):
            raise ValueError("owned hosts must be a contiguous block or the cyclic set r, r+N, ...")
        if nr == 1 and sorted(self.hosts) != list(range(H)):
            raise ValueError("a single rank must own every host")
        self.device = torch.device(device)
        self.rows = t_new * n_heads
        # floats per host: O [rows][d] then lse [rows], padded to 16 B so every slot stays aligned
        self.slot = (self.rows * head_dim + self.rows + 3) // 4 * 4
        self.parts = torch.zeros((H, self.slot), dtype=torch.float32, device=self.device)
        self.ws = {}

    def dims(self, h: int, cache_len: int) -> apb.DecodeDims:
        return apb.DecodeDims(self.H, h, self.t, cache_len, self.hq, self.hk, self.d, self.scale)

    def step(self, q, caches: dict, k_new, v_new, out, out_lse=None, stream=None) -> None:
        """q: [t][hq][d] bf16 (same on every host); caches: {host: (k_cache, v_cache)} for the owned
        hosts ([c_h][hk][d] bf16); k_new/v_new: [t][hk][d] bf16; out: [t][hq][d] bf16."""
        single = self.comm is None or self.comm.nranks == 1
        if self.batch_hosts and self.fuse_merge and single and self.hosts == list(range(self.H)):
            # every host on this rank: one streaming launch + MergeScore over all hosts' splits,
            # straight into out (no per-host partials, nothing to gather)
            kcs, vcs = [caches[h][0] for h in self.hosts], [caches[h][1] for h in self.hosts]
            d = self.dims(0, 0)
            n = apb.decode_hosts_workspace_size(d, [k.shape[0] for k in kcs])
            if self.ws.get("batch") is None or self.ws["batch"].numel() < n:
                self.ws["batch"] = torch.zeros(max(n, 16), dtype=torch.uint8, device=self.device)
            apb.decode_step_hosts(d, q, kcs, vcs, k_new, v_new, out, out_lse, self.ws["batch"], stream=stream)
            return
        if len(self.hosts) > 1 and self.batch_hosts and self.contiguous:
            # every owned host's partial in one streaming launch + one fold (same partials up to
            # the split plan's fp32 summation order)
            h0 = self.hosts[0]
            kcs, vcs = [caches[h][0] for h in self.hosts], [caches[h][1] for h in self.hosts]
            d = self.dims(h0, 0)
            n = apb.decode_hosts_workspace_size(d, [k.shape[0] for k in kcs])
            if self.ws.get("batch") is None or self.ws["batch"].numel() < n:
                self.ws["batch"] = torch.zeros(max(n, 16), dtype=torch.uint8, device=self.device)
            last_owned = self.H - 1 in self.hosts
            apb.decode_attention_hosts(d, q, kcs, vcs, k_new if last_owned else None, v_new if last_owned else None,
                                       self.parts[h0: h0 + len(self.hosts)], self.rows * self.d, self.ws["batch"],
                                       stream=stream)
        else:
            for h in self.hosts:
                kc, vc = caches[h]
                d = self.dims(h, kc.shape[0])
                n = apb.decode_workspace_size(d)
                if self.ws.get(h) is None or self.ws[h].numel() < n:
                    self.ws[h] = torch.zeros(max(n, 16), dtype=torch.uint8, device=self.device)
                slot = self.parts[h]
                apb.decode_attention(d, q, kc, vc, k_new if h == self.H - 1 else None,
                                     v_new if h == self.H - 1 else None, slot[: self.rows * self.d],
                                     slot[self.rows * self.d:], self.ws[h], stream=stream)
        if self.cyclic:  # host h's partial sits in slot h; H/N rounds of one slot per rank
            apb.exchange_partials_cyclic(self.comm, self.H, self.slot, self.parts, stream=stream)
        else:
            per_rank = self.slot * (self.H // (self.comm.nranks if self.comm else 1))
            apb.exchange_partials(self.comm, per_rank, self.parts, stream=stream)
        apb.merge_partials(self.H, self.rows, self.d, self.parts, self.slot, self.parts[:, self.rows * self.d:],
                           self.slot, out, out_lse, stream=stream)
