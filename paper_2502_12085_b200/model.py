"""APB prefill of a Llama-style decoder stack around the hot path.

Alg. apb_prefill per layer and host, every step a libapb call:

    h = RMSNorm(x)                    apb_rmsnorm
    qkv = RoPE_QK(h W_qkv^T)          apb_gemm, ROPE epilogue     (P:708 qkv_proj; positions = local
                                                                   row index, G19)
    hot path                          PrefillRank.layer  (scores, top-l_p, AllGather, attention)
    x += O W_o^T                      apb_gemm, RESIDUAL epilogue (in place)
    h = RMSNorm(x)                    apb_rmsnorm
    a = SiLU(h W_g^T) * (h W_u^T)     apb_gemm, SWIGLU epilogue   (gate/up rows interleaved)   (P:730 FFN)
    x += a W_down^T                   apb_gemm, RESIDUAL epilogue

Every GEMM is libapb's tcgen05 kernel.  fused=False runs the same steps unfused (STORE GEMM +
apb_rope, STORE GEMM + apb_swiglu) — the step-wise parity tests check each step that way, and
the fused epilogues are tested bit-identical to it.

Q, K and V are strided views into one [rows][hq+2hk][d] buffer per host: the projection writes
it once, RoPE rotates Q and K in place, and the hot path reads it through its row strides (the
scoring kernel's A operand x_t = [Q_t | K_t | V_t] is literally the qkv row).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import apb
from .prefill import HostIO, PrefillRank


@dataclass
class ModelShape:
    hidden: int
    inter: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    eps: float = 1e-5
    theta: float = 500000.0  # Llama-3.1 rope_theta (public model card)


@dataclass
class LayerWeights:
    """bf16 device tensors in nn.Linear layout [out][in]: w_qkv = [W_q; W_k; W_v]
    [(hq+2hk)d][hidden], w_o [hidden][hq d], w_gu = [W_gate; W_up] [2I][hidden],
    w_down [hidden][I]; norms bf16 [hidden]; retain: the layer's retaining head (None with the
    random compressor)."""
    attn_norm: torch.Tensor
    w_qkv: torch.Tensor
    w_o: torch.Tensor
    ffn_norm: torch.Tensor
    w_gu: torch.Tensor
    w_down: torch.Tensor
    retain: apb.RetainWeights | None = None
    w_gu_il: torch.Tensor | None = None  # w_gu with gate/up rows interleaved (apb.interleave_gate_up), lazily

    def gate_up_interleaved(self) -> torch.Tensor:
        if self.w_gu_il is None:
            self.w_gu_il = apb.interleave_gate_up(self.w_gu)
        return self.w_gu_il


class ApbModelRank:
    """The hosts of one rank running APB prefill of a decoder stack, one layer at a time."""

    def __init__(self, base: apb.Dims, shape: ModelShape, hosts: list[int], comm: apb.Comm | None = None,
                 device: torch.device | str = "cuda", fused: bool = True, **prefill_kw):
        self.base, self.shape, self.hosts, self.fused = base, shape, list(hosts), fused
        self.device = torch.device(device)
        self.hot = PrefillRank(base, hosts, comm, device, **prefill_kw)
        hq, hk, d = shape.n_heads, shape.n_kv_heads, shape.head_dim
        if (hq, hk, d) != (base.n_heads, base.n_kv_heads, base.head_dim):
            raise ValueError("ModelShape heads / head_dim must match the hot-path dims")
        bf = dict(dtype=torch.bfloat16, device=self.device)
        self.rows = {h: base.with_host(h).rows for h in hosts}
        self.qkv = {h: torch.empty((r, hq + 2 * hk, d), **bf) for h, r in self.rows.items()}
        self.attn = {h: torch.empty((r, hq, d), **bf) for h, r in self.rows.items()}
        self.io = {h: HostIO(q=self.qkv[h][:, :hq], k=self.qkv[h][:, hq:hq + hk], v=self.qkv[h][:, hq + hk:],
                             out=self.attn[h]) for h in hosts}
        mr = max(self.rows.values())
        self.hbuf = torch.empty((mr, shape.hidden), **bf)
        self.gu = None if fused else torch.empty((mr, 2 * shape.inter), **bf)  # unfused path only
        self.act = torch.empty((mr, shape.inter), **bf)

    def attn_in(self, h: int, x: torch.Tensor, lw: LayerWeights, stream=None) -> None:
        """qkv[h] <- RoPE(RMSNorm(x) W_qkv^T) for host h's rows [A; B_h]."""
        s, r = self.shape, self.rows[h]
        hb = self.hbuf[:r]
        apb.rmsnorm(x, lw.attn_norm, s.eps, hb, stream=stream)
        qkv2 = self.qkv[h].view(r, -1)
        if self.fused:
            apb.gemm(hb, lw.w_qkv, qkv2, apb.EPI_ROPE, rope_cols=(s.n_heads + s.n_kv_heads) * s.head_dim,
                     head_dim=s.head_dim, theta=s.theta, stream=stream)
        else:
            apb.gemm(hb, lw.w_qkv, qkv2, apb.EPI_STORE, stream=stream)
            apb.rope(qkv2, s.n_heads + s.n_kv_heads, s.head_dim, s.theta, stream=stream)

    def attn_out_ffn(self, h: int, x: torch.Tensor, lw: LayerWeights, stream=None) -> None:
        """x += O W_o^T;  x += SwiGLU(RMSNorm(x) W_gu^T) W_down^T   (in place)."""
        s, r = self.shape, self.rows[h]
        apb.gemm(self.attn[h].view(r, -1), lw.w_o, x, apb.EPI_RESIDUAL, beta=1.0, stream=stream)
        hb, act = self.hbuf[:r], self.act[:r]
        apb.rmsnorm(x, lw.ffn_norm, s.eps, hb, stream=stream)
        if self.fused:
            apb.gemm(hb, lw.gate_up_interleaved(), act, apb.EPI_SWIGLU, stream=stream)
        else:
            gu = self.gu[:r]
            apb.gemm(hb, lw.w_gu, gu, apb.EPI_STORE, stream=stream)
            apb.swiglu(gu, act, stream=stream)
        apb.gemm(act, lw.w_down, x, apb.EPI_RESIDUAL, beta=1.0, stream=stream)

    def layer(self, xs: dict[int, torch.Tensor], lw: LayerWeights, layer_idx: int = 0, overlap: bool = True,
              events: list | None = None) -> None:
        """One APB prefill layer for every owned host, in place on xs[h] ([rows][hidden] bf16),
        enqueued on the current stream."""
        for h in self.hosts:
            self.attn_in(h, xs[h], lw)
        self.hot.layer(self.io, lw.retain, overlap=overlap, events=events, layer_idx=layer_idx)
        for h in self.hosts:
            self.attn_out_ffn(h, xs[h], lw)
