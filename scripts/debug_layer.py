"""Step-by-step error of the post-attention half of the APB layer (diagnostic)."""
import numpy as np
import torch

import synth
from oracle import layer as OL
from paper_2502_12085_b200 import apb

torch.manual_seed(0)
cfg = synth.CONFIGS["toy"]
hidden, inter = 256, 512
mw = synth.model_weights(cfg, 0, hidden, inter)
W = {k: synth.bf16_bits_to_f64(v) for k, v in mw.items()}
dev = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()
f64 = lambda t: t.float().cpu().double().numpy()
xb = synth.host_hidden(cfg, 0, hidden)
x = synth.bf16_bits_to_f64(xb)
rows = x.shape[0]
attn = OL.bf16(np.random.default_rng(1).standard_normal((rows, cfg.hq * cfg.d)) * 0.5)
xt, at = dev(xb), dev(synth.f32_to_bf16_bits(attn.astype(np.float32)))
wt = {k: dev(v) for k, v in mw.items()}


def ulps(got, ref):
    u = np.maximum(np.abs(ref), 1e-30)
    e = np.abs(got - ref) / (2.0 ** (np.floor(np.log2(u)) - 7))
    return f"max {e.max():.2f} ulp, >1ulp {np.mean(e > 1.0) * 100:.2f}%"


apb.gemm_bf16(at, wt["w_o"], xt, beta=1.0)
x1g = f64(xt)
x1r = OL.bf16(x + attn @ W["w_o"].T)
print("x1 (residual add 1):", ulps(x1g, x1r))
hb = torch.empty_like(xt)
apb.rmsnorm(xt, wt["ffn_norm"], 1e-5, hb)
h2g = f64(hb)
print("h2 from gpu x1:", ulps(h2g, OL.bf16(OL.rmsnorm(x1g, W["ffn_norm"], 1e-5))))
gu = torch.empty((rows, 2 * inter), dtype=torch.bfloat16, device="cuda")
apb.gemm_bf16(hb, wt["w_gu"], gu)
gug = f64(gu)
print("gu from gpu h2:", ulps(gug, OL.bf16(h2g @ W["w_gu"].T)))
act = torch.empty((rows, inter), dtype=torch.bfloat16, device="cuda")
apb.swiglu(gu, act)
actg = f64(act)
print("act from gpu gu:", ulps(actg, OL.bf16(OL.swiglu(gug, inter))))
apb.gemm_bf16(act, wt["w_down"], xt, beta=1.0)
outg = f64(xt)
outr = OL.bf16(x1g + actg @ W["w_down"].T)
print("out from gpu x1, act:", ulps(outg, outr))
prod = actg @ W["w_down"].T
print("  |x1| mean", np.abs(x1g).mean(), " |ffn branch| mean", np.abs(prod).mean())
two = OL.bf16(x1g + OL.bf16(prod))
print("  two-rounding model:", ulps(outg, two), " exact-match", np.mean(outg == two) * 100, "%")
