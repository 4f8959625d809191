#!/usr/bin/env python
"""Time libapb's tcgen05 GEMM (apb_gemm, each fused epilogue) on the Llama-3.1-8B layer shapes of
one host (M = L_A + l_b = 20480 rows at 128K, H = 8) against torch.matmul (cuBLAS) on the same
operands.  Device time per launch, launches queued behind a GPU spin (no host overhead)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_12085_b200 import apb  # noqa: E402


def timed(fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=20480)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--square", type=int, default=0, help="also time an NxNxN STORE GEMM (e.g. 8192)")
    a = ap.parse_args()
    apb.load()
    if a.square:
        n = a.square
        g0 = torch.Generator(device="cuda")
        g0.manual_seed(1)
        A = torch.randn(n, n, generator=g0, device="cuda").to(torch.bfloat16)
        B = torch.randn(n, n, generator=g0, device="cuda").to(torch.bfloat16)
        C = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
        t_o = timed(lambda: apb.gemm(A, B, C, apb.EPI_STORE), a.iters)
        t_r = timed(lambda: torch.matmul(A, B.T), a.iters)
        f = 2.0 * n ** 3
        print(f"square {n}: apb {t_o:.3f} ms {f / t_o / 1e9:.1f} TF/s | cuBLAS {t_r:.3f} ms {f / t_r / 1e9:.1f} TF/s")
    M, H, I, hq, hk, d = a.rows, 4096, 14336, 32, 8, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    rnd = lambda *s, sc=1.0: (torch.randn(s, generator=g, device="cuda") * sc).to(torch.bfloat16)  # noqa: E731
    x = rnd(M, H)
    w_qkv, w_o, w_gu, w_down = rnd((hq + 2 * hk) * d, H, sc=H ** -0.5), rnd(H, hq * d, sc=(hq * d) ** -0.5), \
        rnd(2 * I, H, sc=H ** -0.5), rnd(H, I, sc=I ** -0.5)
    w_gu_il = apb.interleave_gate_up(w_gu)
    qkv = torch.empty(M, (hq + 2 * hk) * d, dtype=torch.bfloat16, device="cuda")
    attn = rnd(M, hq * d)
    act = rnd(M, I)
    res = rnd(M, H)
    cases = {
        "qkv+rope": (lambda: apb.gemm(x, w_qkv, qkv, apb.EPI_ROPE, rope_cols=(hq + hk) * d, head_dim=d,
                                      theta=5e5), lambda: torch.matmul(x, w_qkv.T), M * w_qkv.shape[0] * H),
        "o+residual": (lambda: apb.gemm(attn, w_o, res, apb.EPI_RESIDUAL, beta=1.0),
                       lambda: torch.matmul(attn, w_o.T), M * H * hq * d),
        "gate_up+swiglu": (lambda: apb.gemm(x, w_gu_il, act, apb.EPI_SWIGLU), lambda: torch.matmul(x, w_gu.T),
                           M * 2 * I * H),
        "down+residual": (lambda: apb.gemm(act, w_down, res, apb.EPI_RESIDUAL, beta=1.0),
                          lambda: torch.matmul(act, w_down.T), M * H * I),
    }
    out = {}
    tot_ours = tot_ref = tot_f = 0.0
    for name, (ours, ref, mnk) in cases.items():
        ours()
        ref()
        t_o, t_r = timed(ours, a.iters), timed(ref, a.iters)
        f = 2.0 * mnk
        out[name] = {"ms": round(t_o, 4), "tflops": round(f / t_o / 1e9, 1), "cublas_ms": round(t_r, 4),
                     "cublas_tflops": round(f / t_r / 1e9, 1)}
        tot_ours += t_o
        tot_ref += t_r
        tot_f += f
        print(f"{name:16s} apb {t_o:.3f} ms {f / t_o / 1e9:7.1f} TF/s | cuBLAS (no epilogue) {t_r:.3f} ms "
              f"{f / t_r / 1e9:7.1f} TF/s")
    out["layer"] = {"ms": round(tot_ours, 4), "tflops": round(tot_f / tot_ours / 1e9, 1), "cublas_ms": round(tot_ref, 4),
                    "cublas_tflops": round(tot_f / tot_ref / 1e9, 1), "rows": M}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
