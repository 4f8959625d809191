"""libapb's tcgen05 GEMM (apb_gemm): the fused epilogues are bit-identical to the unfused steps
they replace (STORE GEMM + apb_rope, STORE GEMM + apb_swiglu), across tile tails, head sizes and
position sources; plus determinism.  The product itself is checked against fp64 in
tests/test_gpu_model.py::test_gemm (P:708 qkv_proj, P:730 FFN)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_12085_b200 import apb, build
    build.build()
    apb.load()


def _rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return (torch.randn(shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,heads_rot,heads_all,d,pos", [(300, 6, 8, 128, "offset"), (257, 5, 7, 64, "array"),
                                                         (1024, 40, 48, 128, "offset"), (77, 2, 2, 64, "offset")])
def test_rope_epilogue_equals_gemm_then_rope(M, heads_rot, heads_all, d, pos):
    from paper_2502_12085_b200 import apb
    K = 512
    N = heads_all * d
    a, w = _rand((M, K), 1), _rand((N, K), 2, K ** -0.5)
    positions = None
    off = 0
    if pos == "array":
        positions = torch.randint(0, 1 << 20, (M,), device="cuda", dtype=torch.int32)
    else:
        off = 4096
    ref = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    apb.gemm(a, w, ref, apb.EPI_STORE)
    apb.rope(ref, heads_rot, d, 500000.0, positions=positions, pos_offset=off)
    out = torch.empty_like(ref)
    apb.gemm(a, w, out, apb.EPI_ROPE, rope_cols=heads_rot * d, head_dim=d, theta=500000.0, positions=positions,
             pos_offset=off)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("M,inter,K", [(300, 512, 256), (129, 1024, 4096), (1000, 14336 // 4, 1024)])
def test_swiglu_epilogue_equals_gemm_then_swiglu(M, inter, K):
    from paper_2502_12085_b200 import apb
    a, w = _rand((M, K), 3), _rand((2 * inter, K), 4, K ** -0.5 * 3)
    gu = torch.empty((M, 2 * inter), dtype=torch.bfloat16, device="cuda")
    apb.gemm(a, w, gu, apb.EPI_STORE)
    ref = torch.empty((M, inter), dtype=torch.bfloat16, device="cuda")
    apb.swiglu(gu, ref)
    out = torch.full_like(ref, float("nan"))
    apb.gemm(a, apb.interleave_gate_up(w), out, apb.EPI_SWIGLU)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def test_residual_in_place_strided_and_deterministic():
    """RESIDUAL writes C in place through a row-strided view and leaves the other columns alone;
    two runs are bit-identical."""
    from paper_2502_12085_b200 import apb
    M, N, K = 513, 256, 1024
    a, w = _rand((M, K), 5), _rand((N, K), 6, K ** -0.5)
    base = _rand((M, N + 64), 7)
    outs = []
    for _ in range(2):
        c = base.clone()
        apb.gemm(a, w, c[:, 32:32 + N], apb.EPI_RESIDUAL, beta=1.0)
        outs.append(c)
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    assert torch.equal(outs[0][:, :32], base[:, :32]) and torch.equal(outs[0][:, 32 + N:], base[:, 32 + N:])
    prod = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    apb.gemm(a, w, prod, apb.EPI_STORE)
    ref = (base[:, 32:32 + N].float() + prod.float()).to(torch.bfloat16)  # bf16(C + bf16(AW^T)), G20
    assert torch.equal(outs[0][:, 32:32 + N].view(torch.int16), ref.view(torch.int16))
