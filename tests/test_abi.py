"""libapb C ABI: the library loads on a CPU-only box, exports every symbol include/apb.h declares,
and validates arguments synchronously (config / contract errors) before touching a GPU — and
fails loudly (APB_ERR_CUDA), never silently, when no GPU is present."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

from paper_2502_12085_b200 import apb
from paper_2502_12085_b200 import build as apb_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    apb_build.build()
    return apb.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "apb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apb_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert {"apb_retain_score", "apb_select_topk", "apb_exchange_passing", "apb_attention_fwd"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", apb.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (apb_\w+)", out))
    assert set(names) <= exported, set(names) - exported


def test_binary_is_sm100a_with_tcgen05_and_tma(lib):
    sass = subprocess.run(["cuobjdump", "-sass", apb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", apb.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA loads
    assert "LDTM" in sass and "STTM" in sass  # TMEM <-> registers
    # per function: the prefill kernels (attention, retaining heads) use tcgen05 only; the legacy
    # warp-level mma.sync appears only in the decode GEMV kernel (DESIGN 7b: M = t*g <= 16 rows)
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    assert funcs
    for f in funcs:
        name, body = f.split("\n", 1)
        legacy = "HMMA" in re.sub(r"UTCHMMA", "", body)
        if "attention_kernel" in name or "retain_score_kernel" in name:
            assert "UTCHMMA" in body and not legacy, name
        elif legacy:
            assert "decode_mma_kernel" in name, name
    # the decode streaming kernel's TMA instantiations (template flag true, mangled "Lb1E") read the
    # caches with TMA into an mbarrier ring; the cp.async ones (Lb0E) do not
    dec = [f for f in funcs if "decode_mma_kernel" in f.split("\n", 1)[0]]
    tma = [f for f in dec if "Lb1E" in f.split("\n", 1)[0]]
    assert tma and all("UTMALDG" in f and "SYNCS" in f for f in tma)
    assert all("UTMALDG" not in f for f in dec if "Lb0E" in f.split("\n", 1)[0])
    # the attention kernel stores its output tiles with TMA
    assert any("UTMASTG" in f for f in funcs if "attention_kernel" in f.split("\n", 1)[0])


def _dims(**kw):
    base = dict(n=2048, H=4, host=1, l_a=128, l_p=64, n_heads=4, n_kv_heads=2, head_dim=64)
    base.update(kw)
    return apb.Dims(**base)


def test_status_strings_and_version(lib):
    assert lib.apb_status_string(0) == b"APB_OK"
    assert lib.apb_status_string(5) == b"APB_ERR_NCCL"
    assert apb.version() >= 100


@pytest.mark.parametrize("kw,status", [
    (dict(H=0), apb.ERR_CONFIG),
    (dict(host=4), apb.ERR_CONFIG),
    (dict(host=-1), apb.ERR_CONFIG),
    (dict(l_b=500), apb.ERR_CONFIG),          # n != H * l_b (reading G15)
    (dict(n_heads=3), apb.ERR_CONFIG),        # not a multiple of n_kv_heads
    (dict(l_a=-1), apb.ERR_CONFIG),
    (dict(head_dim=96), apb.ERR_UNSUPPORTED),
])
def test_check_dims_rejects(lib, kw, status):
    with pytest.raises(apb.ApbError) as e:
        apb.check_dims(_dims(**kw))
    assert e.value.status == status


def test_check_dims_accepts_paper_configs(lib):
    apb.check_dims(_dims())
    apb.check_dims(apb.Dims(n=131072, H=8, host=7, l_a=4096, l_p=2048, n_heads=32, n_kv_heads=8, head_dim=128))
    apb.check_dims(apb.Dims(n=131072, H=1, host=0, l_a=4096, l_p=2048, n_heads=32, n_kv_heads=8, head_dim=128))


def test_workspace_sizes(lib):
    d = _dims(host=2)
    assert apb.workspace_size(d, apb.WS_ATTENTION) >= d.l_b * 4 * 64 * 4 + 4 * d.l_b * 4
    assert apb.workspace_size(_dims(host=0), apb.WS_ATTENTION) == 0   # host 1: no passing
    assert apb.workspace_size(_dims(l_p=0), apb.WS_ATTENTION) == 0    # l_p = 0: no passing
    assert apb.workspace_size(d, apb.WS_SELECT) == 0


class _FakeT:
    """Stands in for a device tensor: only data_ptr / stride / shape are read by the binding."""

    is_cuda = True

    def __init__(self, ptr, shape, elem=2, dtype=None, strides=None):
        self._p, self.shape = ptr, shape
        st, s = [], 1
        for x in reversed(shape):
            st.append(s)
            s *= x
        self._st = tuple(strides) if strides is not None else tuple(reversed(st))
        self._e = elem
        self.dtype = dtype or {2: torch.bfloat16, 4: torch.float32}[elem]

    def is_contiguous(self):
        return True

    def __getitem__(self, i):
        return _FakeT(self._p, self.shape[1:], self._e, self.dtype, self._st[1:])

    def data_ptr(self):
        return self._p

    def stride(self, i):
        return self._st[i]

    def dim(self):
        return len(self.shape)

    def numel(self):
        n = 1
        for x in self.shape:
            n *= x
        return n

    def element_size(self):
        return self._e


def test_contract_errors_before_any_gpu_work(lib):
    d = _dims(host=0)
    rows = d.rows
    q = _FakeT(0x10000, (rows, 4, 64)); k = _FakeT(0x20000, (rows, 2, 64)); v = _FakeT(0x30000, (rows, 2, 64))
    out = _FakeT(0x40000, (rows, 4, 64))
    # misaligned q
    with pytest.raises(apb.ApbError) as e:
        apb.attention_fwd(d, _FakeT(0x10002, (rows, 4, 64)), k, v, None, out, stream=0)
    assert e.value.status == apb.ERR_CONTRACT
    # NULL gathered although host > 0 and l_p > 0
    with pytest.raises(apb.ApbError) as e:
        apb.attention_fwd(_dims(host=1), q, k, v, None, out, stream=0)
    assert e.value.status == apb.ERR_CONTRACT
    # weights with the wrong d_in
    w = apb.RetainWeights(w1=_FakeT(0x50000, (1024, 100)), w2=_FakeT(0x60000, (4, 1024), 4))
    with pytest.raises(apb.ApbError) as e:
        apb.retain_score(d, w, q, k, v, _FakeT(0x70000, (2, 512), 4), stream=0)
    assert e.value.status == apb.ERR_CONFIG


def test_binding_validates_tensors_before_the_abi(lib):
    """apb.py checks what a raw pointer cannot carry: one shared K/V row stride,
    dtypes, and that every tensor covers the rows / widths `dims` implies."""
    d = _dims(host=0)
    rows = d.rows
    q = _FakeT(0x10000, (rows, 4, 64)); k = _FakeT(0x20000, (rows, 2, 64)); v = _FakeT(0x30000, (rows, 2, 64))
    out = _FakeT(0x40000, (rows, 4, 64))
    v_wide = _FakeT(0x30000, (rows, 2, 64), strides=(256, 64, 1))
    bad = [
        (q, k, v_wide, out, None),                                          # K/V row strides differ
        (_FakeT(0x10000, (rows, 4, 64), dtype=torch.float16), k, v, out, None),  # not bf16
        (_FakeT(0x10000, (rows - 1, 4, 64)), k, v, out, None),               # too few rows
        (q, _FakeT(0x20000, (rows, 1, 64)), v, out, None),                  # too few KV heads
        (q, k, v, _FakeT(0x40000, (rows, 2, 64)), None),                    # out too narrow
        (q, k, v, out, _FakeT(0x50000, (4, rows - 8), 4)),                  # lse too short
    ]
    for args in bad:
        with pytest.raises(apb.ApbError) as e:
            apb.attention_fwd(d, *args[:3], None, args[3], lse=args[4], stream=0)
        assert e.value.status == apb.ERR_CONTRACT
    with pytest.raises(apb.ApbError) as e:  # scores too small
        apb.select_topk(_dims(host=1), _FakeT(0x70000, (2, 100), 4), k, v, _FakeT(0x80000, (2, 64), 4, torch.int32),
                        _FakeT(0x90000, (2, 2, 64, 64)), stream=0)
    assert e.value.status == apb.ERR_CONTRACT


def test_exchange_plan(lib):
    """apb_exchange_plan: block = one round over contiguous per-rank slot ranges; cyclic = H/N
    rounds of one slot per rank; nothing to do for one rank or l_p = 0."""
    d = apb.Dims(n=131072, H=8, host=0, l_a=4096, l_p=2048, n_heads=32, n_kv_heads=8, head_dim=128)
    slot = 2 * 8 * 2048 * 128
    assert apb.exchange_plan(d, 1, 0) == []
    assert apb.exchange_plan(d.__class__(**{**d.__dict__, "l_p": 0}), 4, 1) == []
    assert apb.exchange_plan(d, 8, 3) == [(3 * slot, 0, slot)]
    assert apb.exchange_plan(d, 2, 1) == [(4 * slot, 0, 4 * slot)]
    assert apb.exchange_plan(d, 2, 1, apb.LAYOUT_CYCLIC) == [(k * 2 * slot + slot, k * 2 * slot, slot) for k in range(4)]
    assert apb.exchange_plan(d, 8, 5, apb.LAYOUT_CYCLIC) == [(5 * slot, 0, slot)]
    for bad, st in (((3, 0), apb.ERR_CONFIG), ((2, 2), apb.ERR_CONFIG), ((0, 0), apb.ERR_CONFIG)):
        with pytest.raises(apb.ApbError) as e:
            apb.exchange_plan(d, *bad)
        assert e.value.status == st
    with pytest.raises(apb.ApbError) as e:
        apb.exchange_plan(d, 2, 0, 7)
    assert e.value.status == apb.ERR_CONFIG


def test_comm_check_null_is_ok(lib):
    assert lib.apb_comm_check(None) == 0
    assert lib.apb_comm_abort(None) == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_fails_loudly_without_gpu(lib):
    d = _dims(host=0)
    rows = d.rows
    q = _FakeT(0x10000, (rows, 4, 64)); k = _FakeT(0x20000, (rows, 2, 64)); v = _FakeT(0x30000, (rows, 2, 64))
    with pytest.raises(apb.ApbError) as e:
        apb.attention_fwd(d, q, k, v, None, _FakeT(0x40000, (rows, 4, 64)), stream=0)
    assert e.value.status == apb.ERR_CUDA


def test_exchange_single_rank_is_noop(lib):
    # comm == NULL (one rank) is a legal no-op that never touches memory
    apb.exchange_passing(None, _dims(), _FakeT(0x10000, (4, 2, 2, 64, 64)), stream=0)


def test_peers_contract_errors(lib):
    """apb_peers_*: configuration errors before any allocation; unopened peers are rejected."""
    import ctypes as C
    h = C.c_void_p()
    buf = C.create_string_buffer(64)
    d = _dims().c()
    assert lib.apb_peers_create(C.byref(d), 9, 0, C.byref(h), buf) == apb.ERR_CONFIG   # > 8 ranks
    assert lib.apb_peers_create(C.byref(d), 3, 0, C.byref(h), buf) == apb.ERR_CONFIG   # 3 does not divide H = 4
    assert lib.apb_peers_create(C.byref(d), 2, 2, C.byref(h), buf) == apb.ERR_CONFIG   # rank out of range
    assert lib.apb_peers_wait(None, 1, 1, None) == apb.ERR_CONTRACT
    assert lib.apb_peers_release(None, 1, None) == apb.ERR_CONTRACT
    assert lib.apb_peers_destroy(None) == apb.OK


def test_attention_hosts_contract_errors_before_any_gpu_work(lib):
    """apb_attention_fwd_hosts validates every host before launching (no GPU needed): a repeated
    host and hosts whose dims differ beyond `host` are APB_ERR_CONFIG, a bad per-host pointer is
    APB_ERR_CONTRACT, n outside [1, 8] is rejected by the binding."""
    def qkvo(host, base=0x100000):
        d = _dims(host=host)
        r = d.rows
        return (d, _FakeT(base, (r, 4, 64)), _FakeT(base + 0x10000, (r, 2, 64)), _FakeT(base + 0x20000, (r, 2, 64)),
                _FakeT(base + 0x30000, (r, 4, 64)))
    a, b = qkvo(1), qkvo(2, 0x200000)
    g = _FakeT(0x300000, (4, 2, 2, 64, 64))
    with pytest.raises(apb.ApbError) as e:   # host 1 twice
        apb.attention_fwd_hosts([a[0], a[0]], [a[1], a[1]], [a[2], a[2]], [a[3], a[3]], g, [a[4], a[4]], stream=0)
    assert e.value.status == apb.ERR_CONFIG
    import dataclasses
    d2 = dataclasses.replace(b[0], l_a=b[0].l_a + 64)   # anchor length differs
    r2 = d2.rows
    with pytest.raises(apb.ApbError) as e:
        apb.attention_fwd_hosts([a[0], d2], [a[1], _FakeT(0x200000, (r2, 4, 64))],
                                [a[2], _FakeT(0x210000, (r2, 2, 64))], [a[3], _FakeT(0x220000, (r2, 2, 64))], g,
                                [a[4], _FakeT(0x230000, (r2, 4, 64))], stream=0)
    assert e.value.status == apb.ERR_CONFIG
    with pytest.raises(apb.ApbError) as e:   # host 2's q misaligned
        apb.attention_fwd_hosts([a[0], b[0]], [a[1], _FakeT(0x200002, b[1].shape)], [a[2], b[2]], [a[3], b[3]], g,
                                [a[4], b[4]], stream=0)
    assert e.value.status == apb.ERR_CONTRACT
    with pytest.raises(apb.ApbError):
        apb.attention_fwd_hosts([], [], [], [], g, [], stream=0)


def test_compress_hosts_contract_errors_before_any_gpu_work(lib):
    """apb_retain_score_hosts / apb_select_topk_hosts: hosts with different dims, a workspace
    smaller than n x apb_retain_workspace_size, and NULL arrays are rejected without a GPU."""
    import dataclasses
    d1, d2 = _dims(host=1), _dims(host=2)
    r = d1.rows
    q = [_FakeT(0x100000, (r, 4, 64)), _FakeT(0x200000, (r, 4, 64))]
    k = [_FakeT(0x110000, (r, 2, 64)), _FakeT(0x210000, (r, 2, 64))]
    v = [_FakeT(0x120000, (r, 2, 64)), _FakeT(0x220000, (r, 2, 64))]
    sc = [_FakeT(0x130000, (2, d1.l_b), 4), _FakeT(0x230000, (2, d1.l_b), 4)]
    w = apb.RetainWeights(w1=_FakeT(0x50000, (256, 8 * 64)), w2=_FakeT(0x60000, (4, 256), 4))
    per = apb.retain_workspace_size(d1, w)
    small = _FakeT(0x400000, (per,), 1, dtype=torch.uint8)
    with pytest.raises(apb.ApbError) as e:   # workspace for one host only
        apb.retain_score_hosts([d1, d2], w, q, k, v, sc, small, stream=0)
    assert e.value.status == apb.ERR_CONTRACT
    big = _FakeT(0x400000, (2 * per,), 1, dtype=torch.uint8)
    d2x = dataclasses.replace(d2, l_p=d2.l_p + 8)
    with pytest.raises(apb.ApbError) as e:
        apb.retain_score_hosts([d1, d2x], w, q, k, v, sc, big, stream=0)
    assert e.value.status == apb.ERR_CONFIG
    idx = [_FakeT(0x500000, (2, d1.l_pp), 4, dtype=torch.int32), _FakeT(0x510000, (2, d1.l_pp), 4, dtype=torch.int32)]
    send = [_FakeT(0x600000, (2, 2, d1.l_pp, 64)), _FakeT(0x700000, (2, 2, d1.l_pp, 64))]
    with pytest.raises(apb.ApbError) as e:   # n_heads differs (nothing the binding sizes by)
        apb.select_topk_hosts([d1, dataclasses.replace(d2, n_heads=6)], sc, k, v, idx, send, stream=0)
    assert e.value.status == apb.ERR_CONFIG
    with pytest.raises(apb.ApbError) as e:   # host 2's send misaligned
        apb.select_topk_hosts([d1, d2], sc, k, v, idx, [send[0], _FakeT(0x700008, (2, 2, d1.l_pp, 64))], stream=0)
    assert e.value.status == apb.ERR_CONTRACT
