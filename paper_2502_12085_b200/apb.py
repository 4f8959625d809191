"""Thin Python binding of libapb (include/apb.h): argument marshalling only.

Every step of the APB hot path runs in libapb's sm_100a kernels (or NCCL for the exchange);
this module only turns torch tensors / streams into pointers, row strides and the C structs.
There is no CPU fallback: if libapb.so cannot be loaded, or a call fails, an ApbError is
raised.  Function names mirror the C entry points:

    retain_score      -> apb_retain_score      (retaining heads)
    select_topk       -> apb_select_topk       (ArgTop-l_p + compaction)
    exchange_passing  -> apb_exchange_passing  (AllGather)
    attention_fwd     -> apb_attention_fwd     (eq:apb)
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libapb.so")

OK, ERR_CONFIG, ERR_CONTRACT, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL = range(6)
LAYOUT_BLOCK, LAYOUT_CYCLIC = 0, 1
EPI_STORE, EPI_RESIDUAL, EPI_SWIGLU, EPI_ROPE = range(4)
PHASE_ALL, PHASE_LOCAL, PHASE_PASSING = 0, 1, 2
WS_RETAIN, WS_SELECT, WS_ATTENTION = 0, 1, 2

EXPORTED = ("apb_retain_score", "apb_select_topk", "apb_exchange_passing", "apb_attention_fwd",
            "apb_comm_get_unique_id", "apb_comm_init", "apb_comm_destroy", "apb_workspace_size",
            "apb_check_dims", "apb_status_string", "apb_last_error", "apb_version", "apb_launch_count",
            "apb_decode_attention", "apb_decode_workspace_size", "apb_merge_partials", "apb_exchange_partials",
            "apb_decode_attention_hosts", "apb_decode_hosts_workspace_size", "apb_exchange_passing_cyclic",
            "apb_decode_step_hosts", "apb_exchange_plan", "apb_comm_check", "apb_comm_abort",
            "apb_exchange_partials_cyclic", "apb_gemm", "apb_retain_workspace_size",
            "apb_peers_create", "apb_peers_open", "apb_peers_gathered", "apb_select_topk_peers", "apb_peers_wait",
            "apb_peers_release", "apb_peers_destroy", "apb_attention_fwd_hosts", "apb_retain_score_hosts",
            "apb_select_topk_hosts")


class ApbError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        self.status = status
        super().__init__(f"{fn} failed: status {status} ({_status_name(status)}): {detail}")


class _Dims(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("H", ctypes.c_int32), ("host", ctypes.c_int32),
                ("l_q", ctypes.c_int32), ("l_a", ctypes.c_int32), ("l_b", ctypes.c_int32),
                ("l_p", ctypes.c_int32), ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("softmax_scale", ctypes.c_float)]


class _DecodeDims(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int32), ("host", ctypes.c_int32), ("t_new", ctypes.c_int32),
                ("cache_len", ctypes.c_int64), ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("softmax_scale", ctypes.c_float)]


class _GemmEpi(ctypes.Structure):
    _fields_ = [("epilogue", ctypes.c_int32), ("beta", ctypes.c_float), ("rope_cols", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("theta", ctypes.c_float), ("positions", ctypes.c_void_p),
                ("pos_offset", ctypes.c_int64)]


class _Weights(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int32), ("d_hidden", ctypes.c_int32), ("n_out", ctypes.c_int32),
                ("w1", ctypes.c_void_p), ("b1", ctypes.c_void_p), ("w2", ctypes.c_void_p),
                ("b2", ctypes.c_void_p)]


_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libapb.so (fails loudly if it is missing — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("APB_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ApbError(ERR_CUDA, "load", f"{path} not built; run `python -m paper_2502_12085_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    dp = ctypes.POINTER(_Dims)
    lib.apb_retain_score.argtypes = [dp, ctypes.POINTER(_Weights), vp, vp, vp, i64, i64, vp, vp, sz, vp]
    lib.apb_select_topk.argtypes = [dp, vp, vp, vp, i64, vp, vp, vp, sz, vp]
    lib.apb_retain_score_hosts.argtypes = [i32, dp, ctypes.POINTER(_Weights), vp, vp, vp, i64, i64, vp, vp, sz, vp]
    lib.apb_select_topk_hosts.argtypes = [i32, dp, vp, vp, vp, i64, vp, vp, vp]
    lib.apb_exchange_passing.argtypes = [vp, dp, vp, vp]
    lib.apb_exchange_passing_cyclic.argtypes = [vp, dp, vp, vp]
    lib.apb_attention_fwd.argtypes = [dp, vp, vp, vp, i64, i64, vp, vp, i64, vp, ctypes.c_int, vp, sz, vp]
    lib.apb_attention_fwd_hosts.argtypes = [i32, dp, vp, vp, vp, i64, i64, vp, vp, i64, vp, ctypes.c_int, vp, vp, vp]
    lib.apb_comm_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.apb_comm_init.argtypes = [ctypes.c_char_p, i32, i32, ctypes.POINTER(vp)]
    lib.apb_comm_destroy.argtypes = [vp]
    lib.apb_workspace_size.argtypes = [dp, ctypes.c_int, ctypes.POINTER(sz)]
    lib.apb_check_dims.argtypes = [dp]
    ddp = ctypes.POINTER(_DecodeDims)
    lib.apb_decode_attention.argtypes = [ddp, vp, vp, vp, i64, vp, vp, i64, vp, vp, vp, sz, vp]
    lib.apb_decode_workspace_size.argtypes = [ddp, ctypes.POINTER(sz)]
    lib.apb_decode_attention_hosts.argtypes = [ddp, i32, vp, vp, vp, i64, vp, vp, vp, i64, vp, i64, i64, vp, sz, vp]
    lib.apb_decode_hosts_workspace_size.argtypes = [ddp, i32, vp, ctypes.POINTER(sz)]
    lib.apb_decode_step_hosts.argtypes = [ddp, vp, vp, vp, i64, vp, vp, vp, i64, vp, vp, vp, sz, vp]
    lib.apb_merge_partials.argtypes = [i32, i64, i32, vp, i64, vp, i64, vp, vp, vp]
    lib.apb_exchange_partials.argtypes = [vp, i64, vp, vp]
    lib.apb_random_scores.argtypes = [dp, ctypes.c_uint64, i32, vp, vp]
    lib.apb_rmsnorm.argtypes = [i64, i32, vp, i64, vp, ctypes.c_float, vp, i64, vp]
    lib.apb_rope.argtypes = [i64, i32, i32, vp, i64, vp, i64, ctypes.c_float, vp]
    lib.apb_swiglu.argtypes = [i64, i32, vp, i64, vp, i64, vp]
    lib.apb_gemm_bf16.argtypes = [i64, i32, i32, vp, i64, vp, i64, vp, i64, ctypes.c_float, vp, sz, vp]
    lib.apb_share_scores.argtypes = [dp, vp, vp]
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.apb_exchange_plan.argtypes = [dp, i32, i32, ctypes.c_int, i32, i64p, i64p, i64p, ctypes.POINTER(i32)]
    lib.apb_comm_check.argtypes = [vp]
    lib.apb_comm_abort.argtypes = [vp]
    lib.apb_exchange_partials_cyclic.argtypes = [vp, i32, i64, vp, vp]
    lib.apb_peers_create.argtypes = [dp, i32, i32, ctypes.POINTER(vp), ctypes.c_char_p]
    lib.apb_peers_open.argtypes = [vp, ctypes.c_char_p]
    lib.apb_peers_gathered.argtypes = [vp, i32, ctypes.POINTER(vp)]
    lib.apb_select_topk_peers.argtypes = [dp, vp, vp, vp, i64, vp, vp, i32, vp]
    lib.apb_peers_wait.argtypes = [vp, i32, i32, vp]
    lib.apb_peers_release.argtypes = [vp, i32, vp]
    lib.apb_peers_destroy.argtypes = [vp]
    lib.apb_retain_workspace_size.argtypes = [dp, ctypes.POINTER(_Weights), ctypes.POINTER(sz)]
    lib.apb_gemm.argtypes = [i64, i32, i32, vp, i64, vp, i64, vp, i64, ctypes.POINTER(_GemmEpi), vp]
    for f in ("apb_random_scores", "apb_share_scores", "apb_rmsnorm", "apb_rope", "apb_swiglu", "apb_gemm_bf16", "apb_retain_score", "apb_select_topk", "apb_exchange_passing", "apb_attention_fwd",
              "apb_comm_get_unique_id", "apb_comm_init", "apb_comm_destroy", "apb_workspace_size",
              "apb_check_dims", "apb_decode_attention", "apb_decode_workspace_size", "apb_merge_partials",
              "apb_exchange_partials", "apb_decode_attention_hosts", "apb_decode_hosts_workspace_size",
              "apb_exchange_passing_cyclic", "apb_decode_step_hosts", "apb_exchange_plan", "apb_comm_check",
              "apb_comm_abort", "apb_exchange_partials_cyclic", "apb_gemm", "apb_retain_workspace_size",
              "apb_peers_create", "apb_peers_open", "apb_peers_gathered", "apb_select_topk_peers", "apb_peers_wait",
              "apb_peers_release", "apb_peers_destroy", "apb_attention_fwd_hosts", "apb_retain_score_hosts",
            "apb_select_topk_hosts"):
        getattr(lib, f).restype = ctypes.c_int
    lib.apb_status_string.argtypes = [ctypes.c_int]
    lib.apb_status_string.restype = ctypes.c_char_p
    lib.apb_last_error.restype = ctypes.c_char_p
    lib.apb_version.restype = ctypes.c_int32
    lib.apb_launch_count.restype = ctypes.c_int64
    _lib = lib
    return lib


def _status_name(s: int) -> str:
    names = ["APB_OK", "APB_ERR_CONFIG", "APB_ERR_CONTRACT", "APB_ERR_UNSUPPORTED", "APB_ERR_CUDA", "APB_ERR_NCCL"]
    return names[s] if 0 <= s < len(names) else "?"


def _check(rc: int, fn: str) -> None:
    if rc != OK:
        raise ApbError(rc, fn, load().apb_last_error().decode(errors="replace"))


# ----------------------------------------------------------------------------- problem dims

@dataclasses.dataclass
class Dims:
    """apb_dims: one host's layer (symbols as the paper)."""
    n: int
    H: int
    host: int
    l_a: int
    l_p: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    l_q: int = 0
    l_b: int | None = None
    softmax_scale: float = 0.0

    def __post_init__(self):
        if self.l_b is None:
            self.l_b = self.n // self.H if self.H > 0 else 0

    @property
    def L_A(self) -> int:
        return 0 if self.host == 0 else self.l_q + self.l_a

    @property
    def l_pp(self) -> int:
        return min(self.l_p, self.l_b)

    @property
    def rows(self) -> int:
        return self.L_A + self.l_b

    @property
    def P(self) -> int:
        return self.host * self.l_pp

    def with_host(self, host: int) -> "Dims":
        return dataclasses.replace(self, host=host)

    def c(self) -> _Dims:
        return _Dims(self.n, self.H, self.host, self.l_q, self.l_a, self.l_b, self.l_p, self.n_heads,
                     self.n_kv_heads, self.head_dim, self.softmax_scale)


@dataclasses.dataclass
class RetainWeights:
    """apb_retain_weights: w1 bf16 [d_hidden][d_in]; b1 fp32 [d_hidden] | None; w2 fp32
    [n_out][d_hidden]; b2 fp32 [n_out] | None (device tensors)."""
    w1: torch.Tensor
    w2: torch.Tensor
    b1: torch.Tensor | None = None
    b2: torch.Tensor | None = None

    def c(self) -> _Weights:
        d_hidden, d_in = self.w1.shape
        return _Weights(d_in, d_hidden, self.w2.shape[0], self.w1.data_ptr(),
                        self.b1.data_ptr() if self.b1 is not None else None, self.w2.data_ptr(),
                        self.b2.data_ptr() if self.b2 is not None else None)


def _rowstride(t: torch.Tensor, name: str) -> int:
    """Row stride (elements) of a [rows][heads][head_dim] (or [rows][width]) tensor whose
    inner dims are dense."""
    if t.dim() == 3:
        if t.stride(2) != 1 or t.stride(1) != t.shape[2]:
            raise ApbError(ERR_CONTRACT, name, "inner dims must be dense [rows][heads][head_dim]")
    elif t.dim() == 2:
        if t.stride(1) != 1:
            raise ApbError(ERR_CONTRACT, name, "last dim must be contiguous")
    return t.stride(0)


def _need(t, name: str, dtype, min_rows: int | None = None, width: int | None = None, dense: bool = False):
    """Validate what the C ABI cannot see from a pointer: device, dtype, and that the tensor
    covers the rows / row width (elements) the call will read or write from `dims`."""
    if t is None:
        raise ApbError(ERR_CONTRACT, name, "is None")
    if not t.is_cuda:
        raise ApbError(ERR_CONTRACT, name, "must be a CUDA tensor")
    if t.dtype != dtype:
        raise ApbError(ERR_CONTRACT, name, f"dtype must be {dtype}, got {t.dtype}")
    if dense and not t.is_contiguous():
        raise ApbError(ERR_CONTRACT, name, "must be contiguous")
    if min_rows is not None and (t.dim() == 0 or t.shape[0] < min_rows):
        raise ApbError(ERR_CONTRACT, name, f"needs >= {min_rows} rows, has {tuple(t.shape)}")
    if width is not None:
        w = t[0].numel() if t.dim() >= 2 else t.numel()
        if w < width:
            raise ApbError(ERR_CONTRACT, name, f"rows must hold >= {width} elements, have {w}")


def _need_numel(t, name: str, dtype, numel: int):
    _need(t, name, dtype, dense=True)
    if t.numel() < numel:
        raise ApbError(ERR_CONTRACT, name, f"needs >= {numel} elements, has {t.numel()}")


def _check_qkv(dims: "Dims", q, k, v) -> int:
    """q [rows][hq][d], k/v [rows][hk][d] bf16 with one shared K/V row stride (the ABI takes
    one kv_row_stride for both).  Returns that stride."""
    rows = dims.rows
    _need(q, "q", torch.bfloat16, rows, dims.n_heads * dims.head_dim)
    _need(k, "k", torch.bfloat16, rows, dims.n_kv_heads * dims.head_dim)
    _need(v, "v", torch.bfloat16, rows, dims.n_kv_heads * dims.head_dim)
    ks, vs = _rowstride(k, "k"), _rowstride(v, "v")
    if ks != vs:
        raise ApbError(ERR_CONTRACT, "k/v", f"K and V must share one row stride ({ks} != {vs})")
    _rowstride(q, "q")
    return ks


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t):
    return None if t is None else t.data_ptr()


# ----------------------------------------------------------------------------- entry points

def workspace_size(dims: Dims, kind: int) -> int:
    out = ctypes.c_size_t(0)
    d = dims.c()
    _check(load().apb_workspace_size(ctypes.byref(d), kind, ctypes.byref(out)), "apb_workspace_size")
    return out.value


def check_dims(dims: Dims) -> None:
    d = dims.c()
    _check(load().apb_check_dims(ctypes.byref(d)), "apb_check_dims")


def retain_workspace_size(dims: Dims, w: RetainWeights) -> int:
    out = ctypes.c_size_t(0)
    d, wc = dims.c(), w.c()
    _check(load().apb_retain_workspace_size(ctypes.byref(d), ctypes.byref(wc), ctypes.byref(out)),
           "apb_retain_workspace_size")
    return out.value


def retain_score(dims: Dims, w: RetainWeights, q, k, v, scores, stream=None, ws="auto") -> None:
    """ws: device workspace (apb_retain_workspace_size bytes) for the CTA-pair GEMM; "auto"
    allocates it (torch caching allocator, on q's device); None runs the single-CTA kernel."""
    _check_qkv(dims, q, k, v)
    _need_numel(scores, "scores", torch.float32, dims.n_kv_heads * dims.l_b)
    _need(w.w1, "w1", torch.bfloat16, dense=True)
    _need(w.w2, "w2", torch.float32, dense=True)
    for b, nm in ((w.b1, "b1"), (w.b2, "b2")):
        if b is not None:
            _need(b, nm, torch.float32, dense=True)
    if w.w2.dim() != 2 or w.w2.shape[1] != w.w1.shape[0]:
        raise ApbError(ERR_CONTRACT, "w2", "must be [n_out][d_hidden]")
    if isinstance(ws, str):
        ws = torch.empty(max(retain_workspace_size(dims, w), 16), dtype=torch.uint8, device=q.device)
    d, wc = dims.c(), w.c()
    _check(load().apb_retain_score(ctypes.byref(d), ctypes.byref(wc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                   _rowstride(q, "q"), _rowstride(k, "k"), scores.data_ptr(), _ptr(ws),
                                   0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
           "apb_retain_score")


def select_topk(dims: Dims, scores, k, v, indices, send, stream=None) -> None:
    _need_numel(scores, "scores", torch.float32, dims.n_kv_heads * dims.l_b)
    if dims.l_pp > 0:
        _need(k, "k", torch.bfloat16, dims.rows, dims.n_kv_heads * dims.head_dim)
        _need(v, "v", torch.bfloat16, dims.rows, dims.n_kv_heads * dims.head_dim)
        if _rowstride(k, "k") != _rowstride(v, "v"):
            raise ApbError(ERR_CONTRACT, "k/v", "K and V must share one row stride")
        _need_numel(indices, "indices", torch.int32, dims.n_kv_heads * dims.l_pp)
        _need_numel(send, "send", torch.bfloat16, 2 * dims.n_kv_heads * dims.l_pp * dims.head_dim)
    d = dims.c()
    _check(load().apb_select_topk(ctypes.byref(d), scores.data_ptr(), k.data_ptr(), v.data_ptr(),
                                  _rowstride(k, "k"), indices.data_ptr(), send.data_ptr(), None, 0,
                                  _stream(stream)), "apb_select_topk")


def _ptrs(xs):
    return (ctypes.c_void_p * len(xs))(*[_ptr(x) for x in xs])


def _same_problem(dims: list[Dims]) -> None:
    if not 1 <= len(dims) <= 8:
        raise ApbError(ERR_CONTRACT, "hosts", "1..8 hosts per launch")


def retain_score_hosts(dims: list[Dims], w: RetainWeights, q: list, k: list, v: list, scores: list, ws,
                       stream=None) -> None:
    """apb_retain_score_hosts: the scoring of several hosts (dims[i].host) in one GEMM launch;
    ws: len(dims) x retain_workspace_size bytes."""
    _same_problem(dims)
    n = len(dims)
    if not len(q) == len(k) == len(v) == len(scores) == n:
        raise ApbError(ERR_CONTRACT, "hosts", "one q/k/v/scores per host")
    for i in range(n):
        _check_qkv(dims[i], q[i], k[i], v[i])
        _need_numel(scores[i], "scores", torch.float32, dims[i].n_kv_heads * dims[i].l_b)
        if _rowstride(q[i], "q") != _rowstride(q[0], "q") or _rowstride(k[i], "k") != _rowstride(k[0], "k"):
            raise ApbError(ERR_CONTRACT, "hosts", "the hosts' q / kv row strides must be equal")
    _need(w.w1, "w1", torch.bfloat16, dense=True)
    _need(w.w2, "w2", torch.float32, dense=True)
    for b, nm in ((w.b1, "b1"), (w.b2, "b2")):
        if b is not None:
            _need(b, nm, torch.float32, dense=True)
    if w.w2.dim() != 2 or w.w2.shape[1] != w.w1.shape[0]:
        raise ApbError(ERR_CONTRACT, "w2", "must be [n_out][d_hidden]")
    _need(ws, "ws", ws.dtype, dense=True)
    cd = (_Dims * n)(*[d.c() for d in dims])
    wc = w.c()
    _check(load().apb_retain_score_hosts(n, cd, ctypes.byref(wc), _ptrs(q), _ptrs(k), _ptrs(v), _rowstride(q[0], "q"),
                                         _rowstride(k[0], "k"), _ptrs(scores), _ptr(ws), ws.numel() * ws.element_size(),
                                         _stream(stream)), "apb_retain_score_hosts")


def select_topk_hosts(dims: list[Dims], scores: list, k: list, v: list, indices: list, send: list,
                      stream=None) -> None:
    """apb_select_topk_hosts: several hosts' selection + compaction in one launch pair."""
    _same_problem(dims)
    n = len(dims)
    if not len(scores) == len(k) == len(v) == len(indices) == len(send) == n:
        raise ApbError(ERR_CONTRACT, "hosts", "one scores/k/v/indices/send per host")
    for i, d in enumerate(dims):
        _need_numel(scores[i], "scores", torch.float32, d.n_kv_heads * d.l_b)
        if d.l_pp > 0:
            _need(k[i], "k", torch.bfloat16, d.rows, d.n_kv_heads * d.head_dim)
            _need(v[i], "v", torch.bfloat16, d.rows, d.n_kv_heads * d.head_dim)
            if _rowstride(k[i], "k") != _rowstride(v[i], "v") or _rowstride(k[i], "k") != _rowstride(k[0], "k"):
                raise ApbError(ERR_CONTRACT, "k/v", "K and V of every host must share one row stride")
            _need_numel(indices[i], "indices", torch.int32, d.n_kv_heads * d.l_pp)
            _need_numel(send[i], "send", torch.bfloat16, 2 * d.n_kv_heads * d.l_pp * d.head_dim)
    cd = (_Dims * n)(*[d.c() for d in dims])
    _check(load().apb_select_topk_hosts(n, cd, _ptrs(scores), _ptrs(k), _ptrs(v), _rowstride(k[0], "k"),
                                        _ptrs(indices), _ptrs(send), _stream(stream)), "apb_select_topk_hosts")


def random_scores(dims: Dims, seed: int, layer: int, scores, stream=None) -> None:
    """The "Rd." compressor (Table 4): scores [n_kv_heads][l_b] fp32 <- seeded uniform [0,1)."""
    _need_numel(scores, "scores", torch.float32, dims.n_kv_heads * dims.l_b)
    d = dims.c()
    _check(load().apb_random_scores(ctypes.byref(d), seed % (1 << 64), layer, scores.data_ptr(), _stream(stream)),
           "apb_random_scores")


def share_scores(dims: Dims, scores, stream=None) -> None:
    """Shared index set: scores rows <- max over KV heads, in place."""
    _need_numel(scores, "scores", torch.float32, dims.n_kv_heads * dims.l_b)
    d = dims.c()
    _check(load().apb_share_scores(ctypes.byref(d), scores.data_ptr(), _stream(stream)), "apb_share_scores")


def attention_fwd(dims: Dims, q, k, v, gathered, out, lse=None, phase: int = PHASE_ALL, ws=None,
                  stream=None) -> None:
    _check_qkv(dims, q, k, v)
    _need(out, "out", torch.bfloat16, dims.rows, dims.n_heads * dims.head_dim)
    if lse is not None:
        _need(lse, "lse", torch.float32, dims.n_heads, dims.rows, dense=True)
        if lse.dim() != 2 or lse.shape[1] != dims.rows:
            raise ApbError(ERR_CONTRACT, "lse", f"must be [n_heads][{dims.rows}]")
    if gathered is not None and dims.P > 0 and phase != PHASE_LOCAL:
        _need_numel(gathered, "gathered", torch.bfloat16, dims.H * 2 * dims.n_kv_heads * dims.l_pp * dims.head_dim)
    if ws is not None:
        _need(ws, "ws", ws.dtype, dense=True)
    d = dims.c()
    _check(load().apb_attention_fwd(ctypes.byref(d), q.data_ptr(), k.data_ptr(), v.data_ptr(), _rowstride(q, "q"),
                                    _rowstride(k, "k"), _ptr(gathered), out.data_ptr(), _rowstride(out, "out"),
                                    _ptr(lse), phase, _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                                    _stream(stream)), "apb_attention_fwd")


def attention_fwd_hosts(dims: list[Dims], q: list, k: list, v: list, gathered, out: list, lse: list | None = None,
                        phase: int = PHASE_ALL, ws: list | None = None, stream=None) -> None:
    """apb_attention_fwd_hosts: the attention of several hosts (dims[i].host) in one launch —
    the same results as one attention_fwd call per host."""
    n = len(dims)
    if not (1 <= n <= 8) or not (len(q) == len(k) == len(v) == len(out) == n):
        raise ApbError(ERR_CONTRACT, "hosts", "1..8 hosts with one q/k/v/out each")
    if lse is not None and len(lse) != n or ws is not None and len(ws) != n:
        raise ApbError(ERR_CONTRACT, "hosts", "lse / ws need one entry per host")
    for i in range(n):
        _check_qkv(dims[i], q[i], k[i], v[i])
        _need(out[i], "out", torch.bfloat16, dims[i].rows, dims[i].n_heads * dims[i].head_dim)
        if lse is not None and lse[i] is not None:
            _need(lse[i], "lse", torch.float32, dims[i].n_heads, dims[i].rows, dense=True)
            if lse[i].dim() != 2 or lse[i].shape[1] != dims[i].rows:
                raise ApbError(ERR_CONTRACT, "lse", f"must be [n_heads][{dims[i].rows}]")
        if ws is not None and ws[i] is not None:
            _need(ws[i], "ws", ws[i].dtype, dense=True)
        if _rowstride(q[i], "q") != _rowstride(q[0], "q") or _rowstride(k[i], "k") != _rowstride(k[0], "k") \
                or _rowstride(out[i], "out") != _rowstride(out[0], "out"):
            raise ApbError(ERR_CONTRACT, "hosts", "the hosts' q / kv / out row strides must be equal")
    if gathered is not None and any(d.P > 0 for d in dims) and phase != PHASE_LOCAL:
        d0 = dims[0]
        _need_numel(gathered, "gathered", torch.bfloat16, d0.H * 2 * d0.n_kv_heads * d0.l_pp * d0.head_dim)
    cd = (_Dims * n)(*[d.c() for d in dims])
    arr = lambda xs: (ctypes.c_void_p * n)(*[_ptr(x) for x in xs])  # noqa: E731
    ws_b = None if ws is None else (ctypes.c_size_t * n)(*[0 if w is None else w.numel() * w.element_size() for w in ws])
    _check(load().apb_attention_fwd_hosts(n, cd, arr(q), arr(k), arr(v), _rowstride(q[0], "q"), _rowstride(k[0], "k"),
                                          _ptr(gathered), arr(out), _rowstride(out[0], "out"),
                                          None if lse is None else arr(lse), phase,
                                          None if ws is None else arr(ws), ws_b, _stream(stream)),
           "apb_attention_fwd_hosts")


# ----------------------------------------------------------------------------- model layer (NEXT #2)

def rmsnorm(x, w, eps: float, out, stream=None) -> None:
    """out = RMSNorm(x) * w over the last dim (x, out: bf16 [rows][dim] row-strided views)."""
    _check(load().apb_rmsnorm(x.shape[0], x.shape[-1], x.data_ptr(), _rowstride(x, "x"), w.data_ptr(), eps,
                              out.data_ptr(), _rowstride(out, "out"), _stream(stream)), "apb_rmsnorm")


def rope(x, n_heads: int, head_dim: int, theta: float, positions=None, pos_offset: int = 0, stream=None) -> None:
    """In-place RoPE on the first n_heads heads of every row of x (bf16 [rows][>= n_heads*head_dim])."""
    _check(load().apb_rope(x.shape[0], n_heads, head_dim, x.data_ptr(), x.stride(0), _ptr(positions), pos_offset,
                           theta, _stream(stream)), "apb_rope")


def swiglu(gu, out, stream=None) -> None:
    """out = SiLU(gu[:, :I]) * gu[:, I:] with I = out.shape[-1]."""
    _check(load().apb_swiglu(gu.shape[0], out.shape[-1], gu.data_ptr(), _rowstride(gu, "gu"), out.data_ptr(),
                             _rowstride(out, "out"), _stream(stream)), "apb_swiglu")


def gemm_bf16(a, w, c, beta: float = 0.0, ws=None, stream=None) -> None:
    """c = a @ w.T (+ beta * c): a bf16 [M][K], w bf16 [N][K], c bf16 [M][N] (row-strided views)."""
    _check(load().apb_gemm_bf16(a.shape[0], w.shape[0], w.shape[1], a.data_ptr(), _rowstride(a, "a"), w.data_ptr(),
                                _rowstride(w, "w"), c.data_ptr(), _rowstride(c, "c"), beta, _ptr(ws),
                                0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
           "apb_gemm_bf16")


def gemm(a, w, c, epilogue: int = EPI_STORE, beta: float = 1.0, rope_cols: int = 0, head_dim: int = 128,
         theta: float = 0.0, positions=None, pos_offset: int = 0, stream=None) -> None:
    """apb_gemm: C = A W^T on libapb's tcgen05 GEMM with a fused epilogue (EPI_STORE, EPI_RESIDUAL
    (C = bf16(beta C + bf16(A W^T))), EPI_SWIGLU (W rows [gate; up] interleaved in 128-row blocks,
    C = act [M][N/2]), EPI_ROPE (rotate the heads in columns [0, rope_cols))).  a bf16 [M][K],
    w bf16 [N][K], c bf16 row-strided views."""
    M, N, K = a.shape[0], w.shape[0], w.shape[1]
    _need(a, "a", torch.bfloat16, M, K)
    _need(w, "w", torch.bfloat16, N, K)
    _need(c, "c", torch.bfloat16, M, N // 2 if epilogue == EPI_SWIGLU else N)
    if positions is not None:
        _need_numel(positions, "positions", torch.int32, M)
    e = _GemmEpi(epilogue, beta if epilogue == EPI_RESIDUAL else 0.0, rope_cols, head_dim, theta, _ptr(positions),
                 pos_offset)
    _check(load().apb_gemm(M, N, K, a.data_ptr(), _rowstride(a, "a"), w.data_ptr(), _rowstride(w, "w"),
                           c.data_ptr(), _rowstride(c, "c"), ctypes.byref(e), _stream(stream)), "apb_gemm")


def interleave_gate_up(w_gu: torch.Tensor, block: int = 128) -> torch.Tensor:
    """[W_gate; W_up] ([2I][hidden]) -> rows interleaved in `block`-row blocks, the weight layout
    apb_gemm's SWIGLU epilogue reads (one 256-wide tile = the gate and up rows of the same 128
    intermediate units).  A one-time weight-layout step (row permutation), not a compute step."""
    two_i, hidden = w_gu.shape
    inter = two_i // 2
    if inter % block:
        raise ApbError(ERR_CONFIG, "interleave_gate_up", f"intermediate size {inter} not a multiple of {block}")
    g = w_gu[:inter].reshape(inter // block, block, hidden)
    u = w_gu[inter:].reshape(inter // block, block, hidden)
    return torch.stack([g, u], dim=1).reshape(two_i, hidden).contiguous()


class Comm:
    """apb_comm: an NCCL communicator owned by libapb.  Build it on every rank from a 128-byte
    id that rank 0 draws with `Comm.unique_id()` and broadcasts (e.g. torch.distributed)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        self._h = ctypes.c_void_p()
        _check(load().apb_comm_init(uid, nranks, rank, ctypes.byref(self._h)), "apb_comm_init")
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load().apb_comm_get_unique_id(buf), "apb_comm_get_unique_id")
        return buf.raw

    @property
    def handle(self):
        return self._h

    def check(self) -> None:
        """Raise ApbError(ERR_NCCL) if an enqueued collective failed asynchronously."""
        _check(load().apb_comm_check(self._h), "apb_comm_check")

    def abort(self) -> None:
        """ncclCommAbort + free (recovery after an asynchronous error)."""
        if self._h:
            h, self._h = self._h, ctypes.c_void_p()
            _check(load().apb_comm_abort(h), "apb_comm_abort")

    def close(self) -> None:
        if self._h:
            _check(load().apb_comm_destroy(self._h), "apb_comm_destroy")
            self._h = ctypes.c_void_p()


class _CudaBuffer:
    """A library-owned device buffer exposed through __cuda_array_interface__ (torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class Peers:
    """apb_peers: the passing-block exchange over peer memory (CUDA IPC within one node), the
    AllGather fused into the compaction.  Construct on every rank, all-gather `handle` (64 bytes)
    across ranks, then call open(handles)."""

    def __init__(self, dims: Dims, nranks: int, rank: int):
        self._h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(64)
        d = dims.c()
        _check(load().apb_peers_create(ctypes.byref(d), nranks, rank, ctypes.byref(self._h), buf), "apb_peers_create")
        self.handle = buf.raw
        self.nranks, self.rank, self.dims = nranks, rank, dims

    def open(self, handles: list[bytes]) -> None:
        _check(load().apb_peers_open(self._h, b"".join(handles)), "apb_peers_open")

    def gathered(self, parity: int) -> torch.Tensor:
        """This rank's gathered buffer for a parity, as a bf16 [H][2][hk][l_p'][d] tensor view."""
        ptr = ctypes.c_void_p()
        _check(load().apb_peers_gathered(self._h, parity, ctypes.byref(ptr)), "apb_peers_gathered")
        d = self.dims
        shape = (d.H, 2, d.n_kv_heads, d.l_pp, d.head_dim)
        t = torch.as_tensor(_CudaBuffer(ptr.value, shape, "<i2"), device="cuda")
        return t.view(torch.bfloat16)

    def select_topk(self, dims: Dims, scores, k, v, indices, epoch: int, stream=None) -> None:
        _need_numel(scores, "scores", torch.float32, dims.n_kv_heads * dims.l_b)
        if _rowstride(k, "k") != _rowstride(v, "v"):
            raise ApbError(ERR_CONTRACT, "k/v", "K and V must share one row stride")
        _need_numel(indices, "indices", torch.int32, dims.n_kv_heads * dims.l_pp)
        d = dims.c()
        _check(load().apb_select_topk_peers(ctypes.byref(d), scores.data_ptr(), k.data_ptr(), v.data_ptr(),
                                            _rowstride(k, "k"), indices.data_ptr(), self._h, epoch, _stream(stream)),
               "apb_select_topk_peers")

    def wait(self, n_slots: int, epoch: int, stream=None) -> None:
        _check(load().apb_peers_wait(self._h, n_slots, epoch, _stream(stream)), "apb_peers_wait")

    def release(self, epoch: int, stream=None) -> None:
        _check(load().apb_peers_release(self._h, epoch, _stream(stream)), "apb_peers_release")

    def close(self) -> None:
        if self._h:
            h, self._h = self._h, ctypes.c_void_p()
            _check(load().apb_peers_destroy(h), "apb_peers_destroy")


def exchange_passing(comm: Comm | None, dims: Dims, gathered, stream=None, cyclic: bool = False) -> None:
    """cyclic: rank r owns hosts r, r+N, ... (apb_exchange_passing_cyclic), else contiguous blocks."""
    if comm is not None and comm.nranks > 1 and dims.l_pp > 0:
        _need_numel(gathered, "gathered", torch.bfloat16, dims.H * 2 * dims.n_kv_heads * dims.l_pp * dims.head_dim)
    d = dims.c()
    fn = "apb_exchange_passing_cyclic" if cyclic else "apb_exchange_passing"
    _check(getattr(load(), fn)(comm.handle if comm is not None else None, ctypes.byref(d),
                               gathered.data_ptr(), _stream(stream)), fn)


def exchange_plan(dims: Dims, nranks: int, rank: int, layout: int = LAYOUT_BLOCK) -> list[tuple[int, int, int]]:
    """apb_exchange_plan: the in-place AllGather rounds of apb_exchange_passing{,_cyclic} for
    `rank` of `nranks`, as (send_offset, recv_offset, count) in bf16 elements of gathered."""
    n = max(dims.H, 1)
    so, ro, ct = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
    rounds = ctypes.c_int32(0)
    d = dims.c()
    _check(load().apb_exchange_plan(ctypes.byref(d), nranks, rank, layout, n, so, ro, ct, ctypes.byref(rounds)),
           "apb_exchange_plan")
    return [(so[i], ro[i], ct[i]) for i in range(rounds.value)]


def launch_count() -> int:
    return int(load().apb_launch_count())


def version() -> int:
    return int(load().apb_version())


# ----------------------------------------------------------------------------- decode step (NEXT #1)

@dataclasses.dataclass
class DecodeDims:
    """apb_decode_dims: one host's decode step (Alg. apb_decode)."""
    H: int
    host: int
    t_new: int
    cache_len: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    softmax_scale: float = 0.0

    def c(self) -> _DecodeDims:
        return _DecodeDims(self.H, self.host, self.t_new, self.cache_len, self.n_heads, self.n_kv_heads,
                           self.head_dim, self.softmax_scale)


def decode_workspace_size(dims: DecodeDims) -> int:
    out = ctypes.c_size_t(0)
    d = dims.c()
    _check(load().apb_decode_workspace_size(ctypes.byref(d), ctypes.byref(out)), "apb_decode_workspace_size")
    return out.value


def decode_attention(dims: DecodeDims, q, k_cache, v_cache, k_new, v_new, part_o, part_lse, ws=None,
                     stream=None) -> None:
    """Host partial (A_h, lse_h) of the new tokens."""
    d = dims.c()
    cs = _rowstride(k_cache, "k_cache") if k_cache is not None and k_cache.numel() else 0
    ns = _rowstride(k_new, "k_new") if k_new is not None else 0
    _check(load().apb_decode_attention(ctypes.byref(d), q.data_ptr(), _ptr(k_cache), _ptr(v_cache), cs,
                                       _ptr(k_new), _ptr(v_new), ns, part_o.data_ptr(), part_lse.data_ptr(),
                                       _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                                       _stream(stream)), "apb_decode_attention")


def _host_arrays(cache_lens, k_caches, v_caches):
    n = len(cache_lens)
    lens = (ctypes.c_int64 * n)(*cache_lens)
    kp = (ctypes.c_void_p * n)(*[_ptr(k) for k in k_caches]) if k_caches is not None else None
    vp = (ctypes.c_void_p * n)(*[_ptr(v) for v in v_caches]) if v_caches is not None else None
    return n, lens, kp, vp


def decode_hosts_workspace_size(dims: DecodeDims, cache_lens: list[int]) -> int:
    out = ctypes.c_size_t(0)
    d = dims.c()
    n, lens, _, _ = _host_arrays(cache_lens, None, None)
    _check(load().apb_decode_hosts_workspace_size(ctypes.byref(d), n, lens, ctypes.byref(out)),
           "apb_decode_hosts_workspace_size")
    return out.value


def decode_attention_hosts(dims: DecodeDims, q, k_caches: list, v_caches: list, k_new, v_new, parts,
                           lse_offset: int, ws=None, stream=None) -> None:
    """Partials of hosts dims.host .. dims.host + len(k_caches) - 1 in one launch (+ one fold):
    host i's O at parts[i][:lse_offset], its lse at parts[i][lse_offset:] (parts fp32 [n][stride])."""
    lens = [k.shape[0] for k in k_caches]
    nz = [k for k in k_caches if k.numel()]
    cs = _rowstride(nz[0], "k_cache") if nz else 0
    for t in list(k_caches) + list(v_caches):
        if t.numel() and _rowstride(t, "cache") != cs:
            raise ValueError("all caches of one call must share a row stride")
    ns = _rowstride(k_new, "k_new") if k_new is not None else 0
    n, lp, kp, vp = _host_arrays(lens, k_caches, v_caches)
    d = dims.c()
    _check(load().apb_decode_attention_hosts(ctypes.byref(d), n, lp, kp, vp, cs, q.data_ptr(), _ptr(k_new),
                                             _ptr(v_new), ns, parts.data_ptr(), parts.stride(0), lse_offset,
                                             _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                                             _stream(stream)), "apb_decode_attention_hosts")


def decode_step_hosts(dims: DecodeDims, q, k_caches: list, v_caches: list, k_new, v_new, out, out_lse=None,
                      ws=None, stream=None) -> None:
    """The whole decode step with every host on this rank (dims.host == 0, len(k_caches) == H):
    one streaming launch + MergeScore straight into bf16 out [t][hq][d] (and lse [t][hq])."""
    lens = [k.shape[0] for k in k_caches]
    nz = [k for k in k_caches if k.numel()]
    cs = _rowstride(nz[0], "k_cache") if nz else 0
    for t in list(k_caches) + list(v_caches):
        if t.numel() and _rowstride(t, "cache") != cs:
            raise ValueError("all caches of one call must share a row stride")
    ns = _rowstride(k_new, "k_new") if k_new is not None else 0
    _, lp, kp, vp = _host_arrays(lens, k_caches, v_caches)
    d = dims.c()
    _check(load().apb_decode_step_hosts(ctypes.byref(d), lp, kp, vp, cs, q.data_ptr(), _ptr(k_new), _ptr(v_new), ns,
                                        out.data_ptr(), _ptr(out_lse), _ptr(ws),
                                        0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
           "apb_decode_step_hosts")


def merge_partials(n_parts: int, rows: int, head_dim: int, parts_o, stride_o: int, parts_lse, stride_lse: int,
                   out, out_lse=None, stream=None) -> None:
    """MergeScore of n_parts partials (fp32) into bf16 out [rows][head_dim]."""
    _check(load().apb_merge_partials(n_parts, rows, head_dim, parts_o.data_ptr(), stride_o, parts_lse.data_ptr(),
                                     stride_lse, out.data_ptr(), _ptr(out_lse), _stream(stream)),
           "apb_merge_partials")


def exchange_partials(comm: "Comm | None", count_per_rank: int, buf, stream=None) -> None:
    """Gather: in-place AllGather of fp32 [nranks][count_per_rank]."""
    _check(load().apb_exchange_partials(comm.handle if comm is not None else None, count_per_rank,
                                        buf.data_ptr(), _stream(stream)), "apb_exchange_partials")


def exchange_partials_cyclic(comm: "Comm | None", H: int, slot_count: int, buf, stream=None) -> None:
    """Gather for cyclic ownership: buf fp32 [H][slot_count], host h in slot h."""
    _check(load().apb_exchange_partials_cyclic(comm.handle if comm is not None else None, H, slot_count,
                                               buf.data_ptr(), _stream(stream)), "apb_exchange_partials_cyclic")
