"""libapb: B200-native (sm_100a) APB prefill hot path (arXiv 2502.12085).

`apb` is the thin ctypes binding of the C ABI in include/apb.h; `prefill` orders the four
calls on CUDA streams for the hosts a rank owns.  All numerics run in libapb.so.
"""
from . import apb  # noqa: F401

__all__ = ["apb"]
