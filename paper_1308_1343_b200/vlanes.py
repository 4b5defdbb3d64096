"""Device versions of the reference's explicit-SIMD stencil listings.

``forward_difference`` and ``centered_difference`` (vlanes.py:342-360) with
the reference's frame rule: every index of the iteration range is written by
exactly one active lane, lanes outside it never store (iterate_masked +
vstore_partial, vlanes.py:322-337, 158-169), and the arithmetic is the
unfused IEEE form (FUSED_FMA = False, vlanes.py:33).  On the B200 the lanes
are the 32 threads of a warp; arrays are 1-D fp64 torch tensors in HBM and
the call is asynchronous on the current stream.
"""
from __future__ import annotations

from . import _lib
from .errors import UsageError
from .grid import stream_ptr


def _check(dst, src, n):
    import torch
    for t in (dst, src):
        if t.dtype != torch.float64 or not t.is_cuda or t.dim() != 1 or not t.is_contiguous():
            raise UsageError("arrays must be contiguous 1-D float64 CUDA tensors")
    if n < 0 or n > src.numel() or n > dst.numel():
        raise UsageError(f"length {n} outside the arrays")


def forward_difference(dst, src, n: int, stream=None) -> None:
    """dst[i] = src[i+1] - src[i] for 0 <= i < n-1."""
    _check(dst, src, n)
    _lib.call("sb_diff1d", 0, dst.data_ptr(), src.data_ptr(), int(n), stream_ptr(stream))


def centered_difference(dst, src, n: int, stream=None) -> None:
    """dst[i] = 0.5 * (src[i+1] - src[i-1]) for 1 <= i < n-1."""
    _check(dst, src, n)
    _lib.call("sb_diff1d", 1, dst.data_ptr(), src.data_ptr(), int(n), stream_ptr(stream))
