"""Device-resident fp64 grids with explicit ghost zones and padded rows.

The reference's kernels close over numpy ``(z, y, x)`` arrays (x contiguous,
``stencil.py:9-10, 42-46``).  On the B200 a box lives in HBM as a torch
storage laid out for coalesced, TMA-friendly access (north_star (a)):

* every row owns ``xpad`` = 16 elements (128 B) before interior x = 0, so the
  interior of every row starts on a 128-byte boundary and the ghost columns
  sit in the tail of the pad;
* the row pitch ``sy`` is a multiple of 16 elements (128 B);
* y and z ghost layers are whole rows / planes (``sz = sy * (ny + 2g)``).

Padding is never read as data and never counted as traffic.  Torch owns all
memory; the C library only receives pointers (``abi()``), as the ownership
contract of SURVEY.md §8(b) requires.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import UsageError

ROW_ALIGN = 16   # elements (128 bytes)


def _round_up(a: int, b: int) -> int:
    return -(-a // b) * b


class DeviceGrid:
    """One box's fp64 grid function in HBM.

    ``lower`` is the index-space coordinate of interior point (0,0,0): kernels
    receive pieces in the caller's coordinates (the reference's array indices,
    or level coordinates of a bboxset box) and subtract it."""

    def __init__(self, extents, ghost: int = 0, device=None, lower=(0, 0, 0)):
        import torch
        nx, ny, nz = (int(e) for e in extents)
        if min(nx, ny, nz) < 0 or ghost < 0 or ghost > ROW_ALIGN:
            raise UsageError(f"bad grid geometry {extents} ghost {ghost}")
        self.extents = (nx, ny, nz)
        self.ghost = int(ghost)
        self.lower = tuple(int(v) for v in lower)
        self.xpad = ROW_ALIGN if ghost > 0 else 0
        self.sy = max(ROW_ALIGN, _round_up(self.xpad + nx + ghost, ROW_ALIGN))
        self.sz = self.sy * (ny + 2 * ghost)
        total = self.sz * (nz + 2 * ghost)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.storage = torch.zeros(max(total, 1), dtype=torch.float64, device=device)
        self.offset = self.xpad + ghost * self.sy + ghost * self.sz
        if (self.storage.data_ptr() + 8 * self.offset) % 128:
            raise UsageError("device allocation is not 128-byte aligned")

    # -- views ------------------------------------------------------------------
    @property
    def device(self):
        return self.storage.device

    @property
    def origin_ptr(self) -> int:
        return self.storage.data_ptr() + 8 * self.offset

    def abi(self) -> _lib.sb_array:
        nx, ny, nz = self.extents
        return _lib.sb_array(self.origin_ptr, self.sy, self.sz, nx, ny, nz, self.ghost, self.xpad)

    def full(self):
        """(nz+2g, ny+2g, nx+2g) strided view including ghosts."""
        nx, ny, nz = self.extents
        g = self.ghost
        return self.storage.as_strided((nz + 2 * g, ny + 2 * g, nx + 2 * g), (self.sz, self.sy, 1),
                                       self.offset - g - g * self.sy - g * self.sz)

    def interior(self):
        nx, ny, nz = self.extents
        return self.storage.as_strided((nz, ny, nx), (self.sz, self.sy, 1), self.offset)

    def nbytes_interior(self) -> int:
        nx, ny, nz = self.extents
        return 8 * nx * ny * nz

    def nbytes_ghosted(self) -> int:
        nx, ny, nz = self.extents
        g = 2 * self.ghost
        return 8 * (nx + g) * (ny + g) * (nz + g)

    # -- transfers (through the C ABI: cudaMemcpy2DAsync on the torch stream) ---
    def upload(self, host: np.ndarray, with_ghosts: bool | None = None, stream=None) -> None:
        a = np.ascontiguousarray(host, dtype=np.float64)
        nx, ny, nz = self.extents
        g = self.ghost
        if with_ghosts is None:
            with_ghosts = a.shape == (nz + 2 * g, ny + 2 * g, nx + 2 * g) and g > 0
        want = (nz + 2 * g, ny + 2 * g, nx + 2 * g) if with_ghosts else (nz, ny, nx)
        if a.shape != want:
            raise UsageError(f"host array shape {a.shape} != {want}")
        _lib.call("sb_copy_h2d", self.abi(), a.ctypes.data, int(bool(with_ghosts)), _stream_ptr(stream))
        _sync(stream)   # pageable host memory: keep `a` alive until the copy is done

    def upload_from_ptr(self, host_ptr: int, with_ghosts: bool, stream=None) -> None:
        """Asynchronous copy from (pinned) host memory the caller keeps alive."""
        _lib.call("sb_copy_h2d", self.abi(), int(host_ptr), int(bool(with_ghosts)), _stream_ptr(stream))

    def download_to_ptr(self, host_ptr: int, with_ghosts: bool = False, stream=None) -> None:
        _lib.call("sb_copy_d2h", int(host_ptr), self.abi(), int(bool(with_ghosts)), _stream_ptr(stream))

    def upload_planes_from_ptr(self, host_ptr: int, with_ghosts: bool, p0: int, p1: int, stream=None) -> None:
        """Asynchronous copy of host planes [p0, p1) (host plane numbering)."""
        _lib.call("sb_copy_h2d_planes", self.abi(), int(host_ptr), int(bool(with_ghosts)), int(p0), int(p1),
                  _stream_ptr(stream))

    def upload_planes_staged(self, host_ptr: int, staging, with_ghosts: bool, p0: int, p1: int,
                             stream=None) -> None:
        """Host planes [p0, p1) via a dense device staging tensor (linear H2D at
        full link speed + on-device unpack into the padded rows)."""
        _lib.call("sb_copy_h2d_planes_staged", self.abi(), int(host_ptr), int(staging.data_ptr()),
                  int(bool(with_ghosts)), int(p0), int(p1), _stream_ptr(stream))

    def staging_buffer(self, with_ghosts: bool = True):
        import torch
        nx, ny, nz = self.extents
        g = self.ghost if with_ghosts else 0
        return torch.empty((nz + 2 * g) * (ny + 2 * g) * (nx + 2 * g), dtype=torch.float64, device=self.device)

    def download_planes_to_ptr(self, host_ptr: int, with_ghosts: bool, p0: int, p1: int, stream=None) -> None:
        _lib.call("sb_copy_d2h_planes", int(host_ptr), self.abi(), int(bool(with_ghosts)), int(p0), int(p1),
                  _stream_ptr(stream))

    def download(self, with_ghosts: bool = False, stream=None) -> np.ndarray:
        nx, ny, nz = self.extents
        g = self.ghost if with_ghosts else 0
        out = np.empty((nz + 2 * g, ny + 2 * g, nx + 2 * g), dtype=np.float64)
        _lib.call("sb_copy_d2h", out.ctypes.data, self.abi(), int(bool(with_ghosts)), _stream_ptr(stream))
        _sync(stream)
        return out

    def fill_(self, value: float) -> "DeviceGrid":
        self.storage.fill_(value)
        return self


def _stream_ptr(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _sync(stream) -> None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    s.synchronize()


def stream_ptr(stream=None) -> int:
    return _stream_ptr(stream)
