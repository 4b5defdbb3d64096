"""The C ABI used the way INTEGRATION.md §2 tells a reference maintainer to
bind it: plain ctypes on libstencil_b200.so with locally declared structs —
no package wrappers — device memory from torch, the reference demo's
``_update_rows`` replaced by ``sb_lap7`` on its array-index space."""
import ctypes as C

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


class sb_array(C.Structure):
    _fields_ = [("origin", C.c_void_p), ("sy", C.c_int64), ("sz", C.c_int64),
                ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("ghost", C.c_int32), ("xpad", C.c_int32)]


class sb_space(C.Structure):
    _fields_ = [("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3)]


class sb_launch(C.Structure):
    _fields_ = [("tile_x", C.c_int32), ("tile_y", C.c_int32), ("z_chunk", C.c_int32), ("flags", C.c_int32)]


@pytest.fixture(scope="module")
def lib():
    from paper_1308_1343_b200 import _build
    lib = C.CDLL(str(_build.build()))
    lib.sb_lap7.argtypes = [sb_array, sb_array, sb_space, C.c_double, C.c_double, sb_launch, C.c_void_p]
    lib.sb_lap7.restype = C.c_int
    lib.sb_last_error.restype = C.c_char_p
    return lib


def _padded(u, g=1):
    """Device copy of a ghosted (n+2g)^3 array with rows padded to an even
    pitch and 2 elements before x = 0, so the interior origin is 16-byte
    aligned (the ABI's layout contract, include/stencil_b200.h)."""
    import torch
    m = u.shape[0]
    xpad, pitch = 2, m + 2 + (m % 2)
    buf = torch.zeros((m, m, pitch), dtype=torch.float64, device="cuda")
    buf[:, :, xpad - g:xpad - g + m] = torch.from_numpy(u).cuda()
    n = m - 2 * g
    arr = sb_array(buf.data_ptr() + 8 * (xpad + g * pitch + g * pitch * m), pitch, pitch * m, n, n, n, g, xpad)
    return buf, arr, xpad - g


def test_ctypes_binding_replaces_update_rows(lib):
    import torch
    n = 16                                       # the reference demo's array is 18^3: 16^3 interior
    u = np.random.default_rng(20130715).random((n + 2,) * 3)
    src_buf, src, x0 = _padded(u)
    dst_buf, dst, _ = _padded(u)
    space = sb_space((0, 0, 0), (n, n, n))       # interior-relative indices of both grids
    c0, c1 = -6.0 / 8.0, 1.0 / 8.0
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.sb_lap7(dst, src, space, c0, c1, sb_launch(64, 8, 16, 0), stream)
    assert rc == 0, lib.sb_last_error()
    torch.cuda.synchronize()
    want = u.copy()
    oracle.lap7_rows(want, u, 1, n + 1, 1, n + 1, 1, n + 1, c0, c1)
    got = dst_buf[:, :, x0:x0 + n + 2].cpu().numpy()
    assert np.ascontiguousarray(got).tobytes() == want.tobytes()


def test_ctypes_binding_reports_usage_errors(lib):
    import torch
    n = 8
    u = np.zeros((n + 2,) * 3)
    a_buf, a, _ = _padded(u)
    b_buf, b, _ = _padded(u)
    rc = lib.sb_lap7(b, a, sb_space((0, 0, 0), (n, n, n)), 1.0, 1.0, sb_launch(64, 99, 16, 0), None)
    assert rc == 1 and b"tile_y" in lib.sb_last_error()
    a.origin = a.origin + 8                      # misaligned origin: a usage error, not a fault
    rc = lib.sb_lap7(b, a, sb_space((0, 0, 0), (n, n, n)), 1.0, 1.0, sb_launch(64, 8, 16, 0), None)
    assert rc == 1 and b"aligned" in lib.sb_last_error()
    torch.cuda.synchronize()
