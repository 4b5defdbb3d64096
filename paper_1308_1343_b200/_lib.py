"""ctypes binding of libstencil_b200.so (include/stencil_b200.h).

This is the only place Python touches the C ABI.  Every entry point returns
a status; ``call`` maps SB_USAGE -> UsageError, SB_RESOURCE -> ResourceError,
SB_CUDA -> DeviceError (the reference's error split, lattice.py:22-27), with
the library's thread-local message.  There is no fallback: if the library
cannot be loaded the hot path raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DeviceError, ResourceError, UsageError

LIB_PATH = Path(__file__).resolve().parent / "libstencil_b200.so"

SB_OK, SB_USAGE, SB_RESOURCE, SB_CUDA = 0, 1, 2, 3
SB_ABI_VERSION = 2   # include/stencil_b200.h
SB_MAX_BOXES = 8
SB_N_D4_OUT = 10
SB_N_VARS = 24
SB_N_TERMS = 64

# every symbol include/stencil_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "sb_abi_version", "sb_last_error", "sb_init", "sb_get_device_info", "sb_diff1d",
    "sb_lap7", "sb_d4_all", "sb_d2_all", "sb_lap4_boxes", "sb_ghost_periodic", "sb_rk4_stage",
    "sb_rhs24", "sb_copy_regions", "sb_copy_h2d", "sb_copy_d2h", "sb_copy_h2d_planes", "sb_copy_d2h_planes",
    "sb_copy_h2d_planes_staged", "sb_rk4_stage_zslab", "sb_rk4_pair", "sb_rk4_pair_zslab", "sb_lap7_iterate",
    "sb_d4_all_boxes", "sb_d2_all_boxes", "sb_rk4_stage_boxes", "sb_release_tables", "sb_enable_peer_access",
    "sb_shutdown",
)
SB_MAX_COPY_JOBS = 64


class sb_array(C.Structure):
    _fields_ = [("origin", C.c_void_p), ("sy", C.c_int64), ("sz", C.c_int64),
                ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("ghost", C.c_int32), ("xpad", C.c_int32)]


class sb_space(C.Structure):
    _fields_ = [("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3)]


class sb_launch(C.Structure):
    _fields_ = [("tile_x", C.c_int32), ("tile_y", C.c_int32), ("z_chunk", C.c_int32), ("flags", C.c_int32)]


class sb_d4_constants(C.Structure):
    _fields_ = [("k1", C.c_double), ("k2", C.c_double), ("k11", C.c_double)]


class sb_box_job(C.Structure):
    _fields_ = [("dst", sb_array), ("src", sb_array), ("space", sb_space)]


class sb_rk4_fields(C.Structure):
    _fields_ = [(n, sb_array) for n in ("phi_s", "pi_s", "phi0", "pi0", "acc_phi", "acc_pi", "phi_out", "pi_out")]


class sb_d4_all_job(C.Structure):
    _fields_ = [("out", sb_array * 10), ("src", sb_array), ("space", sb_space)]


class sb_rk4_box_job(C.Structure):
    _fields_ = [("f", sb_rk4_fields), ("space", sb_space)]


class sb_rk4_constants(C.Structure):
    _fields_ = [("lap", sb_d4_constants), ("half_dt", C.c_double), ("dt", C.c_double), ("dt6", C.c_double)]


class sb_zslab(C.Structure):
    _fields_ = [("lo_phi_out", C.c_void_p), ("lo_dz", C.c_int32), ("hi_phi_out", C.c_void_p), ("hi_dz", C.c_int32)]


class sb_poly(C.Structure):
    _fields_ = [("coef", C.c_void_p), ("p", C.c_void_p), ("q", C.c_void_p)]


class sb_copy_job(C.Structure):
    _fields_ = [("dst", sb_array), ("src", sb_array), ("dst_lo", C.c_int32 * 3), ("src_lo", C.c_int32 * 3),
                ("ext", C.c_int32 * 3)]


class sb_device_info(C.Structure):
    _fields_ = [("device", C.c_int32), ("sm_count", C.c_int32), ("cc_major", C.c_int32), ("cc_minor", C.c_int32),
                ("l2_bytes", C.c_int64), ("smem_optin_bytes", C.c_int64), ("global_mem_bytes", C.c_int64)]


_lib = None
_lock = threading.Lock()


def _declare(lib) -> None:
    vp, i32 = C.c_void_p, C.c_int32
    sig = {
        "sb_abi_version": ([], C.c_int),
        "sb_last_error": ([], C.c_char_p),
        "sb_init": ([C.c_int], C.c_int),
        "sb_get_device_info": ([C.POINTER(sb_device_info)], C.c_int),
        "sb_diff1d": ([i32, vp, vp, i32, vp], C.c_int),
        "sb_lap7": ([sb_array, sb_array, sb_space, C.c_double, C.c_double, sb_launch, vp], C.c_int),
        "sb_lap7_iterate": ([sb_array, sb_array, sb_space, C.c_double, C.c_double, i32, sb_launch, vp], C.c_int),
        "sb_d4_all": ([C.POINTER(sb_array), sb_array, sb_space, sb_d4_constants, sb_launch, vp], C.c_int),
        "sb_d2_all": ([C.POINTER(sb_array), sb_array, sb_space, sb_d4_constants, sb_launch, vp], C.c_int),
        "sb_lap4_boxes": ([C.POINTER(sb_box_job), i32, sb_d4_constants, sb_launch, vp], C.c_int),
        "sb_d4_all_boxes": ([C.POINTER(sb_d4_all_job), i32, sb_d4_constants, sb_launch, vp], C.c_int),
        "sb_d2_all_boxes": ([C.POINTER(sb_d4_all_job), i32, sb_d4_constants, sb_launch, vp], C.c_int),
        "sb_rk4_stage_boxes": ([i32, C.POINTER(sb_rk4_box_job), i32, sb_rk4_constants, sb_launch, vp], C.c_int),
        "sb_release_tables": ([], C.c_int),
        "sb_shutdown": ([], C.c_int),
        "sb_enable_peer_access": ([C.c_int], C.c_int),
        "sb_ghost_periodic": ([sb_array, vp], C.c_int),
        "sb_rk4_stage": ([i32, C.POINTER(sb_rk4_fields), sb_space, sb_rk4_constants, sb_launch, vp], C.c_int),
        "sb_rk4_pair": ([i32, C.POINTER(sb_rk4_fields), sb_space, sb_rk4_constants, sb_launch, vp], C.c_int),
        "sb_rk4_pair_zslab": ([i32, C.POINTER(sb_rk4_fields), sb_space, sb_rk4_constants, sb_launch,
                               C.POINTER(sb_zslab), vp], C.c_int),
        "sb_rk4_stage_zslab": ([i32, C.POINTER(sb_rk4_fields), sb_space, sb_rk4_constants, sb_launch,
                                C.POINTER(sb_zslab), vp], C.c_int),
        "sb_rhs24": ([C.POINTER(sb_array), C.POINTER(sb_array), sb_space, sb_d4_constants, sb_poly, sb_launch, vp],
                     C.c_int),
        "sb_copy_regions": ([C.POINTER(sb_copy_job), i32, vp], C.c_int),
        "sb_copy_h2d": ([sb_array, vp, i32, vp], C.c_int),
        "sb_copy_d2h": ([vp, sb_array, i32, vp], C.c_int),
        "sb_copy_h2d_planes": ([sb_array, vp, i32, i32, i32, vp], C.c_int),
        "sb_copy_d2h_planes": ([vp, sb_array, i32, i32, i32, vp], C.c_int),
        "sb_copy_h2d_planes_staged": ([sb_array, vp, vp, i32, i32, i32, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def library_path() -> Path:
    """The library this process uses: ``STENCIL_B200_LIB`` if set; else the
    tolerance-mode build (FMA contraction, ``libstencil_b200_fma.so``) when
    ``STENCIL_B200_MODE=fma``; else the bit-exact product library."""
    if os.environ.get("STENCIL_B200_LIB"):
        return Path(os.environ["STENCIL_B200_LIB"])
    mode = os.environ.get("STENCIL_B200_MODE", "exact")
    if mode == "fma":
        return Path(LIB_PATH).with_name("libstencil_b200_fma.so")
    if mode != "exact":
        raise UsageError(f"STENCIL_B200_MODE must be 'exact' or 'fma', not {mode!r}")
    return Path(LIB_PATH)


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path) if path else library_path()
            if not p.exists():
                raise DeviceError(f"{p} not built; run __graft_entry__.build() (no CPU fallback exists)")
            lib = C.CDLL(str(p))
            _declare(lib)
            if lib.sb_abi_version() != SB_ABI_VERSION:
                raise DeviceError(f"{p} has ABI version {lib.sb_abi_version()}, this package needs "
                                  f"{SB_ABI_VERSION}: rebuild it (__graft_entry__.build())")
            _lib = lib
        return _lib


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc == SB_OK:
        return
    msg = (lib.sb_last_error() or b"").decode(errors="replace")
    if rc == SB_USAGE:
        raise UsageError(f"{name}: {msg}")
    if rc == SB_RESOURCE:
        raise ResourceError(f"{name}: {msg}")
    raise DeviceError(f"{name}: {msg} (status {rc})")


_inited: set[int] = set()


def shutdown() -> None:
    """sb_shutdown: free the library-owned device memory (box tables, barrier
    counters); the next use on a device re-initialises it."""
    call("sb_shutdown")
    _inited.clear()


def init_current_device() -> None:
    """sb_init on torch's current device, once per device (reserves the
    library's per-device scratch, e.g. sb_lap7_iterate's barrier counters,
    outside any CUDA-graph capture)."""
    import torch
    dev = torch.cuda.current_device()
    if dev not in _inited:
        call("sb_init", dev)
        _inited.add(dev)


def space(lo, hi) -> sb_space:
    s = sb_space()
    for d in range(3):
        s.lo[d] = int(lo[d])
        s.hi[d] = int(hi[d])
    return s


SB_LAUNCH_SCALAR = 1
SB_LAUNCH_PERIODIC_GHOSTS = 2


def launch(tile_x: int, tile_y: int, z_chunk: int, points_per_thread: int = 2, flags: int = 0) -> sb_launch:
    if points_per_thread == 1:
        flags |= SB_LAUNCH_SCALAR
    return sb_launch(int(tile_x), int(tile_y), int(z_chunk), int(flags))


def launch_of(p, flags: int = 0) -> sb_launch:
    """sb_launch of a tuner.LaunchParams (plus extra SB_LAUNCH_* flags)."""
    return launch(p.tile_x, p.tile_y, p.z_chunk, getattr(p, "points_per_thread", 2), flags)


def d4_constants(k) -> sb_d4_constants:
    return sb_d4_constants(float(k.k1), float(k.k2), float(k.k11))
