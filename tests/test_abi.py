"""The C-ABI library builds, loads without a GPU, exports exactly the symbols
include/stencil_b200.h declares, and rejects contract violations with the
reference's error classes before touching the device."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1308_1343_b200 import _build, _lib
from paper_1308_1343_b200.errors import UsageError

HEADER = Path(__file__).resolve().parent.parent / "include" / "stencil_b200.h"


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def test_header_and_binding_agree():
    declared = set(re.findall(r"^\s*SB_API\s+(?:int|const char \*)\s*(sb_\w+)\s*\(", HEADER.read_text(), re.M))
    assert declared == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in _lib.EXPORTS:
        assert hasattr(lib, name), name
    assert lib.sb_abi_version() == _lib.SB_ABI_VERSION == 2


def test_struct_layouts_match_header():
    assert C.sizeof(_lib.sb_array) == 8 + 8 + 8 + 5 * 4 + 4   # padded to 8
    assert C.sizeof(_lib.sb_space) == 24
    assert C.sizeof(_lib.sb_launch) == 16
    assert C.sizeof(_lib.sb_box_job) == 2 * C.sizeof(_lib.sb_array) + 24
    assert C.sizeof(_lib.sb_rk4_fields) == 8 * C.sizeof(_lib.sb_array)


def test_usage_errors_are_raised_without_a_device(lib):
    bad = _lib.sb_array()            # null origin
    with pytest.raises(UsageError, match="null origin"):
        _lib.call("sb_lap7", bad, bad, _lib.space((0, 0, 0), (1, 1, 1)), 0.0, 0.0, _lib.launch(64, 8, 8), None)
    with pytest.raises(UsageError, match="kind"):
        _lib.call("sb_diff1d", 7, None, None, 4, None)
    with pytest.raises(UsageError, match="stage"):
        f = _lib.sb_rk4_fields()
        _lib.call("sb_rk4_stage", 5, C.byref(f), _lib.space((0, 0, 0), (1, 1, 1)), _lib.sb_rk4_constants(),
                  _lib.launch(64, 8, 8), None)


def test_geometry_contract(lib):
    # misaligned origin and a ghost narrower than the stencil radius
    a = _lib.sb_array(8, 32, 32 * 8, 4, 4, 4, 1, 16)
    with pytest.raises(UsageError, match="aligned"):
        _lib.call("sb_ghost_periodic", a, None)
    b = _lib.sb_array(1024, 32, 32 * 6, 4, 4, 4, 1, 16)
    with pytest.raises(UsageError, match="ghost width 1 < stencil radius 2"):
        outs = (_lib.sb_array * 10)(*([b] * 10))
        _lib.call("sb_d4_all", outs, b, _lib.space((0, 0, 0), (4, 4, 4)), _lib.sb_d4_constants(1, 1, 1),
                  _lib.launch(64, 4, 4), None)
    c = _lib.sb_array(1024, 32, 32 * 8, 4, 4, 4, 2, 16)
    with pytest.raises(UsageError, match="inverted"):
        _lib.call("sb_lap7", c, c, _lib.space((0, 0, 3), (4, 4, 1)), 0.0, 0.0, _lib.launch(64, 8, 8), None)
