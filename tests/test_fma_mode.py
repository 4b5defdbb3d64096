"""Tolerance mode (STENCIL_B200_MODE=fma): the same kernels built with FMA
contraction (north_star: bit-exact without FMA, otherwise max relative error
<= 1e-13 in fp64; the reference's FUSED_FMA switch, vlanes.py:33).  The
default library stays bit-exact; this mode is opt-in."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
TOLERANCE = 1e-13   # normwise: max|got - want| / max|want|, per output array


def test_mode_selects_the_fma_library(monkeypatch):
    from paper_1308_1343_b200 import _lib
    from paper_1308_1343_b200.errors import UsageError
    monkeypatch.delenv("STENCIL_B200_LIB", raising=False)
    monkeypatch.setenv("STENCIL_B200_MODE", "fma")
    assert _lib.library_path().name == "libstencil_b200_fma.so"
    monkeypatch.setenv("STENCIL_B200_MODE", "exact")
    assert _lib.library_path().name == "libstencil_b200.so"
    monkeypatch.setenv("STENCIL_B200_MODE", "fast")
    with pytest.raises(UsageError):
        _lib.library_path()


def _check(mode: str) -> dict:
    env = dict(os.environ, STENCIL_B200_MODE=mode)
    env.pop("STENCIL_B200_LIB", None)
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "fma_check.py")], capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_fma_mode_within_tolerance_and_active():
    res = _check("fma")
    assert res["library"] == "libstencil_b200_fma.so"
    assert res["max_error"] <= TOLERANCE, {k: v for k, v in res["errors"].items() if v > TOLERANCE}
    assert not res["all_bit_identical"]          # the contraction really happened


@pytest.mark.gpu
def test_exact_mode_is_bit_identical():
    res = _check("exact")
    assert res["all_bit_identical"] and res["max_error"] == 0.0
