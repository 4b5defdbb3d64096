"""examples/c_abi_demo.c: the library driven from plain C through
include/stencil_b200.h (no Python, no torch in the loop) — it compiles and
links here; on a B200 its sweeps are byte-identical to the same expression
trees evaluated in C on the host."""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def _build(out: Path) -> None:
    from paper_1308_1343_b200 import _build as b
    lib = b.build()
    if shutil.which("gcc") is None or not (CUDA / "include" / "cuda_runtime.h").exists():
        pytest.skip("gcc or the CUDA headers are not available")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-ffp-contract=off", "-I", str(ROOT / "include"), "-I",
           str(CUDA / "include"), str(ROOT / "examples" / "c_abi_demo.c"), "-L", str(lib.parent), "-lstencil_b200",
           "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{lib.parent}:{CUDA / 'lib64'}", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_example_builds_against_the_header(tmp_path):
    _build(tmp_path / "c_abi_demo")
    assert (tmp_path / "c_abi_demo").exists()


@pytest.mark.gpu
def test_c_example_sweeps_are_bit_identical(tmp_path):
    exe = tmp_path / "c_abi_demo"
    _build(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("bit-identical") == 2, r.stdout
