"""Build libstencil_b200.so in-tree with nvcc for sm_100a.

The library is compiled with -fmad=false so no a*b+c in the kernels is ever
contracted into an FMA: the reference's unfused-FMA contract
(vlanes.py:33, vlanes.py:243-249) and numpy's one-rounding-per-op
evaluation (stencil.py:35-39) are what parity is measured against.
STENCIL_B200_MODE=fma selects the tolerance mode instead
(libstencil_b200_fma.so: plain operators, -fmad=true; north_star's "max
relative error <= 1e-13" alternative, the reference's FUSED_FMA switch).
cudart is linked statically (like NCCL does), so the library carries no
runtime-library version dependency beside the driver.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libstencil_b200.so"
SOURCES = ["abi.cu", "lap7.cu", "d4.cu", "rkpair.cu", "ghost.cu", "rhs24.cu", "regions.cu"]
HEADERS = ["common.cuh", "internal.h", "stencil_ops.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libstencil_b200.so")


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE / "stencil_b200.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, variant: str | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Compile every CUDA source and link the shared library (no-op if fresh).

    ``variant``/``defines`` build an experimental copy
    (libstencil_b200_<variant>.so, selected at run time with
    STENCIL_B200_LIB) for A/B measurements; the product library is the
    default build."""
    if variant is None and os.environ.get("STENCIL_B200_MODE") == "fma":
        # tolerance mode: the same sources with FMA contraction (SB_FMA, -fmad=true)
        return build(force, verbose, ptxas_info, "fma", tuple(defines) + ("SB_FMA=1",))
    lib = LIB if variant is None else PKG / f"libstencil_b200_{variant}.so"
    if (variant is None or variant == "fma") and not force and not ptxas_info and not _stale(lib):
        return lib
    cc = nvcc()
    objdir = PKG / ("build" if variant is None else f"build_{variant}")
    objdir.mkdir(exist_ok=True)
    def compile_one(src: str):
        obj = objdir / (src + ".o")
        flags = [("-fmad=true" if f == "-fmad=false" and "SB_FMA=1" in defines else f) for f in NVCC_FLAGS]
        cmd = [cc, *flags, *[f"-D{d}" for d in defines], "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)]
        if ptxas_info:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    # the translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    objs = []
    for src, obj, r in results:
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if ptxas_info and r.stderr:
            print(r.stderr, file=sys.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", *objs, "-o", str(tmp)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
