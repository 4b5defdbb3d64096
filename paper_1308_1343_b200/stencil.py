"""The reference's stencil demo, running on the B200.

Same drivers and semantics as ``pkg/src/stencilrt/stencil.py``: a Jacobi
7-point update per iteration, boundary carried over, run serially
(:55-65), with the naive static split (:68-77) and tuned (:80-94), and the
``bit_identical`` predicate (:97-98).  The field is generated on the host
(``make_field``, :26-28) and uploaded once; the two device buffers ping-pong
(``dst = src.copy()`` at :59 only carries the boundary over, which the
second buffer already holds), and ``iter_seconds`` are CUDA-event times of
the sweep.  Index spaces are the reference's array indices
``IndexSpace((1,1,1), (n-1,n-1,n-1))``.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .grid import DeviceGrid
from .kernels import Laplacian7
from .traverse import IndexSpace, _Timer, run_loop, run_static
from .tuner import TopologyConfig, Tuner, device_setup

C0 = -6.0 / 8.0
C1 = 1.0 / 8.0


def make_field(n: int, seed: int) -> np.ndarray:
    """stencil.py:26-28."""
    return np.random.default_rng(seed).random((n, n, n), dtype=np.float64)


@dataclass
class StencilRun:
    final: np.ndarray
    iter_seconds: list[float] = field(default_factory=list)


def _buffers(n: int, seed: int):
    host = make_field(n, seed)
    a = DeviceGrid((n - 2,) * 3, 1, lower=(1, 1, 1))
    b = DeviceGrid((n - 2,) * 3, 1, lower=(1, 1, 1))
    a.upload(host, with_ghosts=True)
    b.upload(host, with_ghosts=True)
    return a, b


def _space(n: int) -> IndexSpace:
    return IndexSpace((1, 1, 1), (n - 1, n - 1, n - 1))


def run_serial(n: int, iters: int, seed: int, c0: float = C0, c1: float = C1) -> StencilRun:
    src, dst = _buffers(n, seed)
    out = StencilRun(np.empty(0))
    space = _space(n)
    for _ in range(iters):
        k = Laplacian7(dst, src, c0, c1)
        with _Timer(True) as tm:
            k.launch(space, k.default_params)
        out.iter_seconds.append(tm.elapsed())
        src, dst = dst, src
    out.final = src.download(with_ghosts=True)
    return out


def run_naive(n: int, iters: int, seed: int, n_threads: int, c0: float = C0, c1: float = C1) -> StencilRun:
    src, dst = _buffers(n, seed)
    out = StencilRun(np.empty(0))
    space = _space(n)
    for _ in range(iters):
        out.iter_seconds.append(run_static(space, Laplacian7(dst, src, c0, c1), n_threads))
        src, dst = dst, src
    out.final = src.download(with_ghosts=True)
    return out


def run_tuned(n: int, iters: int, seed: int, topo: TopologyConfig, c0: float = C0,
              c1: float = C1, graphed: bool = True) -> tuple[StencilRun, Tuner]:
    """stencil.py:80-94 on the device.  The tuning key adds the grid pitch and
    SM count (tuner.device_setup); with ``graphed`` (default) every tuned
    execution replays a per-launch-shape CUDA graph, so the tuner times the
    sweep itself, not the host launch path (traverse.run_loop)."""
    src, dst = _buffers(n, seed)
    out = StencilRun(np.empty(0))
    space = _space(n)
    k_ab, k_ba = Laplacian7(dst, src, c0, c1), Laplacian7(src, dst, c0, c1)
    setup = replace(device_setup(k_ab, space.extents), n_coarse_threads=topo.n_coarse_threads,
                    n_fine_threads=topo.n_fine_threads)
    tuner = Tuner(topo)
    for _ in range(iters):
        out.iter_seconds.append(run_loop(setup, space, k_ab, tuner, graphed=graphed))
        k_ab, k_ba = k_ba, k_ab
        src, dst = dst, src
    out.final = src.download(with_ghosts=True)
    return out, tuner


def run_graphed(n: int, iters: int, seed: int, c0: float = C0, c1: float = C1, batch: int = 50) -> StencilRun:
    """``run_serial`` with the sweep loop captured in a CUDA graph: one graph
    holds ``batch`` ping-pong pairs (2*batch sweeps); iter_seconds are the
    per-sweep averages of each replay (CUDA events)."""
    from .graphs import SweepGraph
    if iters % 2:
        raise ValueError("run_graphed needs an even iteration count (ping-pong pairs)")
    a, b = _buffers(n, seed)
    space = _space(n)
    ka, kb = Laplacian7(b, a, c0, c1), Laplacian7(a, b, c0, c1)

    def pair():
        ka.launch(space, ka.default_params)
        kb.launch(space, kb.default_params)

    out = StencilRun(np.empty(0))
    pairs = iters // 2
    # the warm-up pair inside SweepGraph advances the state; start from the field again
    g = SweepGraph(pair, repeat=min(batch, max(1, pairs)), warmup=1)
    host = make_field(n, seed)
    a.upload(host, with_ghosts=True)
    b.upload(host, with_ghosts=True)
    done = 0
    while done < pairs:
        if pairs - done >= g.repeat:
            with _Timer(True) as tm:
                g.replay()
            out.iter_seconds += [tm.elapsed() / (2 * g.repeat)] * (2 * g.repeat)
            done += g.repeat
        else:
            with _Timer(True) as tm:
                pair()
            out.iter_seconds += [tm.elapsed() / 2] * 2
            done += 1
    out.final = a.download(with_ghosts=True)
    return out


def run_persistent(n: int, iters: int, seed: int, c0: float = C0, c1: float = C1) -> StencilRun:
    """``run_serial`` as ONE persistent cooperative launch
    (``sb_lap7_iterate``): the CTAs stay resident and meet at a grid barrier
    between sweeps; iter_seconds are the per-sweep average of the launch."""
    a, b = _buffers(n, seed)
    out = StencilRun(np.empty(0))
    if iters > 0:
        k = Laplacian7(b, a, c0, c1)
        with _Timer(True) as tm:
            k.iterate(a, b, _space(n), iters)
        out.iter_seconds = [tm.elapsed() / iters] * iters
    out.final = (b if iters % 2 else a).download(with_ghosts=True)
    return out


def bit_identical(a: np.ndarray, b: np.ndarray) -> bool:
    """stencil.py:97-98."""
    return a.shape == b.shape and a.tobytes() == b.tobytes()
