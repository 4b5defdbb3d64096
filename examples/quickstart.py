"""Quickstart: the reference's loop-iterator API driving B200 kernels.

    python examples/quickstart.py

1. the reference demo's 7-point Jacobi loop through ``run_loop`` + ``Tuner``
   (one launch per sweep, CUDA-event seconds, the reference's tuner);
2. a bboxset level (a box minus its upper octant) swept by the 4th-order
   Laplacian, all boxes in one launch, after an inter-box ghost fill;
3. one classical RK4 step of the periodic wave equation (stage pairs);
4. the ten 4th-order derivatives of a box straight from / to host memory.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1308_1343_b200 import inputs  # noqa: E402
from paper_1308_1343_b200.grid import DeviceGrid  # noqa: E402
from paper_1308_1343_b200.kernels import (FourthOrderAll, LevelGhostSync, LevelLaplacian4, Laplacian7,  # noqa: E402
                                          WaveRK4)
from paper_1308_1343_b200.level import Box, box_difference  # noqa: E402
from paper_1308_1343_b200.traverse import IndexSpace, run_loop  # noqa: E402
from paper_1308_1343_b200.tuner import TopologyConfig, Tuner, device_setup  # noqa: E402


def jacobi(n: int = 66, iters: int = 50) -> float:
    """stencil.py:80-94 (run_tuned) with device grids: returns the best seconds per sweep."""
    field = np.random.default_rng(20130715).random((n, n, n))
    a = DeviceGrid((n - 2,) * 3, 1, lower=(1, 1, 1))
    b = DeviceGrid((n - 2,) * 3, 1, lower=(1, 1, 1))
    a.upload(field, with_ghosts=True)
    b.upload(field, with_ghosts=True)
    space = IndexSpace((1, 1, 1), (n - 1, n - 1, n - 1))
    k_ab, k_ba = Laplacian7(b, a, -6.0 / 8.0, 1.0 / 8.0), Laplacian7(a, b, -6.0 / 8.0, 1.0 / 8.0)
    setup = device_setup(k_ab, space.extents)       # tuning key: site, extents, grid pitch, SM count
    tuner = Tuner(TopologyConfig())
    for _ in range(iters):
        # graphed: each tuned execution replays a per-launch-shape CUDA graph,
        # so the tuner times the sweep itself, not the Python launch path
        run_loop(setup, space, k_ab, tuner, graphed=True)
        k_ab, k_ba = k_ba, k_ab
    return tuner.best(setup)[1]


def level(n: int = 64) -> list[np.ndarray]:
    """A bboxset level: [0,n)^3 minus its upper octant, 3 boxes, ghost 2."""
    outer, hole = inputs.c4_outer_and_hole(n)
    boxes = box_difference(Box(*outer), Box(*hole))
    rng = np.random.default_rng(7)
    srcs, dsts = [], []
    for b in boxes:
        s = DeviceGrid(b.extents, 2, lower=b.lo)
        s.upload(rng.uniform(-1, 1, (b.extents[2], b.extents[1], b.extents[0])))   # interior only
        srcs.append(s)
        dsts.append(DeviceGrid(b.extents, 0, lower=b.lo))
    LevelGhostSync(srcs, boxes)()        # ghosts that lie inside other boxes of the level
    k = LevelLaplacian4(dsts, srcs, inputs.D4Constants.for_spacing(1.0 / n))
    k.launch(None, k.default_params)     # every box, one launch
    return [d.download() for d in dsts]


def wave(n: int = 48) -> tuple[np.ndarray, np.ndarray]:
    phi, pi = inputs.c3_fields(n, 2, seed=1)
    rk = WaveRK4(n, 2, inputs.WaveConstants.for_grid(n))
    rk.phi0.upload(phi, with_ghosts=True)
    rk.pi0.upload(pi, with_ghosts=True)
    rk.fill_ghosts(rk.phi0)
    rk.fill_ghosts(rk.pi0)
    rk.advance()                          # one RK4 step; the new state becomes phi0 / pi0
    return rk.phi0.download(), rk.pi0.download()


def derivatives_from_host(n: int = 64) -> list[np.ndarray]:
    import torch
    u = inputs.c2_field(n, 2, seed=3)
    src = DeviceGrid((n,) * 3, 2)
    outs = [DeviceGrid((n,) * 3, 0) for _ in range(10)]
    k = FourthOrderAll(outs, src, inputs.D4Constants.for_spacing(1.0 / n))
    h_in = torch.from_numpy(u).pin_memory()
    h_out = [torch.empty((n, n, n), dtype=torch.float64).pin_memory() for _ in range(10)]
    k.run_host(h_in.data_ptr(), [t.data_ptr() for t in h_out])
    torch.cuda.synchronize()
    return [t.numpy() for t in h_out]


if __name__ == "__main__":
    print(f"jacobi: best {jacobi() * 1e6:.1f} us per sweep (tuned; each execution an isolated graph-replayed"
          " launch; stencil.run_graphed replays the whole loop from one CUDA graph at ~2 us per sweep)")
    print(f"level: {len(level())} boxes swept")
    phi, pi = wave()
    print(f"wave: |phi| max {np.abs(phi).max():.6f}, |pi| max {np.abs(pi).max():.3e}")
    print(f"derivatives: {len(derivatives_from_host())} outputs back on the host")
