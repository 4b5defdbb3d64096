"""The five BASELINE.json workloads as device problems.

Each problem owns its device grids, uploads its seeded host inputs
(inputs.py) once, and runs one "step" (one pass of the hot path over its
data) through the kernels of kernels.py.  ``updates`` and
``canonical_bytes`` are the per-step figures of SURVEY.md §8(d): every array
the algorithm must read is counted once (ghosted size if its ghosts feed a
stencil) and every array it must write once (interior size); padding never
counts.
"""
from __future__ import annotations

import numpy as np

from . import inputs
from .grid import DeviceGrid
from .kernels import FourthOrderAll, Laplacian7, LevelGhostSync, LevelLaplacian4, Rhs24, WaveRK4
from .level import Box, box_difference
from .traverse import IndexSpace
from .tuner import LaunchParams


def _vol(ext, g=0) -> int:
    v = 1
    for e in ext:
        v *= e + 2 * g
    return v


class C1Laplacian7:
    """Config 1: 7-point 2nd-order Laplacian of one 64^3 box (ghost 1), h = 1/64."""

    name = "c1_lap7"

    def __init__(self, n: int = 64, seed: int | None = None):
        self.n = n
        self.host_u = inputs.c1_field(n, seed)
        self.c0, self.c1 = inputs.c1_constants(n)
        self.updates = n ** 3
        self.canonical_bytes = 8 * (_vol((n,) * 3, 1) + n ** 3)

    def setup(self, device=None):
        n = self.n
        self.src = DeviceGrid((n,) * 3, 1, device)
        self.dst = DeviceGrid((n,) * 3, 0, device)
        self.src.upload(self.host_u, with_ghosts=True)
        self.kernel = Laplacian7(self.dst, self.src, self.c0, self.c1)
        self.space = IndexSpace((0, 0, 0), (n, n, n))
        return self

    def run(self, params: LaunchParams | None = None, stream=None) -> None:
        self.kernel.launch(self.space, params or self.kernel.default_params, stream)

    def outputs(self) -> list[np.ndarray]:
        return [self.dst.download()]


class C2FourthOrder:
    """Config 2: ten 4th-order outputs of one 256^3 box (ghost 2), h = 1/256."""

    name = "c2_d4_all"

    def __init__(self, n: int = 256, seed: int | None = None, g: int = 2):
        self.n, self.g = n, g
        self.host_u = inputs.c2_field(n, g, seed)
        self.k = inputs.D4Constants.for_spacing(1.0 / n)
        self.updates = n ** 3
        self.canonical_bytes = 8 * (_vol((n,) * 3, g) + 10 * n ** 3)

    def setup(self, device=None):
        n = self.n
        self.src = DeviceGrid((n,) * 3, self.g, device)
        self.outs = [DeviceGrid((n,) * 3, 0, device) for _ in range(10)]
        self.src.upload(self.host_u, with_ghosts=True)
        self.kernel = FourthOrderAll(self.outs, self.src, self.k)
        self.space = IndexSpace((0, 0, 0), (n, n, n))
        return self

    def run(self, params: LaunchParams | None = None, stream=None) -> None:
        self.kernel.launch(self.space, params or self.kernel.default_params, stream)

    def outputs(self) -> list[np.ndarray]:
        return [o.download() for o in self.outs]

    # end-to-end through the public API with host buffers
    def e2e_step(self, host_in_ptr: int, host_out_ptrs: list[int], params=None, stream=None,
                 chunk: int | None = 32) -> None:
        if chunk:
            self.kernel.run_host(host_in_ptr, host_out_ptrs, params, chunk)
            return
        self.src.upload_from_ptr(host_in_ptr, True, stream)
        self.run(params, stream)
        for o, p in zip(self.outs, host_out_ptrs):
            o.download_to_ptr(p, False, stream)

    @property
    def h2d_bytes(self) -> int:
        return self.src.nbytes_ghosted()

    @property
    def d2h_bytes(self) -> int:
        return sum(o.nbytes_interior() for o in self.outs)


class C3WaveRK4:
    """Config 3: one classical RK4 step of the scalar wave equation, 384^3
    periodic (ghost 2, refilled before every stage), h = 1/384, dt = h/4."""

    name = "c3_wave_rk4"

    def __init__(self, n: int = 384, seed: int | None = None, g: int = 2, schedule: str = "lap_pairs"):
        self.n, self.g = n, g
        self.schedule = schedule
        self.host_phi, self.host_pi = inputs.c3_fields(n, g, seed)
        self.c = inputs.WaveConstants.for_grid(n)
        self.updates = n ** 3
        # array passes over the interior + the ghost shells of the ghosted reads.
        # SURVEY.md §8(d) counts 34 passes (four stage sweeps); the four-stage
        # schedule here needs 32 (stage 1 does not materialise acc_phi = pi0),
        # the fused pair schedule 14: pair 1 reads phi0, pi0 (ghosted) and
        # writes phi3, pi3, acc_phi, acc_pi; pair 2 reads phi3, phi0, pi3
        # (ghosted), pi0, acc_phi, acc_pi and writes phi', pi'.
        shell = _vol((n,) * 3, g) - n ** 3
        # lap_pairs: pair 1 reads phi0, pi0 (ghosted), writes L1, L2; pair 2
        # reads phi0, pi0, L1, L2 (ghosted) and writes phi', pi'.
        passes, ghosted = {"pairs": (14, 5), "lap_pairs": (10, 6), "stages": (32, 4),
                           "stages_unfused": (32, 4)}[schedule]
        self.canonical_bytes = 8 * (passes * n ** 3 + ghosted * shell)
        self.survey_canonical_bytes = 8 * (34 * n ** 3 + 4 * shell)
        self.ghost_fill_bytes = 8 * 4 * 2 * (_vol((n,) * 3, g) - n ** 3)

    def setup(self, device=None):
        self.rk = WaveRK4(self.n, self.g, self.c, device, schedule=self.schedule)
        self.reset()
        return self

    def reset(self):
        self.rk.phi0.upload(self.host_phi, with_ghosts=True)
        self.rk.pi0.upload(self.host_pi, with_ghosts=True)
        self.rk.fill_ghosts(self.rk.phi0)
        self.rk.fill_ghosts(self.rk.pi0)

    def run(self, params: LaunchParams | None = None, stream=None) -> None:
        self.rk.step(params, stream)

    def outputs(self) -> list[np.ndarray]:
        return [self.rk.phi_b.download(), self.rk.pi_b.download()]

    def phi_with_ghosts(self) -> np.ndarray:
        return self.rk.phi_b.download(with_ghosts=True)


class C4Level:
    """Config 4: 4th-order Laplacian over the bboxset level [0,511]^3 minus its
    upper octant (3 boxes, ghost 2), all boxes in one batched launch."""

    name = "c4_level_lap4"

    def __init__(self, n: int = 512, seed: int | None = None, g: int = 2, boxes=None):
        self.n, self.g = n, g
        if boxes is None:
            outer, hole = inputs.c4_outer_and_hole(n)
            boxes = box_difference(Box(*outer), Box(*hole))
        self.boxes = list(boxes)
        self.host_u = inputs.c4_fields(self.boxes, g, seed)
        self.k = inputs.D4Constants.for_spacing(1.0 / n)
        self.updates = sum(b.volume() for b in self.boxes)
        self.canonical_bytes = 8 * sum(_vol(b.extents, g) + b.volume() for b in self.boxes)

    def setup(self, device=None):
        self.srcs, self.dsts = [], []
        for b, u in zip(self.boxes, self.host_u):
            s = DeviceGrid(b.extents, self.g, device, lower=b.lo)
            s.upload(u, with_ghosts=True)
            self.srcs.append(s)
            self.dsts.append(DeviceGrid(b.extents, 0, device, lower=b.lo))
        self.kernel = LevelLaplacian4(self.dsts, self.srcs, self.k)
        self.ghost_sync = LevelGhostSync(self.srcs, self.boxes)
        return self

    def run(self, params: LaunchParams | None = None, stream=None) -> None:
        self.kernel.launch(None, params or self.kernel.default_params, stream)

    def outputs(self) -> list[np.ndarray]:
        return [d.download() for d in self.dsts]


class C5Rhs24:
    """Config 5: 24 fields on 192^3 (ghost 2); 24 fused 64-term quadratic RHS."""

    name = "c5_rhs24"

    def __init__(self, n: int = 192, seed: int | None = None, g: int = 2):
        self.n, self.g = n, g
        self.host_u = inputs.c5_fields(n, g, seed)
        self.poly = inputs.c5_poly(seed)
        self.k = inputs.D4Constants.for_spacing(1.0 / n)
        self.updates = n ** 3
        self.canonical_bytes = 8 * inputs.N_VARS * (_vol((n,) * 3, g) + n ** 3)
        # algorithmic unfused FP64 operations per step, with every reusable
        # intermediate computed once: per variable and point rx, ry (4 each),
        # Dx, Dy (1 each), Dz (5), Dxx, Dyy, Dzz (7 each), Dxy, Dxz, Dyz (5 each)
        # = 51; per output 64 terms x 2 multiplies + 63 additions
        self.fp64_ops = n ** 3 * (inputs.N_VARS * 51 + inputs.N_VARS * (3 * inputs.N_TERMS - 1))

    def setup(self, device=None):
        n = self.n
        self.ins = []
        for u in self.host_u:
            d = DeviceGrid((n,) * 3, self.g, device)
            d.upload(u, with_ghosts=True)
            self.ins.append(d)
        self.outs = [DeviceGrid((n,) * 3, 0, device) for _ in range(inputs.N_VARS)]
        self.kernel = Rhs24(self.ins, self.outs, self.k, self.poly)
        self.space = IndexSpace((0, 0, 0), (n, n, n))
        return self

    def run(self, params: LaunchParams | None = None, stream=None) -> None:
        self.kernel.launch(self.space, params or self.kernel.default_params, stream)

    def outputs(self) -> list[np.ndarray]:
        return [o.download() for o in self.outs]


CONFIGS = {1: C1Laplacian7, 2: C2FourthOrder, 3: C3WaveRK4, 4: C4Level, 5: C5Rhs24}
