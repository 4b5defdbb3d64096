"""Seeded host-side input generators for the five BASELINE.json configurations.

All inputs are generated on the host with numpy and uploaded once; the
device never generates data.  The reference's own
generator is ``make_field`` (``stencil.py:26-28``: ``default_rng(seed)``);
every config here uses ``np.random.default_rng(SEED_BASE + k)`` with the
reference's default seed ``20130715`` (``cli.py:252``, ``conftest.py:12``).

Arrays are numpy ``(z, y, x)`` with x contiguous, exactly the reference's
layout (``stencil.py:9-10``).  A "ghosted" array of a box with interior
extents (nx, ny, nz) and ghost width g has shape (nz+2g, ny+2g, nx+2g);
interior point (i, j, k) lives at [k+g, j+g, i+g].

Choices the reference does not fix (recorded in DESIGN.md §Oracle):
  * C2 ghost values are the analytic field plus noise at x = (i-g)*h.
  * C3 Gaussian: exp(-r^2 / (2 sigma^2)) with sigma = 0.1, evaluated as a
    separable product; noise is added to the interior, then the periodic
    ghost shell is filled.
  * C5: SeedSequence(seed).spawn(2) -> (field stream, polynomial stream);
    input index of variable v, slot s (0 = value, 1..9 = Dx, Dy, Dz, Dxx,
    Dyy, Dzz, Dxy, Dxz, Dyz) is 10*v + s; every term is c * v_p * v_q.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

SEED_BASE = 20130715

# derivative slot order shared by C2 outputs and C5 inputs
DERIV_NAMES = ("Dx", "Dy", "Dz", "Dxx", "Dyy", "Dzz", "Dxy", "Dxz", "Dyz")
C2_OUTPUT_NAMES = DERIV_NAMES + ("Lap4",)


def seed_for(config: int) -> int:
    return SEED_BASE + config


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- C1: 7-point Laplacian on one 64^3 box, ghost 1 ---------------------------

def c1_field(n: int = 64, seed: int | None = None) -> np.ndarray:
    """(n+2)^3 ghosted field, i.i.d. uniform[-1, 1)."""
    rng = np.random.default_rng(seed_for(1) if seed is None else seed)
    return rng.uniform(-1.0, 1.0, size=(n + 2, n + 2, n + 2))


def c1_constants(n: int = 64) -> tuple[float, float]:
    """C0 = -6/h^2 and C1 = 1/h^2 (``stencil.py:22-23`` with the h^2 scaling)."""
    h = 1.0 / n
    return -6.0 / (h * h), 1.0 / (h * h)


# -- 4th-order constants shared by C2..C5 ------------------------------------

@dataclass(frozen=True)
class D4Constants:
    k1: float    # 1 / (12 h)      first derivative
    k2: float    # 1 / (12 h^2)    second derivative
    k11: float   # 1 / (144 h^2)   mixed derivative

    @staticmethod
    def for_spacing(h: float) -> "D4Constants":
        return D4Constants(1.0 / (12.0 * h), 1.0 / (12.0 * h * h), 1.0 / (144.0 * h * h))


@dataclass(frozen=True)
class D2Constants:
    """2nd-order centred constants: k1 = 1/(2h), k2 = 1/h^2, k11 = 1/(4h^2)."""
    k1: float
    k2: float
    k11: float

    @staticmethod
    def for_spacing(h: float) -> "D2Constants":
        return D2Constants(1.0 / (2.0 * h), 1.0 / (h * h), 1.0 / (4.0 * h * h))


# -- C2: 10 derivative outputs on a 256^3 box, ghost 2 ------------------------

def c2_field(n: int = 256, g: int = 2, seed: int | None = None) -> np.ndarray:
    h = 1.0 / n
    rng = np.random.default_rng(seed_for(2) if seed is None else seed)
    x = (np.arange(n + 2 * g, dtype=np.float64) - g) * h
    s = np.sin(2.0 * np.pi * x)
    u = (s[:, None, None] * s[None, :, None]) * s[None, None, :]
    u += 1e-3 * rng.uniform(-1.0, 1.0, size=u.shape)
    return u


# -- C3: scalar wave, RK4, periodic 384^3, ghost 2 ----------------------------

@dataclass(frozen=True)
class WaveConstants:
    lap: D4Constants
    half_dt: float   # 0.5 * dt
    dt: float
    dt6: float       # dt / 6

    @staticmethod
    def for_grid(n: int) -> "WaveConstants":
        h = 1.0 / n
        dt = 0.25 * h
        return WaveConstants(D4Constants.for_spacing(h), 0.5 * dt, dt, dt / 6.0)


def periodic_fill(a: np.ndarray, g: int) -> None:
    """Refill the ghost shell of a ghosted array periodically, axis by axis
    (x, then y, then z, each over the full extent of the other axes) so edges
    and corners come out as the periodic images of interior points."""
    if g == 0:
        return
    for ax in (2, 1, 0):
        n = a.shape[ax] - 2 * g
        src_lo = [slice(None)] * 3
        dst_lo = [slice(None)] * 3
        src_lo[ax] = slice(n, n + g)          # last g interior planes
        dst_lo[ax] = slice(0, g)
        a[tuple(dst_lo)] = a[tuple(src_lo)]
        src_hi = [slice(None)] * 3
        dst_hi = [slice(None)] * 3
        src_hi[ax] = slice(g, 2 * g)          # first g interior planes
        dst_hi[ax] = slice(n + g, n + 2 * g)
        a[tuple(dst_hi)] = a[tuple(src_hi)]


def c3_fields(n: int = 384, g: int = 2, seed: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    h = 1.0 / n
    sigma = 0.1
    rng = np.random.default_rng(seed_for(3) if seed is None else seed)
    x = np.arange(n, dtype=np.float64) * h
    e = np.exp(-((x - 0.5) ** 2) / (2.0 * sigma * sigma))
    phi = np.zeros((n + 2 * g,) * 3)
    core = (e[:, None, None] * e[None, :, None]) * e[None, None, :]
    core += 1e-6 * rng.uniform(-1.0, 1.0, size=core.shape)
    phi[g:n + g, g:n + g, g:n + g] = core
    periodic_fill(phi, g)
    pi = np.zeros_like(phi)
    return phi, pi


# -- C4: bboxset level [0,511]^3 minus [256,511]^3, ghost 2 -------------------

def c4_outer_and_hole(n: int = 512) -> tuple[tuple, tuple]:
    """Inclusive corners (innermost first) of the level box and its upper octant."""
    outer = ((0, 0, 0), (n - 1, n - 1, n - 1))
    hole = ((n // 2, n // 2, n // 2), (n - 1, n - 1, n - 1))
    return outer, hole


def c4_fields(boxes, g: int = 2, seed: int | None = None) -> list[np.ndarray]:
    """One ghosted uniform[-1,1) array per box, drawn from one stream in box order."""
    rng = np.random.default_rng(seed_for(4) if seed is None else seed)
    out = []
    for b in boxes:
        nx, ny, nz = b.extents
        out.append(rng.uniform(-1.0, 1.0, size=(nz + 2 * g, ny + 2 * g, nx + 2 * g)))
    return out


# -- C5: 24-variable BSSN-like fused RHS --------------------------------------

N_VARS = 24
N_SLOTS = 10                 # value + 9 derivatives
N_INPUTS = N_VARS * N_SLOTS  # 240
N_TERMS = 64


@dataclass(frozen=True)
class PolyTable:
    """out_o = ((t_0 + t_1) + ...) + t_63, t_k = (coef[o,k] * v[p[o,k]]) * v[q[o,k]]."""
    coef: np.ndarray   # (24, 64) float64
    p: np.ndarray      # (24, 64) int32 in [0, 240)
    q: np.ndarray      # (24, 64) int32 in [0, 240)

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.coef, self.p, self.q):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


def c5_streams(seed: int | None = None):
    ss = np.random.SeedSequence(seed_for(5) if seed is None else seed)
    f, p = ss.spawn(2)
    return np.random.default_rng(f), np.random.default_rng(p)


def c5_poly(seed: int | None = None) -> PolyTable:
    _, prng = c5_streams(seed)
    coef = prng.standard_normal((N_VARS, N_TERMS))
    p = prng.integers(0, N_INPUTS, size=(N_VARS, N_TERMS)).astype(np.int32)
    q = prng.integers(0, N_INPUTS, size=(N_VARS, N_TERMS)).astype(np.int32)
    return PolyTable(coef, p, q)


def c5_fields(n: int = 192, g: int = 2, seed: int | None = None) -> list[np.ndarray]:
    frng, _ = c5_streams(seed)
    return [frng.uniform(0.9, 1.1, size=(n + 2 * g,) * 3) for _ in range(N_VARS)]
