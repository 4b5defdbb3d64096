"""numpy restatement of the hot-path arithmetic — TEST INFRASTRUCTURE ONLY.

Every kernel here is written exactly like the reference's ``_update_rows``
(pkg/src/stencilrt/stencil.py:31-39): numpy slice arithmetic over a slab,
one IEEE rounding per ``+ - *`` in the written association, no FMA, host
constants.  Decomposition cannot change a bit (stencil.py:5-7), which the
threaded driver :func:`run_static` (traverse.py:235-260 restated) relies on.

Layout: numpy (z, y, x), x contiguous (stencil.py:9-10).  Ghosted inputs
have ghost width g on every face; interior point (i, j, k) is u[k+g, j+g, i+g].
Regions are (x0, x1, y0, y1, z0, z1) in interior coordinates, half-open.
"""
from __future__ import annotations

import os
import threading

import numpy as np


# -- reference kernels -------------------------------------------------------

def lap7_rows(dst, src, z0, z1, y0, y1, x0, x1, c0, c1) -> None:
    """stencil.py:31-39 with the module constants passed in (C0, C1):
    dst = C0*b + C1*(((xm+xp) + (ym+yp)) + (zm+zp)) on the slab, in array indices."""
    b = src
    dst[z0:z1, y0:y1, x0:x1] = c0 * b[z0:z1, y0:y1, x0:x1] + c1 * (
        (b[z0:z1, y0:y1, x0 - 1:x1 - 1] + b[z0:z1, y0:y1, x0 + 1:x1 + 1])
        + (b[z0:z1, y0 - 1:y1 - 1, x0:x1] + b[z0:z1, y0 + 1:y1 + 1, x0:x1])
        + (b[z0 - 1:z1 - 1, y0:y1, x0:x1] + b[z0 + 1:z1 + 1, y0:y1, x0:x1])
    )


def forward_difference(src: np.ndarray) -> np.ndarray:
    """vlanes.py:342-349: dst[i] = src[i+1] - src[i] for 0 <= i < n-1; other
    entries stay as initialised (0.0, AlignedArray's default fill)."""
    n = len(src)
    dst = np.zeros(n)
    if n >= 2:
        dst[:n - 1] = src[1:] - src[:-1]
    return dst


def centered_difference(src: np.ndarray) -> np.ndarray:
    """vlanes.py:352-360: dst[i] = 0.5 * (src[i+1] - src[i-1]) for 1 <= i < n-1."""
    n = len(src)
    dst = np.zeros(n)
    if n >= 3:
        dst[1:n - 1] = 0.5 * (src[2:] - src[:-2])
    return dst


# -- 4th-order operators (association fixed here) ----------

class _Slab:
    """Shifted views of a ghosted array over an interior region."""

    def __init__(self, u, g, region):
        self.u, self.g = u, g
        self.x0, self.x1, self.y0, self.y1, self.z0, self.z1 = region

    def __call__(self, dz=0, dy=0, dx=0):
        g = self.g
        return self.u[g + self.z0 + dz:g + self.z1 + dz,
                      g + self.y0 + dy:g + self.y1 + dy,
                      g + self.x0 + dx:g + self.x1 + dx]


def _d1u(m2, m1, p1, p2):
    """Unscaled 4th-order first difference: (u[-2] - u[+2]) + 8*(u[+1] - u[-1])."""
    return (m2 - p2) + 8.0 * (p1 - m1)


def _d2(m2, m1, c, p1, p2, k2):
    """((16*(u[-1] + u[+1]) - (u[-2] + u[+2])) - 30*u) * k2."""
    return ((16.0 * (m1 + p1) - (m2 + p2)) - 30.0 * c) * k2


def _rx(U, dz, dy):
    return _d1u(U(dz, dy, -2), U(dz, dy, -1), U(dz, dy, 1), U(dz, dy, 2))


def _ry(U, dz, dx):
    return _d1u(U(dz, -2, dx), U(dz, -1, dx), U(dz, 1, dx), U(dz, 2, dx))


def derivs9(u, g, region, k) -> list[np.ndarray]:
    """Dx, Dy, Dz, Dxx, Dyy, Dzz, Dxy, Dxz, Dyz of a ghosted field over a region.

    Mixed derivatives apply the outer axis' unscaled difference to the inner
    axis' unscaled differences: Dxy = d1u_y(d1u_x)*k11, Dxz = d1u_z(d1u_x)*k11,
    Dyz = d1u_z(d1u_y)*k11."""
    U = _Slab(u, g, region)
    c = U()
    dx = _rx(U, 0, 0) * k.k1
    dy = _ry(U, 0, 0) * k.k1
    dz = _d1u(U(-2), U(-1), U(1), U(2)) * k.k1
    dxx = _d2(U(0, 0, -2), U(0, 0, -1), c, U(0, 0, 1), U(0, 0, 2), k.k2)
    dyy = _d2(U(0, -2), U(0, -1), c, U(0, 1), U(0, 2), k.k2)
    dzz = _d2(U(-2), U(-1), c, U(1), U(2), k.k2)
    dxy = _d1u(_rx(U, 0, -2), _rx(U, 0, -1), _rx(U, 0, 1), _rx(U, 0, 2)) * k.k11
    dxz = _d1u(_rx(U, -2, 0), _rx(U, -1, 0), _rx(U, 1, 0), _rx(U, 2, 0)) * k.k11
    dyz = _d1u(_ry(U, -2, 0), _ry(U, -1, 0), _ry(U, 1, 0), _ry(U, 2, 0)) * k.k11
    return [dx, dy, dz, dxx, dyy, dzz, dxy, dxz, dyz]


def d4_all(outs, u, g, region, k) -> None:
    """Config 2: the nine derivatives and Lap4 = (Dxx + Dyy) + Dzz into
    interior-indexed output arrays over `region`."""
    x0, x1, y0, y1, z0, z1 = region
    ds = derivs9(u, g, region, k)
    lap = (ds[3] + ds[4]) + ds[5]
    for o, v in zip(outs, ds + [lap]):
        o[z0:z1, y0:y1, x0:x1] = v


def derivs9_o2(u, g, region, k) -> list[np.ndarray]:
    """2nd-order centred Dx, Dy, Dz, Dxx, Dyy, Dzz, Dxy, Dxz, Dyz:
    D1 = (u[+1]-u[-1])*k1, D2 = ((u[-1]+u[+1]) - 2u)*k2, D_ab = d_a(d_b)*k11
    with the inner difference b as for 4th order (x for xy/xz, y for yz)."""
    U = _Slab(u, g, region)
    c = U()
    ex = lambda dz, dy: U(dz, dy, 1) - U(dz, dy, -1)
    ey = lambda dz, dx: U(dz, 1, dx) - U(dz, -1, dx)
    dx = ex(0, 0) * k.k1
    dy = ey(0, 0) * k.k1
    dz = (U(1) - U(-1)) * k.k1
    dxx = ((U(0, 0, -1) + U(0, 0, 1)) - 2.0 * c) * k.k2
    dyy = ((U(0, -1) + U(0, 1)) - 2.0 * c) * k.k2
    dzz = ((U(-1) + U(1)) - 2.0 * c) * k.k2
    dxy = (ex(0, 1) - ex(0, -1)) * k.k11
    dxz = (ex(1, 0) - ex(-1, 0)) * k.k11
    dyz = (ey(1, 0) - ey(-1, 0)) * k.k11
    return [dx, dy, dz, dxx, dyy, dzz, dxy, dxz, dyz]


def d2_all(outs, u, g, region, k) -> None:
    """The ten outputs with 2nd-order operators; Lap2 = (Dxx + Dyy) + Dzz."""
    x0, x1, y0, y1, z0, z1 = region
    ds = derivs9_o2(u, g, region, k)
    lap = (ds[3] + ds[4]) + ds[5]
    for o, v in zip(outs, ds + [lap]):
        o[z0:z1, y0:y1, x0:x1] = v


def lap4(out, u, g, region, k2) -> None:
    """Configs 3/4: Lap4 = (Dxx + Dyy) + Dzz."""
    x0, x1, y0, y1, z0, z1 = region
    U = _Slab(u, g, region)
    c = U()
    dxx = _d2(U(0, 0, -2), U(0, 0, -1), c, U(0, 0, 1), U(0, 0, 2), k2)
    dyy = _d2(U(0, -2), U(0, -1), c, U(0, 1), U(0, 2), k2)
    dzz = _d2(U(-2), U(-1), c, U(1), U(2), k2)
    out[z0:z1, y0:y1, x0:x1] = (dxx + dyy) + dzz


# -- config 3: periodic ghosts + classical RK4 ---------------------------------

def periodic_fill(a: np.ndarray, g: int) -> None:
    """Fill the ghost shell axis by axis (x, y, z), each over the full extent
    of the other axes, from the opposite interior faces."""
    if g == 0:
        return
    for ax in (2, 1, 0):
        n = a.shape[ax] - 2 * g
        idx = lambda s: tuple(s if d == ax else slice(None) for d in range(3))
        a[idx(slice(0, g))] = a[idx(slice(n, n + g))]
        a[idx(slice(n + g, n + 2 * g))] = a[idx(slice(g, 2 * g))]


def rk4_step(phi0, pi0, g, c, threads: int = 1):
    """One classical RK4 step of d/dt(phi, pi) = (pi, Lap4 phi), periodic.

    Stage formulas (the device kernels evaluate the same trees):
      s1: L=Lap(phi0); phi2 = phi0 + hdt*pi0; pi2 = pi0 + hdt*L; acc=(pi0, L)
      s2: L=Lap(phi2); phi3 = phi0 + hdt*pi2; pi3 = pi0 + hdt*L; acc += 2*(pi2, L)
      s3: L=Lap(phi3); phi4 = phi0 + dt*pi3;  pi4 = pi0 + dt*L;  acc += 2*(pi3, L)
      s4: L=Lap(phi4); phi' = phi0 + dt6*(acc_phi + pi4); pi' = pi0 + dt6*(acc_pi + L)
    i.e. y' = y0 + (dt/6)*(((k1 + 2k2) + 2k3) + k4).  Inputs are ghosted
    (n+2g)^3 arrays; returns ghosted (phi', pi') whose ghosts are refilled."""
    n = phi0.shape[0] - 2 * g
    I = (slice(g, g + n),) * 3
    k2 = c.lap.k2

    def lap_of(phi):
        a = phi.copy()
        periodic_fill(a, g)
        out = np.empty((n, n, n))
        run_static(lambda z0, z1: lap4(out, a, g, (0, n, 0, n, z0, z1), k2), 0, n, threads)
        return out

    p0, q0 = phi0[I], pi0[I]
    L = lap_of(phi0)
    acc_f, acc_p = q0.copy(), L
    phi_s, pi_s = p0 + c.half_dt * q0, q0 + c.half_dt * L
    for coef in (c.half_dt, c.dt):
        full = np.zeros_like(phi0)
        full[I] = phi_s
        L = lap_of(full)
        acc_f = acc_f + 2.0 * pi_s
        acc_p = acc_p + 2.0 * L
        phi_s, pi_s = p0 + coef * pi_s, q0 + coef * L
    full = np.zeros_like(phi0)
    full[I] = phi_s
    L = lap_of(full)
    phi_new = np.zeros_like(phi0)
    pi_new = np.zeros_like(pi0)
    phi_new[I] = p0 + c.dt6 * (acc_f + pi_s)
    pi_new[I] = q0 + c.dt6 * (acc_p + L)
    periodic_fill(phi_new, g)
    periodic_fill(pi_new, g)
    return phi_new, pi_new


# -- config 5: fused 24-variable right-hand side -------------------------------

def rhs24(outs, ins, g, region, k, poly) -> None:
    """out_o = ((t_0 + t_1) + ...) + t_63 with t_j = (c*v_p)*v_q; input 10*v+s is
    variable v's slot s (0 value, 1..9 the derivs9 order)."""
    x0, x1, y0, y1, z0, z1 = region
    vals = []
    for u in ins:
        vals.append(_Slab(u, g, region)())
        vals.extend(derivs9(u, g, region, k))
    n_out, n_terms = poly.coef.shape
    for o in range(n_out):
        acc = (poly.coef[o, 0] * vals[poly.p[o, 0]]) * vals[poly.q[o, 0]]
        for t in range(1, n_terms):
            acc = acc + (poly.coef[o, t] * vals[poly.p[o, t]]) * vals[poly.q[o, t]]
        outs[o][z0:z1, y0:y1, x0:x1] = acc


# -- threaded static driver (traverse.py:235-260 restated) ----------------------

def host_threads() -> int:
    return len(os.sched_getaffinity(0))


def run_static(fn, z0: int, z1: int, n_threads: int) -> None:
    """Even chunks of [z0, z1) (the outermost dimension), one thread each;
    numpy releases the GIL inside its loops.  fn(za, zb) handles one chunk."""
    n = max(1, min(n_threads, z1 - z0))
    cuts = [z0 + (z1 - z0) * j // n for j in range(n)] + [z1]
    if n == 1:
        fn(z0, z1)
        return
    errs: list[BaseException] = []

    def work(a, b):
        try:
            fn(a, b)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(cuts[j], cuts[j + 1])) for j in range(n) if cuts[j] < cuts[j + 1]]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
