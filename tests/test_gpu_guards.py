"""Write-footprint checks (compute-sanitizer is closed on this pool): every
output grid is allocated with ghost zones and row padding, the whole storage
is filled with a sentinel, and after the kernel only the elements the
kernel is allowed to write may differ — the interior of the swept space
(plus, for the fused periodic refresh, the ghost shell).  Catches stray
stores anywhere in the allocation, not just outside the swept space."""
import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import _build, inputs
from paper_1308_1343_b200.grid import DeviceGrid
from paper_1308_1343_b200.tuner import LaunchParams

pytestmark = pytest.mark.gpu
SENTINEL = -7.25


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()


def guarded(ext, g=2):
    d = DeviceGrid(ext, g)
    d.storage.fill_(SENTINEL)
    return d


def allowed_mask(d: DeviceGrid, region=None, shell=False):
    """Boolean mask over the flat storage: True where writes are allowed."""
    import torch
    m = torch.zeros_like(d.storage, dtype=torch.bool)
    nx, ny, nz = d.extents
    if shell:
        d_full = m.as_strided(d.full().shape, d.full().stride(), d.offset - d.ghost * (1 + d.sy + d.sz))
        d_full.fill_(True)
    x0, x1, y0, y1, z0, z1 = region or (0, nx, 0, ny, 0, nz)
    inner = m.as_strided((nz, ny, nx), (d.sz, d.sy, 1), d.offset)
    inner[z0:z1, y0:y1, x0:x1] = True
    return m


def check_footprint(d: DeviceGrid, mask):
    s = d.storage
    outside = s[~mask]
    assert bool((outside == SENTINEL).all()), f"{int((outside != SENTINEL).sum())} stray writes"


def test_d4_all_footprint():
    from paper_1308_1343_b200.kernels import FourthOrderAll
    from paper_1308_1343_b200.traverse import IndexSpace
    n, g = 40, 2
    u = inputs.c2_field(n, g, seed=3)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    src = DeviceGrid((n,) * 3, g)
    src.upload(u)
    outs = [guarded((n,) * 3) for _ in range(10)]
    region = (3, 37, 1, 39, 2, 38)
    for params in [(32, 4, 4, 2), (64, 2, 7, 1), (128, 1, 16, 2)]:
        FourthOrderAll(outs, src, k).launch(IndexSpace((3, 1, 2), (37, 39, 38)), LaunchParams(*params))
        want = [np.empty((n, n, n)) for _ in range(10)]
        oracle.d4_all(want, u, g, region, k)
        for i, o in enumerate(outs):
            check_footprint(o, allowed_mask(o, region))
            got = o.interior()[2:38, 1:39, 3:37].cpu().numpy()
            assert got.tobytes() == np.ascontiguousarray(want[i][2:38, 1:39, 3:37]).tobytes()


def test_lap4_level_footprint():
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    from paper_1308_1343_b200.level import Box, box_difference
    n, g = 24, 2
    outer, hole = inputs.c4_outer_and_hole(n)
    boxes = box_difference(Box(*outer), Box(*hole))
    fields = inputs.c4_fields(boxes, g, seed=2)
    srcs, dsts = [], []
    for b, u in zip(boxes, fields):
        s = DeviceGrid(b.extents, g, lower=b.lo)
        s.upload(u)
        srcs.append(s)
        d = DeviceGrid(b.extents, g, lower=b.lo)
        d.storage.fill_(SENTINEL)
        dsts.append(d)
    LevelLaplacian4(dsts, srcs, inputs.D4Constants.for_spacing(1.0 / n)).launch(None, LaunchParams(32, 4, 5, 2))
    for d in dsts:
        check_footprint(d, allowed_mask(d))


@pytest.mark.parametrize("schedule", ["pairs", "lap_pairs", "stages"])
def test_rk4_footprint_interior_and_shell(schedule):
    from paper_1308_1343_b200.configs import C3WaveRK4
    n = 20
    p = C3WaveRK4(n=n, seed=9, schedule=schedule).setup()
    rk = p.rk
    for grid in (rk.phi_a, rk.pi_a, rk.phi_b, rk.pi_b, rk.acc_phi, rk.acc_pi):
        grid.storage.fill_(SENTINEL)
    rk.step(LaunchParams(32, 4, 6, 1))
    for grid in (rk.phi_a, rk.pi_a, rk.phi_b, rk.pi_b):
        check_footprint(grid, allowed_mask(grid, shell=True))
    for grid in (rk.acc_phi, rk.acc_pi):
        check_footprint(grid, allowed_mask(grid))


def test_rhs24_footprint():
    from paper_1308_1343_b200.kernels import Rhs24
    from paper_1308_1343_b200.traverse import IndexSpace
    n, g = 11, 2
    fields = inputs.c5_fields(n, g, seed=1)
    ins = []
    for u in fields:
        d = DeviceGrid((n,) * 3, g)
        d.upload(u)
        ins.append(d)
    outs = [guarded((n,) * 3) for _ in range(24)]
    k = inputs.D4Constants.for_spacing(1.0 / n)
    Rhs24(ins, outs, k, inputs.c5_poly(seed=1)).launch(IndexSpace((1, 2, 0), (10, 11, 9)), LaunchParams(32, 24, 4, 1))
    for o in outs:
        check_footprint(o, allowed_mask(o, (1, 10, 2, 11, 0, 9)))


def test_lap7_footprint():
    from paper_1308_1343_b200.kernels import Laplacian7
    from paper_1308_1343_b200.traverse import IndexSpace
    n = 19
    src = DeviceGrid((n,) * 3, 1)
    src.upload(inputs.c1_field(n, seed=4))
    dst = guarded((n,) * 3, 1)
    Laplacian7(dst, src, 1.0, 2.0).launch(IndexSpace((1, 0, 3), (18, 19, 17)), LaunchParams(64, 4, 5))
    check_footprint(dst, allowed_mask(dst, (1, 18, 0, 19, 3, 17)))
