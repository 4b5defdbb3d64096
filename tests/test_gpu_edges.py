"""Edge cases through the C ABI: ragged and odd extents, thin boxes, offset
boxes, empty spaces, single points — every kernel bit-exact vs the oracle."""
import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import _build, inputs
from paper_1308_1343_b200.tuner import LaunchParams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()


def same(a, b):
    return a.shape == b.shape and np.ascontiguousarray(a).tobytes() == np.ascontiguousarray(b).tobytes()


def d4_setup(ext, g=2, seed=0, lower=(0, 0, 0)):
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import FourthOrderAll
    nx, ny, nz = ext
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1, 1, (nz + 2 * g, ny + 2 * g, nx + 2 * g))
    k = inputs.D4Constants.for_spacing(1.0 / 17)
    src = DeviceGrid(ext, g, lower=lower)
    src.upload(u)
    outs = [DeviceGrid(ext, 0, lower=lower).fill_(0.25) for _ in range(10)]
    return u, k, src, outs, FourthOrderAll(outs, src, k)


@pytest.mark.parametrize("ext", [(37, 23, 11), (1, 1, 1), (5, 3, 1), (64, 1, 9), (130, 7, 3)])
@pytest.mark.parametrize("params", [(32, 4, 4, 2), (64, 2, 7, 1), (128, 1, 64, 2)])
def test_d4_all_ragged(ext, params):
    from paper_1308_1343_b200.traverse import IndexSpace
    u, k, src, outs, kern = d4_setup(ext, seed=sum(ext))
    nx, ny, nz = ext
    kern.launch(IndexSpace((0, 0, 0), ext), LaunchParams(*params))
    want = [np.empty((nz, ny, nx)) for _ in range(10)]
    oracle.d4_all(want, u, 2, (0, nx, 0, ny, 0, nz), k)
    for i in range(10):
        assert same(outs[i].download(), want[i]), (ext, params, i)


def test_empty_space_writes_nothing():
    from paper_1308_1343_b200.traverse import IndexSpace
    u, k, src, outs, kern = d4_setup((16, 16, 16))
    kern.launch(IndexSpace((3, 3, 3), (3, 9, 9)), LaunchParams(32, 4, 4, 2))
    for o in outs:
        assert (o.download() == 0.25).all()


def test_offset_box_level_coordinates():
    """A box whose lower corner is (100, -7, 33) in level coordinates."""
    from paper_1308_1343_b200.traverse import IndexSpace
    lower = (100, -7, 33)
    ext = (20, 12, 9)
    u, k, src, outs, kern = d4_setup(ext, seed=4, lower=lower)
    sub = IndexSpace((103, -5, 34), (119, 4, 41))      # local [3,19) x [2,11) x [1,8)
    kern.launch(sub, LaunchParams(32, 4, 3, 2))
    want = [np.full((9, 12, 20), 0.25) for _ in range(10)]
    oracle.d4_all(want, u, 2, (3, 19, 2, 11, 1, 8), k)
    for i in range(10):
        assert same(outs[i].download(), want[i]), i


@pytest.mark.parametrize("schedule", ["lap_pairs", "pairs", "stages"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 30])
def test_rk4_small_and_ragged_periodic(n, schedule):
    from paper_1308_1343_b200.configs import C3WaveRK4
    from paper_1308_1343_b200.errors import UsageError
    g = 2
    if n < g:   # a periodic ghost shell wider than the box is rejected, not mis-filled
        with pytest.raises(UsageError):
            C3WaveRK4(n=n, seed=n, schedule=schedule).setup().run(LaunchParams(32, 4, 5, 1))
        return
    p = C3WaveRK4(n=n, seed=n, schedule=schedule).setup()
    p.run(LaunchParams(32, 4, 5, 1))
    wphi, wpi = oracle.rk4_step(p.host_phi, p.host_pi, g, p.c)
    assert same(p.phi_with_ghosts(), wphi)
    I = (slice(g, g + n),) * 3
    assert same(p.outputs()[1], wpi[I])
    if "pairs" in schedule:   # the pair schedules also refresh pi's ghosts
        assert same(p.rk.pi_b.download(with_ghosts=True), wpi)


@pytest.mark.parametrize("n,zc", [(13, 5), (9, 192), (2, 1)])
def test_rhs24_ragged(n, zc):
    from paper_1308_1343_b200.configs import C5Rhs24
    p = C5Rhs24(n=n, seed=n + 100).setup()
    p.run(LaunchParams(32, 24, zc, 1))
    want = [np.empty((n, n, n)) for _ in range(24)]
    oracle.rhs24(want, p.host_u, 2, (0, n, 0, n, 0, n), p.k, p.poly)
    for o, got in enumerate(p.outputs()):
        assert same(got, want[o]), o


@pytest.mark.parametrize("n", [1, 2, 7])
def test_lap7_tiny(n):
    from paper_1308_1343_b200.configs import C1Laplacian7
    p = C1Laplacian7(n=n, seed=n).setup()
    p.run()
    u = p.host_u
    ref = u.copy()
    oracle.lap7_rows(ref, u, 1, n + 1, 1, n + 1, 1, n + 1, p.c0, p.c1)
    assert same(p.outputs()[0], ref[1:-1, 1:-1, 1:-1])


def test_level_with_more_boxes_than_inline_table():
    """More boxes than SB_MAX_BOXES: one launch through the device-resident
    box table."""
    from paper_1308_1343_b200.configs import C4Level
    from paper_1308_1343_b200.level import Box
    boxes = [Box((8 * i, 0, 0), (8 * i + 6, 5, 4 + i % 3)) for i in range(11)]
    p = C4Level(n=96, seed=8, boxes=boxes).setup()
    p.run(LaunchParams(32, 4, 2, 2))
    for b, u, got in zip(p.boxes, p.host_u, p.outputs()):
        nx, ny, nz = b.extents
        want = np.empty((nz, ny, nx))
        oracle.lap4(want, u, 2, (0, nx, 0, ny, 0, nz), p.k.k2)
        assert same(got, want), b


def test_topology_from_device():
    from paper_1308_1343_b200.tuner import TopologyConfig
    t = TopologyConfig().with_device()
    assert t.sm_count >= 100 and t.smem_per_block >= 200 * 1024 and t.l2_bytes > 50 * 2 ** 20


@pytest.mark.parametrize("seed", range(6))
def test_random_levels_random_launches(seed):
    """Random bboxset-style levels (a random box minus a random box, plus an
    unrelated box at a negative offset), random launch shapes: every box of
    the level matches the oracle."""
    import random

    from paper_1308_1343_b200.configs import C4Level
    from paper_1308_1343_b200.level import Box, box_difference
    rng = random.Random(seed)
    lo = tuple(rng.randint(-20, 20) for _ in range(3))
    ext = tuple(rng.randint(6, 40) for _ in range(3))
    outer = Box(lo, tuple(a + e - 1 for a, e in zip(lo, ext)))
    hlo = tuple(a + rng.randint(1, e - 2) for a, e in zip(lo, ext))
    hole = Box(hlo, tuple(min(a + e - 1, h + rng.randint(0, 10)) for a, e, h in zip(lo, ext, hlo)))
    boxes = box_difference(outer, hole)
    far = tuple(rng.randint(-200, -100) for _ in range(3))
    boxes.append(Box(far, tuple(f + rng.randint(1, 20) for f in far)))
    p = C4Level(n=64, seed=seed, boxes=boxes).setup()
    tx = rng.choice([32, 64, 128])
    pp = rng.choice([1, 2])
    ty = rng.choice([t for t in (1, 2, 4, 8) if (tx // pp) * t % 32 == 0 and (tx // pp) * t <= 512])
    p.run(LaunchParams(tx, ty, rng.randint(1, 40), pp))
    for b, u, got in zip(p.boxes, p.host_u, p.outputs()):
        nx, ny, nz = b.extents
        want = np.empty((nz, ny, nx))
        oracle.lap4(want, u, 2, (0, nx, 0, ny, 0, nz), p.k.k2)
        assert same(got, want), (b, tx, ty, pp)


def test_d4_all_nonfinite_inputs_follow_ieee():
    """NaN and +-Inf in the input propagate as in the reference's numpy
    arithmetic: every finite output and every infinity is bit-identical, and
    the outputs that are NaN on the host are NaN on the device (NaN payloads
    are not part of the contract: x86 propagates the operand's payload, the
    GPU returns the canonical quiet NaN)."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import FourthOrderAll
    from paper_1308_1343_b200.traverse import IndexSpace
    ext = (40, 12, 9)
    nx, ny, nz = ext
    g = 2
    rng = np.random.default_rng(99)
    u = rng.uniform(-1, 1, (nz + 2 * g, ny + 2 * g, nx + 2 * g))
    u[4, 6, 7] = np.nan
    u[7, 3, 30] = np.inf
    u[2, 10, 20] = -np.inf
    u[5, 5, 41] = 1e308            # overflow to inf inside the stencil sums
    k = inputs.D4Constants.for_spacing(1.0 / 17)
    src = DeviceGrid(ext, g)
    src.upload(u)
    outs = [DeviceGrid(ext, 0).fill_(0.25) for _ in range(10)]
    FourthOrderAll(outs, src, k).launch(IndexSpace((0, 0, 0), ext), LaunchParams(32, 4, 4, 2))
    want = [np.empty((nz, ny, nx)) for _ in range(10)]
    with np.errstate(all="ignore"):
        oracle.d4_all(want, u, g, (0, nx, 0, ny, 0, nz), k)
    for i in range(10):
        got = outs[i].download()
        nan_w, nan_g = np.isnan(want[i]), np.isnan(got)
        assert nan_w.any()                    # the NaN reaches every derivative's stencil
        assert np.array_equal(nan_w, nan_g), i
        assert np.array_equal(got[~nan_g].view(np.uint64), want[i][~nan_w].view(np.uint64)), i
        assert np.isinf(want[i]).any() == np.isinf(got).any(), i


@pytest.mark.parametrize("g", [3, 4, 7])
def test_wider_ghost_zones(g):
    """Ghost widths beyond the stencil radius (the TMA maps start at the
    first ghost row, interior at (xpad, g, g)): the ten outputs and the
    level Laplacian read the right points."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    from paper_1308_1343_b200.level import Box
    ext = (29, 14, 10)
    u, k, src, outs, kern = d4_setup(ext, g=g, seed=50 + g)
    kern.launch(kern.full_space(), LaunchParams(64, 2, 4, 2))
    want = [np.empty(ext[::-1]) for _ in range(10)]
    oracle.d4_all(want, u, g, (0, ext[0], 0, ext[1], 0, ext[2]), k)
    for i in range(10):
        assert same(outs[i].download(), want[i]), (g, i)
    boxes = [Box((0, 0, 0), (28, 13, 9)), Box((40, 0, 0), (52, 6, 4))]
    rng = np.random.default_rng(g)
    srcs, hosts, dsts = [], [], []
    for b in boxes:
        nx, ny, nz = b.extents
        a = rng.uniform(-1, 1, (nz + 2 * g, ny + 2 * g, nx + 2 * g))
        d = DeviceGrid(b.extents, g, lower=b.lo)
        d.upload(a, with_ghosts=True)
        srcs.append(d)
        hosts.append(a)
        dsts.append(DeviceGrid(b.extents, 0, lower=b.lo))
    LevelLaplacian4(dsts, srcs, k).launch(None, LaunchParams(32, 4, 3, 2))
    for b, a, d in zip(boxes, hosts, dsts):
        nx, ny, nz = b.extents
        w = np.empty((nz, ny, nx))
        oracle.lap4(w, a, g, (0, nx, 0, ny, 0, nz), k.k2)
        assert same(d.download(), w), (g, b)


@pytest.mark.parametrize("schedule", ["lap_pairs", "stages"])
def test_rk4_periodic_ghost_width_three(schedule):
    """A periodic box with ghost width 3: the fused refresh writes all three
    ghost layers (images at distance up to 3) and the step still equals the
    oracle's (which fills the whole 3-wide shell)."""
    from paper_1308_1343_b200.configs import C3WaveRK4
    n, g = 14, 3
    p = C3WaveRK4(n=n, seed=21, g=g, schedule=schedule).setup()
    p.run(LaunchParams(32, 4, 5, 1))
    wphi, wpi = oracle.rk4_step(p.host_phi, p.host_pi, g, p.c)
    assert same(p.phi_with_ghosts(), wphi)
    I = (slice(g, g + n),) * 3
    assert same(p.outputs()[1], wpi[I])


def _adversarial_poly(seed: int) -> "inputs.PolyTable":
    """Term tables a fixed seed never draws: operand indices at both ends of
    0..239, p == q, one operand reused by every term of an output, signed
    zeros, and coefficients large enough to overflow to +-inf or small
    enough to land in the subnormals."""
    rng = np.random.default_rng(seed)
    n_out, n_t = inputs.N_VARS, inputs.N_TERMS
    coef = rng.standard_normal((n_out, n_t))
    p = rng.integers(0, 240, (n_out, n_t)).astype(np.int32)
    q = rng.integers(0, 240, (n_out, n_t)).astype(np.int32)
    p[0, :], q[0, :] = 0, 239                  # the first and last operand rows
    p[1, :] = q[1, :] = 7                      # v_7 * v_7, 64 times
    coef[2, ::2], coef[2, 1::2] = 0.0, -0.0    # signed zeros
    coef[3, :] = 1e307                         # positive u*u products: the sum overflows to +inf (no inf - inf)
    p[3, :] = q[3, :] = 10 * (np.arange(n_t) % 24)
    coef[4, :] = 1e-310                        # subnormal products
    p[5, :] = np.arange(n_t) % 240
    q[5, :] = 239 - p[5, :]
    coef[6, 10] = np.inf                       # one infinite coefficient
    return inputs.PolyTable(coef, p, q)


@pytest.mark.parametrize("ext,lo,hi", [((13, 7, 5), (0, 0, 0), (13, 7, 5)), ((21, 9, 6), (3, 1, 2), (20, 8, 5))])
def test_rhs24_adversarial_tables_and_subspaces(ext, lo, hi):
    """The config-5 kernel takes any term table: edge operand indices,
    repeated operands, signed zeros, overflow and subnormal products all
    follow the oracle's IEEE evaluation bit for bit, on a ragged box and on a
    sub-space (the outputs outside it keep their sentinel)."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import Rhs24
    from paper_1308_1343_b200.traverse import IndexSpace
    g = 2
    nx, ny, nz = ext
    rng = np.random.default_rng(sum(ext))
    host = [rng.uniform(0.9, 1.1, (nz + 2 * g, ny + 2 * g, nx + 2 * g)) for _ in range(inputs.N_VARS)]
    ins = []
    for u in host:
        d = DeviceGrid(ext, g)
        d.upload(u, with_ghosts=True)
        ins.append(d)
    outs = [DeviceGrid(ext, 0).fill_(-3.25) for _ in range(inputs.N_VARS)]
    poly = _adversarial_poly(sum(ext))
    k = inputs.D4Constants.for_spacing(1.0 / 19)
    with np.errstate(all="ignore"):
        Rhs24(ins, outs, k, poly).launch(IndexSpace(lo, hi), LaunchParams(32, 4, 3, 2))
        want = [np.full((nz, ny, nx), -3.25) for _ in range(inputs.N_VARS)]
        oracle.rhs24(want, host, g, (lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]), k, poly)
    got = [o.download() for o in outs]
    assert np.isinf(want[3][lo[2], lo[1], lo[0]]) and want[2][lo[2], lo[1], lo[0]] == 0.0
    for o in range(inputs.N_VARS):
        assert same(got[o], want[o]), o
