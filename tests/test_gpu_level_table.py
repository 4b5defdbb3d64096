"""Level box tables that scale: a random 128-box level (arbitrary origins
and extents, as BBoxSet.to_bboxes() produces, bboxset.py:313-317) swept by
every multi-box operator — the 4th-order Laplacian (K3), all ten 4th- and
2nd-order outputs (K2) and each RK4 stage (K5) — in ONE launch through the
device-resident box table (blockIdx -> box by binary search), bit-exact
against the oracle box by box."""
import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import _build, _lib, inputs
from paper_1308_1343_b200.errors import UsageError
from paper_1308_1343_b200.grid import DeviceGrid
from paper_1308_1343_b200.level import Box
from paper_1308_1343_b200.tuner import LaunchParams

pytestmark = pytest.mark.gpu
G = 2


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    import torch
    torch.cuda.init()


def random_level(nbox: int, seed: int, region=(150, 110, 90), origin=(-13, 5, 2)) -> list[Box]:
    """A random partition of a box into `nbox` boxes by recursive cuts."""
    rng = np.random.default_rng(seed)
    boxes = [(list(origin), [o + e - 1 for o, e in zip(origin, region)])]
    while len(boxes) < nbox:
        i = int(np.argmax([np.prod([h - l + 1 for l, h in zip(*b)]) for b in boxes]))
        lo, hi = boxes.pop(i)
        ext = [h - l + 1 for l, h in zip(lo, hi)]
        d = int(rng.choice([k for k in range(3) if ext[k] >= 2], p=None))
        cut = int(rng.integers(lo[d] + 1, hi[d] + 1))
        a_hi, b_lo = list(hi), list(lo)
        a_hi[d], b_lo[d] = cut - 1, cut
        boxes += [(lo, a_hi), (b_lo, hi)]
    return [Box(tuple(l), tuple(h)) for l, h in boxes]


def grids(boxes, seed, ghost=G):
    rng = np.random.default_rng(seed)
    out, host = [], []
    for b in boxes:
        nx, ny, nz = b.extents
        u = rng.uniform(-1.0, 1.0, (nz + 2 * ghost, ny + 2 * ghost, nx + 2 * ghost))
        d = DeviceGrid(b.extents, ghost, lower=b.lo)
        d.upload(u, with_ghosts=True)
        out.append(d)
        host.append(u)
    return out, host


class Counter:
    """Counts library calls by entry point (one launch per call)."""

    def __init__(self, monkeypatch):
        self.n = {}
        real = _lib.call

        def counting(name, *a):
            self.n[name] = self.n.get(name, 0) + 1
            return real(name, *a)
        monkeypatch.setattr(_lib, "call", counting)


@pytest.mark.parametrize("params", [LaunchParams(32, 4, 128, 2), LaunchParams(64, 2, 7, 1), LaunchParams(128, 1, 33, 2)])
def test_lap4_128_box_level_one_launch(monkeypatch, params):
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    boxes = random_level(128, 1)
    srcs, host = grids(boxes, 11)
    dsts = [DeviceGrid(b.extents, 0, lower=b.lo).fill_(0.5) for b in boxes]
    k = inputs.D4Constants.for_spacing(1 / 64)
    kern = LevelLaplacian4(dsts, srcs, k)
    cnt = Counter(monkeypatch)
    kern.launch(None, params)
    kern.launch(None, params)          # second launch of the same shape: the cached table
    assert cnt.n == {"sb_lap4_boxes": 2}
    for b, u, d in zip(boxes, host, dsts):
        nx, ny, nz = b.extents
        want = np.empty((nz, ny, nx))
        oracle.lap4(want, u, G, (0, nx, 0, ny, 0, nz), k.k2)
        assert d.download().tobytes() == want.tobytes(), b


@pytest.mark.parametrize("order", [4, 2])
def test_all10_128_box_level_one_launch(monkeypatch, order):
    from paper_1308_1343_b200.kernels import LevelFourthOrderAll
    boxes = random_level(128, 2)
    srcs, host = grids(boxes, 12)
    outs = [[DeviceGrid(b.extents, 0, lower=b.lo).fill_(0.25) for _ in range(10)] for b in boxes]
    k = inputs.D4Constants.for_spacing(1 / 50) if order == 4 else inputs.D2Constants.for_spacing(1 / 50)
    kern = LevelFourthOrderAll(outs, srcs, k, order=order)
    cnt = Counter(monkeypatch)
    kern.launch(None, LaunchParams(32, 4, 16, 2))
    assert sum(cnt.n.values()) == 1
    ref = oracle.d4_all if order == 4 else oracle.d2_all
    for b, u, os_ in zip(boxes, host, outs):
        nx, ny, nz = b.extents
        want = [np.empty((nz, ny, nx)) for _ in range(10)]
        ref(want, u, G, (0, nx, 0, ny, 0, nz), k)
        for i in range(10):
            assert os_[i].download().tobytes() == want[i].tobytes(), (b, inputs.C2_OUTPUT_NAMES[i])


def _stage_oracle(stage, f, c):
    """The stage formulas of oracle.rk4_step (one IEEE rounding per op)."""
    n = f["phi_s"].shape
    g = G
    I = (slice(g, -g),) * 3
    nz, ny, nx = n[0] - 2 * g, n[1] - 2 * g, n[2] - 2 * g
    L = np.empty((nz, ny, nx))
    oracle.lap4(L, f["phi_s"], g, (0, nx, 0, ny, 0, nz), c.lap.k2)
    out = {k: v.copy() for k, v in f.items() if k in ("acc_phi", "acc_pi", "phi_out", "pi_out")}
    if stage == 1:
        out["phi_out"] = f["phi_s"][I] + c.half_dt * f["pi0"]
        out["pi_out"] = f["pi0"] + c.half_dt * L
        out["acc_pi"] = L
    elif stage == 2:
        out["phi_out"] = f["phi0"] + c.half_dt * f["pi_s"]
        out["pi_out"] = f["pi0"] + c.half_dt * L
        out["acc_phi"] = f["pi0"] + 2.0 * f["pi_s"]
        out["acc_pi"] = f["acc_pi"] + 2.0 * L
    elif stage == 3:
        out["phi_out"] = f["phi0"] + c.dt * f["pi_s"]
        out["pi_out"] = f["pi0"] + c.dt * L
        out["acc_phi"] = f["acc_phi"] + 2.0 * f["pi_s"]
        out["acc_pi"] = f["acc_pi"] + 2.0 * L
    else:
        out["phi_out"] = f["phi0"] + c.dt6 * (f["acc_phi"] + f["pi_s"])
        out["pi_out"] = f["pi0"] + c.dt6 * (f["acc_pi"] + L)
    return out


@pytest.mark.parametrize("stage", [1, 2, 3, 4])
def test_rk4_stage_over_level_one_launch(monkeypatch, stage):
    from paper_1308_1343_b200.kernels import LevelRK4Stage
    boxes = random_level(40, 3 + stage, region=(70, 60, 50))
    c = inputs.WaveConstants.for_grid(64)
    rng = np.random.default_rng(20 + stage)
    fields, host = [], []
    for b in boxes:
        nx, ny, nz = b.extents
        f, h = {}, {}
        for name in LevelRK4Stage.NAMES:
            gh = G if name == "phi_s" else 0
            a = rng.uniform(-1, 1, (nz + 2 * gh, ny + 2 * gh, nx + 2 * gh))
            d = DeviceGrid(b.extents, gh, lower=b.lo)
            d.upload(a, with_ghosts=gh > 0)
            f[name], h[name] = d, a
        fields.append(f)
        host.append(h)
    kern = LevelRK4Stage(stage, fields, c)
    cnt = Counter(monkeypatch)
    kern.launch(None, LaunchParams(64, 4, 9, 1))
    assert cnt.n == {"sb_rk4_stage_boxes": 1}
    for b, f, h in zip(boxes, fields, host):
        want = _stage_oracle(stage, h, c)
        for name, w in want.items():
            assert f[name].download().tobytes() == np.ascontiguousarray(w).tobytes(), (b, stage, name)


def test_table_capture_rules_and_release():
    """The first launch of a level shape builds its table (refused inside a
    capture); captured launches of a built shape replay correctly; tables
    can be released and rebuilt."""
    import torch
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    boxes = random_level(20, 9, region=(40, 30, 20))
    srcs, host = grids(boxes, 19)
    dsts = [DeviceGrid(b.extents, 0, lower=b.lo) for b in boxes]
    k = inputs.D4Constants.for_spacing(0.1)
    kern = LevelLaplacian4(dsts, srcs, k)
    p = LaunchParams(32, 4, 8, 2)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with pytest.raises(UsageError):
        with torch.cuda.graph(g, stream=s):
            kern.launch(None, p)
    kern.launch(None, p)
    torch.cuda.synchronize()
    for d in dsts:
        d.fill_(0.0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        kern.launch(None, p)
    g.replay()
    torch.cuda.synchronize()
    for b, u, d in zip(boxes, host, dsts):
        nx, ny, nz = b.extents
        want = np.empty((nz, ny, nx))
        oracle.lap4(want, u, G, (0, nx, 0, ny, 0, nz), k.k2)
        assert d.download().tobytes() == want.tobytes()
    _lib.call("sb_release_tables")
    kern.launch(None, LaunchParams(64, 4, 8, 2))
    torch.cuda.synchronize()


def test_multi_box_error_paths():
    """Periodic refresh and z-slab stores are single-box operations; bad
    tables are usage errors, not crashes."""
    import ctypes as C
    from paper_1308_1343_b200.kernels import LevelRK4Stage
    boxes = random_level(10, 31, region=(30, 20, 20))
    c = inputs.WaveConstants.for_grid(32)
    fields = [{name: DeviceGrid(b.extents, G if name == "phi_s" else 0, lower=b.lo)
               for name in LevelRK4Stage.NAMES} for b in boxes]
    kern = LevelRK4Stage(2, fields, c)
    kern.extra_flags = _lib.SB_LAUNCH_PERIODIC_GHOSTS
    with pytest.raises(UsageError):
        kern.launch(None, LaunchParams(64, 4, 8, 1))
    with pytest.raises(UsageError):
        _lib.call("sb_lap4_boxes", None, 3, _lib.sb_d4_constants(1, 1, 1), _lib.launch(32, 4, 8), 0)
    assert _lib.load().sb_lap4_boxes(None, 0, _lib.sb_d4_constants(1, 1, 1), _lib.launch(32, 4, 8), None) == 0


def test_boxes_with_empty_spaces_are_skipped(monkeypatch):
    """A level sweep clipped to a space that misses most boxes: only the
    touched boxes' points change, still one launch."""
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    from paper_1308_1343_b200.traverse import IndexSpace
    boxes = random_level(24, 41, region=(60, 40, 30), origin=(0, 0, 0))
    srcs, host = grids(boxes, 42)
    dsts = [DeviceGrid(b.extents, 0, lower=b.lo).fill_(7.0) for b in boxes]
    k = inputs.D4Constants.for_spacing(0.05)
    kern = LevelLaplacian4(dsts, srcs, k)
    space = IndexSpace((5, 3, 2), (33, 21, 15))
    cnt = Counter(monkeypatch)
    kern.launch(space, LaunchParams(32, 4, 4, 2))
    assert sum(cnt.n.values()) == 1
    for b, u, d in zip(boxes, host, dsts):
        nx, ny, nz = b.extents
        want = np.full((nz, ny, nx), 7.0)
        lo = [max(b.lo[i], space.lo[i]) - b.lo[i] for i in range(3)]
        hi = [min(b.hi[i] + 1, space.hi[i]) - b.lo[i] for i in range(3)]
        if all(h > l for l, h in zip(lo, hi)):
            oracle.lap4(want, u, G, (lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]), k.k2)
        assert d.download().tobytes() == want.tobytes(), b


@pytest.mark.parametrize("seed", range(4))
def test_random_multi_box_levels_random_shapes(seed):
    """Random levels (9-40 boxes) x random launch shapes (tile 32/64/128,
    tile rows, z chunk, scalar or paired points) for the ten-output set and
    the Laplacian: every box bit-exact (inline table for <= 8 boxes, device
    table above)."""
    from paper_1308_1343_b200.kernels import LevelFourthOrderAll, LevelLaplacian4
    rng = np.random.default_rng(100 + seed)
    nbox = int(rng.integers(9, 41))
    boxes = random_level(nbox, 200 + seed, region=(int(rng.integers(40, 90)), int(rng.integers(20, 50)),
                                                   int(rng.integers(10, 40))), origin=tuple(int(v) for v in
                                                                                           rng.integers(-30, 30, 3)))
    srcs, host = grids(boxes, 300 + seed)
    k = inputs.D4Constants.for_spacing(float(rng.uniform(0.01, 0.1)))
    tx = int(rng.choice([32, 64, 128]))
    np_ = int(rng.choice([1, 2]))
    ty = int(rng.choice([1, 2, 4])) if (tx // np_) * 4 <= 256 else 1
    while (tx // np_) * ty % 32:
        ty *= 2
    p = LaunchParams(tx, ty, int(rng.integers(1, 40)), np_)
    outs = [[DeviceGrid(b.extents, 0, lower=b.lo) for _ in range(10)] for b in boxes]
    LevelFourthOrderAll(outs, srcs, k).launch(None, p)
    dsts = [DeviceGrid(b.extents, 0, lower=b.lo) for b in boxes]
    LevelLaplacian4(dsts, srcs, k).launch(None, p)
    for b, u, os_, d in zip(boxes, host, outs, dsts):
        nx, ny, nz = b.extents
        want = [np.empty((nz, ny, nx)) for _ in range(10)]
        oracle.d4_all(want, u, G, (0, nx, 0, ny, 0, nz), k)
        for i in range(10):
            assert os_[i].download().tobytes() == want[i].tobytes(), (p, b, i)
        assert d.download().tobytes() == want[9].tobytes(), (p, b)
