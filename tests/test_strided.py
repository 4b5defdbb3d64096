"""F3 — strided (coarsened) levels: the boxes of ``BBoxSet.coarsen``
(bboxset.py:387-406) swept in compact lattice coordinates (level.compact_level).
CPU: the compact boxes cover exactly the reference's lattice points.  GPU:
a coarsened config-4-style level swept in one launch equals the oracle on one
global compact field."""
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1308_1343_b200.level import Lattice, compact_level
from paper_1308_1343_b200.errors import UsageError

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def srt():
    if not (REF / "stencilrt").is_dir():
        pytest.skip(f"reference package not installed at {REF}")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import stencilrt.bboxset
    import stencilrt.lattice
    return stencilrt


def coarse_level(srt, n, factor):
    L, B = srt.lattice, srt.bboxset
    outer = L.BBox(L.Point((0, 0, 0)), L.Point((n - 1,) * 3), L.Stride.ones(3))
    hole = L.BBox(L.Point((n // 2,) * 3), L.Point((n - 1,) * 3), L.Stride.ones(3))
    fine = B.BBoxSet.from_bboxes([outer]).difference(B.BBoxSet.from_bboxes([hole]))
    return fine.coarsen(L.Stride(factor))


@pytest.mark.parametrize("factor", [(2, 2, 2), (3, 2, 1), (4, 4, 2)])
def test_compact_boxes_cover_the_reference_lattice_points(srt, factor):
    lvl = coarse_level(srt, 20, factor)
    boxes, lat = compact_level(lvl)
    assert lat.stride == factor
    want = set()
    for b in lvl.to_bboxes():
        want |= {p.coords for p in b.points()}
    got = set()
    for b in boxes:
        for z in range(b.lo[2], b.hi[2] + 1):
            for y in range(b.lo[1], b.hi[1] + 1):
                for x in range(b.lo[0], b.hi[0] + 1):
                    p = lat.to_fine((x, y, z))
                    assert p not in got
                    got.add(p)
    assert got == want
    assert sum(b.volume() for b in boxes) == sum(b.point_count() for b in lvl.to_bboxes())


def test_lattice_round_trip_and_off_lattice_points():
    lat = Lattice((2, 3, 1), (1, 2, 0))
    for k in [(0, 0, 0), (3, -2, 5), (-4, 7, -1)]:
        assert lat.to_compact(lat.to_fine(k)) == k
    with pytest.raises(UsageError):
        lat.to_compact((2, 2, 0))


def test_unit_level_is_unchanged(srt):
    lvl = coarse_level(srt, 16, (1, 1, 1))
    boxes, lat = compact_level(lvl)
    assert lat == Lattice((1, 1, 1), (0, 0, 0))
    assert [(b.lo, b.hi) for b in boxes] == [(tuple(b.lower.coords), tuple(b.upper.coords)) for b in lvl.to_bboxes()]


@pytest.mark.gpu
def test_coarsened_level_swept_in_one_launch(srt):
    """The coarsened 96^3-minus-octant level (stride 2): each compact box's
    source cut from ONE global compact field (ghosts included), the whole
    level swept by LevelLaplacian4 at spacing 2h; every box equals the oracle
    on the global field."""
    import oracle
    from paper_1308_1343_b200 import _build, inputs
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    _build.build()
    n, g = 96, 2
    boxes, lat = compact_level(coarse_level(srt, n, (2, 2, 2)))
    lo = [min(b.lo[d] for b in boxes) for d in range(3)]
    hi = [max(b.hi[d] for b in boxes) for d in range(3)]
    ext = [h - l + 1 for l, h in zip(lo, hi)]
    glob = np.random.default_rng(5).uniform(-1, 1, (ext[2] + 2 * g, ext[1] + 2 * g, ext[0] + 2 * g))
    k = inputs.D4Constants.for_spacing(2.0 / n)
    srcs, dsts = [], []
    for b in boxes:
        s = [b.lo[d] - lo[d] for d in range(3)]
        e = b.extents
        d = DeviceGrid(e, g, lower=b.lo)
        d.upload(glob[s[2]:s[2] + e[2] + 2 * g, s[1]:s[1] + e[1] + 2 * g, s[0]:s[0] + e[0] + 2 * g])
        srcs.append(d)
        dsts.append(DeviceGrid(e, 0, lower=b.lo))
    LevelLaplacian4(dsts, srcs, k).launch(None, LevelLaplacian4.default_params)
    full = np.empty(ext[::-1])
    oracle.lap4(full, glob, g, (0, ext[0], 0, ext[1], 0, ext[2]), k.k2)
    for b, d in zip(boxes, dsts):
        s = [b.lo[i] - lo[i] for i in range(3)]
        e = b.extents
        want = full[s[2]:s[2] + e[2], s[1]:s[1] + e[1], s[0]:s[0] + e[0]]
        assert d.download().tobytes() == np.ascontiguousarray(want).tobytes(), b
