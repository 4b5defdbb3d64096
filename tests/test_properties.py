"""Property tests (hypothesis, as the reference's own suites use it) for the
host-side logic of the path: the level box algebra, the inter-box ghost
schedule, plan partitions, z-slab cuts, rank sharding and the device
launch space.  Point sets are small enough to enumerate."""
import itertools

from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1308_1343_b200 import traverse as tv
from paper_1308_1343_b200.halo import z_cuts
from paper_1308_1343_b200.level import Box, box_difference, expand, ghost_schedule, intersect
from paper_1308_1343_b200.shard import shard_boxes, split_z
from paper_1308_1343_b200.tuner import LaunchSpace, LoopSetup, TopologyConfig

coord = st.integers(-6, 6)
ext = st.integers(1, 6)


@st.composite
def boxes3(draw):
    lo = tuple(draw(coord) for _ in range(3))
    return Box(lo, tuple(l + draw(ext) - 1 for l in lo))


def pts(b: Box) -> set:
    if b.is_empty:
        return set()
    return set(itertools.product(*[range(l, h + 1) for l, h in zip(b.lo, b.hi)]))


@settings(max_examples=150, deadline=None)
@given(boxes3(), boxes3())
def test_box_difference_is_an_exact_disjoint_cover(a, b):
    parts = box_difference(a, b)
    seen: set = set()
    for p in parts:
        q = pts(p)
        assert q and not (q & seen)
        seen |= q
    assert seen == pts(a) - pts(b)
    assert parts == sorted(parts, key=lambda p: (p.lo[::-1], p.hi[::-1]))


@settings(max_examples=150, deadline=None)
@given(boxes3(), boxes3())
def test_intersect_and_expand(a, b):
    assert pts(intersect(a, b)) == pts(a) & pts(b)
    g = 2
    grown = pts(expand(a, g))
    assert all(all(l - g <= c <= h + g for c, l, h in zip(p, a.lo, a.hi)) for p in grown)
    assert len(grown) == (a.extents[0] + 2 * g) * (a.extents[1] + 2 * g) * (a.extents[2] + 2 * g)


@settings(max_examples=100, deadline=None)
@given(boxes3(), boxes3(), st.integers(1, 3))
def test_ghost_schedule_fills_exactly_the_ghosts_inside_the_level(a, b, g):
    level = box_difference(a, b) + ([b] if not intersect(a, b).is_empty else [])
    level = [x for x in level if not x.is_empty]
    covered = set().union(*[pts(x) for x in level]) if level else set()
    sched = ghost_schedule(level, g)
    for i, box in enumerate(level):
        ghosts = (pts(expand(box, g)) - pts(box)) & covered
        got = [pts(c.region) for c in sched if c.dst == i]
        flat = set().union(*got) if got else set()
        assert flat == ghosts
        assert sum(len(r) for r in got) == len(flat)              # no ghost point written twice
        for c in sched:
            if c.dst == i:
                assert pts(c.region) <= pts(level[c.src])          # copied from the source's interior


@settings(max_examples=100, deadline=None)
@given(boxes3(), st.integers(1, 8))
def test_split_z_partitions(box, parts):
    slabs = split_z(box, parts)
    assert sorted(set().union(*[pts(s) for s in slabs])) == sorted(pts(box))
    assert sum(s.volume() for s in slabs) == box.volume()
    th = [s.extents[2] for s in slabs]
    assert max(th) - min(th) <= 1


@settings(max_examples=60, deadline=None)
@given(st.lists(boxes3(), min_size=1, max_size=4), st.integers(1, 5))
def test_shards_own_every_point_once(boxes, world):
    boxes = [b for i, b in enumerate(boxes) if all(intersect(b, o).is_empty for o in boxes[:i])]
    owned = [pts(p) for r in range(world) for p in shard_boxes(boxes, world, r)]
    flat = set().union(*owned)
    assert flat == set().union(*[pts(b) for b in boxes])
    assert sum(len(o) for o in owned) == len(flat)


@settings(max_examples=60, deadline=None)
@given(st.integers(2, 80), st.integers(1, 8), st.integers(1, 3))
def test_z_cuts(n, parts, g):
    if n // parts < g:
        return
    c = z_cuts(n, parts, g)
    assert c[0] == 0 and c[-1] == n and all(b - a >= g for a, b in zip(c, c[1:]))


@settings(max_examples=80, deadline=None)
@given(st.tuples(st.integers(1, 3), st.integers(1, 40), st.integers(1, 40), st.integers(1, 40)),
       st.integers(1, 4), st.integers(1, 16), st.integers(1, 2))
def test_build_plan_partitions(dims_ext, cs, ts, fs):
    d, *e = dims_ext
    e = e[:d]
    space = tv.IndexSpace(tuple(0 for _ in e), tuple(e))
    from paper_1308_1343_b200.tuner import ExecParams
    p = ExecParams(tuple([cs] + [1] * (d - 1)), tuple([ts * 4] + [ts] * (d - 1)), tuple([fs] + [1] * (d - 1)), 4)
    pieces = list(tv.build_plan(space, p).pieces())
    seen: set = set()
    for q in pieces:
        qp = set(itertools.product(*[range(l, h) for l, h in zip(q.lo, q.hi)]))
        assert not (qp & seen)
        seen |= qp
    assert len(seen) == space.volume()


@settings(max_examples=60, deadline=None)
@given(st.integers(8, 300), st.integers(8, 300), st.integers(1, 300))
def test_launch_space_neighbours_stay_valid(nx, ny, nz):
    space = LaunchSpace(kind="d4", max_threads_pair=256, max_threads_scalar=512)
    setup, topo = LoopSetup("prop", (nx, ny, nz)), TopologyConfig()
    p = space.initial(setup, topo)
    for q in space.neighbors(p, setup, topo):
        space.check(q, setup, topo)
    assert p in space.enumerate(setup, topo)
