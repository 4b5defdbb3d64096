"""Host-side loop engine (traverse.py mirror): plan partition exactness,
determinism, lane alignment, errors, and the reference's own tests' shape."""
import itertools
import random

import numpy as np
import pytest

from paper_1308_1343_b200 import traverse as tv
from paper_1308_1343_b200.errors import UsageError
from paper_1308_1343_b200.level import Box
from paper_1308_1343_b200.tuner import ExecParams, LoopSetup, PlanSpace, TopologyConfig, Tuner


def points(space):
    return set(itertools.product(*[range(l, h) for l, h in zip(space.lo, space.hi)]))


def assert_partition(parent, children):
    assert sum(c.volume() for c in children) == parent.volume()
    seen = set()
    for c in children:
        p = points(c)
        assert not (p & seen)
        seen |= p
    assert seen == points(parent)


def test_index_space_contract():
    s = tv.IndexSpace((1, 2, 3), (4, 6, 8))
    assert s.extents == (3, 4, 5) and s.volume() == 60 and s.dim == 3
    with pytest.raises(UsageError):
        tv.IndexSpace((0, 0), (1,))
    with pytest.raises(UsageError):
        tv.IndexSpace((5,), (4,))


def test_bbox_conversion_roundtrip():
    b = Box((0, 2, 4), (7, 9, 11))
    s = tv.index_space_from_bbox(b)
    assert s == tv.IndexSpace((0, 2, 4), (8, 10, 12))
    assert tv.index_space_to_bbox(s) == b
    assert tv.index_space_from_bbox(Box.empty(3)).volume() == 0


def test_example_16x16_plan():
    space = tv.IndexSpace((0, 0), (16, 16))
    p = ExecParams((2, 2), (8, 4), (1, 2), 4)
    plan = tv.build_plan(space, p)
    assert len(plan.blocks) == 4
    for b in plan.blocks:
        assert len(b.tiles) == 2
        for t in b.tiles:
            assert len(t.slices) == 2


@pytest.mark.parametrize("seed", range(40))
def test_random_plans_partition_exactly(seed):
    rng = random.Random(seed)
    d = rng.choice([1, 2, 3])
    lo = tuple(rng.randint(-8, 8) for _ in range(d))
    ext = tuple(rng.randint(1, 24) for _ in range(d))
    space = tv.IndexSpace(lo, tuple(a + e for a, e in zip(lo, ext)))
    setup = LoopSetup("t", ext, "vector", 4, 2)
    topo = TopologyConfig(n_coarse_threads=4, n_fine_threads=2, lane_width=4)
    p = rng.choice(PlanSpace().enumerate(setup, topo))
    plan = tv.build_plan(space, p)
    assert_partition(space, [b.space for b in plan.blocks])
    for b in plan.blocks:
        assert_partition(b.space, [t.space for t in b.tiles])
        for t in b.tiles:
            assert_partition(t.space, list(t.slices))
    # interior x cuts of blocks/slices are multiples of the lane width
    for b in plan.blocks:
        for t in b.tiles:
            for s in t.slices:
                for x in (s.lo[0], s.hi[0]):
                    assert x in (space.lo[0], space.hi[0]) or x % 4 == 0 or x in (t.space.lo[0], t.space.hi[0])
    assert tv.build_plan(space, p) == plan


def test_degenerate_plans_degrade():
    space = tv.IndexSpace((0,), (3,))
    plan = tv.build_plan(space, ExecParams((4,), (3,), (2,), 4))
    assert_partition(space, list(plan.pieces()))


def _stencil_kernel(dst, src):
    def kern(piece):
        (a,), (b,) = piece.lo, piece.hi
        dst[a:b] = 0.5 * (src[a + 1:b + 1] - src[a - 1:b - 1])
    return kern


@pytest.mark.parametrize("workers", [1, 2, 4])
def test_result_independent_of_decomposition(workers):
    rng = np.random.default_rng(3)
    n = 301
    src = rng.uniform(-10, 10, n)
    space = tv.IndexSpace((1,), (n - 1,))
    setup = LoopSetup("c7k", (n - 2,), "vector", 1, 1)
    topo = TopologyConfig(lane_width=4)
    pool = PlanSpace().enumerate(setup, topo)
    ref = None
    for p in random.Random(5).sample(pool, 8):
        dst = np.zeros(n)
        tv.execute_plan(tv.build_plan(space, p), _stencil_kernel(dst, src), workers, 1)
        ref = dst if ref is None else ref
        assert dst.tobytes() == ref.tobytes()


def test_execute_plan_propagates_first_error_and_run_loop_discards_timing():
    space = tv.IndexSpace((0, 0), (16, 16))
    setup = LoopSetup("boom", (16, 16), "vector", 2, 2)
    topo = TopologyConfig(n_coarse_threads=2, n_fine_threads=2, lane_width=4)
    tuner = Tuner(topo)

    def bad(piece):
        raise RuntimeError("kernel failed")
    with pytest.raises(RuntimeError, match="kernel failed"):
        tv.run_loop(setup, space, bad, tuner)
    assert tuner.log == []


def test_run_loop_and_run_static_with_python_kernel():
    n = 64
    src = np.random.default_rng(1).random(n + 2)
    dst = np.zeros(n + 2)
    space = tv.IndexSpace((1,), (n + 1,))
    setup = LoopSetup("loop", (n,), "vector", 2, 1)
    tuner = Tuner(TopologyConfig(n_coarse_threads=2, lane_width=4))
    for _ in range(12):
        el = tv.run_loop(setup, space, _stencil_kernel(dst, src), tuner)
        assert el >= 0
    want = np.zeros(n + 2)
    want[1:n + 1] = 0.5 * (src[2:] - src[:-2])
    assert dst.tobytes() == want.tobytes()
    assert len(tuner.log) == 12 and tuner.log[0]["phase"] == "warmup"
    dst[:] = 0
    assert tv.run_static(space, _stencil_kernel(dst, src), 3) >= 0
    assert dst.tobytes() == want.tobytes()
