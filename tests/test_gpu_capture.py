"""Launch state and CUDA-graph capture: every launch carries all of its
state (no device-global tables another launch can change), so launches with
different data may interleave on several streams, and captured graphs
replay the data they were captured with."""
import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import _build, _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    import torch
    torch.cuda.init()


def _rhs_want(p):
    n = p.n
    want = [np.empty((n, n, n)) for _ in range(24)]
    oracle.rhs24(want, p.host_u, p.g, (0, n, 0, n, 0, n), p.k, p.poly)
    return want


def _check(p, want, what):
    for o, got in enumerate(p.outputs()):
        assert got.tobytes() == want[o].tobytes(), (what, o)


def test_rhs24_tables_interleaved_on_two_streams():
    """Two polynomial tables launched alternately on two streams without
    host synchronisation: each launch uses its own table."""
    import torch
    from paper_1308_1343_b200.configs import C5Rhs24
    a, b = C5Rhs24(n=10, seed=11).setup(), C5Rhs24(n=10, seed=12).setup()
    assert not np.array_equal(a.poly.coef, b.poly.coef)
    wa, wb = _rhs_want(a), _rhs_want(b)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(20):
        with torch.cuda.stream(sa):
            a.run()
        with torch.cuda.stream(sb):
            b.run()
    torch.cuda.synchronize()
    _check(a, wa, "table a")
    _check(b, wb, "table b")


def test_rhs24_graph_replays_its_own_table():
    import torch
    from paper_1308_1343_b200.configs import C5Rhs24
    from paper_1308_1343_b200.graphs import SweepGraph
    a, b = C5Rhs24(n=10, seed=21).setup(), C5Rhs24(n=10, seed=22).setup()
    wa, wb = _rhs_want(a), _rhs_want(b)
    g = SweepGraph(a.run, repeat=2, warmup=1)
    for o in a.outs:
        o.fill_(0.0)
    b.run()                 # a different table launched between capture and replay
    g.replay()
    torch.cuda.synchronize()
    _check(a, wa, "graph a")
    _check(b, wb, "direct b")


def test_lap7_iterate_captured_on_first_use():
    """sb_lap7_iterate's barrier counter comes from the pool sb_init
    reserves, so its first call may be inside a capture."""
    import torch
    from paper_1308_1343_b200 import inputs
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import Laplacian7
    from paper_1308_1343_b200.traverse import IndexSpace
    n, iters = 20, 6
    u = inputs.c1_field(n, 5)
    c0, c1 = inputs.c1_constants(n)
    a, b = DeviceGrid((n,) * 3, 1), DeviceGrid((n,) * 3, 1)
    a.upload(u, with_ghosts=True)
    b.upload(u, with_ghosts=True)
    k = Laplacian7(b, a, c0, c1)
    _lib.init_current_device()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        res = k.iterate(a, b, IndexSpace((0, 0, 0), (n, n, n)), iters)
    graph.replay()
    torch.cuda.synchronize()
    x, y = u.copy(), u.copy()
    for _ in range(iters):
        oracle.lap7_rows(y, x, 1, n + 1, 1, n + 1, 1, n + 1, c0, c1)
        x, y = y, x
    want = x[1:-1, 1:-1, 1:-1]
    assert res.download().tobytes() == np.ascontiguousarray(want).tobytes()


def test_shutdown_releases_and_library_stays_usable():
    """sb_shutdown frees the box tables and barrier counters; the next calls
    allocate again (lap7_iterate, a >8-box level)."""
    import torch
    from paper_1308_1343_b200 import inputs
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import Laplacian7, LevelLaplacian4
    from paper_1308_1343_b200.level import Box
    from paper_1308_1343_b200.traverse import IndexSpace
    from paper_1308_1343_b200.tuner import LaunchParams
    boxes = [Box((6 * i, 0, 0), (6 * i + 4, 5, 6)) for i in range(10)]
    srcs = [DeviceGrid(b.extents, 2, lower=b.lo) for b in boxes]
    dsts = [DeviceGrid(b.extents, 0, lower=b.lo) for b in boxes]
    lvl = LevelLaplacian4(dsts, srcs, inputs.D4Constants.for_spacing(0.1))
    lvl.launch(None, LaunchParams(32, 4, 4, 2))
    n = 12
    u = inputs.c1_field(n, 3)
    c0, c1 = inputs.c1_constants(n)
    a, b = DeviceGrid((n,) * 3, 1), DeviceGrid((n,) * 3, 1)
    a.upload(u, with_ghosts=True)
    b.upload(u, with_ghosts=True)
    k = Laplacian7(b, a, c0, c1)
    k.iterate(a, b, IndexSpace((0, 0, 0), (n, n, n)), 3)
    torch.cuda.synchronize()
    _lib.shutdown()
    for s in srcs:
        s.fill_(1.0)
    lvl.launch(None, LaunchParams(32, 4, 4, 2))
    res = k.iterate(a, b, IndexSpace((0, 0, 0), (n, n, n)), 3)
    torch.cuda.synchronize()
    # a constant field: the 4th-order Laplacian is exactly zero everywhere
    assert all(float(d.interior().abs().max()) == 0.0 for d in dsts)
    assert res.download().shape == (n, n, n)
