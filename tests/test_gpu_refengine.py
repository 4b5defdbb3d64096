"""The drop-in claim, proven against the reference's OWN engine: the
unmodified ``stencilrt`` package (installed under baseline/_ref, see
DESIGN.md §6) drives this repository's device kernel objects through its
plugin type ``Kernel = Callable[[IndexSpace], None]`` (traverse.py:159) —
``run_loop`` with its own ``Tuner`` (traverse.py:220-232), ``execute_plan``
with coarse and fine worker threads (traverse.py:162-209) and
``run_static`` (traverse.py:235-260) — over index spaces and a bboxset level
built by its own ``IndexSpace``/``BBoxSet`` types.  Results must be
byte-identical to the reference goldens.  Skipped (with the reason) when
baseline/_ref is absent."""
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1308_1343_b200 import _build, inputs

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def srt():
    if not (REF / "stencilrt").is_dir():
        pytest.skip(f"reference package not installed at {REF} (pip install --target baseline/_ref)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import stencilrt.bboxset
    import stencilrt.lattice
    import stencilrt.traverse
    import stencilrt.tuner
    _build.build()
    return stencilrt


def _sync():
    import torch
    torch.cuda.synchronize()


@pytest.mark.parametrize("threads", [(1, 1), (2, 2)])
def test_reference_run_loop_tunes_device_lap7(srt, golden, threads):
    """40 executions of the reference's run_loop + Tuner over the C1 box:
    every plan the tuner tries gives the reference's own output bytes."""
    from paper_1308_1343_b200.configs import C1Laplacian7
    T, TU = srt.traverse, srt.tuner
    meta, _ = golden
    p = C1Laplacian7().setup()
    nc, nf = threads
    topo = TU.TopologyConfig(n_coarse_threads=nc, n_fine_threads=nf)
    setup = TU.LoopSetup("laplacian3d", (64, 64, 64), "vector", nc, nf)
    tuner = TU.Tuner(topo)
    space = T.IndexSpace((0, 0, 0), (64, 64, 64))
    for _ in range(40):
        p.dst.fill_(0.0)
        secs = T.run_loop(setup, space, p.kernel, tuner)
        assert secs > 0
        _sync()
        assert inputs.sha256(p.outputs()[0]) == meta["c1"]["output_sha256"]
    assert len(tuner.log) == 40
    assert tuner.best(setup) is not None


def test_reference_execute_plan_and_run_static_drive_d4_all(srt, golden):
    """The ten config-2 outputs through the reference's execute_plan (two
    coarse x two fine workers) and run_static (4 threads) equal the golden."""
    from paper_1308_1343_b200.configs import C2FourthOrder
    T, TU = srt.traverse, srt.tuner
    meta, a = golden
    n = meta["c2"]["n"]
    p = C2FourthOrder(n=n, seed=meta["c2"]["seed"]).setup()
    space = T.IndexSpace((0, 0, 0), (n, n, n))
    setup = TU.LoopSetup("d4_all", (n, n, n), "vector", 2, 2)
    tuner = TU.Tuner(TU.TopologyConfig(n_coarse_threads=2, n_fine_threads=2))
    for _ in range(6):
        for o in p.outs:
            o.fill_(0.0)
        T.execute_plan(T.build_plan(space, tuner.next_params(setup)), p.kernel, 2, 2)
        _sync()
        for i, got in enumerate(p.outputs()):
            assert got.tobytes() == a["c2_out"][i].tobytes(), inputs.C2_OUTPUT_NAMES[i]
    for o in p.outs:
        o.fill_(0.0)
    T.run_static(space, p.kernel, 4)
    _sync()
    for i, got in enumerate(p.outputs()):
        assert got.tobytes() == a["c2_out"][i].tobytes(), inputs.C2_OUTPUT_NAMES[i]


def test_reference_bboxset_level_through_run_static(srt, golden):
    """A level built by the reference's BBoxSet algebra (difference ->
    to_bboxes) feeds the device box table; the reference's run_static
    sweeps the level's bounding space in z chunks (each piece clipped to
    every box), and the outputs equal the golden per-box Laplacians."""
    from paper_1308_1343_b200.configs import C4Level
    from paper_1308_1343_b200.level import boxes_of
    L, B, T = srt.lattice, srt.bboxset, srt.traverse
    meta, a = golden
    n = meta["c4"]["n"]
    outer = L.BBox(L.Point((0, 0, 0)), L.Point((n - 1,) * 3), L.Stride.ones(3))
    hole = L.BBox(L.Point((n // 2,) * 3), L.Point((n - 1,) * 3), L.Stride.ones(3))
    level = B.BBoxSet.from_bboxes([outer]).difference(B.BBoxSet.from_bboxes([hole]))
    boxes = boxes_of(level)
    assert len(boxes) == 3
    p = C4Level(n=n, seed=meta["c4"]["seed"], boxes=boxes).setup()
    space = T.index_space_from_bbox(outer)
    T.run_static(space, p.kernel, 3)
    _sync()
    for j, got in enumerate(p.outputs()):
        assert got.tobytes() == a[f"c4_out{j}"].tobytes(), j
    # the reference's run_loop over the same level space, with its own tuner
    TU = srt.tuner
    setup = TU.LoopSetup("lap4_level", space.extents, "vector", 1, 1)
    tuner = TU.Tuner(TU.TopologyConfig())
    for _ in range(8):
        for d in p.dsts:
            d.fill_(0.0)
        T.run_loop(setup, space, p.kernel, tuner)
        _sync()
        for j, got in enumerate(p.outputs()):
            assert got.tobytes() == a[f"c4_out{j}"].tobytes(), j
