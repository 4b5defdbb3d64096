"""Device parity: every sm_100a kernel, through the C ABI, against the oracle
and the reference's golden vectors — bit-exact (fp64, no FMA contraction,
the reference's association), so the tolerance is zero ulps."""
import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import _build, inputs
from paper_1308_1343_b200.errors import UsageError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    import torch
    torch.cuda.init()


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def first_diff(a, b):
    d = np.argwhere(a.view(np.int64) != b.view(np.int64))
    return None if d.size == 0 else (tuple(d[0]), a[tuple(d[0])], b[tuple(d[0])], len(d))


# -- K0 / K1 ------------------------------------------------------------------

def test_diff1d_matches_reference_vectors(golden):
    import torch
    from paper_1308_1343_b200 import vlanes
    _, a = golden
    off = 0
    for n in a["diff_len"]:
        n = int(n)
        src = torch.tensor(a["diff_in"][off:off + n], device="cuda")
        for fn, key in ((vlanes.forward_difference, "diff_fwd"), (vlanes.centered_difference, "diff_ctr")):
            dst = torch.zeros(n, dtype=torch.float64, device="cuda")
            fn(dst, src, n)
            assert bits_equal(dst.cpu().numpy(), a[key][off:off + n]), (n, key)
        off += n


def test_c1_lap7_matches_reference_hash(golden):
    from paper_1308_1343_b200.configs import C1Laplacian7
    meta, _ = golden
    p = C1Laplacian7().setup()
    p.run()
    out = p.outputs()[0]
    assert inputs.sha256(out) == meta["c1"]["output_sha256"]


@pytest.mark.parametrize("params", [(64, 8, 16), (64, 1, 64), (64, 4, 3), (64, 2, 7)])
def test_c1_lap7_any_launch_shape(golden, params):
    from paper_1308_1343_b200.configs import C1Laplacian7
    from paper_1308_1343_b200.tuner import LaunchParams
    meta, _ = golden
    p = C1Laplacian7().setup()
    p.run(LaunchParams(*params))
    assert inputs.sha256(p.outputs()[0]) == meta["c1"]["output_sha256"]


def test_reference_demo_drivers_bit_identical(golden):
    from paper_1308_1343_b200 import stencil
    from paper_1308_1343_b200.tuner import TopologyConfig
    meta, a = golden
    d = meta["demo"]
    assert bits_equal(stencil.run_serial(16, d["n16_iters"], d["seed"]).final, a["demo16_final"])
    s = stencil.run_serial(64, d["n64_iters"], d["seed"])
    nv = stencil.run_naive(64, d["n64_iters"], d["seed"], 2)
    topo = TopologyConfig(n_coarse_threads=2, n_fine_threads=1, lane_width=4, rng_seed=d["seed"])
    tu, tuner = stencil.run_tuned(64, d["n64_iters"], d["seed"], topo)
    assert inputs.sha256(s.final) == d["n64_final_sha256"]
    assert stencil.bit_identical(s.final, nv.final) and stencil.bit_identical(s.final, tu.final)
    assert len(tuner.log) == d["n64_iters"]


@pytest.mark.parametrize("n,iters", [(64, 100), (16, 8), (19, 7), (64, 1), (130, 6)])
def test_persistent_sweeps_match_serial(golden, n, iters):
    """All sweeps in one cooperative launch (grid barrier between sweeps)
    give the serial driver's bits, odd and even counts, ragged extents."""
    from paper_1308_1343_b200 import stencil
    meta, a = golden
    d = meta["demo"]
    got = stencil.run_persistent(n, iters, d["seed"]).final
    if (n, iters) == (64, d["n64_iters"]):
        assert inputs.sha256(got) == d["n64_final_sha256"]
    if (n, iters) == (16, d["n16_iters"]):
        assert bits_equal(got, a["demo16_final"])
    assert stencil.bit_identical(got, stencil.run_serial(n, iters, d["seed"]).final)


def test_graphed_demo_matches_reference(golden):
    """The CUDA-graph-captured sweep loop gives the reference's bits."""
    from paper_1308_1343_b200 import stencil
    meta, a = golden
    d = meta["demo"]
    g = stencil.run_graphed(64, d["n64_iters"], d["seed"], batch=16)
    assert inputs.sha256(g.final) == d["n64_final_sha256"]
    assert len(g.iter_seconds) == d["n64_iters"]
    g16 = stencil.run_graphed(16, d["n16_iters"], d["seed"], batch=3)
    assert bits_equal(g16.final, a["demo16_final"])


def test_lap7_masked_subspace_writes_only_inside():
    """Odd x origin, ragged extents: only points of the space change (the
    iterate_masked frame rule)."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import Laplacian7
    from paper_1308_1343_b200.traverse import IndexSpace
    n = 37
    u = inputs.c1_field(n, seed=5)
    src = DeviceGrid((n,) * 3, 1)
    src.upload(u)
    dst = DeviceGrid((n,) * 3, 0).fill_(0.125)
    space = IndexSpace((3, 1, 2), (36, 30, 35))
    Laplacian7(dst, src, -3.0, 0.5)(space)
    got = dst.download()
    want = np.full((n, n, n), 0.125)
    tmp = u.copy()
    oracle.lap7_rows(tmp, u, 3, 36, 2, 31, 4, 37, -3.0, 0.5)
    want[2:35, 1:30, 3:36] = tmp[3:36, 2:31, 4:37]
    assert bits_equal(got, want), first_diff(got, want)


# -- K2 -------------------------------------------------------------------------

def _d4_oracle(u, n, g, k, region=None):
    region = region or (0, n, 0, n, 0, n)
    x0, x1, y0, y1, z0, z1 = region
    outs = [np.full((n, n, n), np.nan) for _ in range(10)]
    oracle.d4_all(outs, u, g, region, k)
    return [o[z0:z1, y0:y1, x0:x1] for o in outs]


def test_c2_small_golden(golden):
    from paper_1308_1343_b200.configs import C2FourthOrder
    from paper_1308_1343_b200.tuner import LaunchParams
    meta, a = golden
    p = C2FourthOrder(n=meta["c2"]["n"], seed=meta["c2"]["seed"]).setup()
    for params in [(32, 2, 8), (64, 4, 4), (128, 2, 3)]:
        p.run(LaunchParams(*params))
        for i, got in enumerate(p.outputs()):
            assert bits_equal(got, a["c2_out"][i]), (params, inputs.C2_OUTPUT_NAMES[i], first_diff(got, a["c2_out"][i]))


@pytest.mark.parametrize("params", [(64, 4, 32), (32, 8, 16), (128, 2, 64), (64, 1, 5), (64, 2, 40)])
def test_c2_medium_vs_oracle(params):
    from paper_1308_1343_b200.configs import C2FourthOrder
    from paper_1308_1343_b200.tuner import LaunchParams
    n = 72
    p = C2FourthOrder(n=n, seed=123).setup()
    p.run(LaunchParams(*params))
    want = _d4_oracle(p.host_u, n, 2, p.k)
    for i, got in enumerate(p.outputs()):
        assert bits_equal(got, want[i]), (params, inputs.C2_OUTPUT_NAMES[i], first_diff(got, want[i]))


def test_c2_full_size_slabs_and_identities():
    """256^3: z slabs at both faces and the middle against the oracle; every
    point: Lap4 == (Dxx + Dyy) + Dzz bitwise; launch shapes agree bitwise."""
    import torch
    from paper_1308_1343_b200.configs import C2FourthOrder
    from paper_1308_1343_b200.tuner import LaunchParams
    p = C2FourthOrder().setup()
    n = p.n
    p.run(LaunchParams(64, 4, 32))
    outs = [o.interior() for o in p.outs]
    assert torch.equal((outs[3] + outs[4]) + outs[5], outs[9])
    for z0, z1 in ((0, 3), (127, 130), (253, 256)):
        want = _d4_oracle(p.host_u, n, 2, p.k, (0, n, 0, n, z0, z1))
        for i in range(10):
            got = outs[i][z0:z1].cpu().numpy()
            assert bits_equal(got, want[i]), (z0, inputs.C2_OUTPUT_NAMES[i], first_diff(got, want[i]))
    ref = [o.clone() for o in outs]
    p.run(LaunchParams(32, 8, 256))
    for i in range(10):
        assert torch.equal(outs[i], ref[i])


def test_d4_masked_subspace_writes_only_inside():
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import FourthOrderAll
    from paper_1308_1343_b200.traverse import IndexSpace
    from paper_1308_1343_b200.tuner import LaunchParams
    n, g = 41, 2
    u = inputs.c2_field(n, g, seed=9)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    src = DeviceGrid((n,) * 3, g)
    src.upload(u)
    outs = [DeviceGrid((n,) * 3, 0).fill_(0.125) for _ in range(10)]
    kern = FourthOrderAll(outs, src, k)
    space = IndexSpace((5, 3, 1), (40, 38, 39))
    kern.launch(space, LaunchParams(64, 4, 7))
    want = [np.full((n, n, n), 0.125) for _ in range(10)]
    oracle.d4_all(want, u, g, (5, 40, 3, 38, 1, 39), k)
    for i in range(10):
        got = outs[i].download()
        assert bits_equal(got, want[i]), (inputs.C2_OUTPUT_NAMES[i], first_diff(got, want[i]))


# -- K3 ---------------------------------------------------------------------------

def test_c4_small_level_golden(golden):
    from paper_1308_1343_b200.configs import C4Level
    from paper_1308_1343_b200.tuner import LaunchParams
    meta, a = golden
    p = C4Level(n=meta["c4"]["n"], seed=meta["c4"]["seed"]).setup()
    p.run(LaunchParams(64, 8, 4))
    for j, got in enumerate(p.outputs()):
        assert bits_equal(got, a[f"c4_out{j}"]), (j, first_diff(got, a[f"c4_out{j}"]))


def test_c4_full_level_slabs():
    from paper_1308_1343_b200.configs import C4Level
    from paper_1308_1343_b200.tuner import LaunchParams
    p = C4Level().setup()
    p.run(LaunchParams(64, 8, 32))
    for b, u, d in zip(p.boxes, p.host_u, p.dsts):
        nx, ny, nz = b.extents
        inter = d.interior()
        for z0, z1 in ((0, 2), (nz // 2 - 1, nz // 2 + 1), (nz - 2, nz)):
            want = np.empty((z1 - z0, ny, nx))
            full = np.empty((nz, ny, nx))
            oracle.lap4(full, u, 2, (0, nx, 0, ny, z0, z1), p.k.k2)
            want = full[z0:z1]
            got = inter[z0:z1].cpu().numpy()
            assert bits_equal(got, want), (b, z0, first_diff(got, want))


def test_level_sweep_through_run_loop():
    """A bboxset level swept by the engine: tuner-driven launches are bit-identical."""
    from paper_1308_1343_b200.configs import C4Level
    from paper_1308_1343_b200.traverse import run_loop
    from paper_1308_1343_b200.tuner import LoopSetup, TopologyConfig, Tuner
    p = C4Level(n=64, seed=4).setup()
    p.run()
    want = p.outputs()
    tuner = Tuner(TopologyConfig())
    setup = LoopSetup(p.kernel.site_id, p.kernel.full_space().extents)
    for _ in range(12):
        for d in p.dsts:
            d.fill_(0.0)
        run_loop(setup, p.kernel.full_space(), p.kernel, tuner)
        for w, got in zip(want, p.outputs()):
            assert bits_equal(got, w)
    assert len(tuner.log) == 12


# -- K4 / K5 ----------------------------------------------------------------------

def test_ghost_periodic_is_wrap_image():
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import PeriodicGhosts
    n, g = 19, 2
    a = np.random.default_rng(1).random((n + 2 * g,) * 3)
    d = DeviceGrid((n,) * 3, g)
    d.upload(a)
    PeriodicGhosts(d)()
    want = a.copy()
    oracle.periodic_fill(want, g)
    got = d.download(with_ghosts=True)
    assert bits_equal(got, want), first_diff(got, want)


def test_c3_small_golden(golden):
    from paper_1308_1343_b200.configs import C3WaveRK4
    from paper_1308_1343_b200.tuner import LaunchParams
    meta, a = golden
    p = C3WaveRK4(n=meta["c3"]["n"], seed=meta["c3"]["seed"]).setup()
    p.run(LaunchParams(64, 8, 4))
    phi, pi = p.outputs()
    assert bits_equal(phi, a["c3_phi1"]), first_diff(phi, a["c3_phi1"])
    assert bits_equal(pi, a["c3_pi1"]), first_diff(pi, a["c3_pi1"])


@pytest.mark.parametrize("schedule", ["pairs", "lap_pairs", "stages", "stages_unfused"])
@pytest.mark.parametrize("params", [(64, 4, 16, 2), (128, 2, 48, 1), (32, 8, 5, 1)])
def test_c3_medium_vs_oracle(schedule, params):
    """Interior and (fused) periodic ghost shell of phi after one RK4 step."""
    from paper_1308_1343_b200.configs import C3WaveRK4
    from paper_1308_1343_b200.tuner import LaunchParams
    n, g = 48, 2
    fused = schedule != "stages_unfused"
    p = C3WaveRK4(n=n, seed=77, schedule=schedule).setup()
    p.run(LaunchParams(*params))
    phi, pi = p.outputs()
    wphi, wpi = oracle.rk4_step(p.host_phi, p.host_pi, g, p.c)
    I = (slice(g, g + n),) * 3
    assert bits_equal(phi, wphi[I]), first_diff(phi, wphi[I])
    assert bits_equal(pi, wpi[I]), first_diff(pi, wpi[I])
    if fused:
        full = p.phi_with_ghosts()
        assert bits_equal(full, wphi), first_diff(full, wphi)


@pytest.mark.parametrize("schedule", ["pairs", "lap_pairs", "stages", "stages_unfused"])
def test_c3_two_steps_advance(schedule):
    """advance() twice equals two oracle steps (ghosts carried by the fused refill)."""
    from paper_1308_1343_b200.configs import C3WaveRK4
    n, g = 24, 2
    p = C3WaveRK4(n=n, seed=5, schedule=schedule).setup()
    p.rk.advance()
    p.rk.advance()
    a, b = oracle.rk4_step(p.host_phi, p.host_pi, g, p.c)
    a, b = oracle.rk4_step(a, b, g, p.c)
    I = (slice(g, g + n),) * 3
    got = p.rk.phi0.download()
    assert bits_equal(got, a[I]), first_diff(got, a[I])
    assert bits_equal(p.rk.pi0.download(), b[I])


def test_c3_full_size_zero_state_and_shapes_agree():
    """384^3: phi = pi = 0 stays exactly 0; two launch shapes agree bitwise on
    the real initial data."""
    import torch
    from paper_1308_1343_b200.configs import C3WaveRK4
    from paper_1308_1343_b200.tuner import LaunchParams
    p = C3WaveRK4().setup()
    p.run(LaunchParams(64, 8, 32))
    a = [t.interior().clone() for t in (p.rk.phi_b, p.rk.pi_b)]
    p.run(LaunchParams(128, 4, 96))
    b = [t.interior() for t in (p.rk.phi_b, p.rk.pi_b)]
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert torch.isfinite(a[0]).all()
    p.rk.phi0.fill_(0.0)
    p.rk.pi0.fill_(0.0)
    p.run()
    assert int(torch.count_nonzero(p.rk.phi_b.interior())) == 0
    assert int(torch.count_nonzero(p.rk.pi_b.interior())) == 0


# -- K6 ---------------------------------------------------------------------------

def test_c5_small_golden(golden):
    from paper_1308_1343_b200.configs import C5Rhs24
    meta, a = golden
    p = C5Rhs24(n=meta["c5"]["n"], seed=meta["c5"]["seed"]).setup()
    p.run()
    for o, got in enumerate(p.outputs()):
        assert bits_equal(got, a["c5_out"][o]), (o, first_diff(got, a["c5_out"][o]))


def test_c5_medium_vs_oracle():
    from paper_1308_1343_b200.configs import C5Rhs24
    n, g = 18, 2
    p = C5Rhs24(n=n, seed=55).setup()
    p.run()
    want = [np.empty((n, n, n)) for _ in range(24)]
    oracle.rhs24(want, p.host_u, g, (0, n, 0, n, 0, n), p.k, p.poly)
    for o, got in enumerate(p.outputs()):
        assert bits_equal(got, want[o]), (o, first_diff(got, want[o]))


def test_c5_full_size_slab():
    from paper_1308_1343_b200.configs import C5Rhs24
    p = C5Rhs24().setup()
    p.run()
    n = p.n
    for z0, z1 in ((0, 1), (95, 97), (191, 192)):
        want = [np.empty((n, n, n)) for _ in range(24)]
        oracle.rhs24(want, p.host_u, 2, (0, n, 0, n, z0, z1), p.k, p.poly)
        for o in range(24):
            got = p.outs[o].interior()[z0:z1].cpu().numpy()
            assert bits_equal(got, want[o][z0:z1]), (z0, o)


# -- errors -----------------------------------------------------------------------

def test_bad_launch_params_raise_usage_error():
    from paper_1308_1343_b200.configs import C2FourthOrder
    from paper_1308_1343_b200.tuner import LaunchParams
    p = C2FourthOrder(n=16, seed=1).setup()
    with pytest.raises(UsageError):
        p.run(LaunchParams(48, 4, 4))
    with pytest.raises(UsageError):
        p.run(LaunchParams(64, 16, 4))   # 512 consumer threads > d4_all limit


def test_level_ghost_sync_matches_global_field():
    """F1: after the inter-box ghost fill every ghost point that lies inside
    the level equals the neighbouring box's interior value; others untouched."""
    from paper_1308_1343_b200.configs import C4Level
    n, g = 40, 2
    p = C4Level(n=n, seed=3).setup()
    glob = np.full((n, n, n), np.nan)
    for b, u in zip(p.boxes, p.host_u):
        nx, ny, nz = b.extents
        glob[b.lo[2]:b.hi[2] + 1, b.lo[1]:b.hi[1] + 1, b.lo[0]:b.hi[0] + 1] = u[g:g + nz, g:g + ny, g:g + nx]
    p.ghost_sync()
    assert p.ghost_sync.points() > 0
    for b, u, s in zip(p.boxes, p.host_u, p.srcs):
        got = s.download(with_ghosts=True)
        want = u.copy()
        nx, ny, nz = b.extents
        for kz in range(nz + 2 * g):
            for ky in range(ny + 2 * g):
                z, y = b.lo[2] - g + kz, b.lo[1] - g + ky
                if not (0 <= z < n and 0 <= y < n):
                    continue
                xs = np.arange(b.lo[0] - g, b.hi[0] + g + 1)
                ok = (xs >= 0) & (xs < n)
                row = np.where(ok, glob[z, y, np.clip(xs, 0, n - 1)], np.nan)
                fill = ~np.isnan(row)
                want[kz, ky, fill] = row[fill]
        assert bits_equal(got, want), first_diff(got, want)


@pytest.mark.parametrize("chunk", [None, 16, 100])
def test_c2_host_pipeline_matches_device_run(chunk):
    """run_host (chunked H2D / sweep / D2H on three streams) returns the same
    bits as the resident sweep, and uploads the whole input."""
    import torch
    from paper_1308_1343_b200.configs import C2FourthOrder
    n = 72
    p = C2FourthOrder(n=n, seed=31).setup()
    p.run()
    want = p.outputs()
    p.src.fill_(0.0)
    for o in p.outs:
        o.fill_(0.0)
    h_in = torch.from_numpy(p.host_u).pin_memory()
    h_out = [torch.empty((n, n, n), dtype=torch.float64).pin_memory() for _ in range(10)]
    for _ in range(2):
        p.e2e_step(h_in.data_ptr(), [t.data_ptr() for t in h_out], chunk=chunk)
    torch.cuda.synchronize()
    for w, h in zip(want, h_out):
        assert bits_equal(h.numpy(), w)
    assert bits_equal(p.src.download(with_ghosts=True), p.host_u)


def test_d2_all_golden_and_oracle(golden):
    """2nd-order ten-output sweep: reference-vlanes golden (n=8) and the
    oracle at n=40 on several launch shapes, sub-space included."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import SecondOrderAll
    from paper_1308_1343_b200.traverse import IndexSpace
    from paper_1308_1343_b200.tuner import LaunchParams
    meta, a = golden
    m = meta["c2_order2"]
    for n, u, want_all in ((m["n"], a["c2o2_in"], None), (40, inputs.c2_field(40, 2, seed=44), None)):
        k = inputs.D2Constants.for_spacing(1.0 / n)
        src = DeviceGrid((n,) * 3, 2)
        src.upload(u)
        outs = [DeviceGrid((n,) * 3, 0).fill_(0.5) for _ in range(10)]
        kern = SecondOrderAll(outs, src, k)
        for params in [(32, 4, 4, 2), (64, 2, 7, 1)]:
            kern.launch(IndexSpace((0, 0, 0), (n, n, n)), LaunchParams(*params))
            want = [np.empty((n, n, n)) for _ in range(10)]
            oracle.d2_all(want, u, 2, (0, n, 0, n, 0, n), k)
            for i in range(10):
                got = outs[i].download()
                assert bits_equal(got, want[i]), (n, params, i, first_diff(got, want[i]))
                if n == m["n"]:
                    assert bits_equal(got, a["c2o2_out"][i])


def test_launch_plan_equals_execute_plan_piece_by_piece():
    """kernel.launch_plan(build_plan(...)) — one launch over the plan's space —
    writes exactly what execute_plan writes piece by piece (traverse.py:130-209)."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import FourthOrderAll
    from paper_1308_1343_b200.traverse import IndexSpace, build_plan, execute_plan
    from paper_1308_1343_b200.tuner import ExecParams
    rng = np.random.default_rng(41)
    ext, g = (45, 19, 13), 2
    u = rng.uniform(-1, 1, (ext[2] + 2 * g, ext[1] + 2 * g, ext[0] + 2 * g))
    k = inputs.D4Constants.for_spacing(1.0 / 45)
    src = DeviceGrid(ext, g, lower=(3, -2, 5))
    src.upload(u)
    space = IndexSpace((4, -1, 6), (44, 15, 17))
    plan = build_plan(space, ExecParams((2, 1, 2), (16, 8, 4), (2, 1, 1), 4))
    outs = []
    for run in ("pieces", "plan"):
        o = [DeviceGrid(ext, 0, lower=(3, -2, 5)).fill_(0.5) for _ in range(10)]
        kern = FourthOrderAll(o, src, k)
        if run == "pieces":
            execute_plan(plan, kern, 2, 2)
        else:
            kern.launch_plan(plan)
        outs.append([x.download() for x in o])
    for a, b in zip(*outs):
        assert a.tobytes() == b.tobytes()
    assert not np.all(outs[1][9] == 0.5)
