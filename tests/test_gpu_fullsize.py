"""Whole-volume parity at the BASELINE.json shapes — every output point of
every config compared bit for bit with the oracle (the reference's contract
is whole-array byte identity: ``bit_identical``, stencil.py:97-98;
criterion 9, test_acceptance.py:217-231).  Tolerance: zero ulps.

The oracle runs on all host threads through its static z split
(traverse.py:235-260 restated, oracle.run_static): config 3 one RK4 step of
384^3 in a few seconds, config 5 (~44 G numpy ops) in about 15 s on the GPU
box's 16 threads.  Each comparison reports the first differing point."""
import numpy as np
import pytest

import oracle
from oracle.stencils import host_threads
from paper_1308_1343_b200 import _build, inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    import torch
    torch.cuda.init()


def _same(got: np.ndarray, want: np.ndarray, what) -> None:
    got, want = np.ascontiguousarray(got), np.ascontiguousarray(want)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    if got.tobytes() != want.tobytes():
        d = np.argwhere(got.view(np.int64) != want.view(np.int64))
        i = tuple(d[0])
        pytest.fail(f"{what}: {len(d)} points differ; first (z,y,x)={i}: got {got[i]!r} want {want[i]!r}")


def _threads() -> int:
    return host_threads()


# -- config 2: all ten outputs of the whole 256^3 box ---------------------------

@pytest.mark.parametrize("shape", [None, (32, 4, 4, 2)])   # default launch / the bench's tuned shape
def test_c2_whole_volume_all_ten_outputs(shape):
    from paper_1308_1343_b200.configs import C2FourthOrder
    from paper_1308_1343_b200.tuner import LaunchParams
    p = C2FourthOrder().setup()
    p.run(None if shape is None else LaunchParams(*shape))
    n, g = p.n, p.g
    want = [np.empty((n, n, n)) for _ in range(10)]
    oracle.run_static(lambda z0, z1: oracle.d4_all(want, p.host_u, g, (0, n, 0, n, z0, z1), p.k), 0, n, _threads())
    for i, got in enumerate(p.outputs()):
        _same(got, want[i], f"C2 {inputs.C2_OUTPUT_NAMES[i]}")


# -- config 3: one and two RK4 steps of the whole 384^3 periodic box -------------

@pytest.fixture(scope="module")
def c3_oracle():
    from paper_1308_1343_b200.configs import C3WaveRK4
    prob = C3WaveRK4()
    one = oracle.rk4_step(prob.host_phi, prob.host_pi, prob.g, prob.c, threads=_threads())
    return prob, one


@pytest.mark.parametrize("schedule", ["lap_pairs", "pairs", "stages"])
def test_c3_whole_volume_one_step_with_ghost_shells(c3_oracle, schedule):
    """phi' and pi' including their ghost shells (the fused schedules refresh
    them in the same launches; the four-stage schedule refreshes phi's)."""
    from paper_1308_1343_b200.configs import C3WaveRK4
    prob, (wphi, wpi) = c3_oracle
    p = C3WaveRK4(schedule=schedule)
    p.host_phi, p.host_pi = prob.host_phi, prob.host_pi
    p.setup()
    p.run()
    g, n = p.g, p.n
    I = (slice(g, g + n),) * 3
    _same(p.phi_with_ghosts(), wphi, f"C3[{schedule}] phi' with ghosts")
    phi, pi = p.outputs()
    _same(pi, wpi[I], f"C3[{schedule}] pi' interior")
    if "pairs" in schedule:
        _same(p.rk.pi_b.download(with_ghosts=True), wpi, f"C3[{schedule}] pi' ghost shell")


def test_c3_whole_volume_two_steps_advance(c3_oracle):
    """advance() twice on the full box: the second step starts from the
    ghost shells the first one wrote (no separate refill)."""
    from paper_1308_1343_b200.configs import C3WaveRK4
    prob, (wphi, wpi) = c3_oracle
    a, b = oracle.rk4_step(wphi, wpi, prob.g, prob.c, threads=_threads())
    p = C3WaveRK4()
    p.host_phi, p.host_pi = prob.host_phi, prob.host_pi
    p.setup()
    p.rk.advance()
    p.rk.advance()
    _same(p.rk.phi0.download(with_ghosts=True), a, "C3 two steps phi with ghosts")
    _same(p.rk.pi0.download(with_ghosts=True), b, "C3 two steps pi with ghosts")


# -- config 4: the whole 512^3 level (3 boxes, one launch) ----------------------

def test_c4_whole_level():
    from paper_1308_1343_b200.configs import C4Level
    p = C4Level().setup()
    p.run()
    for j, (b, u, got) in enumerate(zip(p.boxes, p.host_u, p.outputs())):
        nx, ny, nz = b.extents
        want = np.empty((nz, ny, nx))
        oracle.run_static(lambda z0, z1: oracle.lap4(want, u, p.g, (0, nx, 0, ny, z0, z1), p.k.k2), 0, nz,
                          _threads())
        _same(got, want, f"C4 box {j} {b}")


# -- config 5: all 24 right-hand sides of the whole 192^3 box --------------------

def test_c5_whole_volume_all_24_outputs():
    from paper_1308_1343_b200.configs import C5Rhs24
    p = C5Rhs24().setup()
    p.run()
    n, g = p.n, p.g
    want = [np.empty((n, n, n)) for _ in range(24)]

    def planes(z0, z1):      # two planes at a time: 240 operand arrays per thread stay small
        for z in range(z0, z1, 2):
            oracle.rhs24(want, p.host_u, g, (0, n, 0, n, z, min(z1, z + 2)), p.k, p.poly)

    oracle.run_static(planes, 0, n, _threads())
    for o, got in enumerate(p.outputs()):
        _same(got, want[o], f"C5 output {o}")


def test_c2_second_order_set_whole_volume():
    """north_star (c)'s 2nd-order operator set (sb_d2_all) over the whole
    256^3 box, all ten outputs."""
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import SecondOrderAll
    n, g = 256, 2
    u = inputs.c2_field(n, g)
    k = inputs.D2Constants.for_spacing(1.0 / n)
    src = DeviceGrid((n,) * 3, g)
    src.upload(u, with_ghosts=True)
    outs = [DeviceGrid((n,) * 3, 0) for _ in range(10)]
    kern = SecondOrderAll(outs, src, k)
    kern.launch(kern.full_space(), kern.default_params)
    want = [np.empty((n, n, n)) for _ in range(10)]
    oracle.run_static(lambda z0, z1: oracle.d2_all(want, u, g, (0, n, 0, n, z0, z1), k), 0, n, _threads())
    for i, o in enumerate(outs):
        _same(o.download(), want[i], f"C2 order-2 {inputs.C2_OUTPUT_NAMES[i]}")
