"""Generate the golden fixtures that pin the oracle — run HERE, with the
reference at /root/reference (it does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything in tests/golden/{golden.json,golden.npz} comes out of the
reference's own code:

1. config 1: ``stencilrt.stencil._update_rows`` (stencil.py:31-39) with its
   module constants set to C0 = -6/h^2, C1 = 1/h^2 on the seeded 66^3
   config-1 field (SHA-256 of input and output), plus a small case stored
   whole;
2. the reference's stencil demo ``run_serial`` (stencil.py:55-65), n=16 x 8
   iterations stored whole, n=64 x 100 iterations (criterion 9) by hash —
   ``run_naive``/``run_tuned`` are checked equal to it here;
3. vlanes ``forward_difference``/``centered_difference`` (vlanes.py:342-360)
   on the criterion-6 inputs (lengths 1..129, random.Random(960000));
4. configs 2-5 at small sizes, evaluated lane by lane with the reference's
   vlanes API (iterate_masked / vload_off / vadd / vsub / vmul /
   vstore_partial) and driven through the reference's traverse engine
   (build_plan + execute_plan with several parameter settings and worker
   counts; outputs must agree bit for bit across all of them).  The
   expression trees are SURVEY.md App. A, written here independently of
   oracle/stencils.py;
5. config 4's level decomposition: BBoxSet([0,511]^3).difference(upper
   octant).to_bboxes(), and the same for a 16^3 level used in tests.
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import stencilrt.stencil as st  # noqa: E402
import stencilrt.vlanes as vl  # noqa: E402
from stencilrt.bboxset import BBoxSet  # noqa: E402
from stencilrt.lattice import BBox, Point, Stride  # noqa: E402
from stencilrt.traverse import IndexSpace, build_plan, execute_plan  # noqa: E402
from stencilrt.tuner import LoopSetup, TopologyConfig, enumerate_valid_params  # noqa: E402

from paper_1308_1343_b200 import inputs  # noqa: E402

W = 4
PAD = W + 4


# -- vlanes helpers ---------------------------------------------------------------

class LaneGrid:
    """A ghosted numpy array as one vlanes.AlignedArray per (z, y) row."""

    def __init__(self, a: np.ndarray):
        self.shape = a.shape
        self.rows = {(z, y): vl.AlignedArray.from_values(list(a[z, y, :]), W, PAD)
                     for z in range(a.shape[0]) for y in range(a.shape[1])}

    def load(self, z, y, i, dx):
        return vl.vload_off(dx, self.rows[(z, y)], i + dx)

    def to_numpy(self) -> np.ndarray:
        out = np.empty(self.shape)
        for (z, y), r in self.rows.items():
            out[z, y, :] = r.to_list()
        return out


def blank(shape) -> LaneGrid:
    return LaneGrid(np.zeros(shape))


c = lambda v: vl.vset1(v, W)
add, sub, mul = vl.vadd, vl.vsub, vl.vmul


def d1u(m2, m1, p1, p2):
    return add(sub(m2, p2), mul(c(8.0), sub(p1, m1)))


def d2(m2, m1, cc, p1, p2, k2):
    return mul(sub(sub(mul(c(16.0), add(m1, p1)), add(m2, p2)), mul(c(30.0), cc)), c(k2))


def slots(G: LaneGrid, z, y, i, k):
    """value + 9 derivatives at lanes i..i+W-1 of row (z, y)."""
    L = lambda dz, dy, dx: G.load(z + dz, y + dy, i, dx)
    rx = lambda dz, dy: d1u(L(dz, dy, -2), L(dz, dy, -1), L(dz, dy, 1), L(dz, dy, 2))
    ry = lambda dz, dx: d1u(L(dz, -2, dx), L(dz, -1, dx), L(dz, 1, dx), L(dz, 2, dx))
    cc = L(0, 0, 0)
    return [
        cc,
        mul(rx(0, 0), c(k.k1)),
        mul(ry(0, 0), c(k.k1)),
        mul(d1u(L(-2, 0, 0), L(-1, 0, 0), L(1, 0, 0), L(2, 0, 0)), c(k.k1)),
        d2(L(0, 0, -2), L(0, 0, -1), cc, L(0, 0, 1), L(0, 0, 2), k.k2),
        d2(L(0, -2, 0), L(0, -1, 0), cc, L(0, 1, 0), L(0, 2, 0), k.k2),
        d2(L(-2, 0, 0), L(-1, 0, 0), cc, L(1, 0, 0), L(2, 0, 0), k.k2),
        mul(d1u(rx(0, -2), rx(0, -1), rx(0, 1), rx(0, 2)), c(k.k11)),
        mul(d1u(rx(-2, 0), rx(-1, 0), rx(1, 0), rx(2, 0)), c(k.k11)),
        mul(d1u(ry(-2, 0), ry(-1, 0), ry(1, 0), ry(2, 0)), c(k.k11)),
    ]


def sweep(piece_fn, shape_ghosted, g, n_settings=4, seed=0):
    """Run piece_fn over the interior through the reference's build_plan +
    execute_plan with several params/worker counts; return the common result."""
    nz, ny, nx = (s - 2 * g for s in shape_ghosted)
    space = IndexSpace((g, g, g), (g + nx, g + ny, g + nz))
    setup = LoopSetup("golden", space.extents, "vector", 2, 1)
    topo = TopologyConfig(n_coarse_threads=2, n_fine_threads=1, lane_width=W)
    pool = enumerate_valid_params(setup, topo)
    rng = random.Random(seed)
    picks = rng.sample(pool, min(n_settings, len(pool)))
    ref = None
    for params in picks:
        for workers in (1, 2):
            got = piece_fn(lambda kern: execute_plan(build_plan(space, params), kern, workers, 1))
            got = [np.asarray(a) for a in got]
            if ref is None:
                ref = got
            else:
                for a, b in zip(ref, got):
                    assert a.tobytes() == b.tobytes(), ("decomposition changed bits", params, workers)
    return ref


def rows_of(piece):
    (x0, y0, z0), (x1, y1, z1) = piece.lo, piece.hi
    for z in range(z0, z1):
        for y in range(y0, y1):
            for i, m in vl.iterate_masked(x0, x1, W):
                yield z, y, i, m


def strip(a: np.ndarray, g: int) -> np.ndarray:
    return a[g:-g, g:-g, g:-g].copy() if g else a


# -- config 2 ---------------------------------------------------------------------------

def golden_c2(n=8, g=2):
    u = inputs.c2_field(n, g, seed=inputs.seed_for(2) + 1000)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    G = LaneGrid(u)

    def run(execute):
        outs = [blank(u.shape) for _ in range(10)]

        def kern(piece):
            for z, y, i, m in rows_of(piece):
                s = slots(G, z, y, i, k)
                vals = s[1:] + [add(add(s[4], s[5]), s[6])]
                for o, v in zip(outs, vals):
                    vl.vstore_partial(o.rows[(z, y)], i, v, m)
        execute(kern)
        return [strip(o.to_numpy(), g) for o in outs]
    return u, sweep(run, u.shape, g)


def slots_o2(G: LaneGrid, z, y, i, k):
    """2nd-order: value + 9 derivatives (d = u[+1] - u[-1], D2 = ((u[-1]+u[+1]) - 2u) k2)."""
    L = lambda dz, dy, dx: G.load(z + dz, y + dy, i, dx)
    ex = lambda dz, dy: sub(L(dz, dy, 1), L(dz, dy, -1))
    ey = lambda dz, dx: sub(L(dz, 1, dx), L(dz, -1, dx))
    sec = lambda m, cc, p: mul(sub(add(m, p), mul(c(2.0), cc)), c(k.k2))
    cc = L(0, 0, 0)
    return [
        cc,
        mul(ex(0, 0), c(k.k1)),
        mul(ey(0, 0), c(k.k1)),
        mul(sub(L(1, 0, 0), L(-1, 0, 0)), c(k.k1)),
        sec(L(0, 0, -1), cc, L(0, 0, 1)),
        sec(L(0, -1, 0), cc, L(0, 1, 0)),
        sec(L(-1, 0, 0), cc, L(1, 0, 0)),
        mul(sub(ex(0, 1), ex(0, -1)), c(k.k11)),
        mul(sub(ex(1, 0), ex(-1, 0)), c(k.k11)),
        mul(sub(ey(1, 0), ey(-1, 0)), c(k.k11)),
    ]


def golden_c2_order2(n=8, g=2):
    u = inputs.c2_field(n, g, seed=inputs.seed_for(2) + 2000)
    k = inputs.D2Constants.for_spacing(1.0 / n)
    G = LaneGrid(u)

    def run(execute):
        outs = [blank(u.shape) for _ in range(10)]

        def kern(piece):
            for z, y, i, m in rows_of(piece):
                s = slots_o2(G, z, y, i, k)
                vals = s[1:] + [add(add(s[4], s[5]), s[6])]
                for o, v in zip(outs, vals):
                    vl.vstore_partial(o.rows[(z, y)], i, v, m)
        execute(kern)
        return [strip(o.to_numpy(), g) for o in outs]
    return u, sweep(run, u.shape, g, n_settings=2)


# -- config 4 (and the Lap4 operator of config 3) ---------------------------------

def lap4_lanes(G, z, y, i, k2):
    L = lambda dz, dy, dx: G.load(z + dz, y + dy, i, dx)
    cc = L(0, 0, 0)
    dxx = d2(L(0, 0, -2), L(0, 0, -1), cc, L(0, 0, 1), L(0, 0, 2), k2)
    dyy = d2(L(0, -2, 0), L(0, -1, 0), cc, L(0, 1, 0), L(0, 2, 0), k2)
    dzz = d2(L(-2, 0, 0), L(-1, 0, 0), cc, L(1, 0, 0), L(2, 0, 0), k2)
    return add(add(dxx, dyy), dzz)


def lap4_grid(u, g, k2):
    G = LaneGrid(u)

    def run(execute):
        out = blank(u.shape)

        def kern(piece):
            for z, y, i, m in rows_of(piece):
                vl.vstore_partial(out.rows[(z, y)], i, lap4_lanes(G, z, y, i, k2), m)
        execute(kern)
        return [strip(out.to_numpy(), g)]
    return sweep(run, u.shape, g, n_settings=2)[0]


def level_boxes(n):
    outer = BBox(Point((0, 0, 0)), Point((n - 1,) * 3), Stride.ones(3))
    hole = BBox(Point((n // 2,) * 3), Point((n - 1,) * 3), Stride.ones(3))
    boxes = BBoxSet.from_bboxes([outer]).difference(BBoxSet.from_bboxes([hole])).to_bboxes()
    return [[list(b.lower.coords), list(b.upper.coords)] for b in boxes]


def ghost_regions(n, g):
    """Per box of the level, the reference bboxset algebra's ghost-sync
    region: (expand(box, g) ∩ level) \\ box, as its canonical box list."""
    outer = BBox(Point((0, 0, 0)), Point((n - 1,) * 3), Stride.ones(3))
    hole = BBox(Point((n // 2,) * 3), Point((n - 1,) * 3), Stride.ones(3))
    lvl = BBoxSet.from_bboxes([outer]).difference(BBoxSet.from_bboxes([hole]))
    out = []
    for b in lvl.to_bboxes():
        grown = BBoxSet.from_bboxes([b.expand(Point((g,) * 3), Point((g,) * 3))])
        ghost = grown.intersection(lvl).difference(BBoxSet.from_bboxes([b]))
        out.append([[list(r.lower.coords), list(r.upper.coords)] for r in ghost.to_bboxes()])
    return out


def golden_c4(n=16, g=2):
    from paper_1308_1343_b200.level import Box
    boxes = [Box(tuple(lo), tuple(hi)) for lo, hi in level_boxes(n)]
    fields = inputs.c4_fields(boxes, g, seed=inputs.seed_for(4) + 1000)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    outs = [lap4_grid(u, g, k.k2) for u in fields]
    return boxes, fields, outs


# -- config 3 ---------------------------------------------------------------------------

def fill(a, g):
    """Periodic ghost copy (exact), axis by axis."""
    for ax in (2, 1, 0):
        n = a.shape[ax] - 2 * g
        sl = lambda s: tuple(s if d == ax else slice(None) for d in range(3))
        a[sl(slice(0, g))] = a[sl(slice(n, n + g))]
        a[sl(slice(n + g, n + 2 * g))] = a[sl(slice(g, 2 * g))]


def golden_c3(n=8, g=2):
    phi0, pi0 = inputs.c3_fields(n, g, seed=inputs.seed_for(3) + 1000)
    cst = inputs.WaveConstants.for_grid(n)
    I = (slice(g, g + n),) * 3

    def combine(fn, *arrays):
        """Apply a lane-wise function to interior rows of interior arrays."""
        out = np.zeros((n, n, n))
        for z in range(n):
            for y in range(n):
                rows = [vl.AlignedArray.from_values(list(a[z, y, :]), W, PAD) for a in arrays]
                dst = vl.AlignedArray(n, W, PAD)
                for i, m in vl.iterate_masked(0, n, W):
                    vs = [vl.vload_aligned(r, i) for r in rows]
                    vl.vstore_partial(dst, i, fn(*vs), m)
                out[z, y, :] = dst.to_list()
        return out

    def lap(phi_int):
        a = np.zeros((n + 2 * g,) * 3)
        a[I] = phi_int
        fill(a, g)
        return lap4_grid(a, g, cst.lap.k2)

    p0, q0 = phi0[I].copy(), pi0[I].copy()
    hdt, dt, dt6 = c(cst.half_dt), c(cst.dt), c(cst.dt6)
    L = lap(p0)
    acc_f, acc_p = q0.copy(), L
    phi_s = combine(lambda a, b: add(a, mul(hdt, b)), p0, q0)
    pi_s = combine(lambda a, b: add(a, mul(hdt, b)), q0, L)
    for coef in (hdt, dt):
        L = lap(phi_s)
        acc_f = combine(lambda a, b: add(a, mul(c(2.0), b)), acc_f, pi_s)
        acc_p = combine(lambda a, b: add(a, mul(c(2.0), b)), acc_p, L)
        phi_s, pi_s = (combine(lambda a, b: add(a, mul(coef, b)), p0, pi_s),
                       combine(lambda a, b: add(a, mul(coef, b)), q0, L))
    L = lap(phi_s)
    phi_new = combine(lambda a, af, ps: add(a, mul(dt6, add(af, ps))), p0, acc_f, pi_s)
    pi_new = combine(lambda a, ap, l: add(a, mul(dt6, add(ap, l))), q0, acc_p, L)
    return phi0, pi0, phi_new, pi_new


# -- config 5 ---------------------------------------------------------------------------

def golden_c5(n=4, g=2):
    fields = inputs.c5_fields(n, g, seed=inputs.seed_for(5) + 1000)
    poly = inputs.c5_poly(seed=inputs.seed_for(5) + 1000)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    Gs = [LaneGrid(u) for u in fields]
    shape = fields[0].shape

    def run(execute):
        outs = [blank(shape) for _ in range(inputs.N_VARS)]

        def kern(piece):
            for z, y, i, m in rows_of(piece):
                vals = []
                for G in Gs:
                    vals.extend(slots(G, z, y, i, k))
                for o in range(inputs.N_VARS):
                    term = lambda t: mul(mul(c(float(poly.coef[o, t])), vals[poly.p[o, t]]), vals[poly.q[o, t]])
                    acc = term(0)
                    for t in range(1, inputs.N_TERMS):
                        acc = add(acc, term(t))
                    vl.vstore_partial(outs[o].rows[(z, y)], i, acc, m)
        execute(kern)
        return [strip(o.to_numpy(), g) for o in outs]
    return fields, poly, sweep(run, shape, g, n_settings=2)


# -- main ------------------------------------------------------------------------------------

def main():
    assert vl.FUSED_FMA is False
    meta: dict = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src (stencilrt)",
                  "numpy": np.__version__}
    arrays: dict = {}

    # 1. config 1 through the reference's own _update_rows
    n = 64
    u = inputs.c1_field(n)
    c0, c1 = inputs.c1_constants(n)
    st.C0, st.C1 = c0, c1
    dst = u.copy()
    st._update_rows(dst, u, 1, n + 1, 1, n + 1, 1, n + 1)
    meta["c1"] = {"n": n, "c0": c0, "c1": c1, "seed": inputs.seed_for(1),
                  "input_sha256": inputs.sha256(u), "output_sha256": inputs.sha256(dst[1:-1, 1:-1, 1:-1])}
    small = inputs.c1_field(10, seed=7)
    cs0, cs1 = inputs.c1_constants(10)
    st.C0, st.C1 = cs0, cs1
    d = small.copy()
    st._update_rows(d, small, 1, 11, 1, 11, 1, 11)
    arrays["c1_small_in"], arrays["c1_small_out"] = small, d[1:-1, 1:-1, 1:-1].copy()
    meta["c1_small"] = {"n": 10, "seed": 7, "c0": cs0, "c1": cs1}

    # 2. the reference demo (C0 = -6/8, C1 = 1/8)
    st.C0, st.C1 = -6.0 / 8.0, 1.0 / 8.0
    demo = st.run_serial(16, 8, 20130715)
    arrays["demo16_final"] = demo.final
    topo = TopologyConfig(n_coarse_threads=2, n_fine_threads=1, lane_width=4, rng_seed=20130715)
    s64 = st.run_serial(64, 100, 20130715)
    nv = st.run_naive(64, 100, 20130715, 2)
    tu, _ = st.run_tuned(64, 100, 20130715, topo)
    assert st.bit_identical(s64.final, nv.final) and st.bit_identical(s64.final, tu.final)
    meta["demo"] = {"n16_iters": 8, "n64_iters": 100, "seed": 20130715,
                    "n64_final_sha256": inputs.sha256(s64.final), "c0": st.C0, "c1": st.C1}

    # 3. vlanes criterion-6 vectors
    rng = random.Random(960_000)
    ins, fwd, ctr, lens = [], [], [], []
    for m in range(1, 130):
        vals = [rng.uniform(-1e6, 1e6) for _ in range(m)]
        src = vl.AlignedArray.from_values(vals, W)
        a = vl.AlignedArray(m, W)
        vl.forward_difference(a, src, m)
        b = vl.AlignedArray(m, W)
        vl.centered_difference(b, src, m)
        ins += vals
        fwd += a.to_list()
        ctr += b.to_list()
        lens.append(m)
    arrays["diff_in"], arrays["diff_fwd"], arrays["diff_ctr"] = map(np.array, (ins, fwd, ctr))
    arrays["diff_len"] = np.array(lens, dtype=np.int64)

    # 4. configs 2-5 through vlanes + traverse
    u2, outs2 = golden_c2()
    arrays["c2_in"] = u2
    arrays["c2_out"] = np.stack(outs2)
    meta["c2"] = {"n": 8, "g": 2, "seed": inputs.seed_for(2) + 1000}

    u2b, outs2b = golden_c2_order2()
    arrays["c2o2_in"] = u2b
    arrays["c2o2_out"] = np.stack(outs2b)
    meta["c2_order2"] = {"n": 8, "g": 2, "seed": inputs.seed_for(2) + 2000}

    phi0, pi0, phin, pin = golden_c3()
    arrays["c3_phi0"], arrays["c3_pi0"], arrays["c3_phi1"], arrays["c3_pi1"] = phi0, pi0, phin, pin
    meta["c3"] = {"n": 8, "g": 2, "seed": inputs.seed_for(3) + 1000}

    boxes, f4, o4 = golden_c4()
    for j, (f, o) in enumerate(zip(f4, o4)):
        arrays[f"c4_in{j}"], arrays[f"c4_out{j}"] = f, o
    meta["c4"] = {"n": 16, "g": 2, "seed": inputs.seed_for(4) + 1000,
                  "boxes": [[list(b.lo), list(b.hi)] for b in boxes]}
    meta["c4_level512_boxes"] = level_boxes(512)
    meta["c4_ghost_regions_n12_g2"] = ghost_regions(12, 2)

    f5, poly5, o5 = golden_c5()
    arrays["c5_in"] = np.stack(f5)
    arrays["c5_out"] = np.stack(o5)
    arrays["c5_coef"], arrays["c5_p"], arrays["c5_q"] = poly5.coef, poly5.p, poly5.q
    meta["c5"] = {"n": 4, "g": 2, "seed": inputs.seed_for(5) + 1000}
    meta["c5_full_poly_sha256"] = inputs.c5_poly().digest()

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("wrote", HERE / "golden.npz", HERE / "golden.json")


if __name__ == "__main__":
    main()
