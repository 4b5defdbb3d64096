"""Tolerance mode check: run configs 2-5 on small boxes with the library in
the current mode (STENCIL_B200_MODE=fma for the FMA-contracted build) and
print, per output, the normwise relative error against the bit-exact CPU
oracle, max|got - want| / max|want|, as one JSON object (north_star: "max
relative error <= 1e-13 in fp64" when FMA contraction is on).

    STENCIL_B200_MODE=fma python tools/fma_check.py [--full]

``--full`` uses the BASELINE.json shapes (256^3, 384^3, the 512^3 level,
192^3) with the oracle on all host threads.
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402  (checker)
from oracle.stencils import host_threads  # noqa: E402
from paper_1308_1343_b200 import _build, _lib  # noqa: E402
from paper_1308_1343_b200.configs import C2FourthOrder, C3WaveRK4, C4Level, C5Rhs24  # noqa: E402


def rel(got, want) -> float:
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def main(full: bool = False) -> dict:
    _build.build()
    out = {"library": _lib.library_path().name, "errors": {}, "bit_identical": {}, "full_size": full}
    err, same = out["errors"], out["bit_identical"]
    thr = host_threads()

    n = 256 if full else 48
    p = C2FourthOrder(n=n, seed=None if full else 1).setup()
    p.run()
    want = [np.empty((n,) * 3) for _ in range(10)]
    oracle.run_static(lambda a, b: oracle.d4_all(want, p.host_u, 2, (0, n, 0, n, a, b), p.k), 0, n, thr)
    for i, (g, w) in enumerate(zip(p.outputs(), want)):
        err[f"c2_out{i}"], same[f"c2_out{i}"] = rel(g, w), g.tobytes() == w.tobytes()

    n = 384 if full else 40
    r = C3WaveRK4(n=n, seed=None if full else 3).setup()
    r.run()
    wphi, wpi = oracle.rk4_step(r.host_phi, r.host_pi, 2, r.c, threads=thr)
    I = (slice(2, 2 + n),) * 3
    for nm, g, w in (("c3_phi", r.outputs()[0], wphi[I]), ("c3_pi", r.outputs()[1], wpi[I])):
        err[nm], same[nm] = rel(g, w), g.tobytes() == w.tobytes()

    lv = C4Level(n=512 if full else 24, seed=None if full else 4).setup()
    lv.run()
    for b, (u, g) in enumerate(zip(lv.host_u, lv.outputs())):
        nz, ny, nx = g.shape
        w = np.empty_like(g)
        oracle.run_static(lambda a, bb: oracle.lap4(w, u, 2, (0, nx, 0, ny, a, bb), lv.k.k2), 0, nz, thr)
        err[f"c4_box{b}"], same[f"c4_box{b}"] = rel(g, w), g.tobytes() == w.tobytes()

    n = 192 if full else 8
    f = C5Rhs24(n=n, seed=None if full else 5).setup()
    f.run()
    want = [np.empty((n,) * 3) for _ in range(24)]

    def planes(a, b):
        for z in range(a, b, 2):
            oracle.rhs24(want, f.host_u, 2, (0, n, 0, n, z, min(b, z + 2)), f.k, f.poly)
    oracle.run_static(planes, 0, n, thr)
    for o, (g, w) in enumerate(zip(f.outputs(), want)):
        err[f"c5_out{o}"], same[f"c5_out{o}"] = rel(g, w), g.tobytes() == w.tobytes()
    out["max_error"] = max(err.values())
    out["all_bit_identical"] = all(same.values())
    return out


if __name__ == "__main__":
    print(json.dumps(main(full="--full" in sys.argv)))
