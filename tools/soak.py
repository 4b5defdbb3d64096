"""Randomised soak of the multi-box kernels against the oracle: random
levels (1-60 boxes, arbitrary origins and ragged extents), random clipping
spaces, random launch shapes (tile 32/64/128, rows, z chunk, scalar/paired)
for the ten-output set (4th and 2nd order), the Laplacian and RK4 stage 2 —
every box bit-exact.  python tools/soak.py [iterations] > profiles/r02/soak.json"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import oracle
    from paper_1308_1343_b200 import _build, inputs
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import LevelFourthOrderAll, LevelLaplacian4
    from paper_1308_1343_b200.traverse import IndexSpace
    from paper_1308_1343_b200.tuner import LaunchParams
    from test_gpu_level_table import random_level
    _build.build()
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    G = 2
    fails, done = [], 0
    for it in range(iters):
        rng = np.random.default_rng(10_000 + it)
        nbox = int(rng.integers(1, 61))
        region = tuple(int(v) for v in rng.integers(12, 70, 3))
        origin = tuple(int(v) for v in rng.integers(-40, 40, 3))
        try:
            boxes = random_level(nbox, 20_000 + it, region=region, origin=origin)
        except ValueError:
            continue
        srcs, host = [], []
        for b in boxes:
            nx, ny, nz = b.extents
            u = rng.uniform(-1, 1, (nz + 2 * G, ny + 2 * G, nx + 2 * G))
            d = DeviceGrid(b.extents, G, lower=b.lo)
            d.upload(u, with_ghosts=True)
            srcs.append(d)
            host.append(u)
        order = int(rng.choice([2, 4]))
        h = float(rng.uniform(0.01, 0.2))
        k = inputs.D4Constants.for_spacing(h) if order == 4 else inputs.D2Constants.for_spacing(h)
        tx = int(rng.choice([32, 64, 128]))
        npp = int(rng.choice([1, 2]))
        ty = int(rng.choice([1, 2, 4, 8]))
        while (tx // npp) * ty > 256:
            ty //= 2
        while (tx // npp) * ty % 32:
            ty *= 2
        p = LaunchParams(tx, ty, int(rng.integers(1, 70)), npp)
        lo = [min(b.lo[d] for b in boxes) for d in range(3)]
        hi = [max(b.hi[d] + 1 for b in boxes) for d in range(3)]
        clip = None
        if rng.random() < 0.5:
            a = [int(rng.integers(lo[d], hi[d])) for d in range(3)]
            c = [int(rng.integers(a[d] + 1, hi[d] + 1)) for d in range(3)]
            clip = IndexSpace(tuple(a), tuple(c))
        outs = [[DeviceGrid(b.extents, 0, lower=b.lo).fill_(3.5) for _ in range(10)] for b in boxes]
        dsts = [DeviceGrid(b.extents, 0, lower=b.lo).fill_(3.5) for b in boxes]
        LevelFourthOrderAll(outs, srcs, k, order=order).launch(clip, p)
        if order == 4:
            LevelLaplacian4(dsts, srcs, k).launch(clip, p)
        ok = True
        for b, u, os_, d in zip(boxes, host, outs, dsts):
            nx, ny, nz = b.extents
            want = [np.full((nz, ny, nx), 3.5) for _ in range(10)]
            r = [0, nx, 0, ny, 0, nz]
            if clip is not None:
                r = []
                for dd in range(3):
                    r += [max(b.lo[dd], clip.lo[dd]) - b.lo[dd], min(b.hi[dd] + 1, clip.hi[dd]) - b.lo[dd]]
            if r[1] > r[0] and r[3] > r[2] and r[5] > r[4]:
                (oracle.d4_all if order == 4 else oracle.d2_all)(want, u, G, tuple(r), k)
            for i in range(10):
                ok &= os_[i].download().tobytes() == want[i].tobytes()
            if order == 4:
                ok &= d.download().tobytes() == want[9].tobytes()
        done += 1
        if not ok:
            fails.append({"iter": it, "boxes": nbox, "params": p.flat(), "order": order, "clip": clip is not None})
        print(json.dumps({"iter": it, "boxes": nbox, "params": p.flat(), "order": order, "clip": clip is not None,
                          "ok": ok}), file=sys.stderr)
    print(json.dumps({"iterations": done, "failures": fails}, indent=1))


if __name__ == "__main__":
    main()
