"""Time the two Laplacian-pair launches of config 3 (pair LA = stages 1+2,
pair LB = stages 3+4) separately over launch shapes: can the two launches
of a step prefer different shapes?  CUDA events, median of reps; every shape
is checked bit-identical to the default step.

    python tools/c3_pair_shapes.py > profiles/r02/c3_pair_shapes.json
"""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_1308_1343_b200 import _build
    from paper_1308_1343_b200.configs import C3WaveRK4
    from paper_1308_1343_b200.tuner import LaunchParams
    _build.build()
    p = C3WaveRK4().setup()
    rk = p.rk
    rk.step()
    ref = [t.full().clone() for t in (rk.phi_b, rk.pi_b)]
    shapes = [(32, 4, 64, 1), (32, 8, 64, 1), (32, 2, 64, 1), (64, 2, 64, 1), (64, 4, 64, 1), (32, 4, 32, 1),
              (32, 4, 96, 1), (32, 8, 64, 2), (64, 4, 64, 2), (32, 4, 64, 2), (64, 8, 64, 2), (128, 2, 64, 2),
              (64, 4, 32, 2), (32, 16, 64, 2)]
    reps = 60
    out = {}
    for s in shapes:
        lp = LaunchParams(*s)
        res = {}
        try:
            for k, args in ((3, (rk.phi0, rk.pi0, rk.phi_a, rk.pi_a)), (4, (rk.phi_a, rk.pi_a, rk.phi_b, rk.pi_b))):
                for _ in range(3):
                    rk.pair(3, rk.phi0, rk.pi0, rk.phi_a, rk.pi_a, lp)
                    rk.pair(4, rk.phi_a, rk.pi_a, rk.phi_b, rk.pi_b, lp)
                ms = []
                for _ in range(reps):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    rk.pair(k, *args, lp)
                    b.record()
                    b.synchronize()
                    ms.append(a.elapsed_time(b))
                res["LA" if k == 3 else "LB"] = statistics.median(ms)
            torch.cuda.synchronize()
            res["bits_equal"] = all(torch.equal(x.full(), y) for x, y in zip((rk.phi_b, rk.pi_b), ref))
        except Exception as e:  # noqa: BLE001
            res["error"] = str(e)[:200]
        out["x".join(map(str, s))] = res
        print(json.dumps({"shape": s, **res}), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
