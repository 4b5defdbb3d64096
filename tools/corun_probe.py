"""Do config 3's two Laplacian-pair kernels overlap when co-resident?

Two independent 384^3 problems X and Y.  Times (CUDA events, median of 20):
  serial   : LA(X); LB(X)                       on one stream
  corun    : LA(X) on stream 1  ||  LB(Y) on stream 2   (independent data)
  LA alone, LB alone
If corun < LA + LB, a z-chunked pipeline (LA of chunk k+1 beside LB of
chunk k) could hide part of one kernel behind the other.

    python tools/corun_probe.py > profiles/r02/c3_corun_probe.json
"""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_1308_1343_b200.configs import C3WaveRK4
    X = C3WaveRK4().setup()
    Y = C3WaveRK4(seed=11).setup()
    rx, ry = X.rk, Y.rk
    p = rx.params
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def LA(r, st):
        r.pair(3, r.phi0, r.pi0, r.phi_a, r.pi_a, p, st)

    def LB(r, st):
        r.pair(4, r.phi_a, r.pi_a, r.phi_b, r.pi_b, p, st)

    def timed(fn, reps=20):
        cur = torch.cuda.current_stream()
        ts = []
        for k in range(reps + 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            fn()
            cur.wait_stream(s1)
            cur.wait_stream(s2)
            b.record(cur)
            b.synchronize()
            if k >= 3:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    LA(rx, s1)
    LA(ry, s1)
    torch.cuda.synchronize()
    res = {
        "LA_alone_ms": timed(lambda: LA(rx, s1)),
        "LB_alone_ms": timed(lambda: LB(rx, s1)),
        "serial_LA_LB_ms": timed(lambda: (LA(rx, s1), LB(rx, s1))),
        "corun_LAx_LBy_ms": timed(lambda: (LA(rx, s1), LB(ry, s2))),
        "serial_LAx_LBy_ms": timed(lambda: (LA(rx, s1), LB(ry, s1))),
    }
    res["corun_gain"] = 1 - res["corun_LAx_LBy_ms"] / res["serial_LAx_LBy_ms"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
