"""Cost of the z-slab decomposition with fused halo stores (F4, halo.py) on
one GPU: config 3 (384^3 periodic RK4, Laplacian pairs) as R = 1, 2, 4, 8
slabs in one process.  Every slab's pair launches write their two boundary
planes straight into the neighbours' ghost planes (sb_rk4_pair_zslab).

Reported per R (CUDA events around CUDA-graph replays, median over reps,
inputs resident):
  * step_ms      — all R slabs' launches back to back (the whole box's work
                   on this one GPU: the decomposition's total overhead);
  * slab0_ms     — the launches of one slab alone (the per-GPU work of an
                   R-GPU run, without the inter-GPU barrier and NVLink
                   latency, which one GPU cannot measure);
  * bits_equal   — the result equals the single-box schedule's bit for bit;
  * launch       — the z chunk (64 / 32 / 16) with the fastest slab0_ms
                   (thin slabs need shorter chunks to fill the GPU).
This is a one-GPU measurement of the decomposition, not a multi-GPU run.

    python tools/zslab_probe.py > gpurun_out/zslab_probe.json
"""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    from paper_1308_1343_b200 import _build, inputs
    from paper_1308_1343_b200.graphs import SweepGraph
    from paper_1308_1343_b200.halo import WaveRK4Slabs, launch_pair
    from paper_1308_1343_b200.kernels import WaveRK4
    from paper_1308_1343_b200.tuner import LaunchParams

    _build.build()
    n, g, reps = 384, 2, 30
    c = inputs.WaveConstants.for_grid(n)
    phi, pi = inputs.c3_fields(n, g)

    def timed(fn) -> float:
        """Device time of fn's launches: captured 10x into a CUDA graph (no
        host launch overhead in the number), median of reps replays / 10."""
        g = SweepGraph(fn, repeat=10)
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b) / 10)
        return statistics.median(ms)

    box = WaveRK4(n, g, c, schedule="lap_pairs")
    box.phi0.upload(phi, with_ghosts=True)
    box.pi0.upload(pi, with_ghosts=True)
    box.step()
    torch.cuda.synchronize()
    ref = box.phi_b.download(), box.pi_b.download()
    out = {"config": "c3 384^3 periodic RK4, Laplacian pairs, 32x4/z64/p1", "single_box_ms": timed(box.step),
           "rows": []}
    del box
    torch.cuda.empty_cache()

    for R in (1, 2, 4, 8):
        sl = WaveRK4Slabs(n, R, g, c, schedule="lap_pairs")
        sl.upload(phi, pi)
        sl.step()
        torch.cuda.synchronize()
        same = all(__import__("numpy").array_equal(a, b) for a, b in
                   zip(ref, (sl.result("phi_b"), sl.result("pi_b"))))
        s0 = sl.slabs[0]
        lo, hi = sl.slabs[-1], sl.slabs[1 % R]

        def slab0():
            for pair in sl.launches:
                out_, out2 = pair[3], pair[4]
                launch_pair(s0, pair, c, sl.params, (getattr(lo, out_).origin_ptr, getattr(lo, out2).origin_ptr),
                            lo.nz, (getattr(hi, out_).origin_ptr, getattr(hi, out2).origin_ptr), -s0.nz)

        best = None
        for zc in (64, 32, 16):
            sl.params = LaunchParams(32, 4, zc, 1)
            cand = {"z_chunk": zc, "step_ms": timed(sl.step), "slab0_ms": timed(slab0)}
            if best is None or cand["slab0_ms"] < best["slab0_ms"]:
                best = cand
        row = {"slabs": R, "slab_planes": s0.nz, "launch": f"32x4/z{best['z_chunk']}/p1", "step_ms": best["step_ms"],
               "slab0_ms": best["slab0_ms"], "bits_equal": bool(same)}
        row["step_overhead_vs_box"] = row["step_ms"] / out["single_box_ms"] - 1.0
        row["projected_speedup_R_gpus"] = out["single_box_ms"] / row["slab0_ms"]
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
        del sl
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
