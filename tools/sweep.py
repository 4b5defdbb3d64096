"""Time one configuration's kernel over a list of launch shapes (CUDA events,
median of reps), checking that every shape produces the same bits.

    python tools/sweep.py --config 2 [--shapes all|default] [--reps 20]

Prints one JSON line per shape and a summary with the best shape.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shapes", default="all")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--graph", action="store_true", help="time reps launches captured in one CUDA graph")
    ap.add_argument("--flags", type=int, default=0, help="extra SB_LAUNCH_* flags for the kernel")
    ap.add_argument("--schedule", default=None, help="config 3: RK4 schedule (kernels.WaveRK4.SCHEDULES)")
    args = ap.parse_args()

    import torch

    from paper_1308_1343_b200 import _build
    from paper_1308_1343_b200.configs import CONFIGS
    from paper_1308_1343_b200.tuner import LaunchParams, LoopSetup, TopologyConfig

    _build.build()
    kw = {"n": args.n} if args.n else {}
    if args.schedule:
        kw["schedule"] = args.schedule
    prob = CONFIGS[args.config](**kw).setup()
    kern = getattr(prob, "kernel", None)
    if kern is not None and args.flags:
        kern.extra_flags = args.flags
    if kern is not None:
        space = kern.launch_space()
        ext = kern.full_space().extents
    else:
        from paper_1308_1343_b200.kernels import RK4_SPACE
        space = RK4_SPACE
        ext = (prob.n,) * 3
    setup = LoopSetup(f"c{args.config}", ext)
    topo = TopologyConfig()
    shapes = space.enumerate(setup, topo) if args.shapes == "all" else [space.initial(setup, topo)]
    if args.shapes not in ("all", "default"):
        shapes = [LaunchParams(*map(int, s.split(","))) for s in args.shapes.split(";")]

    def outs():
        return [t.clone() for t in _device_outputs(prob)]

    prob.run(shapes[0])
    ref = outs()
    results = []
    for p in shapes:
        prob.run(p)
        got = outs()
        same = all(torch.equal(a, b) for a, b in zip(ref, got))
        for _ in range(3):
            prob.run(p)
        if args.graph:
            from paper_1308_1343_b200.graphs import SweepGraph
            g = SweepGraph(lambda: prob.run(p), repeat=args.reps)
            ms = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b) / args.reps)
            med = statistics.median(ms)
        else:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.reps + 1)]
            ev[0].record()
            for i in range(args.reps):
                prob.run(p)
                ev[i + 1].record()
            torch.cuda.synchronize()
            ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.reps)]
            med = statistics.median(ms)
        r = {"shape": p.flat(), "ms": med, "gpts": prob.updates / med / 1e6,
             "gbs": prob.canonical_bytes / med / 1e6, "bits_equal": same}
        results.append(r)
        print(json.dumps(r), flush=True)
    best = min(results, key=lambda r: r["ms"])
    print(json.dumps({"config": args.config, "best": best, "n_shapes": len(results),
                      "all_bits_equal": all(r["bits_equal"] for r in results)}))


def _device_outputs(prob):
    if hasattr(prob, "outs"):
        return [o.interior() for o in prob.outs]
    if hasattr(prob, "dsts"):
        return [d.interior() for d in prob.dsts]
    if hasattr(prob, "dst"):
        return [prob.dst.interior()]
    if hasattr(prob, "rk"):
        return [prob.rk.phi_b.interior(), prob.rk.pi_b.interior()]
    raise ValueError("unknown problem")


if __name__ == "__main__":
    main()
