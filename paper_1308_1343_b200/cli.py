"""Command line: the reference's ``stencil-bench`` harness on the B200.

Mirrors ``stencilrt stencil-bench`` (cli.py:185-209, flags cli.py:246-285):
run the 7-point Jacobi demo serially, with the naive static split and
tuned, check the outputs are bit-identical, write the per-iteration CSV
``impl,iter,elapsed_ns,phase,is_best`` and print the summary; exit 0 when
bit-identical, 1 otherwise, 2 on usage/resource errors (cli.py:288-295).
The device adds two implementations: ``graphed`` (the same sweeps captured
in a CUDA graph) and ``persistent`` (all sweeps in one cooperative launch
with a grid barrier between them).  ``config-bench`` times one BASELINE.json
configuration (1..5) with the run-time tuner.  ``tune-sim`` runs the
tuner against a synthetic cost surface (reference cli.py:212-226; no GPU).

    python -m paper_1308_1343_b200 stencil-bench --extent 64 --iters 100 --threads 2
    python -m paper_1308_1343_b200 config-bench --config 2 --iters 50
    python -m paper_1308_1343_b200 tune-sim --seeds 100 --iters 50 --space launch
"""
from __future__ import annotations

import argparse
import json
import sys
from dataclasses import replace
from pathlib import Path

from .errors import ResourceError, UsageError
from .tuner import TopologyConfig


def _topology(args) -> TopologyConfig:
    topo = TopologyConfig.from_file(args.topology) if args.topology else TopologyConfig()
    over = {}
    if args.threads is not None:
        over["n_coarse_threads"] = args.threads
    if args.fine_threads is not None:
        over["n_fine_threads"] = args.fine_threads
    if args.lane_width is not None:
        over["lane_width"] = args.lane_width
    if args.seed is not None:
        over["rng_seed"] = args.seed
    return replace(topo, **over) if over else topo


def _med(xs):
    return sorted(xs)[len(xs) // 2]


def cmd_stencil_bench(args) -> int:
    from . import stencil
    topo = _topology(args)
    n, iters = args.extent, args.iters
    serial = stencil.run_serial(n, iters, args.seed)
    naive = stencil.run_naive(n, iters, args.seed, topo.n_coarse_threads)
    tuned, tuner = stencil.run_tuned(n, iters, args.seed, topo)
    graphed = stencil.run_graphed(n, iters - iters % 2, args.seed) if iters >= 2 else None
    persistent = stencil.run_persistent(n, iters, args.seed)
    ok = stencil.bit_identical(serial.final, naive.final) and stencil.bit_identical(serial.final, tuned.final)
    ok = ok and stencil.bit_identical(serial.final, persistent.final)
    if graphed is not None and iters % 2 == 0:
        ok = ok and stencil.bit_identical(serial.final, graphed.final)
    rows = ["impl,iter,elapsed_ns,phase,is_best"]
    rows += [f"serial,{i},{int(t * 1e9)},," for i, t in enumerate(serial.iter_seconds)]
    rows += [f"naive,{i},{int(t * 1e9)},," for i, t in enumerate(naive.iter_seconds)]
    rows += [f"tuned,{i},{int(t * 1e9)},{r['phase']},{r['is_best']}"
             for i, (t, r) in enumerate(zip(tuned.iter_seconds, tuner.log))]
    if graphed is not None:
        rows += [f"graphed,{i},{int(t * 1e9)},," for i, t in enumerate(graphed.iter_seconds)]
    rows += [f"persistent,{i},{int(t * 1e9)},," for i, t in enumerate(persistent.iter_seconds)]
    if args.out:
        Path(args.out).write_text("\n".join(rows) + "\n")
    tail = max(1, min(20, iters // 2))
    print(f"stencil-bench {n}^3 x{iters}: outputs bit-identical: {ok}")
    line = (f"median seconds/iter: serial {_med(serial.iter_seconds):.6f}  naive {_med(naive.iter_seconds):.6f}  "
            f"tuned(last {tail}) {_med(tuned.iter_seconds[-tail:]):.6f}")
    if graphed is not None:
        line += f"  graphed {_med(graphed.iter_seconds):.6f}"
    if persistent.iter_seconds:
        line += f"  persistent {_med(persistent.iter_seconds):.6f}"
    print(line)
    return 0 if ok else 1


def cmd_config_bench(args) -> int:
    import torch

    from .configs import CONFIGS
    from .traverse import _Timer, run_loop
    from .tuner import LoopSetup, Tuner
    if args.config not in CONFIGS:
        raise UsageError(f"unknown config {args.config} (1..5)")
    prob = CONFIGS[args.config](seed=args.seed_config).setup()
    kern = getattr(prob, "kernel", None) or prob.rk
    space = kern.launch_space()
    ext = kern.full_space().extents if hasattr(kern, "full_space") else (prob.n,) * 3
    # device tuning key (tuner.device_setup): site, extents, grid pitch, SM count
    pitch = kern.pitch_class() if hasattr(kern, "pitch_class") else prob.rk.phi0.sy
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    setup = LoopSetup(f"config{args.config}", ext, pitch=pitch, sm_count=sms)
    tuner = Tuner(_topology(args))
    default = getattr(kern, "default_params", None) or getattr(kern, "params")
    tuner.prime(setup, space, default)

    class _Step:
        def launch_space(self):
            return space

        def launch(self, _space, params, stream=None):
            prob.run(params, stream)

    step = _Step()
    for _ in range(args.tune):
        run_loop(setup, None, step, tuner)
    best, _ = tuner.best(setup) if args.tune > 1 else (default, None)
    best = best or default
    times = []
    for _ in range(args.iters):
        with _Timer(True) as tm:
            prob.run(best)
        times.append(tm.elapsed())
    torch.cuda.synchronize()
    med = _med(times)
    print(json.dumps({"config": args.config, "params": best.flat(), "ms": med * 1e3,
                      "gpts": prob.updates / med / 1e9, "algorithmic_gbs": prob.canonical_bytes / med / 1e9}))
    return 0


def cmd_tune_sim(args) -> int:
    from . import tunesim
    case = tunesim.launch_case if args.space == "launch" else tunesim.plan_case
    topo, setup, surf, space = case()
    if args.topology:
        topo = TopologyConfig.from_file(args.topology)
    r = tunesim.simulate(args.seeds, args.iters, topo, setup, surf, space)
    print(f"tune-sim ({args.space} space): optimum {r.optimum:.4f}, {r.converged}/{args.seeds} seeds within 10% "
          f"in <= {args.iters} evals (median {r.median_evals_to_target})")
    if args.out:
        Path(args.out).write_text(r.csv())
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1308_1343_b200")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p, extent, iters):
        p.add_argument("--seed", type=int, default=20130715)
        p.add_argument("--extent", type=int, default=extent)
        p.add_argument("--iters", type=int, default=iters)
        p.add_argument("--threads", type=int, default=None)
        p.add_argument("--fine-threads", dest="fine_threads", type=int, default=None)
        p.add_argument("--lane-width", dest="lane_width", type=int, default=None)
        p.add_argument("--topology", type=str, default=None)
        p.add_argument("--out", type=str, default=None)

    p = sub.add_parser("stencil-bench", help="7-point Jacobi demo: serial, static split, tuned, graphed")
    common(p, 64, 100)
    p.set_defaults(fn=cmd_stencil_bench)
    p = sub.add_parser("config-bench", help="time one BASELINE.json configuration with the run-time tuner")
    common(p, 0, 20)
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--tune", type=int, default=30)
    p.add_argument("--seed-config", dest="seed_config", type=int, default=None)
    p.set_defaults(fn=cmd_config_bench)
    p = sub.add_parser("tune-sim", help="tuner simulation on a synthetic cost surface")
    p.add_argument("--seeds", type=int, default=100)
    p.add_argument("--iters", type=int, default=50)
    p.add_argument("--space", choices=("plan", "launch"), default="plan")
    p.add_argument("--topology", type=str, default=None)
    p.add_argument("--out", type=str, default=None)
    p.set_defaults(fn=cmd_tune_sim)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (UsageError, ResourceError) as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
