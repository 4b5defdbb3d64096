"""Every BASELINE.json configuration on the B200 next to the reference's CPU
path (the oracle port: numpy expression trees in the reference's
_update_rows style, static thread split over all host cores).

    python tools/config_table.py [--cpu-seconds 8] > profiles/r01/config_table.json

GPU: median of CUDA-event timings of back-to-back launches at the kernels'
default (swept) launch shapes, inputs resident in HBM (config 1: launches
replayed from a CUDA graph — it is launch-bound), with the SM clock and
clock-event reasons sampled through NVML while timing.  CPU: a bounded sample of each workload
(stated per row), timed with perf_counter, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402  (checker / CPU baseline only)
from oracle.stencils import host_threads  # noqa: E402
from paper_1308_1343_b200 import inputs  # noqa: E402


def gpu_time(prob, reps=20, graph=False):
    """Median per-launch time of back-to-back launches (events between them);
    with graph=True the launches are replayed from one CUDA graph (for the
    launch-bound config 1)."""
    import torch
    for _ in range(3):
        prob.run()
    if graph:
        from paper_1308_1343_b200.graphs import SweepGraph
        g = SweepGraph(prob.run, repeat=reps)
        ms = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b) / reps)
        return statistics.median(ms) / 1e3
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        prob.run()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps)) / 1e3


def timed(fn, seconds):
    n, el = 0, 0.0
    while el < seconds or n == 0:
        t0 = time.perf_counter()
        fn()
        el += time.perf_counter() - t0
        n += 1
    return el / n


def cpu_c1(threads, seconds):
    n = 64
    u = inputs.c1_field(n)
    c0, c1 = inputs.c1_constants(n)
    dst = u.copy()
    t = timed(lambda: oracle.run_static(lambda a, b: oracle.lap7_rows(dst, u, 1 + a, 1 + b, 1, n + 1, 1, n + 1, c0, c1),
                                        0, n, threads), seconds)
    return n ** 3 / t, "whole 64^3 sweep"


def cpu_c2(threads, seconds, planes=8):
    n, g = 256, 2
    u = inputs.c2_field(n, g)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    outs = [np.empty((n, n, n)) for _ in range(10)]
    t = timed(lambda: oracle.run_static(lambda a, b: oracle.d4_all(outs, u, g, (0, n, 0, n, a, b), k), 100,
                                        100 + planes, threads), seconds)
    return planes * n * n / t, f"{planes} z-planes of the 256^3 box"


def cpu_c3(threads, seconds, n=96):
    g = 2
    phi, pi = inputs.c3_fields(n, g)
    c = inputs.WaveConstants.for_grid(n)
    t = timed(lambda: oracle.rk4_step(phi, pi, g, c, threads), seconds)
    return n ** 3 / t, f"one RK4 step of a {n}^3 periodic box (same per-point arithmetic as 384^3)"


def cpu_c4(threads, seconds, planes=8):
    from paper_1308_1343_b200.level import Box, box_difference
    outer, hole = inputs.c4_outer_and_hole(512)
    b = box_difference(Box(*outer), Box(*hole))[0]
    nx, ny, nz = b.extents
    g = 2
    u = np.random.default_rng(4).uniform(-1, 1, (planes + 4, ny + 4, nx + 4))
    k = inputs.D4Constants.for_spacing(1.0 / 512)
    out = np.empty((planes, ny, nx))
    t = timed(lambda: oracle.run_static(lambda a, z1: oracle.lap4(out, u, g, (0, nx, 0, ny, a, z1), k.k2), 0, planes,
                                        threads), seconds)
    return planes * nx * ny / t, f"{planes} z-planes of the 512x512x256 box of the level"


def cpu_c5(threads, seconds, planes=2):
    n, g = 192, 2
    fields = [f[: planes + 4] for f in inputs.c5_fields(n, g)]
    poly = inputs.c5_poly()
    k = inputs.D4Constants.for_spacing(1.0 / n)
    outs = [np.empty((planes, n, n)) for _ in range(24)]
    t = timed(lambda: oracle.run_static(lambda a, b: oracle.rhs24(outs, fields, g, (0, n, 0, n, a, b), k, poly), 0,
                                        planes, threads), seconds)
    return planes * n * n / t, f"{planes} z-planes of the 192^3 box (all 24 fields and outputs)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    args = ap.parse_args()
    import torch

    from paper_1308_1343_b200 import _build
    from paper_1308_1343_b200.configs import CONFIGS
    _build.build()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    copy_peak = float(peaks.get("hbm_gbs", 6650.0))
    threads = host_threads()
    cpu = {1: cpu_c1, 2: cpu_c2, 3: cpu_c3, 4: cpu_c4, 5: cpu_c5}
    rows = []
    sys.path.insert(0, str(ROOT))
    from bench import ClockSampler   # NVML SM clock + clock-event reasons while timing
    for k, cls in CONFIGS.items():
        prob = cls().setup()
        with ClockSampler(torch.cuda.current_device()) as clk:
            t = gpu_time(prob, reps=100 if k == 1 else (20 if k != 5 else 5), graph=(k == 1))
        gpts = prob.updates / t / 1e9
        cpu_pts, sample = cpu[k](threads, args.cpu_seconds)
        rows.append({"config": k, "name": cls.name, "gpu_s": t, "gpu_gpts": gpts,
                     "algorithmic_bytes": prob.canonical_bytes, "algorithmic_gbs": prob.canonical_bytes / t / 1e9,
                     "frac_of_measured_copy": prob.canonical_bytes / t / 1e9 / copy_peak,
                     "cpu_gpts": cpu_pts / 1e9, "cpu_sample": sample, "cpu_threads": threads,
                     "gpu_over_cpu": gpts / (cpu_pts / 1e9), "clocks": clk.summary()})
        del prob
        torch.cuda.empty_cache()
    print(json.dumps({"gpu": torch.cuda.get_device_name(0), "host_threads": threads,
                      "cpu_model": _cpu_model(), "rows": rows}, indent=1))


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if __name__ == "__main__":
    main()
