"""The reference's own CPU stencil path next to the oracle port, on the same
host (only where /root/reference exists — this is the build container, not
the GPU box): justifies timing the port as the CPU baseline on the GPU box.

    PYTHONPATH=/root/reference/pkg/src python tools/ref_vs_port.py > profiles/r01/ref_vs_port.json

Config 1 (the reference's only implemented kernel, 66^3 with a 1-point
boundary = 64^3 interior): median seconds per sweep of the reference's
run_serial / run_naive (all host threads) / run_tuned (after 40 tuning
iterations), and of the port (oracle.lap7_rows, serial and through
oracle.run_static with the same thread count), plus bit-identity.
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from oracle.stencils import host_threads  # noqa: E402

try:
    from stencilrt import stencil as ref
    from stencilrt.tuner import TopologyConfig
except ImportError:
    sys.exit("run with PYTHONPATH=/root/reference/pkg/src (the reference package)")

n, iters, seed = 66, 60, 20130715
threads = host_threads()
res = {"host_threads": threads, "cpu": os.uname().machine, "n": n, "iters": iters}

s = ref.run_serial(n, iters, seed)
res["ref_run_serial_s"] = statistics.median(s.iter_seconds)
nv = ref.run_naive(n, iters, seed, threads)
res["ref_run_naive_s"] = statistics.median(nv.iter_seconds)
topo = TopologyConfig(n_coarse_threads=threads, n_fine_threads=1)
tu, _ = ref.run_tuned(n, iters, seed, topo)
res["ref_run_tuned_last20_s"] = statistics.median(tu.iter_seconds[-20:])

u = ref.make_field(n, seed)
c0, c1 = ref.C0, ref.C1


def port_serial(src):
    dst = src.copy()
    t0 = time.perf_counter()
    oracle.lap7_rows(dst, src, 1, n - 1, 1, n - 1, 1, n - 1, c0, c1)
    return dst, time.perf_counter() - t0


def port_static(src):
    dst = src.copy()
    t0 = time.perf_counter()
    oracle.run_static(lambda a, b: oracle.lap7_rows(dst, src, a, b, 1, n - 1, 1, n - 1, c0, c1), 1, n - 1, threads)
    return dst, time.perf_counter() - t0


for name, fn in (("port_serial_s", port_serial), ("port_static_s", port_static)):
    src, ts = u.copy(), []
    for _ in range(iters):
        src, t = fn(src)
        ts.append(t)
    res[name] = statistics.median(ts)
    res[name[:-2] + "_bit_identical_to_ref"] = bool(src.tobytes() == s.final.tobytes())
pts = (n - 2) ** 3
for k in list(res):
    if k.endswith("_s"):
        res[k[:-2] + "_mpts"] = pts / res[k] / 1e6
print(json.dumps(res, indent=1))
