"""How much of a graph-replayed, event-bracketed config-1 sweep (run_loop's
graphed path) is the sweep?  Times graphs holding [event, event],
[event, sweep, event], [event, sweep x2, event] and [event, sweep x10, event]
(CUDA events inside the graph), median of 200 replays each.

    python tools/event_overhead_probe.py > profiles/r02/event_overhead.json
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
    from paper_1308_1343_b200 import stencil
    from paper_1308_1343_b200.kernels import Laplacian7

    n = 66
    src, dst = stencil._buffers(n, 1)
    space = stencil._space(n)
    k = Laplacian7(dst, src, stencil.C0, stencil.C1)
    p = k.default_params
    s = torch.cuda.Stream()
    res = {}
    for nk in (0, 1, 2, 10):
        a = torch.cuda.Event(enable_timing=True, external=True)
        b = torch.cuda.Event(enable_timing=True, external=True)
        with torch.cuda.stream(s):
            k.launch(space, p, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            a.record(s)
            for _ in range(nk):
                k.launch(space, p, stream=s)
            b.record(s)
        ts = []
        for _ in range(220):
            with torch.cuda.stream(s):
                g.replay()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[f"graph_events_{nk}_sweeps_us"] = statistics.median(ts[20:])
    # events on the stream around an eager launch / around a graph replay of the bare sweep
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=s):
        k.launch(space, p, stream=s)
    for name, fn in (("stream_events_eager_sweep_us", lambda: k.launch(space, p, stream=s)),
                     ("stream_events_graph_sweep_us", g1.replay)):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(220):
            with torch.cuda.stream(s):
                a.record(s)
                fn()
                b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[name] = statistics.median(ts[20:])
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
