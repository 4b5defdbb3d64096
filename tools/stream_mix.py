"""HBM throughput of config 2's stream mix under different access shapes
(tools/csrc/stream_mix.cu -> tools/libstream.so): write-only with 1 or 10
output streams, and 1 read + 10 writes with 1/4/8 loads in flight per
thread, over a range of grid sizes.  Modes 0/1: every CTA owns a
contiguous chunk of each stream; modes 2/3 (write-only / 1 read): the whole
grid sweeps each stream as one coalesced front.  Bytes = algorithmic (8 B per element
per stream)."""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libstream.so"))
lib.stream_launch.argtypes = [C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_longlong, C.c_int, C.c_int,
                              C.c_int, C.c_void_p]
n = 256 ** 3
x = torch.rand(n + 4 * 260 * 260, dtype=torch.float64, device="cuda")
outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(10)]
ptrs = (C.c_void_p * 10)(*[o.data_ptr() for o in outs])
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream
res = {}


def run(mode, unroll, nout, blocks, threads):
    f = lambda: lib.stream_launch(mode, unroll, x.data_ptr(), ptrs, n, nout, blocks, threads, st)
    for _ in range(3):
        f()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
    ev[0].record()
    for i in range(20):
        f()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
    return 8 * n * (nout + (mode in (1, 3))) / ms / 1e6


CASES = ((0, 1, 1), (0, 4, 1), (0, 1, 10), (0, 4, 10), (1, 1, 10), (1, 4, 10), (1, 8, 10),
         (2, 1, 1), (2, 4, 1), (2, 1, 10), (2, 4, 10), (3, 1, 10), (3, 4, 10), (3, 8, 10), (3, 4, 1))
for mode, unroll, nout in CASES:
    for bps, threads in ((4, 256), (8, 256), (16, 128), (2, 512), (32, 64)):
        res[f"mode{mode}_u{unroll}_w{nout}_{bps}x{threads}"] = run(mode, unroll, nout, sms * bps, threads)
best = {}
for k, v in res.items():
    key = k.rsplit("_", 1)[0]
    best[key] = max(best.get(key, 0), v)
print(json.dumps({"best_GBs": best, "all_GBs": res}, indent=1))
