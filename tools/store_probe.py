"""HBM write throughput of config 2's output mix by store instruction
(tools/csrc/store_probe.cu -> tools/libstoreprobe.so): width 8/16/32 bytes
per thread (st.global[.v2|.v4].f64), hint none / .cs / L1::no_allocate,
front (grid-stride) vs d4_all's tile pattern (TX x 4 tile, z4 chunk, x tiles
fastest), 1 or 10 output streams, with or without the read stream.  Beside
them: torch's fill of one 1.34 GB buffer and of the ten 134 MB outputs.
Bytes = algorithmic (8 B per element per stream); median of 20 launches.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
        -o tools/libstoreprobe.so tools/csrc/store_probe.cu
    python tools/store_probe.py > gpurun_out/store_probe.json
"""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libstoreprobe.so"))
lib.store_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p),
                            C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_void_p]
n = 256 ** 3
x = torch.rand(n, dtype=torch.float64, device="cuda")
outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(10)]
ptrs = (C.c_void_p * 10)(*[o.data_ptr() for o in outs])
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream


def timed(f, nbytes, reps=20):
    for _ in range(3):
        f()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        f()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    return round(nbytes / ms / 1e6, 1)


res = {}
big = torch.empty(10 * n, dtype=torch.float64, device="cuda")
res["torch_fill_1x1.34GB"] = timed(lambda: big.fill_(1.5), 80 * n)
res["torch_fill_10x134MB"] = timed(lambda: [o.fill_(1.5) for o in outs], 80 * n)
del big
HINTS = {0: "none", 1: "cs", 2: "na"}
for read in (0, 1):
    for nout in (1, 10):
        for w in (8, 16, 32):
            for h in (0, 1, 2):
                nbytes = 8 * n * (nout + read)
                best = 0
                for bps, thr in ((4, 256), (8, 256), (16, 128), (2, 512)):
                    f = lambda: lib.store_probe(w, h, 0, read, 0, x.data_ptr(), ptrs, n, nout, sms * bps, thr, st)
                    best = max(best, timed(f, nbytes))
                res[f"front_r{read}_w{nout}_{w}B_{HINTS[h]}"] = best
                if nout == 10:
                    for tx in (32, 64, 128):
                        if tx // (w // 8) * 4 < 32:
                            continue
                        f = lambda: lib.store_probe(w, h, 1, read, tx, x.data_ptr(), ptrs, n, nout, 0, 0, st)
                        res[f"tile{tx}_r{read}_w{nout}_{w}B_{HINTS[h]}"] = timed(f, nbytes)
assert torch.cuda.synchronize() is None
print(json.dumps(res, indent=1))
