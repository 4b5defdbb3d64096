"""HBM ceiling of config 2's traffic mix (1 read + 10 write streams of 256^3
doubles), measured with a trivial grid-stride kernel (tools/csrc/mix_ceiling.cu)."""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libmix.so"))
lib.mix_launch.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_void_p]
n = 256 ** 3
x = torch.rand(n, dtype=torch.float64, device="cuda")
outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(10)]
ptrs = (C.c_void_p * 10)(*[o.data_ptr() for o in outs])
res = {}
for nout in (1, 5, 10):
    for blocks, threads in ((148 * 8, 256), (148 * 16, 256), (148 * 4, 512)):
        def run():
            lib.mix_launch(x.data_ptr(), ptrs, n, nout, blocks, threads, torch.cuda.current_stream().cuda_stream)
        for _ in range(3):
            run()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        ev[0].record()
        for i in range(20):
            run()
            ev[i + 1].record()
        torch.cuda.synchronize()
        ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
        res[f"read1_write{nout}_{blocks}x{threads}"] = 8 * n * (1 + nout) / ms / 1e6
print(json.dumps(res))
