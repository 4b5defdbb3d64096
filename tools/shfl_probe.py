"""SHFL vs LDS data path (tools/csrc/shfl_probe.cu -> tools/libshfl_probe.so):
per-SM rates of LDS.64 (wavefronts), SHFL.32, and both in one loop.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \\
         tools/csrc/shfl_probe.cu -o tools/libshfl_probe.so
    python tools/shfl_probe.py > profiles/r02/shfl_probe.json
"""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libshfl_probe.so"))
lib.probe.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(1 << 12, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
clk = 1.965e9


def timed(which, blocks, threads, iters, reps=7):
    for _ in range(2):
        lib.probe(which, out.data_ptr(), blocks, threads, iters, st)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        lib.probe(which, out.data_ptr(), blocks, threads, iters, st)
        ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps)) * 1e-3


res = {}
iters, threads, bps = 4096, 256, 4
b = sms * bps
warps = b * threads // 32
for which, name, lds, shfl in ((0, "lds_only", 8, 0), (1, "shfl8_only", 0, 8), (2, "lds8_shfl8", 8, 8),
                               (3, "lds8_shfl4", 8, 4), (4, "lds8_shfl16", 8, 16)):
    s = timed(which, b, threads, iters)
    per_clk_sm = lambda n: warps * iters * n / s / sms / clk
    res[name] = {"ms": s * 1e3, "lds_wavefronts_per_clk_sm": per_clk_sm(lds) * 2,
                 "shfl_instr_per_clk_sm": per_clk_sm(shfl)}
print(json.dumps(res, indent=1))
