"""FP64-pipe and shared-memory ceilings for the config-5 roofline
(tools/csrc/pipe_ceiling.cu, built to tools/libpipe.so):

* fp64: DMUL+DADD chains (unfused, -fmad=false), FP64 ops / s;
* lds: LDS.64 of 32 consecutive doubles per warp instruction (2 wavefronts),
  shared-memory wavefronts / s.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -shared \\
         -Xcompiler -fPIC tools/csrc/pipe_ceiling.cu -o tools/libpipe.so
    python tools/pipe_ceiling.py > profiles/r01/pipe_ceiling.json
"""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libpipe.so"))
for f in (lib.fp64_launch, lib.lds_launch):
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(1 << 16, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps)) * 1e-3


res = {"sm_count": sms}
best = 0.0
for blocks_per_sm, threads in ((4, 256), (8, 256), (2, 1024), (16, 128)):
    iters = 4096
    b = sms * blocks_per_sm
    s = timed(lambda: lib.fp64_launch(out.data_ptr(), b, threads, iters, st))
    ops = b * threads * iters * 8 * 2
    res[f"fp64_{blocks_per_sm}x{threads}_tops"] = ops / s / 1e12
    best = max(best, ops / s)
res["fp64_ops_per_s"] = best
res["fp64_ops_per_clk_per_sm"] = best / sms / 1.965e9
best = 0.0
for blocks_per_sm, threads in ((4, 256), (2, 1024), (8, 128)):
    iters = 4096
    b = sms * blocks_per_sm
    s = timed(lambda: lib.lds_launch(out.data_ptr(), b, threads, iters, st))
    wavefronts = b * (threads // 32) * iters * 8 * 2
    res[f"lds_{blocks_per_sm}x{threads}_gwf"] = wavefronts / s / 1e9
    best = max(best, wavefronts / s)
res["smem_wavefronts_per_s"] = best
res["smem_wavefronts_per_clk_per_sm"] = best / sms / 1.965e9
print(json.dumps(res, indent=1))
