"""Read/write phase separation probe (tools/csrc/phase_probe.cu ->
tools/libphaseprobe.so): one CTA per SM reads a chunk per phase into shared
memory and writes it to 1 or 10 outputs, with (sync=1) or without (sync=0) a
grid barrier between the chip-wide read and write halves of each phase.
Config 2's volume (256^3 doubles per stream); bytes = algorithmic; median of
20 launches.  Beside it: torch's copy of the same 134 MB.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
        -o tools/libphaseprobe.so tools/csrc/phase_probe.cu
    python tools/phase_probe.py > gpurun_out/phase_probe.json
"""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libphaseprobe.so"))
lib.phase_probe.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_longlong, C.c_int, C.c_int, C.c_int,
                            C.c_void_p]
n = 256 ** 3
x = torch.rand(n, dtype=torch.float64, device="cuda")
outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(10)]
ptrs = (C.c_void_p * 10)(*[o.data_ptr() for o in outs])
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream


def timed(f, nbytes, reps=20):
    for _ in range(3):
        r = f()
        assert r is None or isinstance(r, torch.Tensor) or r == 0, r
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        f()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    return round(nbytes / ms / 1e6, 1)


res = {"torch_copy_134MB": timed(lambda: outs[0].copy_(x), 16 * n)}
for nout in (1, 10):
    for chunk in (32768, 65536, 131072, 196608):
        for sync in (0, 1):
            f = lambda: lib.phase_probe(sync, x.data_ptr(), ptrs, n, nout, chunk, sms, st)
            res[f"w{nout}_chunk{chunk // 1024}K_sync{sync}"] = timed(f, 8 * n * (nout + 1))
print(json.dumps(res, indent=1))
