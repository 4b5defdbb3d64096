"""TMA bulk-tensor stores vs st.global for config 2's output mix
(tools/csrc/tma_store_probe.cu -> tools/libtmastoreprobe.so, beside
tools/libstoreprobe.so's STG tile kernels in the same session).  Bytes =
algorithmic (8 B per element per stream: 10 writes [+ 1 read]); median of
20 launches.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \\
        -o tools/libtmastoreprobe.so tools/csrc/tma_store_probe.cu -lcuda
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \\
        -o tools/libstoreprobe.so tools/csrc/store_probe.cu
    python tools/tma_store_probe.py > gpurun_out/tma_store_probe.json
"""
import ctypes as C
import json
import statistics
from pathlib import Path

import torch

here = Path(__file__).resolve().parent
tma = C.CDLL(str(here / "libtmastoreprobe.so"))
tma.tma_store_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_int,
                                C.c_void_p]
stg = C.CDLL(str(here / "libstoreprobe.so"))
stg.store_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p),
                            C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_void_p]
n = 256 ** 3
x = torch.rand(n, dtype=torch.float64, device="cuda")
outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(10)]
ptrs = (C.c_void_p * 10)(*[o.data_ptr() for o in outs])
st = torch.cuda.current_stream().cuda_stream


def timed(f, nbytes, reps=20):
    for _ in range(3):
        assert f() == 0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        f()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    return round(nbytes / ms / 1e6, 1)


res = {}
# correctness of one TMA variant: output k = (k+1) * input
assert tma.tma_store_probe(32, 1, 2, 0, x.data_ptr(), ptrs, 10, st) == 0
torch.cuda.synchronize()
res["tma_bits_ok"] = all(torch.equal(outs[k], x * (k + 1)) for k in (0, 9))
for rnd in range(2):
    for read in (0, 1):
        nbytes = 8 * n * (10 + read)
        res[f"r{rnd}_stg_tile32_r{read}_16B_cs"] = timed(
            lambda: stg.store_probe(16, 1, 1, read, 32, x.data_ptr(), ptrs, n, 10, 0, 0, st), nbytes)
        for tx in (32, 64, 128):
            for nbuf in (1, 2, 4):
                if tx == 128 and nbuf == 4:
                    continue   # 160 KB of staging
                for hint in (0, 1):
                    res[f"r{rnd}_tma_tile{tx}_r{read}_buf{nbuf}_{'evict_first' if hint else 'nohint'}"] = timed(
                        lambda: tma.tma_store_probe(tx, read, nbuf, hint, x.data_ptr(), ptrs, 10, st), nbytes)
print(json.dumps(res, indent=1))
