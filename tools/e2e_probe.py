"""Where does the config-2 end-to-end step's time go?  Times the public
host pipeline at several chunk sizes, the raw transfers alone, and
H2D + D2H concurrently."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1308_1343_b200.configs import C2FourthOrder  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


p = C2FourthOrder().setup()
n = p.n
h_in = torch.from_numpy(p.host_u).pin_memory()
h_out = [torch.empty((n, n, n), dtype=torch.float64).pin_memory() for _ in range(10)]
ptrs = [t.data_ptr() for t in h_out]
res = {}
for chunk in (None, 16, 32, 64, 128):
    res[f"e2e_chunk{chunk}_ms"] = timed(lambda: p.e2e_step(h_in.data_ptr(), ptrs, chunk=chunk))
res["d2h_only_ms"] = timed(lambda: [o.download_to_ptr(q, False) for o, q in zip(p.outs, ptrs)])
res["h2d_only_ms"] = timed(lambda: p.src.upload_from_ptr(h_in.data_ptr(), True))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    p.src.upload_from_ptr(h_in.data_ptr(), True, s1)
    for o, q in zip(p.outs, ptrs):
        o.download_to_ptr(q, False, s2)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


res["h2d_and_d2h_concurrent_ms"] = timed(both)
flat = torch.empty(10 * n ** 3, dtype=torch.float64).pin_memory()
dflat = torch.empty(10 * n ** 3, dtype=torch.float64, device="cuda")
res["torch_d2h_1.34GB_ms"] = timed(lambda: flat.copy_(dflat, non_blocking=True))
print(json.dumps(res))
