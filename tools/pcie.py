"""Host<->device copy bandwidth with pinned memory: one stream vs several
concurrent streams (copy engines), H2D and D2H, 1.34 GB total."""
import json

import torch

n = 10 * 256 ** 3
dev = torch.empty(n, dtype=torch.float64, device="cuda")
host = torch.empty(n, dtype=torch.float64).pin_memory()
res = {}
for direction in ("d2h", "h2d"):
    for k in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(k)]
        parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]

        def run():
            for s, (a, b) in zip(streams, parts):
                with torch.cuda.stream(s):
                    if direction == "d2h":
                        host[a:b].copy_(dev[a:b], non_blocking=True)
                    else:
                        dev[a:b].copy_(host[a:b], non_blocking=True)
            torch.cuda.synchronize()
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[f"{direction}_streams{k}_GBs"] = 3 * 8 * n / e0.elapsed_time(e1) / 1e6
print(json.dumps(res))
