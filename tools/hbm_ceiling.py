"""HBM ceilings for the traffic mix of the stencil sweeps (torch kernels,
CUDA events, median of 20): write-only fill of 1.34 GB (config 2's ten
outputs), and copy (read+write) of 1 GiB, for context next to
MEASURED_PEAKS.json's copy figure."""
import json
import statistics

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))


def main():
    n = 10 * 256 ** 3
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    ms = timed(lambda: out.fill_(1.0))
    res = {"fill_1.34GB_GBs": 8 * n / ms / 1e6}
    a = torch.empty(2 ** 27, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    ms = timed(lambda: b.copy_(a))
    res["copy_1GiB_rw_GBs"] = 2 * 8 * a.numel() / ms / 1e6
    print(json.dumps(res))


if __name__ == "__main__":
    main()
