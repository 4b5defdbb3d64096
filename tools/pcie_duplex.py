"""Full-duplex PCIe probe for the config-2 end-to-end step: pinned H2D of
the 140.6 MB ghosted input and D2H of the 1.342 GB outputs, alone and
concurrently on two streams (torch copies).  python tools/pcie_duplex.py"""
import torch, json
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
n_in, n_out = 140_608_000 // 8, 1_342_177_280 // 8
hin = torch.empty(n_in, dtype=torch.float64).pin_memory(); din = torch.empty(n_in, dtype=torch.float64, device="cuda")
hout = torch.empty(n_out, dtype=torch.float64).pin_memory(); dout = torch.empty(n_out, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2): hout.copy_(dout, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
big_in = torch.empty(n_out, dtype=torch.float64).pin_memory(); dbig = torch.empty(n_out, dtype=torch.float64, device="cuda")
def both_big():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): dbig.copy_(big_in, non_blocking=True)
    with torch.cuda.stream(s2): hout.copy_(dout, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
r = {"h2d_140MB_ms": timed(lambda: din.copy_(hin, non_blocking=True)),
     "d2h_1342MB_ms": timed(lambda: hout.copy_(dout, non_blocking=True)),
     "both_ms": timed(both),
     "h2d_1342MB_ms": timed(lambda: dbig.copy_(big_in, non_blocking=True)),
     "both_1342MB_each_ms": timed(both_big)}
print(json.dumps(r))
