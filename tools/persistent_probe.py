import json, torch, sys
sys.path.insert(0, '.')
from paper_1308_1343_b200 import stencil
from paper_1308_1343_b200.kernels import Laplacian7
from paper_1308_1343_b200.tuner import LaunchParams
n = 66
a, b = stencil._buffers(n, 1)
k = Laplacian7(b, a, stencil.C0, stencil.C1)
sp = stencil._space(n)
res = {}
for p in [(64, 8, 4), (64, 8, 8), (64, 4, 4), (64, 4, 2), (64, 2, 2), (64, 8, 16), (64, 8, 64), (64, 4, 8), (64, 2, 4), (64, 1, 4)]:
    lp = LaunchParams(*p)
    k.iterate(a, b, sp, 10, lp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); k.iterate(a, b, sp, 2000, lp); e1.record(); torch.cuda.synchronize()
    res[str(p)] = e0.elapsed_time(e1) / 2000 * 1e3
print(json.dumps(res, indent=0))
