"""F1 inter-box ghost fill on the config-4 level (3 boxes, ghost 2): bytes
moved per fill and device time — 20 fills captured in a CUDA graph and
replayed (one fill is far shorter than its Python launch path, so timing
single host-issued fills would measure the host)."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1308_1343_b200.configs import C4Level  # noqa: E402
from paper_1308_1343_b200.graphs import SweepGraph  # noqa: E402
from paper_1308_1343_b200.kernels import LevelGhostSync  # noqa: E402

p = C4Level().setup()
sync = LevelGhostSync(p.srcs, p.boxes)
g = SweepGraph(sync, repeat=20)
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e-3 / 20)
t = statistics.median(ts)
pts = sync.points()
print(json.dumps({"regions": len(sync.schedule), "points": pts, "bytes_moved": 16 * pts, "median_us": t * 1e6,
                  "GBs": 16 * pts / t / 1e9, "launches": -(-len(sync.schedule) // 64)}))
