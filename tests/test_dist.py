"""Multi-rank path on CPU: world-size-2 gloo processes each sweep their shard
of a level's boxes (no data-path collective), results gathered and compared
with the single-process sweep; max-over-ranks timing reduction."""
import os

import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import inputs
from paper_1308_1343_b200.level import Box, box_difference
from paper_1308_1343_b200.shard import shard_boxes, split_z


def level(n):
    outer, hole = inputs.c4_outer_and_hole(n)
    return box_difference(Box(*outer), Box(*hole))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_cover_every_point_once(world):
    boxes = level(32)
    owned = [shard_boxes(boxes, world, r) for r in range(world)]
    pts = set()
    total = 0
    for part in owned:
        for b in part:
            total += b.volume()
            for z in range(b.lo[2], b.hi[2] + 1):
                for y in range(b.lo[1], b.hi[1] + 1):
                    row = {(x, y, z) for x in range(b.lo[0], b.hi[0] + 1)}
                    assert not (row & pts)
                    pts |= row
    assert total == sum(b.volume() for b in boxes) == len(pts)
    loads = [sum(b.volume() for b in part) for part in owned]
    assert max(loads) <= 1.5 * (total / world) + max(b.volume() for b in boxes) / world


def test_split_z():
    b = Box((0, 0, 3), (4, 4, 12))
    parts = split_z(b, 4)
    assert sum(p.volume() for p in parts) == b.volume()
    assert parts[0].lo[2] == 3 and parts[-1].hi[2] == 12


def _worker(rank, world, port, n, g, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    boxes = level(n)
    fields = inputs.c4_fields(boxes, g, seed=99)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    mine = shard_boxes(boxes, world, rank)
    results = {}
    for piece in mine:
        j = next(i for i, b in enumerate(boxes) if all(b.lo[d] <= piece.lo[d] and piece.hi[d] <= b.hi[d] for d in range(3)))
        b = boxes[j]
        nx, ny, nz = b.extents
        out = np.full((nz, ny, nx), np.nan)
        region = tuple(v for d in range(3) for v in (piece.lo[d] - b.lo[d], piece.hi[d] + 1 - b.lo[d]))
        oracle.lap4(out, fields[j], g, region, k.k2)
        z0, z1 = region[4], region[5]
        results[(j, z0, z1)] = out[z0:z1]
    gathered = [None] * world
    dist.all_gather_object(gathered, results)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((gathered, float(t.item())))
    dist.destroy_process_group()


def test_gloo_world2_level_sweep_matches_single_process():
    import torch.multiprocessing as mp
    n, g, world = 24, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, g, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    boxes = level(n)
    fields = inputs.c4_fields(boxes, g, seed=99)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    for j, (b, u) in enumerate(zip(boxes, fields)):
        nx, ny, nz = b.extents
        want = np.empty((nz, ny, nx))
        oracle.lap4(want, u, g, (0, nx, 0, ny, 0, nz), k.k2)
        got = np.full((nz, ny, nx), np.nan)
        for part in gathered:
            for (jj, z0, z1), arr in part.items():
                if jj == j:
                    got[z0:z1] = arr
        assert got.tobytes() == want.tobytes()
