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
from conftest import free_port


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
    port = free_port()
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


@pytest.mark.gpu
@pytest.mark.parametrize("impl", ["ours", "reference"])
def test_bench_under_torchrun_two_ranks(impl):
    """bench.py launched the way the driver launches N>1 (torchrun, one
    process per rank), both ranks on the one GPU here with the gloo backend
    (plumbing only: the ranks never wait on each other's kernels): rank 0
    prints exactly one JSON line with the whole-job value."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(root / "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--impl", impl]
    if impl == "ours":
        cmd += ["--tune", "0", "--no-cpu", "--e2e-steps", "3", "--sustained-steps", "0"]
    env = dict(os.environ, STENCIL_BENCH_BACKEND="gloo")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    rec = json.loads(lines[0])
    assert rec["value"] > 0 and rec["n_gpus"] == 2
    if impl == "ours":
        assert rec["scaling"] == "weak" and rec["gpu_launches"] == 3
        # config 3 as two z-slabs, one per rank, halo planes stored into the
        # other rank's ghost planes through CUDA IPC (host-ordered: ranks share the GPU)
        zs = rec["zslab"]["fused"]
        assert zs.get("bit_exact_vs_single_gpu") is True, zs
        assert zs["ms_per_step"] > 0
    else:
        assert rec["impl"] == "reference"


def _device_worker(rank, world, port, n, g, q):
    """One rank: its shard of the level's boxes swept by the DEVICE kernel
    (LevelLaplacian4, one launch for the shard), results gathered."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1308_1343_b200 import _build
    from paper_1308_1343_b200.grid import DeviceGrid
    from paper_1308_1343_b200.kernels import LevelLaplacian4
    _build.build()
    boxes = level(n)
    fields = inputs.c4_fields(boxes, g, seed=99)
    k = inputs.D4Constants.for_spacing(1.0 / n)
    mine = shard_boxes(boxes, world, rank)
    srcs, dsts, keys = [], [], []
    for piece in mine:
        j = next(i for i, b in enumerate(boxes) if all(b.lo[d] <= piece.lo[d] and piece.hi[d] <= b.hi[d] for d in range(3)))
        b = boxes[j]
        # the piece's source with ghosts, cut from its box's field
        z0, z1 = piece.lo[2] - b.lo[2], piece.hi[2] + 1 - b.lo[2]
        s = DeviceGrid(piece.extents, g, lower=piece.lo)
        s.upload(fields[j][z0:z1 + 2 * g])
        srcs.append(s)
        dsts.append(DeviceGrid(piece.extents, 0, lower=piece.lo))
        keys.append((j, z0, z1))
    LevelLaplacian4(dsts, srcs, k).launch(None, LevelLaplacian4.default_params)
    results = {key: d.download() for key, d in zip(keys, dsts)}
    gathered = [None] * world
    dist.all_gather_object(gathered, results)
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_device_kernels_shard_the_level():
    """world-size-2 gloo: each rank sweeps its shard of the config-4-style
    level with the device kernel (ranks share the one GPU; no kernel waits
    on another rank); the gathered outputs equal the single-box oracle."""
    import torch.multiprocessing as mp
    n, g, world = 40, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_device_worker, args=(r, world, port, n, g, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
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
        assert got.tobytes() == want.tobytes(), j
