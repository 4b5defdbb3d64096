"""F4: z-slab decomposition with the halo written by the producing stage into
the neighbour's ghost planes — single-process slabs (GPU), two processes
sharing buffers over CUDA IPC on one GPU (GPU), slab bookkeeping (CPU)."""
import os

import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import inputs
from paper_1308_1343_b200.errors import UsageError
from paper_1308_1343_b200.halo import z_cuts
from conftest import free_port


def test_z_cuts():
    assert z_cuts(384, 8, 2) == [0, 48, 96, 144, 192, 240, 288, 336, 384]
    assert z_cuts(10, 3, 2) == [0, 3, 6, 10]
    with pytest.raises(UsageError):
        z_cuts(6, 4, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["fused", "staged"])
@pytest.mark.parametrize("schedule", ["stages", "lap_pairs", "pairs"])
@pytest.mark.parametrize("parts", [1, 2, 3])
def test_slabs_one_process_match_global_oracle(parts, schedule, transport):
    """Fused: the kernels store the boundary planes into the neighbours'
    ghost planes; staged: into local send blocks that a device copy (NCCL
    send/recv across ranks) moves there — same bits either way."""
    from paper_1308_1343_b200 import _build
    from paper_1308_1343_b200.halo import WaveRK4Slabs
    _build.build()
    n, g = 24, 2
    phi0, pi0 = inputs.c3_fields(n, g, seed=40 + parts)
    c = inputs.WaveConstants.for_grid(n)
    sl = WaveRK4Slabs(n, parts, g, c, schedule=schedule, transport=transport)
    sl.upload(phi0, pi0)
    sl.step()
    wphi, wpi = oracle.rk4_step(phi0, pi0, g, c)
    I = (slice(g, g + n),) * 3
    assert sl.result("phi_b").tobytes() == np.ascontiguousarray(wphi[I]).tobytes()
    assert sl.result("pi_b").tobytes() == np.ascontiguousarray(wpi[I]).tobytes()
    # every slab's ghost shell (incl. the z planes written by its neighbours)
    for s, full in zip(sl.slabs, sl.result("phi_b", with_ghosts=True)):
        want = wphi[s.z0:s.z0 + s.nz + 2 * g]
        assert full.tobytes() == np.ascontiguousarray(want).tobytes(), s.z0
    if schedule != "stages":   # the pair schedules also carry pi's ghosts across slabs
        for s, full in zip(sl.slabs, sl.result("pi_b", with_ghosts=True)):
            want = wpi[s.z0:s.z0 + s.nz + 2 * g]
            assert full.tobytes() == np.ascontiguousarray(want).tobytes(), s.z0


def _ipc_worker(rank, world, port, q, schedule):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1308_1343_b200.halo import ZSlabRank
    n, g = 20, 2
    phi0, pi0 = inputs.c3_fields(n, g, seed=77)
    c = inputs.WaveConstants.for_grid(n)
    me = ZSlabRank(n, rank, world, g, c, dist, schedule=schedule)
    me.slab.upload(phi0, pi0)
    me.barrier()
    me.step()
    got = me.slab.phi_b.download(with_ghosts=True)
    got_pi = me.slab.pi_b.download(with_ghosts=True)
    dist.barrier()
    q.put((rank, me.slab.z0, got, got_pi))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["stages", "lap_pairs"])
def test_two_ranks_ipc_on_one_gpu(schedule):
    """Two processes, one slab each, neighbour ghost planes written through
    CUDA IPC mappings; kernels never wait on each other (host barrier)."""
    import torch.multiprocessing as mp
    from paper_1308_1343_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, schedule)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, g = 20, 2
    phi0, pi0 = inputs.c3_fields(n, g, seed=77)
    wphi, wpi = oracle.rk4_step(phi0, pi0, g, inputs.WaveConstants.for_grid(n))
    for rank, z0, got, got_pi in res:
        want = wphi[z0:z0 + got.shape[0]]
        assert got.tobytes() == np.ascontiguousarray(want).tobytes(), rank
        if schedule != "stages":
            want = wpi[z0:z0 + got_pi.shape[0]]
            assert got_pi.tobytes() == np.ascontiguousarray(want).tobytes(), rank
