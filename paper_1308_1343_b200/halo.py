"""F4 — z-slab decomposition of one periodic box.

A 384^3 periodic box split along z into R slabs needs exactly one exchange
per RK stage: the 2 planes next to each slab face go to the neighbouring
slab's ghost planes.  Instead of a separate exchange step (pack, NCCL
send/recv, unpack), the stage kernel that produces phi writes those planes
straight into the neighbour's phi ghost planes as part of its stores
(``sb_rk4_stage_zslab``): over NVLink when the neighbour is another GPU
(peer-mapped pointers via CUDA IPC), as plain stores when it is another slab
on the same GPU.  The only synchronisation left is "every slab finished
stage s" before stage s+1 reads its ghosts — a barrier, no data movement.

The stage pairs (``sb_rk4_pair_zslab``) work the same way with two launches
and two barriers per step instead of four: both outputs of a pair launch
(L1, L2 — or phi3, pi3 — and then phi', pi') write their boundary planes
into the neighbours' ghost planes, since each feeds a stencil of the next
launch.

The exchange has two transports:

* ``"fused"`` (default) — the stores above: the boundary planes land in the
  neighbour's ghost planes from inside the kernel (peer memory);
* ``"staged"`` — the NCCL baseline: the kernel writes the same boundary
  planes (with their x/y periodic images) into two local send blocks laid
  out exactly like a neighbour's g ghost planes, and a transport moves each
  block into the neighbour's contiguous ghost-plane block — a device copy
  between slabs of one process, ``ncclSend``/``ncclRecv`` (torch
  ``batch_isend_irecv``) between ranks.

* :class:`WaveRK4Slabs` — R slabs in one process (one GPU): both transports
  exercised end to end without extra GPUs.
* :class:`ZSlabRank` — one slab per process/rank; for ``"fused"`` the
  neighbour buffers are mapped with CUDA IPC handles exchanged through
  ``torch.distributed`` objects.  Ranks are ordered between launches either
  on the host (``sync="host"``: device synchronise + ``dist.barrier``, what
  ranks sharing one GPU must use) or on the device (``sync="device"``: a
  one-element all-reduce on the launching stream — it completes on a rank
  only after every rank's previous kernel has completed, so no host round
  trip; NCCL only).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from .errors import UsageError
from .grid import DeviceGrid, stream_ptr
from .inputs import WaveConstants
from .tuner import LaunchParams

BUFFERS = ("phi0", "pi0", "phi_a", "pi_a", "phi_b", "pi_b", "acc_phi", "acc_pi")
# (stage, phi_s, pi_s, phi_out, pi_out) of one classical RK4 step
STAGES = ((1, "phi0", "pi0", "phi_a", "pi_a"), (2, "phi_a", "pi_a", "phi_b", "pi_b"),
          (3, "phi_b", "pi_b", "phi_a", "pi_a"), (4, "phi_a", "pi_a", "phi_b", "pi_b"))
# (pair, phi_s, pi_s, phi_out, pi_out) of the pair schedules (kernels.WaveRK4)
PAIRS = {"lap_pairs": ((3, "phi0", "pi0", "phi_a", "pi_a"), (4, "phi_a", "pi_a", "phi_b", "pi_b")),
         "pairs": ((1, "phi0", "pi0", "phi_a", "pi_a"), (2, "phi_a", "pi_a", "phi_b", "pi_b"))}
SCHEDULES = ("stages", "lap_pairs", "pairs")


def _launches(schedule: str):
    if schedule not in SCHEDULES:
        raise UsageError(f"unknown z-slab RK4 schedule {schedule!r}")
    return STAGES if schedule == "stages" else PAIRS[schedule]


def z_cuts(n: int, parts: int, ghost: int) -> list[int]:
    """Even z cuts of [0, n) into `parts` slabs, each at least `ghost` thick."""
    if parts < 1 or n // parts < ghost:
        raise UsageError(f"{parts} slabs of a {n}-plane box would be thinner than the ghost width {ghost}")
    return [n * j // parts for j in range(parts)] + [n]


class Slab:
    """One z-slab's RK4 state: interior (n, n, nz), ghost g, level z offset z0."""

    def __init__(self, n: int, z0: int, nz: int, ghost: int, device=None):
        self.n, self.z0, self.nz, self.g = n, z0, nz, ghost
        for name in BUFFERS:
            setattr(self, name, DeviceGrid((n, n, nz), ghost, device, lower=(0, 0, z0)))

    def upload(self, phi_global, pi_global) -> None:
        """Take this slab's planes (with z ghosts) from global ghosted arrays."""
        g, z0, nz = self.g, self.z0, self.nz
        self.phi0.upload(phi_global[z0:z0 + nz + 2 * g], with_ghosts=True)
        self.pi0.upload(pi_global[z0:z0 + nz + 2 * g], with_ghosts=True)


def _fields(s: Slab, phi_s: str, pi_s: str, phi_out: str, pi_out: str) -> _lib.sb_rk4_fields:
    return _lib.sb_rk4_fields(getattr(s, phi_s).abi(), getattr(s, pi_s).abi(), s.phi0.abi(), s.pi0.abi(),
                              s.acc_phi.abi(), s.acc_pi.abi(), getattr(s, phi_out).abi(), getattr(s, pi_out).abi())


def _consts(c: WaveConstants) -> _lib.sb_rk4_constants:
    return _lib.sb_rk4_constants(_lib.d4_constants(c.lap), c.half_dt, c.dt, c.dt6)


def launch_stage(s: Slab, stage: tuple, c: WaveConstants, params: LaunchParams, lo_ptr: int, lo_dz: int,
                 hi_ptr: int, hi_dz: int, stream=None) -> None:
    st, phi_s, pi_s, phi_out, pi_out = stage
    f = _fields(s, phi_s, pi_s, phi_out, pi_out)
    zs = _lib.sb_zslab(lo_ptr, lo_dz, hi_ptr, hi_dz)
    _lib.call("sb_rk4_stage_zslab", st, C.byref(f), _lib.space((0, 0, 0), (s.n, s.n, s.nz)), _consts(c),
              _lib.launch_of(params, _lib.SB_LAUNCH_PERIODIC_GHOSTS), C.byref(zs), stream_ptr(stream))


def launch_pair(s: Slab, pair: tuple, c: WaveConstants, params: LaunchParams, lo: tuple, lo_dz: int, hi: tuple,
                hi_dz: int, stream=None) -> None:
    """One pair launch of slab s; lo / hi = (phi_out, pi_out) origins of the
    lower / upper neighbours."""
    k, phi_s, pi_s, phi_out, pi_out = pair
    f = _fields(s, phi_s, pi_s, phi_out, pi_out)
    zs = (_lib.sb_zslab * 2)(_lib.sb_zslab(lo[0], lo_dz, hi[0], hi_dz), _lib.sb_zslab(lo[1], lo_dz, hi[1], hi_dz))
    _lib.call("sb_rk4_pair_zslab", k, C.byref(f), _lib.space((0, 0, 0), (s.n, s.n, s.nz)), _consts(c),
              _lib.launch_of(params, _lib.SB_LAUNCH_PERIODIC_GHOSTS), zs, stream_ptr(stream))


def _default_params(schedule: str) -> LaunchParams:
    return LaunchParams(64, 4, 16, 1) if schedule == "stages" else LaunchParams(32, 4, 64, 1)


TRANSPORTS = ("fused", "staged")


def ghost_block(grid: DeviceGrid, side: str):
    """The g contiguous ghost planes below (``"lo"``) or above (``"hi"``) the
    interior of `grid`, as a flat view of its storage (whole planes, padding
    included)."""
    g, sz, nz = grid.ghost, grid.sz, grid.extents[2]
    k0 = 0 if side == "lo" else nz + g
    return grid.storage[k0 * sz:(k0 + g) * sz]


class SendBlocks:
    """Local send blocks of one slab output (staged transport): ``lo`` holds
    the planes destined for the lower neighbour's upper ghost planes, ``hi``
    those for the upper neighbour's lower ghost planes; ``targets(nz_lo)``
    are the (lo, hi) origins to hand the kernel in place of peer origins."""

    def __init__(self, like: DeviceGrid):
        import torch
        self.g, self.sz, self.sy, self.xpad = like.ghost, like.sz, like.sy, like.xpad
        self.lo = torch.empty(self.g * self.sz, dtype=torch.float64, device=like.device)
        self.hi = torch.empty(self.g * self.sz, dtype=torch.float64, device=like.device)

    def targets(self, nz_lo: int) -> tuple[int, int]:
        inner = 8 * (self.xpad + self.g * self.sy)   # interior origin of a plane within a block
        # lower neighbour's planes [nz_lo, nz_lo + g) -> block planes [0, g)
        lo = self.lo.data_ptr() + inner - 8 * nz_lo * self.sz
        # upper neighbour's planes [-g, 0) -> block planes [0, g)
        hi = self.hi.data_ptr() + inner + 8 * self.g * self.sz
        return lo, hi


class WaveRK4Slabs:
    """R z-slabs of one periodic n^3 box in one process.  Each stage launch of
    slab r writes its boundary planes into slabs r-1 / r+1 (ring): directly
    (``transport="fused"``) or through its send blocks and a device copy
    (``"staged"``)."""

    def __init__(self, n: int, parts: int, ghost: int, c: WaveConstants, device=None, schedule: str = "stages",
                 transport: str = "fused"):
        if transport not in TRANSPORTS:
            raise UsageError(f"unknown z-slab transport {transport!r}")
        self.n, self.g, self.c = n, ghost, c
        self.schedule = schedule
        self.transport = transport
        self.launches = _launches(schedule)
        cuts = z_cuts(n, parts, ghost)
        self.slabs = [Slab(n, cuts[j], cuts[j + 1] - cuts[j], ghost, device) for j in range(parts)]
        self.params = _default_params(schedule)
        if transport == "staged":
            outs = {name for st in self.launches for name in (st[3], st[4] if schedule != "stages" else st[3])}
            self.send = [{name: SendBlocks(getattr(s, name)) for name in outs} for s in self.slabs]

    def upload(self, phi_global, pi_global) -> None:
        for s in self.slabs:
            s.upload(phi_global, pi_global)

    def step(self, params: LaunchParams | None = None, stream=None) -> None:
        import torch
        p = params or self.params
        R = len(self.slabs)
        for stage in self.launches:
            out, out2 = stage[3], stage[4]
            names = (out,) if self.schedule == "stages" else (out, out2)
            for r, s in enumerate(self.slabs):
                lo, hi = self.slabs[(r - 1) % R], self.slabs[(r + 1) % R]
                if self.transport == "staged":
                    t = [self.send[r][nm].targets(lo.nz) for nm in names]
                    lo_t, hi_t = tuple(x[0] for x in t), tuple(x[1] for x in t)
                else:
                    lo_t = tuple(getattr(lo, nm).origin_ptr for nm in names)
                    hi_t = tuple(getattr(hi, nm).origin_ptr for nm in names)
                if self.schedule == "stages":
                    launch_stage(s, stage, self.c, p, lo_t[0], lo.nz, hi_t[0], -s.nz, stream)
                else:
                    launch_pair(s, stage, self.c, p, lo_t, lo.nz, hi_t, -s.nz, stream)
            if self.transport == "staged":   # every slab's blocks to its neighbours' ghost planes
                with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
                    for r in range(R):
                        lo, hi = self.slabs[(r - 1) % R], self.slabs[(r + 1) % R]
                        for nm in names:
                            ghost_block(getattr(lo, nm), "hi").copy_(self.send[r][nm].lo)
                            ghost_block(getattr(hi, nm), "lo").copy_(self.send[r][nm].hi)

    def result(self, name: str = "phi_b", with_ghosts: bool = False):
        import numpy as np
        parts = [getattr(s, name).download(with_ghosts=with_ghosts) for s in self.slabs]
        if not with_ghosts:
            return np.concatenate(parts, axis=0)
        return parts


class ZSlabRank:
    """This rank's slab of a z-decomposed periodic box (one slab per rank).

    ``transport="fused"``: neighbour buffers are CUDA-IPC-mapped (peer memory
    over NVLink on a multi-GPU node) and the kernels store the boundary
    planes into them; ``"staged"``: local send blocks and NCCL send/recv
    (``dist`` must be an NCCL group).  ``sync="host"`` orders launches with a
    device synchronise + ``dist.barrier`` (required when ranks share a GPU),
    ``"device"`` with a one-element all-reduce on the stream (NCCL)."""

    def __init__(self, n: int, rank: int, world: int, ghost: int, c: WaveConstants, dist, device=None,
                 schedule: str = "stages", transport: str = "fused", sync: str = "host"):
        import torch
        if transport not in TRANSPORTS or sync not in ("host", "device"):
            raise UsageError(f"bad z-slab transport/sync {transport!r}/{sync!r}")
        self.n, self.g, self.c = n, ghost, c
        self.rank, self.world, self.dist = rank, world, dist
        self.schedule, self.transport, self.sync = schedule, transport, sync
        self.launches = _launches(schedule)
        cuts = z_cuts(n, world, ghost)
        self.slab = Slab(n, cuts[rank], cuts[rank + 1] - cuts[rank], ghost, device)
        self.params = _default_params(schedule)
        self.lo, self.hi = (rank - 1) % world, (rank + 1) % world
        shared = ("phi_a", "phi_b") if schedule == "stages" else ("phi_a", "pi_a", "phi_b", "pi_b")
        self._keep = []
        self.peer: dict[tuple[int, str], int] = {}
        self.peer_nz: dict[int, int] = {}
        if transport == "fused":
            mine = {name: (getattr(self.slab, name).storage.untyped_storage()._share_cuda_(),
                           getattr(self.slab, name).offset) for name in shared}
        else:
            mine = {}
            self.send = {name: SendBlocks(getattr(self.slab, name)) for name in shared}
        everyone = [None] * world
        dist.all_gather_object(everyone, (self.slab.nz, mine))
        for r in {self.lo, self.hi}:
            nz_r, handles = everyone[r]
            self.peer_nz[r] = nz_r
            for name, (h, off) in handles.items():
                if r == rank:
                    ptr = getattr(self.slab, name).origin_ptr
                else:
                    st = torch.UntypedStorage._new_shared_cuda(*h)
                    self._keep.append(st)
                    ptr = st.data_ptr() + 8 * off
                    # our kernels store into the neighbour's memory: peer
                    # access from OUR device to the owner's (a no-op when the
                    # ranks share a GPU)
                    with torch.cuda.device(self.slab.phi0.device):
                        _lib.call("sb_enable_peer_access", st.device.index)
                self.peer[(r, name)] = ptr
        if sync == "device":
            self._token = torch.zeros(1, dtype=torch.float32, device=self.slab.phi0.device)

    def barrier(self) -> None:
        if self.sync == "device":
            self.dist.all_reduce(self._token)
            return
        import torch
        torch.cuda.synchronize()
        self.dist.barrier()

    def _exchange(self, names) -> None:
        """Staged transport: my send blocks to the neighbours' ghost planes and
        theirs into mine, one grouped NCCL send/recv (sends ordered lo, hi;
        receives from hi, lo — the order every peer pair matches)."""
        d = self.dist
        ops = []
        for nm in names:
            grid, blk = getattr(self.slab, nm), self.send[nm]
            ops += [d.P2POp(d.isend, blk.lo, self.lo), d.P2POp(d.isend, blk.hi, self.hi),
                    d.P2POp(d.irecv, ghost_block(grid, "hi"), self.hi), d.P2POp(d.irecv, ghost_block(grid, "lo"), self.lo)]
        for w in d.batch_isend_irecv(ops):
            w.wait()

    def step(self, params: LaunchParams | None = None) -> None:
        p = params or self.params
        lo, hi = self.lo, self.hi
        for stage in self.launches:
            out, out2 = stage[3], stage[4]
            names = (out,) if self.schedule == "stages" else (out, out2)
            if self.transport == "staged":
                t = [self.send[nm].targets(self.peer_nz[lo]) for nm in names]
                lo_t, hi_t = tuple(x[0] for x in t), tuple(x[1] for x in t)
            else:
                lo_t = tuple(self.peer[(lo, nm)] for nm in names)
                hi_t = tuple(self.peer[(hi, nm)] for nm in names)
            if self.schedule == "stages":
                launch_stage(self.slab, stage, self.c, p, lo_t[0], self.peer_nz[lo], hi_t[0], -self.slab.nz)
            else:
                launch_pair(self.slab, stage, self.c, p, lo_t, self.peer_nz[lo], hi_t, -self.slab.nz)
            if self.transport == "staged":
                self._exchange(names)
            else:
                self.barrier()
