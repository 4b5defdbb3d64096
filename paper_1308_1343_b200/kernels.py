"""Device stencil kernels behind the reference's ``Kernel`` plugin type.

The reference plugs arithmetic into its loop iterator as
``Kernel = Callable[[IndexSpace], None]`` (traverse.py:159), e.g.
``_piece_kernel(dst, src)`` around ``_update_rows`` (stencil.py:31-46).
Each class here is such a callable — ``kernel(piece)`` launches the B200
kernel over that piece, so the reference's ``execute_plan``/``run_static``
drive it unchanged — and additionally exposes the fast path the device
engine uses: ``launch(space, params)`` covers a whole index space (or a
whole level) in one launch with a :class:`~.tuner.LaunchParams` tile shape,
and ``launch_space()`` names the tunable space for the GPU tuner.

Index spaces are in the caller's coordinates; each kernel subtracts the
grid's ``lower`` (so the reference's array-index pieces work for the demo,
and level coordinates work for bboxset boxes).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import UsageError
from .grid import DeviceGrid, stream_ptr
from .inputs import N_TERMS, N_VARS, D4Constants, PolyTable, WaveConstants
from .traverse import IndexSpace
from .tuner import LaunchParams, LaunchSpace

# launch spaces: thread caps mirror max_threads() in csrc/d4.cu (register budgets)
D4_ALL_SPACE = LaunchSpace(kind="d4_all", max_threads_pair=256, max_threads_scalar=512, rx_buffer=True)
D4_SPACE = LaunchSpace(kind="lap4", max_threads_pair=512, max_threads_scalar=512)
RK4_SPACE = LaunchSpace(kind="rk4", max_threads_pair=256, max_threads_scalar=512)
LAP7_SPACE = LaunchSpace(kind="lap7", max_threads_pair=256, radius=1, stages=0, tile_xs=(64,), z_min=1,
                         tile_ys=(1, 2, 4, 8), points=(2,))


def _local(space: IndexSpace, grid: DeviceGrid) -> _lib.sb_space:
    if space.dim != 3:
        raise UsageError("device stencil kernels sweep 3-D index spaces")
    lo = tuple(a - o for a, o in zip(space.lo, grid.lower))
    hi = tuple(b - o for b, o in zip(space.hi, grid.lower))
    return _lib.space(lo, hi)


def _interior_space(grid: DeviceGrid) -> IndexSpace:
    return IndexSpace(grid.lower, tuple(l + e for l, e in zip(grid.lower, grid.extents)))


class DeviceKernel:
    """Common behaviour of the device kernels (plugin + fast path)."""

    site_id = "kernel"
    space_kind = D4_SPACE
    idempotent = True    # outputs are a pure function of the inputs (run_loop may replay a launch)
    extra_flags = 0   # SB_LAUNCH_* flags added to every launch (tools/sweep.py --flags)
    default_params: LaunchParams = LaunchParams(64, 8, 32)

    def launch_space(self) -> LaunchSpace:
        return self.space_kind

    def __call__(self, piece: IndexSpace) -> None:
        self.launch(piece, self.default_params)

    def launch_plan(self, plan, params: LaunchParams | None = None, stream=None) -> None:
        """The fast path for a reference plan (``build_plan``, traverse.py:130-156):
        its pieces partition ``plan.space``, so executing all of them is ONE
        launch over that space (tiles = CTAs) — the result ``execute_plan``
        would produce piece by piece, bit for bit."""
        self.launch(plan.space, params or self.default_params, stream=stream)

    def launch(self, space: IndexSpace, params: LaunchParams, stream=None) -> None:
        raise NotImplementedError

    def full_space(self) -> IndexSpace:
        raise NotImplementedError

    def pitch_class(self) -> int:
        """Row pitch (elements) of the swept source grid: part of the device
        tuning key (tuner.device_setup)."""
        for name in ("src", "srcs", "ins", "fields"):
            g = getattr(self, name, None)
            if g is None:
                continue
            if isinstance(g, list):
                g = g[0]["phi_s"] if isinstance(g[0], dict) else g[0]
            return g.sy
        return 0

    # host-path caches: the ctypes argument structs of a launch are built once
    # per (space, params) — the grids of a kernel object never move
    def _space_arg(self, space: IndexSpace, grid: DeviceGrid) -> _lib.sb_space:
        cache = self.__dict__.setdefault("_space_cache", {})
        key = (tuple(space.lo), tuple(space.hi))
        a = cache.get(key)
        if a is None:
            if len(cache) > 256:
                cache.clear()
            a = cache[key] = _local(space, grid)
        return a

    def _launch_arg(self, params: LaunchParams, flags: int = 0) -> _lib.sb_launch:
        cache = self.__dict__.setdefault("_launch_cache", {})
        key = (params, flags | self.extra_flags)
        a = cache.get(key)
        if a is None:
            a = cache[key] = _lib.launch_of(params, flags | self.extra_flags)
        return a


class Laplacian7(DeviceKernel):
    """K1 — ``_update_rows`` (stencil.py:31-39): dst = C0*b + C1*(sum of 6 neighbours)."""

    site_id = "laplacian3d"
    space_kind = LAP7_SPACE
    # best of the CUDA-graph sweep at 64^3 (profiles/r01/v12_sweep_c1_graph.log)
    default_params = LaunchParams(64, 8, 2)

    def __init__(self, dst: DeviceGrid, src: DeviceGrid, c0: float, c1: float):
        if src.ghost < 1:
            raise UsageError("7-point stencil needs ghost width >= 1")
        if dst.lower != src.lower or dst.extents != src.extents:
            raise UsageError("dst and src must cover the same box")
        self.dst, self.src, self.c0, self.c1 = dst, src, float(c0), float(c1)
        self._abi = (dst.abi(), src.abi())

    def full_space(self) -> IndexSpace:
        return _interior_space(self.src)

    def launch(self, space: IndexSpace, params: LaunchParams, stream=None) -> None:
        _lib.call("sb_lap7", self._abi[0], self._abi[1], self._space_arg(space, self.src), self.c0, self.c1,
                  self._launch_arg(params), stream_ptr(stream))

    def iterate(self, a: DeviceGrid, b: DeviceGrid, space: IndexSpace, iters: int,
                params: LaunchParams | None = None, stream=None) -> DeviceGrid:
        """``iters`` Jacobi sweeps a -> b -> a ... in one persistent launch
        (``sb_lap7_iterate``); returns the grid holding the result."""
        if a.extents != b.extents or a.lower != b.lower:
            raise UsageError("a and b must cover the same box")
        _lib.init_current_device()
        _lib.call("sb_lap7_iterate", a.abi(), b.abi(), _local(space, a), self.c0, self.c1, int(iters),
                  _lib.launch_of(params or self.default_params, self.extra_flags), stream_ptr(stream))
        return b if iters % 2 else a


class FourthOrderAll(DeviceKernel):
    """K2 — all ten 4th-order outputs of a box (config 2): Dx Dy Dz Dxx Dyy Dzz Dxy Dxz Dyz Lap4."""

    site_id = "d4_all"
    space_kind = D4_ALL_SPACE
    # best of the full launch-space sweep at 256^3 on B200 (profiles/r01/v2_sweep_c2.jsonl)
    default_params = LaunchParams(32, 4, 4, 2)

    def __init__(self, outs: list[DeviceGrid], src: DeviceGrid, k: D4Constants):
        if len(outs) != _lib.SB_N_D4_OUT:
            raise UsageError("need 10 output grids")
        if src.ghost < 2:
            raise UsageError("4th-order stencils need ghost width >= 2")
        self.outs, self.src, self.k = list(outs), src, k
        self._out_abi = (_lib.sb_array * 10)(*[o.abi() for o in self.outs])

    def full_space(self) -> IndexSpace:
        return _interior_space(self.src)

    def launch(self, space: IndexSpace, params: LaunchParams, stream=None) -> None:
        if not hasattr(self, "_src_abi"):
            self._src_abi, self._k_abi = self.src.abi(), _lib.d4_constants(self.k)
        _lib.call("sb_d4_all", self._out_abi, self._src_abi, self._space_arg(space, self.src), self._k_abi,
                  self._launch_arg(params), stream_ptr(stream))

    def run_host(self, host_in_ptr: int, host_out_ptrs: list[int], params: LaunchParams | None = None,
                 chunk: int = 32) -> None:
        """Whole-box sweep from/to host memory (pinned for overlap): the
        ghosted input goes up, the box is swept and the ten outputs come back
        z chunk by z chunk on three streams, so the uploads, the sweeps and the
        downloads of different chunks overlap.  Ordered after the current
        stream's prior work; the current stream waits for the last download."""
        import torch
        p = params or self.default_params
        if not hasattr(self, "_streams"):
            self._streams = tuple(torch.cuda.Stream() for _ in range(3))
            self._staging = self.src.staging_buffer(True)
        up, cmp, down = self._streams
        cur = torch.cuda.current_stream()
        for s in self._streams:
            s.wait_stream(cur)
        cmp.wait_stream(down)     # outputs of a previous call are fully downloaded
        up.wait_stream(cmp)       # and its sweeps are done reading the input
        g = self.src.ghost
        lo = self.src.lower
        nx, ny, nz = self.src.extents
        have = 0
        for z0 in range(0, nz, chunk):
            z1 = min(nz, z0 + chunk)
            need = z1 + 2 * g                       # ghosted planes [0, z1 + 2g) feed planes < z1
            self.src.upload_planes_staged(host_in_ptr, self._staging, True, have, need, up)
            have = need
            ev = torch.cuda.Event()
            ev.record(up)
            cmp.wait_event(ev)
            space = IndexSpace((lo[0], lo[1], lo[2] + z0), (lo[0] + nx, lo[1] + ny, lo[2] + z1))
            self.launch(space, p, cmp)
            ev = torch.cuda.Event()
            ev.record(cmp)
            down.wait_event(ev)
            for o, ptr in zip(self.outs, host_out_ptrs):
                o.download_planes_to_ptr(ptr, False, z0, z1, down)
        cur.wait_stream(down)


class SecondOrderAll(FourthOrderAll):
    """K2' — the ten outputs with the 2nd-order centred operators
    (constants: inputs.D2Constants)."""

    site_id = "d2_all"

    def launch(self, space: IndexSpace, params: LaunchParams, stream=None) -> None:
        if not hasattr(self, "_src_abi"):
            self._src_abi, self._k_abi = self.src.abi(), _lib.d4_constants(self.k)
        _lib.call("sb_d2_all", self._out_abi, self._src_abi, self._space_arg(space, self.src), self._k_abi,
                  self._launch_arg(params), stream_ptr(stream))


class Laplacian4(DeviceKernel):
    """K3 — 4th-order Laplacian of one box; see :class:`LevelLaplacian4` for levels."""

    site_id = "lap4"
    space_kind = D4_SPACE
    default_params = LaunchParams(32, 4, 128, 2)

    def __init__(self, dst: DeviceGrid, src: DeviceGrid, k: D4Constants):
        if src.ghost < 2:
            raise UsageError("4th-order stencils need ghost width >= 2")
        self.dst, self.src, self.k = dst, src, k

    def full_space(self) -> IndexSpace:
        return _interior_space(self.src)

    def launch(self, space: IndexSpace, params: LaunchParams, stream=None) -> None:
        job = _lib.sb_box_job(self.dst.abi(), self.src.abi(), _local(space, self.src))
        _lib.call("sb_lap4_boxes", C.byref(job), 1, _lib.d4_constants(self.k),
                  _lib.launch_of(params, self.extra_flags), stream_ptr(stream))


def _clip(box: IndexSpace, space) -> IndexSpace | None:
    lo = tuple(max(a, b) for a, b in zip(box.lo, space.lo))
    hi = tuple(min(a, b) for a, b in zip(box.hi, space.hi))
    return None if any(h <= l for l, h in zip(lo, hi)) else IndexSpace(lo, hi)


def _array_of(owner, ctype, jobs):
    """The ctypes array of a (cached) job list, built once per list."""
    cache = owner.__dict__.setdefault("_array_cache", {})
    a = cache.get(id(jobs))
    if a is None or a[0] is not jobs:
        a = cache[id(jobs)] = (jobs, (ctype * len(jobs))(*jobs))
    return a[1]


class _LevelKernel(DeviceKernel):
    """A kernel over every box of a refinement level in ONE launch through
    the device box table (blockIdx -> (box, tile); up to SB_MAX_BOXES boxes
    travel in the launch parameters, larger levels use a table the library
    builds on the first launch of a shape and caches).  ``launch`` sweeps each
    box's interior (clipped to ``space`` when one is given, level
    coordinates); ``__call__(piece)`` sweeps the part of ``piece`` inside
    each box — so the reference's execute_plan/run_static can drive it."""

    def _boxes(self):
        raise NotImplementedError

    def _job(self, i: int, space: IndexSpace):
        raise NotImplementedError

    def full_space(self) -> IndexSpace:
        grids = [b[0] for b in self._boxes()]
        lo = tuple(min(g.lower[d] for g in grids) for d in range(3))
        hi = tuple(max(g.lower[d] + g.extents[d] for g in grids) for d in range(3))
        return IndexSpace(lo, hi)

    def _jobs(self, space):
        jobs = []
        for i, (grid, _) in enumerate(self._boxes()):
            box = _interior_space(grid)
            if space is not None:
                box = _clip(box, space)
                if box is None:
                    continue
            jobs.append(self._job(i, box))
        return jobs

    def launch(self, space: IndexSpace | None, params: LaunchParams, stream=None) -> None:
        cache = self.__dict__.setdefault("_jobs_cache", {})
        key = None if space is None else (tuple(space.lo), tuple(space.hi))
        jobs = cache.get(key)
        if jobs is None:
            if len(cache) > 256:
                cache.clear()
                self.__dict__.pop("_array_cache", None)
            jobs = cache[key] = self._jobs(space)
        if jobs:
            self._run(jobs, params, stream)

    def __call__(self, piece: IndexSpace) -> None:
        self.launch(piece, self.default_params)


class LevelLaplacian4(_LevelKernel):
    """K3 over a whole refinement level (config 4): every box in ONE launch."""

    site_id = "lap4_level"
    space_kind = D4_SPACE
    # best of the sweep on the config-4 level (profiles/r01/v2_sweep_c4.jsonl)
    default_params = LaunchParams(32, 4, 128, 2)

    def __init__(self, dsts: list[DeviceGrid], srcs: list[DeviceGrid], k: D4Constants):
        if len(dsts) != len(srcs) or not srcs:
            raise UsageError("need one dst per src box")
        for s in srcs:
            if s.ghost < 2:
                raise UsageError("4th-order stencils need ghost width >= 2")
        self.dsts, self.srcs, self.k = list(dsts), list(srcs), k

    def _boxes(self):
        return [(s, d) for s, d in zip(self.srcs, self.dsts)]

    def _job(self, i, box):
        s, d = self.srcs[i], self.dsts[i]
        return _lib.sb_box_job(d.abi(), s.abi(), _local(box, s))

    def _run(self, jobs, params, stream) -> None:
        arr = _array_of(self, _lib.sb_box_job, jobs)
        _lib.call("sb_lap4_boxes", arr, len(jobs), _lib.d4_constants(self.k), self._launch_arg(params),
                  stream_ptr(stream))


class LevelFourthOrderAll(_LevelKernel):
    """K2 over a level: the ten 4th-order outputs of every box in one launch
    (``sb_d4_all_boxes``; ``order=2`` selects the 2nd-order set)."""

    site_id = "d4_all_level"
    space_kind = D4_ALL_SPACE
    default_params = LaunchParams(32, 4, 4, 2)

    def __init__(self, outs: list[list[DeviceGrid]], srcs: list[DeviceGrid], k: D4Constants, order: int = 4):
        if len(outs) != len(srcs) or not srcs or any(len(o) != _lib.SB_N_D4_OUT for o in outs):
            raise UsageError("need ten output grids per src box")
        if order not in (2, 4):
            raise UsageError("order must be 2 or 4")
        for s in srcs:
            if s.ghost < 2:
                raise UsageError("the stencils need ghost width >= 2")
        self.outs, self.srcs, self.k, self.order = [list(o) for o in outs], list(srcs), k, order

    def _boxes(self):
        return [(s, o) for s, o in zip(self.srcs, self.outs)]

    def _job(self, i, box):
        s = self.srcs[i]
        j = _lib.sb_d4_all_job()
        for a, o in enumerate(self.outs[i]):
            j.out[a] = o.abi()
        j.src = s.abi()
        j.space = _local(box, s)
        return j

    def _run(self, jobs, params, stream) -> None:
        arr = _array_of(self, _lib.sb_d4_all_job, jobs)
        _lib.call("sb_d4_all_boxes" if self.order == 4 else "sb_d2_all_boxes", arr, len(jobs),
                  _lib.d4_constants(self.k), self._launch_arg(params), stream_ptr(stream))


class LevelRK4Stage(_LevelKernel):
    """K5 over a level: one classical RK4 stage (1..4) of the wave equation
    on every box in one launch (``sb_rk4_stage_boxes``).  ``fields[i]`` is
    box i's dict of grids phi_s, pi_s, phi0, pi0, acc_phi, acc_pi, phi_out,
    pi_out (phi_s ghosts filled beforehand, e.g. by LevelGhostSync)."""

    site_id = "rk4_level"
    space_kind = RK4_SPACE
    idempotent = False   # stages 2-3 update the RK accumulators in place
    default_params = LaunchParams(64, 4, 16, 1)
    NAMES = ("phi_s", "pi_s", "phi0", "pi0", "acc_phi", "acc_pi", "phi_out", "pi_out")

    def __init__(self, stage: int, fields: list[dict], c: WaveConstants):
        if stage not in (1, 2, 3, 4):
            raise UsageError("stage must be 1..4")
        if not fields:
            raise UsageError("need at least one box")
        self.stage, self.fields, self.c = stage, list(fields), c

    def _boxes(self):
        return [(f["phi_s"], f) for f in self.fields]

    def _job(self, i, box):
        f = self.fields[i]
        j = _lib.sb_rk4_box_job()
        j.f = _lib.sb_rk4_fields(*[f[n].abi() for n in self.NAMES])
        j.space = _local(box, f["phi_s"])
        return j

    def _run(self, jobs, params, stream) -> None:
        arr = _array_of(self, _lib.sb_rk4_box_job, jobs)
        c = _lib.sb_rk4_constants(_lib.d4_constants(self.c.lap), self.c.half_dt, self.c.dt, self.c.dt6)
        _lib.call("sb_rk4_stage_boxes", self.stage, arr, len(jobs), c, _lib.launch_of(params, self.extra_flags),
                  stream_ptr(stream))


class LevelGhostSync:
    """F1 — fill every box's ghost zone from the interiors of the other boxes
    of its level (schedule: level.ghost_schedule), all copies of a chunk of
    up to SB_MAX_COPY_JOBS regions in one launch."""

    def __init__(self, grids: list[DeviceGrid], boxes=None):
        from .level import Box, ghost_schedule
        if not grids:
            raise UsageError("need at least one grid")
        g = min(d.ghost for d in grids)
        if boxes is None:
            boxes = [Box(d.lower, tuple(l + e - 1 for l, e in zip(d.lower, d.extents))) for d in grids]
        self.grids = list(grids)
        self.schedule = ghost_schedule(list(boxes), g)
        jobs = []
        for c in self.schedule:
            dst, src = self.grids[c.dst], self.grids[c.src]
            j = _lib.sb_copy_job()
            j.dst, j.src = dst.abi(), src.abi()
            for d in range(3):
                j.dst_lo[d] = c.region.lo[d] - dst.lower[d]
                j.src_lo[d] = c.region.lo[d] - src.lower[d]
                j.ext[d] = c.region.hi[d] - c.region.lo[d] + 1
            jobs.append(j)
        self._jobs = jobs

    def points(self) -> int:
        return sum(c.region.volume() for c in self.schedule)

    def __call__(self, stream=None) -> None:
        for i in range(0, len(self._jobs), _lib.SB_MAX_COPY_JOBS):
            chunk = self._jobs[i:i + _lib.SB_MAX_COPY_JOBS]
            arr = (_lib.sb_copy_job * len(chunk))(*chunk)
            _lib.call("sb_copy_regions", arr, len(chunk), stream_ptr(stream))


class PeriodicGhosts:
    """K4 — periodic refill of a grid's ghost shell."""

    def __init__(self, grid: DeviceGrid):
        self.grid = grid

    def __call__(self, stream=None) -> None:
        _lib.call("sb_ghost_periodic", self.grid.abi(), stream_ptr(stream))


class WaveRK4:
    """One classical RK4 step of d/dt(phi, pi) = (pi, Lap4 phi) on a periodic
    box.  ``schedule``:

    * ``"lap_pairs"`` (default) — K5b, two launches per step with the
      stages fused in pairs (temporal blocking) and only the stage
      Laplacians L1, L2 stored between them (10 array passes);
    * ``"pairs"`` — K5b storing phi3, pi3 and the two RK accumulators
      between the launches (14 array passes);
    * ``"stages"`` — K5, four stage launches (32 passes);
    * ``"stages_unfused"`` — four stage launches each preceded by the
      stand-alone K4 periodic ghost refill.

    Every schedule gives the same bits.  The fused schedules refresh the
    periodic ghost shells of the phi (and, for pairs, pi) they produce, so
    after :meth:`fill_ghosts` of the initial state no ghost pass runs."""

    site_id = "wave_rk4"
    SCHEDULES = ("pairs", "lap_pairs", "stages", "stages_unfused")

    def __init__(self, n: int, ghost: int, c: WaveConstants, device=None, schedule: str = "lap_pairs"):
        if schedule not in self.SCHEDULES:
            raise UsageError(f"unknown RK4 schedule {schedule!r}")
        self.n, self.g, self.c = n, ghost, c
        self.schedule = schedule
        mk = lambda: DeviceGrid((n, n, n), ghost, device)
        self.phi0, self.pi0 = mk(), mk()
        self.phi_a, self.pi_a, self.phi_b, self.pi_b = mk(), mk(), mk(), mk()
        self.acc_phi, self.acc_pi = mk(), mk()
        # best of the sweeps at 384^3: pairs profiles/r01/v9_c3_lap_pairs_ab.log,
        # stages profiles/r01/v4_c3_rk2_ab.log
        self.params = LaunchParams(32, 4, 64, 1) if "pairs" in schedule else LaunchParams(64, 4, 16, 1)

    @property
    def fused_ghosts(self) -> bool:
        return self.schedule != "stages_unfused"

    def launch_space(self) -> LaunchSpace:
        return RK4_SPACE

    def _consts(self) -> _lib.sb_rk4_constants:
        return _lib.sb_rk4_constants(_lib.d4_constants(self.c.lap), self.c.half_dt, self.c.dt, self.c.dt6)

    def fill_ghosts(self, grid: DeviceGrid, stream=None) -> None:
        _lib.call("sb_ghost_periodic", grid.abi(), stream_ptr(stream))

    def _fields(self, phi_s, pi_s, phi_out, pi_out) -> _lib.sb_rk4_fields:
        return _lib.sb_rk4_fields(phi_s.abi(), pi_s.abi(), self.phi0.abi(), self.pi0.abi(), self.acc_phi.abi(),
                                  self.acc_pi.abi(), phi_out.abi(), pi_out.abi())

    def _whole(self):
        n = self.n
        return _lib.space((0, 0, 0), (n, n, n))

    def stage(self, s: int, phi_s: DeviceGrid, pi_s: DeviceGrid, phi_out: DeviceGrid, pi_out: DeviceGrid,
              params: LaunchParams, stream=None) -> None:
        if not self.fused_ghosts:
            self.fill_ghosts(phi_s, stream)
        f = self._fields(phi_s, pi_s, phi_out, pi_out)
        flags = _lib.SB_LAUNCH_PERIODIC_GHOSTS if self.fused_ghosts else 0
        _lib.call("sb_rk4_stage", s, C.byref(f), self._whole(), self._consts(), _lib.launch_of(params, flags),
                  stream_ptr(stream))

    def pair(self, k: int, phi_s: DeviceGrid, pi_s: DeviceGrid, phi_out: DeviceGrid, pi_out: DeviceGrid,
             params: LaunchParams, stream=None) -> None:
        f = self._fields(phi_s, pi_s, phi_out, pi_out)
        _lib.call("sb_rk4_pair", k, C.byref(f), self._whole(), self._consts(),
                  _lib.launch_of(params, _lib.SB_LAUNCH_PERIODIC_GHOSTS), stream_ptr(stream))

    def step(self, params: LaunchParams | None = None, stream=None) -> tuple[DeviceGrid, DeviceGrid]:
        """One RK4 step from (phi0, pi0) (ghost shells filled); returns the grids
        holding the new state."""
        p = params or self.params
        if self.schedule == "pairs":
            self.pair(1, self.phi0, self.pi0, self.phi_a, self.pi_a, p, stream)
            self.pair(2, self.phi_a, self.pi_a, self.phi_b, self.pi_b, p, stream)
            return self.phi_b, self.pi_b
        if self.schedule == "lap_pairs":
            # phi_a / pi_a hold L1 / L2 between the two launches
            self.pair(3, self.phi0, self.pi0, self.phi_a, self.pi_a, p, stream)
            self.pair(4, self.phi_a, self.pi_a, self.phi_b, self.pi_b, p, stream)
            return self.phi_b, self.pi_b
        self.stage(1, self.phi0, self.pi0, self.phi_a, self.pi_a, p, stream)
        self.stage(2, self.phi_a, self.pi_a, self.phi_b, self.pi_b, p, stream)
        self.stage(3, self.phi_b, self.pi_b, self.phi_a, self.pi_a, p, stream)
        self.stage(4, self.phi_a, self.pi_a, self.phi_b, self.pi_b, p, stream)
        return self.phi_b, self.pi_b

    def advance(self, params: LaunchParams | None = None, stream=None) -> None:
        """Step and make the new state the start of the next step."""
        phi, pi = self.step(params, stream)
        if not self.fused_ghosts:
            self.fill_ghosts(phi, stream)
        if "pairs" not in self.schedule:
            self.fill_ghosts(pi, stream)     # pi's ghosts are only refreshed by the pair schedules
        self.phi0, self.phi_b = phi, self.phi0
        self.pi0, self.pi_b = pi, self.pi0


class Rhs24(DeviceKernel):
    """K6 — config-5 fused 24-variable right-hand side."""

    site_id = "rhs24"
    # the CTA shape is fixed (8 x 4 columns, one warp per field / output =
    # 768 threads, written here as a 32 x 24 scalar tile); only z_chunk is tuned
    space_kind = LaunchSpace(kind="rhs24", tile_xs=(32,), tile_ys=(24,), points=(1,), max_threads_scalar=768)
    default_params = LaunchParams(32, 24, 192, 1)   # profiles/r01/v2_sweep_c5.jsonl

    def __init__(self, ins: list[DeviceGrid], outs: list[DeviceGrid], k: D4Constants, poly: PolyTable):
        if len(ins) != N_VARS or len(outs) != N_VARS:
            raise UsageError("need 24 input and 24 output grids")
        for g in ins:
            if g.ghost < 2:
                raise UsageError("4th-order stencils need ghost width >= 2")
        self.ins, self.outs, self.k = list(ins), list(outs), k
        self._coef = np.ascontiguousarray(poly.coef, dtype=np.float64).reshape(N_VARS * N_TERMS)
        self._p = np.ascontiguousarray(poly.p, dtype=np.int32).reshape(-1)
        self._q = np.ascontiguousarray(poly.q, dtype=np.int32).reshape(-1)
        self._in = (_lib.sb_array * N_VARS)(*[g.abi() for g in self.ins])
        self._out = (_lib.sb_array * N_VARS)(*[g.abi() for g in self.outs])

    def full_space(self) -> IndexSpace:
        return _interior_space(self.ins[0])

    def launch(self, space: IndexSpace, params: LaunchParams, stream=None) -> None:
        poly = _lib.sb_poly(self._coef.ctypes.data, self._p.ctypes.data, self._q.ctypes.data)
        _lib.call("sb_rhs24", self._in, self._out, _local(space, self.ins[0]), _lib.d4_constants(self.k), poly,
                  _lib.launch_of(params, self.extra_flags), stream_ptr(stream))
