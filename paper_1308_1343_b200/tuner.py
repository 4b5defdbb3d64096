"""Run-time loop auto-tuner: random-restart hill climbing, per loop setup.

Host-side mirror of the reference's LoopControl tuner
(``pkg/src/stencilrt/tuner.py``).  The optimiser state machine behaves like
the reference's (``tuner.py:356-487``): per-setup RNG seeded from
``"{seed}:{site}:{extents}"`` (:387), the first execution of a setup is a
discarded warm-up (:444-448), each setting keeps a median of its last 5
samples (:31, :449-451), the climb recentres on every new best (:402-407),
at a local optimum it jumps to a random setting with probability
``p_restart`` (:418-425), and an excursion sample worse than
``abort_factor`` x best returns to the best at once (:398-400, :458-463).

What changes for the B200 is the parameter space the machine walks.  A
space object supplies ``initial``/``neighbors``/``random``/``enumerate``:

* :class:`PlanSpace` — the reference's CPU split space (coarse split, tile,
  fine split, lane width; ``tuner.py:114-346``), kept for the per-piece
  compatibility path of ``traverse.execute_plan``;
* :class:`LaunchSpace` — the device space: CTA tile (x, y) and z chunk of
  the z-streaming sm_100a kernels (north_star (d)), with the hardware
  invariants (tile_x in {32, 64, 128}, threads and shared memory per CTA).

Best settings can be persisted per (kernel, box shape, GPU) in a small JSON
cache (:class:`TuningCache`), the tuner persistence the paper lists as
future work.
"""
from __future__ import annotations

import json
import math
import os
import random
import statistics
from collections import deque
from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Protocol

from .errors import UsageError

MEDIAN_WINDOW = 5


def default_lane_width() -> int:
    """SIMD width W of the reference (vlanes.py:36-37: env LANE_WIDTH, default 4)."""
    return int(os.environ.get("LANE_WIDTH", "4"))


@dataclass(frozen=True)
class TopologyConfig:
    """Hardware description plus tuner constants (reference tuner.py:34-75),
    extended with the device facts the launch space needs."""

    cache_size_bytes: int = 262144
    cache_line_bytes: int = 64
    n_coarse_threads: int = 1
    n_fine_threads: int = 1
    lane_width: int = field(default_factory=default_lane_width)
    p_restart: float = 0.05
    abort_factor: float = 1.5
    rng_seed: int = 12345
    # device keys (B200 defaults; refreshed from the device when available)
    sm_count: int = 148
    smem_per_block: int = 232448
    l2_bytes: int = 132644864

    _INT_KEYS = ("cache_size_bytes", "cache_line_bytes", "n_coarse_threads", "n_fine_threads",
                 "lane_width", "rng_seed", "sm_count", "smem_per_block", "l2_bytes")
    _FLOAT_KEYS = ("p_restart", "abort_factor")

    @staticmethod
    def from_file(path: str | Path) -> "TopologyConfig":
        """``key = value`` lines with ``#`` comments (reference README format)."""
        vals: dict = {}
        for raw in Path(path).read_text().splitlines():
            line = raw.partition("#")[0].strip()
            if not line:
                continue
            key, sep, val = line.partition("=")
            if not sep:
                raise UsageError(f"malformed topology line: {raw!r}")
            key, val = key.strip(), val.strip()
            if key in TopologyConfig._INT_KEYS:
                vals[key] = int(val)
            elif key in TopologyConfig._FLOAT_KEYS:
                vals[key] = float(val)
            else:
                raise UsageError(f"unknown topology key: {key}")
        return TopologyConfig(**vals)

    @property
    def cache_line_elems(self) -> int:
        return max(1, self.cache_line_bytes // 8)

    def with_device(self) -> "TopologyConfig":
        """This topology with sm_count / shared memory / L2 of the current
        CUDA device (the run-time discovery the reference leaves to a file,
        tuner.py:38-40)."""
        from . import _lib
        info = _lib.sb_device_info()
        _lib.call("sb_get_device_info", _lib.C.byref(info))
        return replace(self, sm_count=int(info.sm_count), smem_per_block=int(info.smem_optin_bytes),
                       l2_bytes=int(info.l2_bytes))


@dataclass(frozen=True)
class LoopSetup:
    """Tuning identity (reference tuner.py:78-96); equal setups share history.

    Device setups add what changes the best launch shape on a GPU beside the
    extents: the row pitch of the swept source grid (``pitch``,
    elements; 0 = not a device setup) and the device's SM count
    (``sm_count``).  Both default to 0, so the reference's CPU setups, their
    RNG seeds and logs are unchanged; ``device_setup`` builds a device key."""

    site_id: str
    extents: tuple[int, ...]
    alignment: str = "vector"   # none | vector | cache_line
    n_coarse_threads: int = 1
    n_fine_threads: int = 1
    pitch: int = 0
    sm_count: int = 0

    def __post_init__(self) -> None:
        if any(e <= 0 for e in self.extents):
            raise UsageError(f"extents must be positive: {self.extents}")
        if self.alignment not in ("none", "vector", "cache_line"):
            raise UsageError(f"unknown alignment class {self.alignment!r}")

    @property
    def dim(self) -> int:
        return len(self.extents)


def _rng_key(seed: int, setup: LoopSetup) -> str:
    """Per-setup RNG stream key (reference tuner.py:387); device setups also
    key on pitch and SM count."""
    k = f"{seed}:{setup.site_id}:{setup.extents}"
    if setup.pitch or setup.sm_count:
        k += f":{setup.pitch}:{setup.sm_count}"
    return k


def device_setup(kernel, extents=None) -> LoopSetup:
    """The LoopSetup of a device kernel: site, extents (default: the kernel's
    full space), the row pitch of its swept source grid and the SM count of
    the current device."""
    import torch
    ext = tuple(extents) if extents is not None else kernel.full_space().extents
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return LoopSetup(kernel.site_id, ext, pitch=int(kernel.pitch_class()), sm_count=int(sms))


@dataclass(frozen=True)
class ExecParams:
    """The reference's CPU split parameters (tuner.py:99-111)."""

    coarse_split: tuple[int, ...]
    tile_size: tuple[int, ...]
    fine_split: tuple[int, ...]
    vector_width: int

    def flat(self) -> str:
        j = lambda t: "x".join(str(v) for v in t)
        return f"{j(self.coarse_split)}/{j(self.tile_size)}/{j(self.fine_split)}/w{self.vector_width}"


@dataclass(frozen=True)
class LaunchParams:
    """One point of the device space: CTA tile (x, y), z planes per CTA, and
    x points per thread (2 = one 16-byte pair, the device's SIMD width W)."""

    tile_x: int
    tile_y: int
    z_chunk: int
    points_per_thread: int = 2

    def flat(self) -> str:
        return f"{self.tile_x}x{self.tile_y}/z{self.z_chunk}/p{self.points_per_thread}"


class ParamSpace(Protocol):
    def initial(self, setup: LoopSetup, topo: TopologyConfig): ...
    def neighbors(self, p, setup: LoopSetup, topo: TopologyConfig) -> list: ...
    def random(self, setup: LoopSetup, topo: TopologyConfig, rng: random.Random): ...
    def enumerate(self, setup: LoopSetup, topo: TopologyConfig) -> list: ...
    def check(self, p, setup: LoopSetup, topo: TopologyConfig) -> None: ...


def _prod(xs) -> int:
    return math.prod(xs)


def _prime_factors_desc(n: int) -> list[int]:
    fs, f = [], 2
    while f * f <= n:
        while n % f == 0:
            fs.append(f)
            n //= f
        f += 1
    if n > 1:
        fs.append(n)
    return sorted(fs, reverse=True)


def _with(t: tuple, i: int, v: int) -> tuple:
    lst = list(t)
    lst[i] = v
    return tuple(lst)


# -- the reference's CPU plan space --------------------------------------------

class PlanSpace:
    """Coarse split x tile x fine split at a fixed lane width (tuner.py:114-346)."""

    @staticmethod
    def inner_unit(setup: LoopSetup, topo: TopologyConfig) -> int:
        w = topo.lane_width
        if setup.alignment == "cache_line":
            return math.lcm(topo.cache_line_elems, w)
        return w

    def check(self, p: ExecParams, setup: LoopSetup, topo: TopologyConfig) -> None:
        d = setup.dim
        if not (len(p.coarse_split) == len(p.tile_size) == len(p.fine_split) == d):
            raise UsageError("parameter vectors disagree with setup dimension")
        if _prod(p.coarse_split) != setup.n_coarse_threads:
            raise UsageError(f"coarse split {p.coarse_split} does not use {setup.n_coarse_threads} threads")
        if _prod(p.fine_split) != setup.n_fine_threads:
            raise UsageError(f"fine split {p.fine_split} does not use {setup.n_fine_threads} threads")
        if p.vector_width != topo.lane_width:
            raise UsageError(f"vector width {p.vector_width} != configured {topo.lane_width}")
        for axis, (t, e) in enumerate(zip(p.tile_size, setup.extents)):
            if not 1 <= t <= e:
                raise UsageError(f"tile size {t} out of range 1..{e} in dim {axis}")
        unit = self.inner_unit(setup, topo)
        if p.tile_size[0] % unit and p.tile_size[0] != setup.extents[0]:
            raise UsageError(f"innermost tile {p.tile_size[0]} neither multiple of {unit} "
                             f"nor whole extent {setup.extents[0]}")

    @staticmethod
    def factorizations(n: int, d: int) -> list[tuple[int, ...]]:
        if d == 1:
            return [(n,)]
        return [(a,) + rest for a in range(1, n + 1) if n % a == 0
                for rest in PlanSpace.factorizations(n // a, d - 1)]

    def _splits(self, threads: int, setup: LoopSetup) -> list[tuple[int, ...]]:
        every = self.factorizations(threads, setup.dim)
        fit = [c for c in every if all(ci <= ei for ci, ei in zip(c, setup.extents))]
        return fit if fit else every

    def _tiles(self, setup: LoopSetup, topo: TopologyConfig, axis: int) -> list[int]:
        e = setup.extents[axis]
        t = self.inner_unit(setup, topo) if axis == 0 else 1
        out = []
        while t < e:
            out.append(t)
            t *= 2
        return out + [e]

    def enumerate(self, setup: LoopSetup, topo: TopologyConfig) -> list[ExecParams]:
        coarse = self._splits(setup.n_coarse_threads, setup)
        fine = self._splits(setup.n_fine_threads, setup)
        tiles: list[tuple] = [()]
        for axis in range(setup.dim):
            tiles = [t + (v,) for t in tiles for v in self._tiles(setup, topo, axis)]
        return [ExecParams(c, t, f, topo.lane_width) for t in tiles for c in coarse for f in fine]

    def random(self, setup: LoopSetup, topo: TopologyConfig, rng: random.Random) -> ExecParams:
        coarse = self._splits(setup.n_coarse_threads, setup)
        fine = self._splits(setup.n_fine_threads, setup)
        tile = tuple(rng.choice(self._tiles(setup, topo, a)) for a in range(setup.dim))
        return ExecParams(rng.choice(coarse), tile, rng.choice(fine), topo.lane_width)

    @staticmethod
    def _greedy(threads: int, ext: tuple[int, ...]) -> list[int]:
        """Give each prime factor (largest first) to the outer dimension with the
        most room left; the innermost dimension is tried last."""
        d = len(ext)
        split = [1] * d
        order = list(range(d - 1, 0, -1)) + [0] if d > 1 else [0]
        for f in _prime_factors_desc(threads):
            best, room = None, 0.0
            for i in order:
                r = ext[i] / (split[i] * f)
                if r >= 1 and r > room:
                    best, room = i, r
            if best is None:
                best = max(range(d), key=lambda i: ext[i] / split[i])
            split[best] *= f
        return split

    @staticmethod
    def _snap_inner(t: int, extent: int, unit: int, floor: int) -> int:
        if extent < unit:
            return extent
        t = max(min(t, extent), min(floor, extent))
        if t % unit and t != extent:
            t = max(unit, t - t % unit)
        return t

    def initial(self, setup: LoopSetup, topo: TopologyConfig) -> ExecParams:
        ext, w = setup.extents, topo.lane_width
        unit = self.inner_unit(setup, topo)
        coarse = self._greedy(setup.n_coarse_threads, ext)
        tile = [max(1, -(-e // c)) for e, c in zip(ext, coarse)]
        tile[0] = self._snap_inner(tile[0], ext[0], unit, 2 * w)
        budget = max(1, topo.cache_size_bytes // 16)     # half the cache, in doubles
        while _prod(tile) > budget:
            outer = [(tile[i], i) for i in range(1, setup.dim) if tile[i] > 1]
            if outer:
                i = max(outer)[1]
                tile[i] = max(1, tile[i] // 2)
            elif tile[0] > max(unit, 2 * w) and tile[0] % (2 * unit) == 0:
                tile[0] //= 2
            else:
                break
        tile[0] = self._snap_inner(tile[0], ext[0], unit, 2 * w)
        fine = self._greedy(setup.n_fine_threads, tuple(tile))
        return ExecParams(tuple(coarse), tuple(tile), tuple(fine), w)

    def _moves(self, split: tuple[int, ...], setup: LoopSetup) -> list[tuple[int, ...]]:
        out = []
        for i in range(len(split)):
            for j in range(len(split)):
                if i == j or split[j] == 1:
                    continue
                f = min(_prime_factors_desc(split[j]))
                if split[i] * f <= setup.extents[i]:
                    out.append(_with(_with(split, j, split[j] // f), i, split[i] * f))
        return out

    def neighbors(self, p: ExecParams, setup: LoopSetup, topo: TopologyConfig) -> list[ExecParams]:
        unit = self.inner_unit(setup, topo)
        cand: list[ExecParams] = []
        for i in range(setup.dim):
            floor = unit if i == 0 else 1
            e, t = setup.extents[i], p.tile_size[i]
            if t < e:
                cand.append(replace(p, tile_size=_with(p.tile_size, i, min(2 * t, e))))
            down = max(floor, (t // 2) // floor * floor)
            if down < t:
                cand.append(replace(p, tile_size=_with(p.tile_size, i, down)))
        cand += [replace(p, coarse_split=s) for s in self._moves(p.coarse_split, setup)]
        cand += [replace(p, fine_split=s) for s in self._moves(p.fine_split, setup)]
        return _valid_unique(self, p, cand, setup, topo)


def _valid_unique(space, p, cand, setup, topo) -> list:
    seen, out = {p}, []
    for q in cand:
        if q in seen:
            continue
        try:
            space.check(q, setup, topo)
        except UsageError:
            continue
        seen.add(q)
        out.append(q)
    return out


# Module-level forms of the reference's plan-space functions, same names and
# signatures (tuner.py:130, 190, 212, 221, 297), over the CPU plan space;
# pinned against the reference by tests/golden/tuner_golden.json.
_PLAN_SPACE = PlanSpace()


def check_params(p: ExecParams, setup: LoopSetup, topo: TopologyConfig) -> None:
    """Raise UsageError unless p satisfies every invariant for this setup."""
    _PLAN_SPACE.check(p, setup, topo)


def enumerate_valid_params(setup: LoopSetup, topo: TopologyConfig) -> list[ExecParams]:
    return _PLAN_SPACE.enumerate(setup, topo)


def random_params(setup: LoopSetup, topo: TopologyConfig, rng: random.Random) -> ExecParams:
    return _PLAN_SPACE.random(setup, topo, rng)


def params_initial(setup: LoopSetup, topo: TopologyConfig) -> ExecParams:
    return _PLAN_SPACE.initial(setup, topo)


def neighbors(p: ExecParams, setup: LoopSetup, topo: TopologyConfig) -> list[ExecParams]:
    return _PLAN_SPACE.neighbors(p, setup, topo)


# -- the device launch space ---------------------------------------------------

@dataclass(frozen=True)
class LaunchSpace:
    """CTA tile x/y and z chunk of a z-streaming sm_100a stencil kernel.

    Threads per CTA are (tile_x / points_per_thread) * tile_y, a multiple of 32
    bounded by ``max_threads_pair`` / ``max_threads_scalar`` (the register
    budget of the kernel variant); ``smem_bytes(tile_x, tile_y)`` is the
    shared memory a CTA needs."""

    kind: str = "d4"
    max_threads_pair: int = 512
    max_threads_scalar: int = 512
    points: tuple[int, ...] = (2, 1)
    radius: int = 2
    rx_buffer: bool = False     # d4_all keeps a double-buffered rx plane in smem
    stages: int = 4
    tile_xs: tuple[int, ...] = (32, 64, 128)
    tile_ys: tuple[int, ...] = (1, 2, 4, 8, 16, 32)
    z_min: int = 4              # smallest z chunk (powers of two from here, then the whole extent)

    def smem_bytes(self, tx: int, ty: int) -> int:
        w, h = tx + 2 * self.radius, ty + 2 * self.radius
        stage = -(-(w * h) // 16) * 16 * 8
        extra = 2 * h * tx * 8 if self.rx_buffer else 0
        return 128 + self.stages * stage + extra

    def _z_values(self, nz: int) -> list[int]:
        vals, z = [], self.z_min
        while z < nz:
            vals.append(z)
            z *= 2
        return vals + [nz]

    def check(self, p: LaunchParams, setup: LoopSetup, topo: TopologyConfig) -> None:
        if p.tile_x not in self.tile_xs:
            raise UsageError(f"tile_x {p.tile_x} not in {self.tile_xs}")
        if p.tile_y < 1 or p.z_chunk < 1:
            raise UsageError("tile_y and z_chunk must be positive")
        if p.tile_y not in self.tile_ys:
            # e.g. rhs24's CTA shape is fixed: other tile heights would be the same kernel
            raise UsageError(f"tile_y {p.tile_y} not in {self.tile_ys}")
        if p.points_per_thread not in self.points:
            raise UsageError(f"points_per_thread {p.points_per_thread} not in {self.points}")
        cap = self.max_threads_pair if p.points_per_thread == 2 else self.max_threads_scalar
        threads = (p.tile_x // p.points_per_thread) * p.tile_y
        if threads % 32 or threads > cap:
            raise UsageError(f"{threads} threads per CTA not a multiple of 32 in 32..{cap}")
        if p.tile_y + 2 * self.radius > 256:
            raise UsageError("tile_y exceeds the TMA box limit")
        if self.smem_bytes(p.tile_x, p.tile_y) > topo.smem_per_block:
            raise UsageError("tile needs more shared memory than a CTA may use")
        nz = setup.extents[2] if setup.dim >= 3 else 1
        if p.z_chunk > max(nz, 1):
            raise UsageError(f"z_chunk {p.z_chunk} exceeds extent {nz}")

    def enumerate(self, setup: LoopSetup, topo: TopologyConfig) -> list[LaunchParams]:
        nz = setup.extents[2] if setup.dim >= 3 else 1
        out = []
        for pp in self.points:
            for tx in self.tile_xs:
                for ty in self.tile_ys:
                    for zc in self._z_values(nz):
                        p = LaunchParams(tx, ty, zc, pp)
                        try:
                            self.check(p, setup, topo)
                        except UsageError:
                            continue
                        out.append(p)
        return out

    def random(self, setup: LoopSetup, topo: TopologyConfig, rng: random.Random) -> LaunchParams:
        return rng.choice(self.enumerate(setup, topo))

    def initial(self, setup: LoopSetup, topo: TopologyConfig) -> LaunchParams:
        """64-wide tiles (a row of doubles is 512 bytes), the first listed
        points-per-thread, tile_y up to 8, z chunk chosen so the grid covers
        the SMs >= 4 times."""
        valid = self.enumerate(setup, topo)
        if not valid:
            raise UsageError(f"no valid launch parameters for {setup}")
        nx, ny = setup.extents[0], setup.extents[1] if setup.dim >= 2 else 1
        nz = setup.extents[2] if setup.dim >= 3 else 1
        pp = next((q for q in self.points if any(p.points_per_thread == q for p in valid)), valid[0].points_per_thread)
        mine = [p for p in valid if p.points_per_thread == pp]
        tx = 64 if any(p.tile_x == 64 for p in mine) else mine[0].tile_x
        ty = max((p.tile_y for p in mine if p.tile_x == tx and p.tile_y <= 8), default=mine[0].tile_y)
        cols = -(-nx // tx) * -(-ny // ty)
        zc = nz
        for cand in sorted({p.z_chunk for p in mine}, reverse=True):
            zc = cand
            if cols * -(-nz // cand) >= 4 * topo.sm_count:
                break
        p = LaunchParams(tx, ty, zc, pp)
        self.check(p, setup, topo)
        return p

    def neighbors(self, p: LaunchParams, setup: LoopSetup, topo: TopologyConfig) -> list[LaunchParams]:
        nz = setup.extents[2] if setup.dim >= 3 else 1
        cand = []
        for f in ("tile_x", "tile_y", "z_chunk"):
            v = getattr(p, f)
            cand.append(replace(p, **{f: v * 2}))
            if v > 1:
                cand.append(replace(p, **{f: v // 2}))
        if p.z_chunk != nz:
            cand.append(replace(p, z_chunk=nz))
        for q in self.points:
            if q != p.points_per_thread:
                # same threads per CTA: trade tile_y against points per thread
                cand.append(replace(p, points_per_thread=q))
                cand.append(replace(p, points_per_thread=q, tile_y=max(1, p.tile_y * p.points_per_thread // q)))
        return _valid_unique(self, p, cand, setup, topo)


# -- the optimiser state machine -----------------------------------------------

_INITIAL, _CLIMBING, _EXCURSION = "initial", "climbing", "excursion"


@dataclass
class _State:
    rng: random.Random
    space: object
    current: object
    phase: str = _INITIAL
    center: object = None
    pending: list = field(default_factory=list)
    best_params: object = None
    best_time: float = float("inf")
    samples: dict = field(default_factory=dict)
    warmed_up: bool = False
    last_elapsed: float | None = None
    executions: int = 0


class Tuner:
    """Per-setup optimisation state plus a CSV-able execution log.

    Single coordinating thread (reference tuner.py:371-377): ``next_params``
    and ``record_timing`` are called between executions only.
    """

    def __init__(self, topo: TopologyConfig, space=None, cache: "TuningCache | None" = None):
        self.topo = topo
        self.default_space = space if space is not None else PlanSpace()
        self.cache = cache
        self._states: dict[LoopSetup, _State] = {}
        self.log: list[dict] = []

    def _state(self, setup: LoopSetup, space=None) -> _State:
        st = self._states.get(setup)
        if st is None:
            sp = space if space is not None else self.default_space
            rng = random.Random(_rng_key(self.topo.rng_seed, setup))
            start = sp.initial(setup, self.topo)
            if self.cache is not None:
                cached = self.cache.get(setup, sp)
                if cached is not None:
                    start = cached
            st = _State(rng=rng, space=sp, current=start)
            self._states[setup] = st
        return st

    def prime(self, setup: LoopSetup, space, start) -> None:
        """Start a not-yet-seen setup's climb at `start` (e.g. a kernel's
        measured default) instead of the space's heuristic."""
        if setup in self._states:
            return
        space.check(start, setup, self.topo)
        rng = random.Random(_rng_key(self.topo.rng_seed, setup))
        self._states[setup] = _State(rng=rng, space=space, current=start)

    def space_of(self, setup: LoopSetup):
        return self._states[setup].space if setup in self._states else None

    def next_params(self, setup: LoopSetup, space=None):
        """Advance the state machine; return the setting to execute next."""
        st = self._state(setup, space)
        if st.best_params is None:
            return st.current
        if st.phase == _EXCURSION and self.should_abort_excursion(setup, st.last_elapsed):
            st.pending.clear()
            return self._settle(st)
        if st.center != st.best_params:
            st.phase, st.center = _CLIMBING, st.best_params
            st.pending = st.space.neighbors(st.best_params, setup, self.topo)
            st.rng.shuffle(st.pending)
        if st.pending:
            st.current = st.pending.pop()
            return st.current
        if st.phase == _EXCURSION:
            return self._settle(st)
        if st.rng.random() < self.topo.p_restart:
            jump = st.space.random(setup, self.topo, st.rng)
            st.phase, st.center = _EXCURSION, jump
            st.pending = st.space.neighbors(jump, setup, self.topo)
            st.rng.shuffle(st.pending)
            st.current = jump
            return jump
        st.current = st.best_params
        return st.current

    @staticmethod
    def _settle(st: _State):
        st.phase, st.center, st.current = _CLIMBING, st.best_params, st.best_params
        return st.current

    def record_timing(self, setup: LoopSetup, params, elapsed: float) -> None:
        if not (math.isfinite(elapsed) and elapsed >= 0):
            raise UsageError(f"rejecting non-finite or negative timing {elapsed!r}")
        st = self._states.get(setup)
        if st is None:
            raise UsageError("record_timing before next_params for this setup")
        st.executions += 1
        if not st.warmed_up:
            st.warmed_up = True
            self._log(setup, st, params, elapsed, "warmup")
            return
        window = st.samples.setdefault(params, deque(maxlen=MEDIAN_WINDOW))
        window.append(elapsed)
        med = statistics.median(window)
        if med < st.best_time:
            st.best_time, st.best_params = med, params
            if self.cache is not None:
                self.cache.put(setup, st.space, params, med)
        st.last_elapsed = elapsed
        self._log(setup, st, params, elapsed, st.phase)

    def should_abort_excursion(self, setup: LoopSetup, latest: float | None) -> bool:
        st = self._states[setup]
        if latest is None or st.best_time == float("inf"):
            return False
        return latest > self.topo.abort_factor * st.best_time

    def best(self, setup: LoopSetup):
        st = self._states[setup]
        return st.best_params, st.best_time

    def phase(self, setup: LoopSetup) -> str:
        return self._states[setup].phase

    def _log(self, setup, st, params, elapsed, phase) -> None:
        self.log.append({"setup_id": setup.site_id, "params": params.flat(),
                         "elapsed_ns": int(elapsed * 1e9), "phase": phase,
                         "is_best": int(params == st.best_params)})

    def write_log(self, path: str | Path) -> None:
        rows = ["setup_id,params,elapsed_ns,phase,is_best"]
        rows += [f"{r['setup_id']},{r['params']},{r['elapsed_ns']},{r['phase']},{r['is_best']}" for r in self.log]
        Path(path).write_text("\n".join(rows) + "\n")


# -- persistence ----------------------------------------------------------------

class TuningCache:
    """Best device launch parameters per (site, extents, GPU), kept in JSON."""

    def __init__(self, path: str | Path, device_key: str = "B200"):
        self.path = Path(path)
        self.device_key = device_key
        self._d: dict = {}
        if self.path.exists():
            try:
                self._d = json.loads(self.path.read_text())
            except (OSError, ValueError):
                self._d = {}

    def _key(self, setup: LoopSetup) -> str:
        k = f"{self.device_key}|{setup.site_id}|{'x'.join(map(str, setup.extents))}"
        if setup.pitch or setup.sm_count:
            k += f"|sy{setup.pitch}|sm{setup.sm_count}"
        return k

    def get(self, setup: LoopSetup, space):
        if not isinstance(space, LaunchSpace):
            return None
        e = self._d.get(self._key(setup))
        if not e:
            return None
        p = LaunchParams(*e["params"])
        try:
            space.check(p, setup, TopologyConfig())
        except UsageError:
            return None
        return p

    def put(self, setup: LoopSetup, space, params, seconds: float) -> None:
        if not isinstance(params, LaunchParams):
            return
        self._d[self._key(setup)] = {"params": [params.tile_x, params.tile_y, params.z_chunk,
                                                params.points_per_thread], "seconds": seconds}
        tmp = self.path.with_suffix(".tmp")
        tmp.write_text(json.dumps(self._d, indent=1, sort_keys=True))
        os.replace(tmp, self.path)
