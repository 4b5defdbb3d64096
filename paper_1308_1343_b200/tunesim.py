"""Tuner simulation on synthetic cost surfaces (the reference's ``tune-sim``,
cli.py:212-226, and acceptance criterion 8, test_acceptance.py:199-214).

Wall-clock timings are replaced by a deterministic cost over the parameter
vector so the tuner's behaviour can be asserted: a convex bowl in log2 tile
sizes, a multiplicative cliff once a tile outgrows the modelled cache, a
penalty for an unfavourable thread split, and a far-away decoy basin slightly
worse than the optimum (pure hill climbing from the wrong side stays there;
random restarts with the excursion-abort rule get out).  ``PlanSpace``
surfaces use ``ExecParams``; ``LaunchSpace`` surfaces use ``LaunchParams``
(tile_x, tile_y, z_chunk), the device tuner's space.
"""
from __future__ import annotations

import math
import statistics
from dataclasses import dataclass, field, replace

from .tuner import ExecParams, LaunchParams, LoopSetup, PlanSpace, TopologyConfig, Tuner


def _bowl(tiles, centre) -> float:
    return sum((math.log2(t) - math.log2(c)) ** 2 for t, c in zip(tiles, centre))


@dataclass(frozen=True)
class BowlSurface:
    """Cost model over ExecParams (PlanSpace) or LaunchParams (LaunchSpace)."""

    opt: tuple[int, ...] = (32, 16, 8)
    decoy: tuple[int, ...] = (4, 2, 64)
    weight: float = 0.3
    decoy_depth: float = 1.2
    decoy_weight: float = 0.7
    cliff_volume: int = 16384
    cliff_factor: float = 3.0
    split_penalty: float = 0.5

    def _tiles(self, p) -> tuple[int, ...]:
        if isinstance(p, LaunchParams):
            return (p.tile_x, p.tile_y, p.z_chunk)
        return tuple(p.tile_size)

    def _split_ok(self, p) -> bool:
        if isinstance(p, LaunchParams):
            return p.points_per_thread == 2
        return tuple(p.coarse_split) == tuple(sorted(p.coarse_split))

    def cost(self, p) -> float:
        tiles = self._tiles(p)
        main = 1.0 + self.weight * _bowl(tiles, self.opt)
        if math.prod(tiles) > self.cliff_volume:
            main *= self.cliff_factor
        decoy = self.decoy_depth + self.decoy_weight * _bowl(tiles, self.decoy)
        return min(main, decoy) + (0.0 if self._split_ok(p) else self.split_penalty)


@dataclass
class SeedResult:
    seed: int
    best_cost: float
    evals_to_target: int | None
    total_cost: float


@dataclass
class SimReport:
    optimum: float
    evals: int
    results: list[SeedResult] = field(default_factory=list)

    @property
    def converged(self) -> int:
        return sum(r.evals_to_target is not None for r in self.results)

    @property
    def median_evals_to_target(self) -> float | None:
        hit = [r.evals_to_target for r in self.results if r.evals_to_target is not None]
        return statistics.median(hit) if hit else None

    def csv(self) -> str:
        rows = ["seed,best_cost,evals_to_within_10pct,total_cost"]
        rows += [f"{r.seed},{r.best_cost:.6f},{r.evals_to_target},{r.total_cost:.6f}" for r in self.results]
        return "\n".join(rows) + "\n"


def simulate(seeds: int, evals: int, topo: TopologyConfig, setup: LoopSetup, surface: BowlSurface,
             space=None, target: float = 1.10) -> SimReport:
    """Run the tuner ``evals`` times per seed against ``surface``; a seed
    converges when the tuner's current best is within ``target`` x the
    optimum over the whole space."""
    sp = space if space is not None else PlanSpace()
    optimum = min(surface.cost(p) for p in sp.enumerate(setup, topo))
    report = SimReport(optimum, evals)
    for seed in range(seeds):
        tuner = Tuner(replace(topo, rng_seed=seed), space=sp)
        reach, total = None, 0.0
        for e in range(1, evals + 1):
            p = tuner.next_params(setup)
            c = surface.cost(p)
            total += c
            tuner.record_timing(setup, p, c)
            best = tuner.best(setup)[0]
            if reach is None and best is not None and surface.cost(best) <= target * optimum:
                reach = e
        best = tuner.best(setup)[0]
        report.results.append(SeedResult(seed, surface.cost(best) if best is not None else math.inf, reach, total))
    return report


def plan_case(topo: TopologyConfig | None = None) -> tuple[TopologyConfig, LoopSetup, BowlSurface, PlanSpace]:
    """The criterion-8 setting: a 128^3 loop, 4 coarse threads, W = 4."""
    topo = topo or TopologyConfig(n_coarse_threads=4, lane_width=4)
    setup = LoopSetup("synthetic", (128, 128, 128), n_coarse_threads=topo.n_coarse_threads)
    return topo, setup, BowlSurface(), PlanSpace()


def launch_case(topo: TopologyConfig | None = None):
    """The device launch space of the config-2 kernel on a 256^3 box, optimum
    at 32 x 4 columns / z-chunk 4 / two points per thread, decoy at 128 x 1 / 64."""
    from .kernels import D4_ALL_SPACE
    topo = topo or TopologyConfig()
    setup = LoopSetup("synthetic_launch", (256, 256, 256))
    surf = BowlSurface(opt=(32, 4, 4), decoy=(128, 1, 64), cliff_volume=1 << 30)
    return topo, setup, surf, D4_ALL_SPACE
