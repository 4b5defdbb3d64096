"""Multi-GPU sharding of a level's boxes.

The stencil sweep partitions into independent units — the boxes of a
level, each read and written only by its own kernel — so N GPUs run with
no data-path collective: each rank sweeps its share of the boxes (or of
the z planes of a box) and the only communication is measurement plumbing
(a barrier and the max-over-ranks time).  Halo exchange between z-slabs of
one box is the next step (§8(f) F4) and is not needed for this.
"""
from __future__ import annotations

from .level import Box


def split_z(box: Box, parts: int) -> list[Box]:
    """Cut a box into `parts` z-slabs of near-equal thickness."""
    z0, z1 = box.lo[2], box.hi[2] + 1
    parts = max(1, min(parts, z1 - z0))
    cuts = [z0 + (z1 - z0) * j // parts for j in range(parts)] + [z1]
    return [Box(box.lo[:2] + (cuts[j],), box.hi[:2] + (cuts[j + 1] - 1,)) for j in range(parts)]


def shard_boxes(boxes: list[Box], world: int, rank: int) -> list[Box]:
    """Deterministic balanced assignment of box pieces to ranks.

    Boxes are cut into z-slabs so that there are at least `world` pieces of
    comparable volume, then dealt largest-first to the least-loaded rank
    (ties -> lowest rank).  Every point of every box is owned by exactly one
    rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    total = sum(b.volume() for b in boxes)
    if total == 0:
        return []
    target = total / world
    pieces: list[Box] = []
    for b in boxes:
        parts = max(1, round(b.volume() / target)) if world > 1 else 1
        pieces.extend(split_z(b, parts))
    pieces.sort(key=lambda b: (-b.volume(), tuple(reversed(b.lo))))
    load = [0] * world
    owned: list[list[Box]] = [[] for _ in range(world)]
    for p in pieces:
        r = min(range(world), key=lambda i: (load[i], i))
        owned[r].append(p)
        load[r] += p.volume()
    return owned[rank]
