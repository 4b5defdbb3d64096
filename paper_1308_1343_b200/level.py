"""Refinement levels as box lists, and the device box table.

The reference represents a level as a ``BBoxSet`` (bboxset.py) and hands the
loop iterator one box at a time through ``index_space_from_bbox``
(traverse.py:59-65).  The hot path only needs the level's canonical disjoint
decomposition, ``BBoxSet.from_bboxes(...).difference(...).to_bboxes()``
(bboxset.py:259-294, 352-353, 313-317); the set algebra itself is host-side
integer logic and out of scope.

:func:`boxes_of` accepts any object with ``to_bboxes()`` (the reference's
``BBoxSet``), a list of reference ``BBox`` objects, or a list of :class:`Box`.
Strided (coarsened) levels — ``BBoxSet.coarsen`` (bboxset.py:387-406), whose
boxes hold the points ``offset + k * stride`` — are swept in compact lattice
coordinates (:func:`compact_level`): a grid function on a strided box is
stored one value per lattice point, the stencil's neighbours at +-stride are
the compact neighbours at +-1, and the spacing is ``h * stride``; the kernels
are unchanged.  ``as_box`` keeps rejecting strided boxes exactly like the
reference's ``index_space_from_bbox`` (traverse.py:63-64).
:func:`box_difference` produces, for the single-box-minus-box case config 4
uses, the same sorted slab decomposition the reference returns (outermost
dimension split first; verified against the reference in
tests/golden/make_golden.py).
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import UsageError


@dataclass(frozen=True)
class _Pt:
    coords: tuple[int, ...]


@dataclass(frozen=True)
class Box:
    """Inclusive, unit-stride box, innermost dimension first (lattice.py:104)."""

    lo: tuple[int, ...]
    hi: tuple[int, ...]

    @staticmethod
    def empty(dim: int) -> "Box":
        return Box((0,) * dim, (-1,) * dim)

    @property
    def is_empty(self) -> bool:
        return any(h < l for l, h in zip(self.lo, self.hi))

    @property
    def dim(self) -> int:
        return len(self.lo)

    # duck-typing with the reference's BBox
    @property
    def lower(self):
        return _Pt(self.lo)

    @property
    def upper(self):
        return _Pt(self.hi)

    @property
    def stride(self):
        return _Pt((1,) * self.dim)

    @property
    def extents(self) -> tuple[int, ...]:
        return tuple(max(0, h - l + 1) for l, h in zip(self.lo, self.hi))

    def volume(self) -> int:
        v = 1
        for e in self.extents:
            v *= e
        return v


def as_box(b) -> Box:
    if isinstance(b, Box):
        return b
    lower = tuple(b.lower.coords)
    upper = tuple(b.upper.coords)
    if b.is_empty:
        return Box.empty(len(lower))
    if any(s != 1 for s in b.stride.steps):
        raise UsageError("only unit-stride boxes can be swept")
    return Box(lower, upper)


def boxes_of(level) -> list[Box]:
    """Canonical box list of a level: ``level.to_bboxes()`` or an iterable."""
    raw = level.to_bboxes() if hasattr(level, "to_bboxes") else list(level)
    return [b for b in (as_box(x) for x in raw) if not b.is_empty]


@dataclass(frozen=True)
class Lattice:
    """The sub-lattice ``offset + k * stride`` of a strided level and the map
    between its fine coordinates and compact coordinates k."""

    stride: tuple[int, ...]
    offset: tuple[int, ...]

    def to_compact(self, p) -> tuple[int, ...]:
        out = []
        for x, o, st in zip(p, self.offset, self.stride):
            if (x - o) % st:
                raise UsageError(f"point {tuple(p)} is not on the lattice {self}")
            out.append((x - o) // st)
        return tuple(out)

    def to_fine(self, k) -> tuple[int, ...]:
        return tuple(o + c * st for c, o, st in zip(k, self.offset, self.stride))


def compact_level(level) -> tuple[list[Box], Lattice]:
    """The boxes of a (possibly strided) level in compact lattice coordinates
    and the lattice: ``level.to_bboxes()`` (or a list of reference BBoxes
    sharing one stride and anchor, bboxset.py:240-263).  Unit-stride levels
    come back unchanged with a unit lattice."""
    raw = [b for b in (level.to_bboxes() if hasattr(level, "to_bboxes") else list(level)) if not b.is_empty]
    if not raw:
        return [], Lattice((1, 1, 1), (0, 0, 0))
    stride = tuple(getattr(raw[0].stride, "steps", getattr(raw[0].stride, "coords", None)))
    if hasattr(level, "offset"):
        offset = tuple(o % st for o, st in zip(level.offset.coords, stride))
    else:
        offset = tuple(l % st for l, st in zip(raw[0].lower.coords, stride))
    lat = Lattice(stride, offset)
    boxes = []
    for b in raw:
        st = tuple(getattr(b.stride, "steps", getattr(b.stride, "coords", None)))
        if st != stride:
            raise UsageError("a level's boxes must share one stride")
        boxes.append(Box(lat.to_compact(b.lower.coords), lat.to_compact(b.upper.coords)))
    return boxes, lat


def box_difference(a: Box, b: Box) -> list[Box]:
    """Disjoint boxes covering a \\ b, split outermost dimension first, sorted by
    (lower, upper) compared outermost-first — the order of the reference's
    ``to_bboxes`` for this case."""
    if a.is_empty:
        return []
    lo = [max(x, y) for x, y in zip(a.lo, b.lo)]
    hi = [min(x, y) for x, y in zip(a.hi, b.hi)]
    if b.is_empty or any(h < l for l, h in zip(lo, hi)):
        return [a]
    pieces = []
    cur_lo, cur_hi = list(a.lo), list(a.hi)
    for d in reversed(range(a.dim)):            # outermost first
        if cur_lo[d] < lo[d]:
            p_hi = list(cur_hi)
            p_hi[d] = lo[d] - 1
            pieces.append(Box(tuple(cur_lo), tuple(p_hi)))
        if hi[d] < cur_hi[d]:
            p_lo = list(cur_lo)
            p_lo[d] = hi[d] + 1
            pieces.append(Box(tuple(p_lo), tuple(cur_hi)))
        cur_lo[d], cur_hi[d] = lo[d], hi[d]
    key = lambda bx: (tuple(reversed(bx.lo)), tuple(reversed(bx.hi)))
    return sorted(pieces, key=key)


def intersect(a: Box, b: Box) -> Box:
    lo = tuple(max(x, y) for x, y in zip(a.lo, b.lo))
    hi = tuple(min(x, y) for x, y in zip(a.hi, b.hi))
    return Box(lo, hi) if all(l <= h for l, h in zip(lo, hi)) else Box.empty(a.dim)


def expand(b: Box, g: int) -> Box:
    """Grow a box by g points on every face (the reference's BBox expand,
    lattice.py:156-191, at unit stride)."""
    return Box(tuple(v - g for v in b.lo), tuple(v + g for v in b.hi))


@dataclass(frozen=True)
class GhostCopy:
    """Ghost points of box `dst` that lie in the interior of box `src`."""

    dst: int
    src: int
    region: Box


def ghost_schedule(boxes: list[Box], g: int) -> list[GhostCopy]:
    """The inter-box ghost-fill schedule of a level:
    for every ordered pair of distinct boxes, expand(dst, g) ∩ src.  Boxes of
    a level are disjoint, so each such region lies in dst's ghost zone and in
    src's interior; ghost points outside every box (the level boundary) are
    not touched."""
    out = []
    for i, a in enumerate(boxes):
        grown = expand(a, g)
        for j, b in enumerate(boxes):
            if i == j:
                continue
            r = intersect(grown, b)
            if not r.is_empty:
                out.append(GhostCopy(i, j, r))
    return out
