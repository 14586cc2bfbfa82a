"""Integer boxes and fields over boxes (oracle data model; TEST INFRASTRUCTURE ONLY).

Index tuples are in ARRAY order (i3, i2, i1): the last entry is x1, the fastest index.
Boxes are half-open: cells lo <= i < hi.  A Field is a dense fp64 array over a box; its
element [0,0,0] is the global cell `box.lo`.

Paper references: cells, i = (x - h/2)/h, PAPER.md:66-68 (§2); regions as grown / clipped
boxes, PAPER.md:187-210 (§4).
"""
from __future__ import annotations

import itertools

import numpy as np


class Box:
    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        self.lo = tuple(int(v) for v in lo)
        self.hi = tuple(int(v) for v in hi)

    # -- predicates / sizes ------------------------------------------------------------
    @property
    def empty(self) -> bool:
        return any(h <= l for l, h in zip(self.lo, self.hi))

    @property
    def shape(self):
        return tuple(max(0, h - l) for l, h in zip(self.lo, self.hi))

    @property
    def volume(self) -> int:
        s = self.shape
        return s[0] * s[1] * s[2]

    def contains(self, other: "Box") -> bool:
        if other.empty:
            return True
        return all(a <= b for a, b in zip(self.lo, other.lo)) and all(
            a >= b for a, b in zip(self.hi, other.hi))

    def contains_cell(self, i) -> bool:
        return all(l <= v < h for l, v, h in zip(self.lo, i, self.hi))

    # -- algebra -----------------------------------------------------------------------
    def grow(self, j: int) -> "Box":
        """grow(b, j): every face moved out by j cells ("grown by J_k h_k")."""
        return Box([l - j for l in self.lo], [h + j for h in self.hi])

    def intersect(self, o: "Box") -> "Box":
        return Box([max(a, b) for a, b in zip(self.lo, o.lo)],
                   [min(a, b) for a, b in zip(self.hi, o.hi)])

    def refine(self) -> "Box":
        """The 8^n children of every cell (N_k = 2 N_{k-1})."""
        return Box([2 * l for l in self.lo], [2 * h for h in self.hi])

    def coarsen_inner(self) -> "Box":
        """Largest coarse box whose refinement lies inside self (all 8 children inside)."""
        return Box([-((-l) // 2) for l in self.lo], [h // 2 for h in self.hi])

    def cells(self):
        return itertools.product(*[range(l, h) for l, h in zip(self.lo, self.hi)])

    def __eq__(self, o):
        if not isinstance(o, Box):
            return NotImplemented
        if self.empty and o.empty:
            return True
        return self.lo == o.lo and self.hi == o.hi

    def __hash__(self):
        return hash((self.lo, self.hi))

    def __repr__(self):
        return f"Box({self.lo}, {self.hi})"


class Field:
    """fp64 values over a storage box; cells never written hold NaN (sentinel)."""

    __slots__ = ("box", "a")

    def __init__(self, box: Box, fill: float = np.nan, array=None):
        self.box = box
        if array is not None:
            assert array.shape == box.shape
            self.a = np.ascontiguousarray(array, dtype=np.float64)
        else:
            self.a = np.full(box.shape, fill, dtype=np.float64)

    def _sl(self, b: Box):
        assert self.box.contains(b), f"{b} outside storage {self.box}"
        return tuple(slice(l - s, h - s) for l, h, s in zip(b.lo, b.hi, self.box.lo))

    def __getitem__(self, b: Box) -> np.ndarray:
        return self.a[self._sl(b)]

    def __setitem__(self, b: Box, v):
        self.a[self._sl(b)] = v

    def copy(self) -> "Field":
        return Field(self.box, array=self.a.copy())

    def at(self, i) -> float:
        return float(self.a[tuple(v - s for v, s in zip(i, self.box.lo))])
