"""Exact-integer closed forms for the lattice workloads (test-side pins; no fp64 path).

A lattice workload is "cube index a in prod [0, n_d) plus one of T type offsets
o_t". Scaling every coordinate by an integer D makes the offsets integers O_t and,
for the configs here, D*rmin an integer R. Then the pair test of Eq. filter_cond
(PAPER.md:263-270), |c_i - c_j| < rmin (strict; reading R1), becomes the
integer test |D*delta + O_t - O_s|^2 < R^2 over integer cube offsets delta, and

    nnz = sum_{s,t} sum_{delta: test} prod_d max(0, n_d - |delta_d|)

counts every ordered pair exactly (each cube a with a+delta inside the grid).
These numbers do not touch the oracle's floating-point code; they pin it.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Lattice:
    n: tuple          # cubes per dimension
    offsets: tuple    # integer type offsets O_t (scaled by D)
    D: int            # scale
    R: int            # D * rmin (integer)

    @property
    def dim(self):
        return len(self.n)

    def _deltas(self):
        m = self.R // self.D + 2
        return itertools.product(range(-m, m + 1), repeat=self.dim)

    def nnz(self) -> int:
        total = 0
        R2 = self.R * self.R
        for Os in self.offsets:
            for Ot in self.offsets:
                for dl in self._deltas():
                    d2 = sum((self.D * dl[k] + Ot[k] - Os[k]) ** 2 for k in range(self.dim))
                    if d2 < R2:
                        total += math.prod(max(0, self.n[k] - abs(dl[k])) for k in range(self.dim))
        return total

    def interior(self, s: int):
        """(count, sorted exact squared distances (scaled by D^2)) of an interior row of type s."""
        R2 = self.R * self.R
        Os = self.offsets[s]
        d2s = []
        for Ot in self.offsets:
            for dl in self._deltas():
                d2 = sum((self.D * dl[k] + Ot[k] - Os[k]) ** 2 for k in range(self.dim))
                if d2 < R2:
                    d2s.append(d2)
        return len(d2s), sorted(d2s)

    def interior_hs(self, s: int) -> float:
        """Interior row sum, sum (rmin - |d|) over the exact neighbour set (math.fsum)."""
        _, d2s = self.interior(s)
        return math.fsum((self.R - math.sqrt(d2)) / self.D for d2 in d2s)


def quads(nx, ny):          # config 1: centroid (i+1/2, j+1/2), rmin 1.5
    return Lattice((nx, ny), ((1, 1),), 2, 3)


def hexes(nx, ny, nz, R=4):  # config 3: centroid (i,j,k)+1/2, rmin 2 -> R = 4 (D = 2)
    return Lattice((nx, ny, nz), ((1, 1, 1),), 2, R)


def tris_right(nx, ny, R=15):
    """Config 2 triangles ("right" diagonal): offsets (2/3,1/3) and (1/3,2/3); D = 6, rmin 2.5 -> R = 15."""
    return Lattice((nx, ny), ((4, 2), (2, 4)), 6, R)


def kuhn(nx, ny, nz, R=6):
    """Config 5 Kuhn tets: offset (2 e_s1 + e_s2 + (1,1,1))/4 for the 6 permutations; D = 4, rmin 1.5 -> R = 6."""
    offs = []
    for s in itertools.permutations(range(3)):
        o = [1, 1, 1]
        o[s[0]] += 2
        o[s[1]] += 1
        offs.append(tuple(o))
    return Lattice((nx, ny, nz), tuple(offs), 4, R)
