"""Oracle BLR data model (test infrastructure only).

Restates core.py: a factor pair ``LR(u, v)`` means ``u @ v.T``
(core.py:31-66, rank = u.shape[1], rank 0 = structural zero), and a grid of
b x b cells with a fixed low-rank/dense kind map (core.py:90-189).  Dense
payloads are float64 ndarrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class LR:
    """u (rows x r) times v (cols x r) transposed (core.py:31-57)."""

    u: np.ndarray
    v: np.ndarray

    @property
    def rank(self) -> int:
        return self.u.shape[1]

    @property
    def rows(self) -> int:
        return self.u.shape[0]

    @property
    def cols(self) -> int:
        return self.v.shape[0]

    def dense(self) -> np.ndarray:  # core.py:53-56
        if self.rank == 0:
            return np.zeros((self.rows, self.cols))
        return self.u @ self.v.T


def is_lr(x) -> bool:
    return isinstance(x, LR)


def empty_lr(rows: int, cols: int) -> LR:
    return LR(np.zeros((rows, 0)), np.zeros((cols, 0)))


def zero_cell(b: int, lowrank: bool):
    """core.py:77-81: rank-0 factors for low-rank cells, dense zeros else."""
    return empty_lr(b, b) if lowrank else np.zeros((b, b))


def to_dense(x) -> np.ndarray:  # core.py:84-87
    return x.dense() if is_lr(x) else x


def weak_map(p: int, q: int) -> np.ndarray:  # core.py:123-128
    lr = np.ones((p, q), dtype=bool)
    d = min(p, q)
    lr[np.arange(d), np.arange(d)] = False
    return lr


class Grid:
    """p x q cells plus the low-rank kind map (core.py:90-189)."""

    def __init__(self, m: int, n: int, b: int, lowrank: np.ndarray, cells):
        if m % b or n % b:
            raise ValueError(f"block size {b} must divide {m} x {n}")
        self.m, self.n, self.b = m, n, b
        self.lowrank = np.asarray(lowrank, dtype=bool).copy()
        if self.lowrank.shape != (self.p, self.q):
            raise ValueError("kind map shape mismatch")
        d = min(self.p, self.q)
        if self.lowrank[np.arange(d), np.arange(d)].any():
            raise ValueError("diagonal blocks must be dense")
        self.cells = cells

    @property
    def p(self) -> int:
        return self.m // self.b

    @property
    def q(self) -> int:
        return self.n // self.b

    def __getitem__(self, ij):
        return self.cells[ij[0]][ij[1]]

    def __setitem__(self, ij, val):
        self.cells[ij[0]][ij[1]] = val

    def clone(self) -> "Grid":  # core.py:179-189
        cells = [
            [LR(c.u.copy(), c.v.copy()) if is_lr(c) else c.copy() for c in row]
            for row in self.cells
        ]
        return Grid(self.m, self.n, self.b, self.lowrank, cells)

    def dense(self) -> np.ndarray:  # core.py:192-201
        b = self.b
        out = np.empty((self.m, self.n))
        for i in range(self.p):
            for j in range(self.q):
                out[i * b:(i + 1) * b, j * b:(j + 1) * b] = to_dense(self[i, j])
        return out

    def rank_map(self) -> np.ndarray:
        """Rank per cell; -1 for dense cells."""
        r = np.full((self.p, self.q), -1, dtype=np.int64)
        for i in range(self.p):
            for j in range(self.q):
                if is_lr(self[i, j]):
                    r[i, j] = self[i, j].rank
        return r

    def max_rank(self) -> int:  # core.py:204-211
        rm = self.rank_map()
        return int(max(0, rm.max()))

    def nbytes(self) -> int:  # core.py:214-224
        e = 0
        for row in self.cells:
            for c in row:
                e += 2 * self.b * c.rank if is_lr(c) else self.b * self.b
        return 8 * e


def from_reference(a) -> Grid:
    """Convert a reference ``blrqr.BlrMatrix`` (tests only)."""
    s = a.structure
    cells = []
    for row in a.blocks:
        out = []
        for blk in row:
            if hasattr(blk, "u"):
                out.append(LR(np.array(blk.u), np.array(blk.v)))
            else:
                out.append(np.array(blk))
        cells.append(out)
    return Grid(s.m, s.n, s.b, s.admissible, cells)
