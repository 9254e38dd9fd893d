"""Device-resident BLR grid and reflector stores (HBM layout).

Layout: one FP64 pool per grid; cell (i, j) owns
  dense cell : b*b doubles, column-major, at off_u[c]
  low-rank   : U (b x cap) at off_u[c], V (b x cap) at off_v[c] = off_u[c] + b*cap
plus an int32 rank per cell and a uint8 kind map.  cap defaults to b, so no
update can overflow; smaller caps trade memory for an overflow check.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from .core import BlrMatrix, BlrStructure, LowRankBlock, is_lowrank


def _f(a: np.ndarray) -> np.ndarray:
    """column-major flat copy of a 2-D array"""
    return np.asarray(a, dtype=np.float64).ravel(order="F")


_POOL = None


def _host_parallel(fn, n: int, min_chunk: int = 64) -> None:
    """fn(lo, hi) over [0, n) in chunks on a host thread pool (numpy copies
    release the GIL); serial for small n."""
    global _POOL
    workers = min(32, os.cpu_count() or 1)
    if n <= min_chunk or workers == 1:
        fn(0, n)
        return
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=workers)
    step = max(min_chunk, -(-n // (4 * workers)))
    list(_POOL.map(lambda lo: fn(lo, min(n, lo + step)), range(0, n, step)))


class DeviceGrid:
    """p x q BLR grid resident on the GPU."""

    def __init__(self, m: int, n: int, b: int, lowrank: np.ndarray, cap: int | None = None,
                 min_lr_slab: int = 0):
        rt = _lib.runtime()
        self.m, self.n, self.b = m, n, b
        self.p, self.q = m // b, n // b
        self.cap = int(cap if cap is not None else b)
        kind = np.asarray(lowrank, dtype=bool)
        self.kind_host = kind.copy()
        lr_slab = max(2 * b * self.cap, min_lr_slab)
        sizes = np.where(kind.ravel(), lr_slab, b * b).astype(np.int64)
        off = np.zeros(self.p * self.q, dtype=np.int64)
        off[1:] = np.cumsum(sizes)[:-1]
        offv = np.where(kind.ravel(), off + b * self.cap, -1)
        self.pool_size = int(sizes.sum())
        dev = rt.dev
        self.kind = torch.from_numpy(kind.ravel().astype(np.uint8)).to(dev)
        self.rank = torch.from_numpy(np.where(kind.ravel(), 0, -1).astype(np.int32)).to(dev)
        self.off_u = torch.from_numpy(off).to(dev)
        self.off_v = torch.from_numpy(offv).to(dev)
        self.off_u_host, self.off_v_host = off, offv
        self.pool = torch.zeros(self.pool_size, dtype=torch.float64, device=dev)

    # -- ctypes view -----------------------------------------------------
    def cstruct(self) -> _lib.Grid:
        return _lib.Grid(self.p, self.q, self.b, self.cap, self.kind.data_ptr(), self.rank.data_ptr(),
                         self.pool.data_ptr(), self.off_u.data_ptr(), self.off_v.data_ptr())

    @property
    def structure(self) -> BlrStructure:
        return BlrStructure(self.m, self.n, self.b, self.kind_host.copy())

    def rank_map(self) -> np.ndarray:
        return self.rank.cpu().numpy().reshape(self.p, self.q).copy()

    def clone(self) -> "DeviceGrid":
        g = DeviceGrid.__new__(DeviceGrid)
        g.__dict__.update(self.__dict__)
        g.kind = self.kind.clone()
        g.rank = self.rank.clone()
        g.pool = self.pool.clone()
        g.kind_host = self.kind_host.copy()
        return g

    # -- host <-> device ----------------------------------------------------
    def _stage_offsets(self, ranks: np.ndarray) -> tuple[np.ndarray, int]:
        b = self.b
        kind = self.kind_host.ravel()
        sz = np.where(kind, 2 * b * np.maximum(ranks, 0), b * b).astype(np.int64)
        off = np.zeros_like(sz)
        off[1:] = np.cumsum(sz)[:-1]
        return off, int(sz.sum())

    def _pack(self, stage: torch.Tensor, offs: np.ndarray, to_grid: bool) -> None:
        lib = _lib.load()
        od = torch.from_numpy(offs).to(stage.device)
        g = self.cstruct()
        _lib.check(lib.blrqr_grid_pack(C.byref(g), stage.data_ptr(), od.data_ptr(), int(to_grid),
                                       _lib.stream_ptr()), "grid_pack")

    @classmethod
    def from_host(cls, a: BlrMatrix, cap: int | None = None, pinned: bool = True) -> "DeviceGrid":
        """Upload a host BlrMatrix: cells are packed column-major into the
        runtime's persistent pinned staging buffer by a host thread pool, sent
        with one H2D copy and scattered into the slabs by the pack kernel."""
        s = a.structure
        g = cls(s.m, s.n, s.b, s.admissible, cap)
        flat = [x for row in a.blocks for x in row]
        ranks = np.array([x.rank if is_lowrank(x) else -1 for x in flat], dtype=np.int32)
        if (ranks > g.cap).any():
            raise ValueError("input rank exceeds the slab capacity")
        offs, tot = g._stage_offsets(ranks)
        b = s.b
        rt = _lib.runtime()
        pin = rt.pinned(tot) if pinned else torch.empty(max(tot, 1), dtype=torch.float64)
        host = pin.numpy()

        def pack(lo, hi):
            for c in range(lo, hi):
                x, o = flat[c], int(offs[c])
                if ranks[c] >= 0:
                    r = int(ranks[c])
                    host[o:o + b * r].reshape(r, b)[...] = x.u.T
                    host[o + b * r:o + 2 * b * r].reshape(r, b)[...] = x.v.T
                else:
                    host[o:o + b * b].reshape(b, b)[...] = np.asarray(x).T

        _host_parallel(pack, len(flat))
        stage = torch.empty(max(tot, 1), dtype=torch.float64, device=g.pool.device)
        stage[:tot].copy_(pin[:tot], non_blocking=pinned)
        if pinned:
            rt.pinned_in_flight()
        g.rank.copy_(torch.from_numpy(ranks))
        g._pack(stage, offs, True)
        return g

    def to_host(self) -> BlrMatrix:
        """Download into a host BlrMatrix (pack kernel, one D2H copy into the
        pinned staging buffer, thread-parallel unpack into fresh arrays)."""
        rt = _lib.runtime()
        ranks = self.rank.cpu().numpy()
        offs, tot = self._stage_offsets(ranks)
        stage = torch.empty(max(tot, 1), dtype=torch.float64, device=self.pool.device)
        self._pack(stage, offs, False)
        pin = rt.pinned(tot)
        pin[:tot].copy_(stage[:tot])
        host = pin.numpy()
        b = self.b
        kind = self.kind_host.ravel()
        cells = [None] * (self.p * self.q)

        def unpack(lo, hi):
            for c in range(lo, hi):
                o = int(offs[c])
                if kind[c]:
                    r = int(ranks[c])
                    u = np.empty((b, r))
                    v = np.empty((b, r))
                    u[...] = host[o:o + b * r].reshape(r, b).T
                    v[...] = host[o + b * r:o + 2 * b * r].reshape(r, b).T
                    cells[c] = LowRankBlock(u, v)
                else:
                    d = np.empty((b, b))
                    d[...] = host[o:o + b * b].reshape(b, b).T
                    cells[c] = d

        _host_parallel(unpack, len(cells))
        blocks = [cells[i * self.q:(i + 1) * self.q] for i in range(self.p)]
        return BlrMatrix(self.structure, blocks)

    @classmethod
    def from_dense(cls, dense, b: int, admissible: np.ndarray, eps: float, fallback: float = 0.5,
                   cap: int | None = None, colmajor: bool = False) -> "DeviceGrid":
        """GPU dense_to_blr (core.py:227-259).  ``dense`` is a host ndarray or
        a CUDA tensor (row-major m x n; ``colmajor=True`` if its storage is
        already column-major, e.g. a symmetric matrix)."""
        rt = _lib.runtime()
        lib = rt.lib
        if isinstance(dense, np.ndarray):
            m, n = dense.shape
            dt = torch.from_numpy(np.ascontiguousarray(dense)).to(rt.dev)
        else:
            m, n = dense.shape
            dt = dense
        adm = np.asarray(admissible, dtype=bool)
        g = cls(m, n, b, adm, cap, min_lr_slab=b * b)
        # cap < fallback*b is allowed: a tile whose rank lands in (cap, fallback*b]
        # raises (rank-overflow status) instead of silently changing kind
        cm = dt if colmajor else dt.t().contiguous()  # column-major m x n, lda = m
        ws, per, nct = rt.workspace(b, g.cap)
        st = g.cstruct()
        _lib.check(lib.blrqr_dense_to_blr(cm.data_ptr(), m, C.byref(st), g.kind.data_ptr(), eps,
                                          fallback, ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(),
                                          _lib.stream_ptr()), "dense_to_blr")
        rt.harvest()
        g.kind_host = g.kind.cpu().numpy().astype(bool).reshape(g.p, g.q)
        del cm
        return g


class DeviceRefl:
    """Householder reflector store for the tiled / blocked methods."""

    def __init__(self, grid: DeviceGrid):
        b, p, q = grid.b, grid.p, grid.q
        kind = grid.kind_host
        y_off = np.full(p * q, -1, dtype=np.int64)
        t_off = np.full(p * q, -1, dtype=np.int64)
        o = 0
        for k in range(q):
            c = k * q + k
            y_off[c] = o; o += b * b
            t_off[c] = o; o += b * b
            for i in range(k + 1, p):
                c = i * q + k
                t_off[c] = o; o += b * b
                if not kind[i, k]:
                    y_off[c] = o; o += b * b
        dev = grid.pool.device
        self.grid = grid
        self.y_off_host, self.t_off_host = y_off, t_off
        self.y_off = torch.from_numpy(y_off).to(dev)
        self.t_off = torch.from_numpy(t_off).to(dev)
        self.yrank = torch.full((p * q,), -1, dtype=torch.int32, device=dev)
        self.pool = torch.zeros(o, dtype=torch.float64, device=dev)
        self.wpool = None
        self.wrank = None

    def enable_split_traps(self) -> None:
        """Allocate the per-cell w slots used by the split ApplyTrap tasks of
        the dynamic scheduler (2 slots of 2*b*cap doubles per cell)."""
        if self.wpool is None:
            g = self.grid
            self.wslot = 2 * g.b * g.cap
            # two slots per cell, by the parity of k (tasks.cuh w_index)
            self.wpool = torch.empty(2 * g.p * g.q * self.wslot, dtype=torch.float64, device=g.pool.device)
            self.wrank = torch.zeros(2 * g.p * g.q, dtype=torch.int32, device=g.pool.device)

    def cstruct(self) -> _lib.Refl:
        return _lib.Refl(self.pool.data_ptr(), self.y_off.data_ptr(), self.t_off.data_ptr(),
                         self.yrank.data_ptr(), self.wpool.data_ptr() if self.wpool is not None else None,
                         self.wrank.data_ptr() if self.wrank is not None else None,
                         getattr(self, "wslot", 0))

    def mat(self, off: int, rows: int, cols: int) -> np.ndarray:
        """Download a column-major rows x cols matrix at pool offset ``off``."""
        x = self.pool[off:off + rows * cols].cpu().numpy()
        return np.ascontiguousarray(x.reshape(cols, rows).T)
