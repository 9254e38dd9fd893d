"""Low-rank arithmetic with the reference API (lowrank.py), computed on the GPU.

Every function keeps the reference's name, arguments, return types and
errors; the numerics run in libblrqr.so (rounded addition = fused QR/QR/core
GEMM/one-sided-Jacobi-SVD/truncation/back-transform per CTA; compression =
truncated column-pivoted QR per CTA).  The batched variants take many
operand pairs in one launch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import Block, LowRankBlock

__all__ = ["ToleranceConfig", "compress_rrqr", "compress_to_lowrank", "rounded_add", "rounded_add_batched",
           "compress_batched", "lr_add_into_dense", "lr_times_dense", "lr_times_lr", "NOISE_FLOOR"]

NOISE_FLOOR = 64 * np.finfo(float).eps  # lowrank.py:170


@dataclass(frozen=True)
class ToleranceConfig:
    """lowrank.py:30-41."""

    epsilon: float
    dense_fallback_fraction: float = 0.5

    def __post_init__(self):
        if not 0 < self.epsilon < 1:
            raise ValueError("epsilon must lie in (0, 1)")
        if not 0 < self.dense_fallback_fraction <= 1:
            raise ValueError("dense_fallback_fraction must lie in (0, 1]")


def _dev(x: np.ndarray) -> torch.Tensor:
    """column-major device copy (shape (cols, rows) row-major = x column-major)"""
    rt = _lib.runtime()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64).T)).to(rt.dev)


def _host(t: torch.Tensor, rows: int, cols: int) -> np.ndarray:
    return np.ascontiguousarray(t[: rows * cols].reshape(cols, rows).cpu().numpy().T) if rows * cols else \
        np.zeros((rows, cols))


def _ptrs(ts) -> torch.Tensor:
    rt = _lib.runtime()
    return torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=rt.dev)


def rounded_add_batched(pairs, cfg: ToleranceConfig) -> list[LowRankBlock]:
    """Rounded additions of many (a, bk) LowRankBlock pairs of equal shape."""
    if not pairs:
        return []
    rt = _lib.runtime()
    m, n = pairs[0][0].rows, pairs[0][0].cols
    for a, bk in pairs:
        if (a.rows, a.cols) != (bk.rows, bk.cols) or (a.rows, a.cols) != (m, n):
            raise ValueError("operands must have equal dimensions")
    cap = max(min(m, n, a.rank + bk.rank) for a, bk in pairs)
    cap = max(cap, 1)
    keep = []

    def up(x):
        t = _dev(x) if x.size else torch.zeros(1, dtype=torch.float64, device=rt.dev)
        keep.append(t)
        return t

    ua = [up(a.u) for a, _ in pairs]
    va = [up(a.v) for a, _ in pairs]
    ub = [up(bk.u) for _, bk in pairs]
    vb = [up(bk.v) for _, bk in pairs]
    ra = torch.tensor([a.rank for a, _ in pairs], dtype=torch.int32, device=rt.dev)
    rb = torch.tensor([bk.rank for _, bk in pairs], dtype=torch.int32, device=rt.dev)
    uo = [torch.empty(m * cap, dtype=torch.float64, device=rt.dev) for _ in pairs]
    vo = [torch.empty(n * cap, dtype=torch.float64, device=rt.dev) for _ in pairs]
    ro = torch.zeros(len(pairs), dtype=torch.int32, device=rt.dev)
    ws, per, nct = rt.workspace(max(m, n), cap)
    lib = rt.lib
    pa = [_ptrs(x) for x in (ua, va, ub, vb, uo, vo)]  # held until the launch is enqueued
    _lib.check(lib.blrqr_rounded_add_batched(
        len(pairs), m, n, pa[0].data_ptr(), pa[1].data_ptr(), ra.data_ptr(), pa[2].data_ptr(),
        pa[3].data_ptr(), rb.data_ptr(), pa[4].data_ptr(), pa[5].data_ptr(), ro.data_ptr(), cap,
        cfg.epsilon, ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
        "rounded_add")
    rt.harvest()
    ranks = ro.cpu().numpy()
    out = []
    for t, (a, bk) in enumerate(pairs):
        r = int(ranks[t])
        if a.rank == 0 and bk.rank == 0:  # lowrank.py:186-187
            out.append(LowRankBlock(a.u, a.v))
            continue
        out.append(LowRankBlock(_host(uo[t], m, r), _host(vo[t], n, r)))
    return out


def rounded_add(a: LowRankBlock, bk: LowRankBlock, cfg: ToleranceConfig) -> LowRankBlock:
    """Alg. 6 recompressed sum (lowrank.py:173-221)."""
    if (a.rows, a.cols) != (bk.rows, bk.cols):
        raise ValueError("operands must have equal dimensions")
    return rounded_add_batched([(a, bk)], cfg)[0]


def compress_batched(tiles, epsilon: float, max_rank: int) -> list:
    """Truncated RRQR of many equal-shape tiles: (u, v) or None (rank > max_rank)."""
    if not tiles:
        return []
    rt = _lib.runtime()
    m, n = tiles[0].shape
    k = min(m, n)
    a = [_dev(t) for t in tiles]
    uo = [torch.empty(m * k, dtype=torch.float64, device=rt.dev) for _ in tiles]
    vo = [torch.empty(n * k, dtype=torch.float64, device=rt.dev) for _ in tiles]
    ro = torch.zeros(len(tiles), dtype=torch.int32, device=rt.dev)
    ws, per, nct = rt.workspace(max(m, n), k)
    pa = [_ptrs(x) for x in (a, uo, vo)]
    _lib.check(rt.lib.blrqr_compress_batched(
        len(tiles), m, n, pa[0].data_ptr(), pa[1].data_ptr(), pa[2].data_ptr(), ro.data_ptr(), k,
        epsilon, max_rank, ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
        "compress")
    rt.harvest()
    out = []
    for t, r in enumerate(ro.cpu().numpy()):
        r = int(r)
        if r < 0:
            out.append(None)
        else:
            out.append((_host(uo[t], m, r), _host(vo[t], n, r)))
    return out


def compress_rrqr(a: np.ndarray, cfg: ToleranceConfig) -> Block:
    """lowrank.py:138-150: LowRankBlock, or ``a`` itself when the rank would
    exceed dense_fallback_fraction * min(m, n)."""
    m, n = a.shape
    out = compress_batched([a], cfg.epsilon, int(cfg.dense_fallback_fraction * min(m, n)))[0]
    return a if out is None else LowRankBlock(*out)


def compress_to_lowrank(a: np.ndarray, epsilon: float) -> LowRankBlock:
    """lowrank.py:153-158 (no dense fallback)."""
    out = compress_batched([a], epsilon, min(a.shape))[0]
    assert out is not None
    return LowRankBlock(*out)


def _product(op, m, k, n, u=None, v=None, r=0, d=None, u2=None, v2=None, r2=0, out_rows=0, out_cols=0):
    rt = _lib.runtime()
    ou = torch.zeros(max(out_rows, 1), dtype=torch.float64, device=rt.dev)
    ov = torch.zeros(max(out_cols, 1), dtype=torch.float64, device=rt.dev)
    orank = torch.zeros(1, dtype=torch.int32, device=rt.dev)
    ws, per, _ = rt.workspace(max(m, k, n), max(r, r2, 1))
    _lib.check(rt.lib.blrqr_lr_product(op, m, k, n, _lib.ptr(u), _lib.ptr(v), r, _lib.ptr(d), _lib.ptr(u2),
                                       _lib.ptr(v2), r2, ou.data_ptr(), ov.data_ptr(), orank.data_ptr(), ws, per,
                                       rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
               "lr_product")
    rt.harvest()
    return ou, ov, int(orank.item())


def lr_add_into_dense(d: np.ndarray, a: LowRankBlock) -> np.ndarray:
    """lowrank.py:224-231."""
    if d.shape != (a.rows, a.cols):
        raise ValueError("operands must have equal dimensions")
    if a.rank == 0:
        return d.copy()
    m, n = d.shape
    ou, _, _ = _product(0, m, a.rank, n, _dev(a.u), _dev(a.v), a.rank, _dev(d), out_rows=m * n)
    return _host(ou, m, n)


def lr_times_dense(a: LowRankBlock, d: np.ndarray, side: str) -> LowRankBlock:
    """lowrank.py:234-261."""
    if side == "right":
        if a.cols != d.shape[0]:
            raise ValueError("inner dimensions do not conform")
        if a.rank == 0:
            return LowRankBlock(a.u, np.zeros((d.shape[1], 0)))
        k, n = d.shape
        _, ov, r = _product(1, a.rows, k, n, None, _dev(a.v), a.rank, _dev(d), out_cols=n * a.rank)
        return LowRankBlock(a.u, _host(ov, n, r))
    if side == "left":
        if d.shape[1] != a.rows:
            raise ValueError("inner dimensions do not conform")
        if a.rank == 0:
            return LowRankBlock(np.zeros((d.shape[0], 0)), a.v)
        m, k = d.shape
        ou, ov, r = _product(2, m, k, a.cols, _dev(a.u), _dev(a.v), a.rank, _dev(d),
                             out_rows=m * a.rank, out_cols=a.cols * a.rank)
        return LowRankBlock(_host(ou, m, r), _host(ov, a.cols, r))
    raise ValueError(f"side must be 'left' or 'right', got {side!r}")


def lr_times_lr(a: LowRankBlock, bk: LowRankBlock) -> LowRankBlock:
    """lowrank.py:264-287."""
    if a.cols != bk.rows:
        raise ValueError("inner dimensions do not conform")
    if a.rank == 0 or bk.rank == 0:
        return LowRankBlock(np.zeros((a.rows, 0)), np.zeros((bk.cols, 0)))
    m, k, n = a.rows, a.cols, bk.cols
    rmax = max(a.rank, bk.rank)
    ou, ov, r = _product(3, m, k, n, _dev(a.u), _dev(a.v), a.rank, None, _dev(bk.u), _dev(bk.v), bk.rank,
                         out_rows=m * rmax, out_cols=n * rmax)
    return LowRankBlock(_host(ou, m, r), _host(ov, n, r))
