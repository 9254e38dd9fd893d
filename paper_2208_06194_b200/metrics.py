"""Accuracy metrics with the reference API (metrics.py), on the GPU, without
the reference's n <= 8192 guard (metrics.py:21, 79-82).

Q is materialised on the device by applying the stored reflectors to the
identity slab (libblrqr ``blrqr_apply_q``: 64-column chunks, one CTA each,
the reference's application order, factorize.py:295-352 / 461-524); MGS
keeps Q explicit.  Res = ||Q R - A||_F / ||A||_F and Orth = ||Q^T Q - I||_F /
sqrt(n) (metrics.py:84-88) then use library FP64 GEMMs (torch.matmul) in
column chunks -- the metric, not the factorization.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _lib
from .core import max_rank, memory_footprint

__all__ = ["AccuracyReport", "materialize_q_device", "res_orth_device", "compute_metrics", "kappa_fro"]


@dataclass
class AccuracyReport:
    """metrics.py:25-42."""

    algorithm: str
    m: int
    n: int
    b: int
    epsilon: float
    res: float
    orth: float
    max_rank: int
    memory_bytes: int
    flops: dict = field(default_factory=dict)
    flops_total: int = 0
    wall_ms: dict = field(default_factory=dict)
    kappa_f: float | None = None

    def to_json(self, indent: int | None = 2) -> str:
        return json.dumps(asdict(self), indent=indent, sort_keys=True)


def blr_dense_device(grid) -> torch.Tensor:
    """Column-major dense expansion of a DeviceGrid, returned as the row-major
    tensor of its transpose (shape n x m)."""
    rt = _lib.runtime()
    out = torch.empty((grid.n, grid.m), dtype=torch.float64, device=rt.dev)
    gs = grid.cstruct()
    _lib.check(rt.lib.blrqr_blr_to_dense(C.byref(gs), out.data_ptr(), grid.m, _lib.stream_ptr()), "blr_to_dense")
    return out


def materialize_q_device(f) -> torch.Tensor:
    """Q^T (n x m row-major = Q column-major) of a DeviceFactorization."""
    if f.method == "mgs":
        return blr_dense_device(f.qg)
    g = f.g
    rt = _lib.runtime()
    m, n = g.m, min(g.n, g.m)
    qt = torch.zeros((n, m), dtype=torch.float64, device=rt.dev)
    qt.diagonal().fill_(1.0)  # column-major identity slab
    ws, per, nct = rt.workspace(g.b, g.cap)
    gs, rs = g.cstruct(), f.rf.cstruct()
    method = 0 if f.method == "tiled-hh" else 1
    _lib.check(rt.lib.blrqr_apply_q(C.byref(gs), C.byref(rs), method, qt.data_ptr(), m, n, 0, ws, per, nct,
                                    rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()), "apply_q")
    rt.harvest()
    return qt


def res_orth_device(f, a_dense: torch.Tensor, chunk: int = 8192) -> tuple[float, float]:
    """(Res, Orth) for a DeviceFactorization against the original dense A
    (row-major m x n tensor on the device)."""
    qt = materialize_q_device(f)  # (n, m) = Q^T
    rt_ = blr_dense_device(f.r_device())  # (n, n) = R^T
    n = qt.shape[0]
    num = torch.zeros((), dtype=torch.float64, device=qt.device)
    orth = torch.zeros((), dtype=torch.float64, device=qt.device)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        # columns c0:c1 of Q R are rows c0:c1 of (Q R)^T = R^T[c0:c1] @ Q^T
        # R^T is n x m for a tall grid (m > n): only its first n columns meet Q^T
        qr_t = rt_[c0:c1, :n] @ qt
        num += torch.sum((qr_t - a_dense[:, c0:c1].T) ** 2)
        g = qt[c0:c1] @ qt.T
        g[:, c0:c1].diagonal().sub_(1.0)
        orth += torch.sum(g * g)
    den = torch.linalg.norm(a_dense)
    return float(torch.sqrt(num) / den), float(torch.sqrt(orth) / np.sqrt(n))


def kappa_fro(dense: np.ndarray) -> float:
    """metrics.py:59-66."""
    sigma = np.linalg.svd(dense, compute_uv=False)
    if sigma[-1] == 0:
        return float("inf")
    return float(np.sqrt(np.sum(sigma ** 2)) * np.sqrt(np.sum(sigma ** -2.0)))


def compute_metrics(a_dense: np.ndarray, result, epsilon: float, flops=None, wall_ms=None,
                    with_kappa: bool = False) -> AccuracyReport:
    """metrics.py:69-109 for a host FactorizationResult: the result is
    uploaded, Q materialised and Res/Orth evaluated on the GPU (any n)."""
    from .device import DeviceGrid, DeviceRefl
    from .factorize import DeviceFactorization

    rt = _lib.runtime()
    m, n = a_dense.shape
    f = DeviceFactorization.__new__(DeviceFactorization)
    f.method = result.algorithm
    f.rt = rt
    if result.algorithm == "mgs":
        f.qg = DeviceGrid.from_host(result.q_explicit)
        f.rg = DeviceGrid.from_host(result.r)
        f.g = f.rg
    else:
        f.g = DeviceGrid.from_host(result.r)
        f.rf = DeviceRefl(f.g)
        _upload_reflectors(f, result)
    a = torch.from_numpy(np.ascontiguousarray(a_dense)).to(rt.dev)
    res, orth = res_orth_device(f, a)
    kappa = kappa_fro(a_dense) if with_kappa else None
    fl = dict(flops or {})
    return AccuracyReport(result.algorithm, m, n, result.r.b, epsilon, res, orth, max_rank(result.r),
                          memory_footprint(result.r), fl, sum(fl.values()), dict(wall_ms or {}), kappa)


def _upload_reflectors(f, result) -> None:
    """Host reflector containers -> device reflector store + Ytilde slabs."""
    g, rf = f.g, f.rf
    b, q = g.b, g.q

    def put(off, mat):
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(mat, dtype=np.float64).T).ravel()).to(rf.pool.device)
        rf.pool[off:off + x.numel()] = x

    def put_ytilde(i, k, y):
        c = i * q + k
        if hasattr(y, "u"):
            r = y.rank
            ou, ov = int(g.off_u_host[c]), int(g.off_v_host[c])
            if r:
                g.pool[ou:ou + b * r] = torch.from_numpy(np.ascontiguousarray(y.u.T).ravel()).to(g.pool.device)
                g.pool[ov:ov + b * r] = torch.from_numpy(np.ascontiguousarray(y.v.T).ravel()).to(g.pool.device)
            rf.yrank[c] = r
        else:
            put(int(rf.y_off_host[c]), y)
            rf.yrank[c] = -1

    if result.q_tiles is not None:
        for k, w in result.q_tiles.diag.items():
            c = k * q + k
            put(int(rf.y_off_host[c]), w.y)
            put(int(rf.t_off_host[c]), w.t)
        for (i, k), (y, t) in result.q_tiles.updates.items():
            put(int(rf.t_off_host[i * q + k]), t)
            put_ytilde(i, k, y)
    else:
        for col in result.q_columns:
            k = col.col
            c = k * q + k
            put(int(rf.t_off_host[c]), col.t)
            for i, y in col.entries:
                if i == k:
                    put(int(rf.y_off_host[c]), y)
                else:
                    put_ytilde(i, k, y)
