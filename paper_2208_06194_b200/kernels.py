"""Dense panel kernels with the reference API (kernels.py), run on the GPU.

qr_compact_wy = blocked Householder QR (LAPACK reflector convention) with
the full forward-columnwise T built blockwise from V^T V (kernels.py:87-103);
tp_qr = triangular-pentagonal QR with l = 0 (kernels.py:131-155);
mgs_panel_qr = right-looking MGS with the reference's per-column operation
order (kernels.py:192-225).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .lowrank import _dev, _host

__all__ = ["WYReflector", "TPReflector", "RankDeficiencyWarning", "qr_compact_wy", "apply_wy",
           "apply_wy_transpose", "tp_qr", "apply_tp", "apply_tp_transpose", "mgs_panel_qr"]


class RankDeficiencyWarning(UserWarning):
    """Panel column collapsed below the representable range during MGS."""


@dataclass
class WYReflector:
    """Q = I - y t y^T (kernels.py:38-59)."""

    y: np.ndarray
    t: np.ndarray

    @property
    def rows(self) -> int:
        return self.y.shape[0]

    @property
    def cols(self) -> int:
        return self.y.shape[1]

    def q_matrix(self) -> np.ndarray:
        return np.eye(self.rows) - self.y @ self.t @ self.y.T


@dataclass
class TPReflector:
    """Q = I - [I; y] t [I; y]^T (kernels.py:62-84)."""

    y: np.ndarray
    t: np.ndarray

    @property
    def bot_rows(self) -> int:
        return self.y.shape[0]

    @property
    def cols(self) -> int:
        return self.y.shape[1]

    def q_matrix(self) -> np.ndarray:
        n, k = self.cols, self.bot_rows
        yf = np.vstack([np.eye(n), self.y])
        return np.eye(n + k) - yf @ self.t @ yf.T


def _buf(n: int) -> torch.Tensor:
    return torch.zeros(max(n, 1), dtype=torch.float64, device=_lib.runtime().dev)


def qr_compact_wy(a: np.ndarray):
    m, n = a.shape
    if m < n:
        raise ValueError(f"panel must be tall: got {m} x {n}")
    rt = _lib.runtime()
    y, t, r = _buf(m * n), _buf(n * n), _buf(n * n)
    ws, per, nct = rt.workspace(max(m, 64), n, m)
    ad = _dev(a)  # keep operands alive until the (async) launch has consumed them
    # the tiled DiagQR routine on a CTA team (blrqr_panel_team op 0)
    _lib.check(rt.lib.blrqr_panel_team(0, m, n, ad.data_ptr(), None, y.data_ptr(), t.data_ptr(), r.data_ptr(), ws,
                                       per, nct, rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
               "geqrt")
    rt.harvest()
    return WYReflector(_host(y, m, n), _host(t, n, n)), _host(r, n, n)


def _check_rows(ref_rows: int, c: np.ndarray, what: str) -> None:
    if c.ndim != 2 or c.shape[0] != ref_rows:
        raise ValueError(f"{what}: operand rows {c.shape} do not match {ref_rows}")


def _apply_wy(ref: WYReflector, c: np.ndarray, transpose: bool) -> np.ndarray:
    m, n = ref.y.shape
    nc = c.shape[1]
    if nc == 0:
        return c.copy()
    rt = _lib.runtime()
    cd = _dev(c)
    ws, per, _ = rt.workspace(max(m, 64), max(n, nc), m)
    yd, td = _dev(ref.y), _dev(ref.t)
    _lib.check(rt.lib.blrqr_apply_wy(m, n, nc, yd.data_ptr(), td.data_ptr(), cd.data_ptr(),
                                     int(transpose), ws, per, rt.status.data_ptr(), rt.flops.data_ptr(),
                                     _lib.stream_ptr()), "apply_wy")
    rt.harvest()
    return _host(cd.reshape(-1), m, nc)


def apply_wy(ref: WYReflector, c: np.ndarray) -> np.ndarray:
    _check_rows(ref.rows, c, "apply_wy")
    return _apply_wy(ref, c, False)


def apply_wy_transpose(ref: WYReflector, c: np.ndarray) -> np.ndarray:
    _check_rows(ref.rows, c, "apply_wy_transpose")
    return _apply_wy(ref, c, True)


def tp_qr(r_top: np.ndarray, a_bot: np.ndarray):
    n = r_top.shape[0]
    if r_top.shape != (n, n):
        raise ValueError("top block must be square upper triangular")
    if a_bot.ndim != 2 or a_bot.shape[1] != n:
        raise ValueError(f"bottom block has {a_bot.shape[1]} cols, expected {n}")
    k = a_bot.shape[0]
    if k == 0:
        return TPReflector(np.zeros((0, n)), np.zeros((n, n))), r_top.copy()
    rt = _lib.runtime()
    rn, y, t = _buf(n * n), _buf(k * n), _buf(n * n)
    ws, per, nct = rt.workspace(max(n, k, 64), n, n + k)
    rtd, abd = _dev(r_top), _dev(a_bot)
    # the tiled UpdateQR routine on a CTA team (blrqr_panel_team op 1)
    _lib.check(rt.lib.blrqr_panel_team(1, k, n, rtd.data_ptr(), abd.data_ptr(), rn.data_ptr(), y.data_ptr(),
                                       t.data_ptr(), ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(),
                                       _lib.stream_ptr()), "tpqrt")
    rt.harvest()
    return TPReflector(_host(y, k, n), _host(t, n, n)), _host(rn, n, n)


def _apply_tp(ref: TPReflector, c_top: np.ndarray, c_bot: np.ndarray, transpose: bool):
    k, n = ref.y.shape
    _check_rows(n, c_top, "apply_tp top")
    _check_rows(k, c_bot, "apply_tp bottom")
    if c_top.shape[1] != c_bot.shape[1]:
        raise ValueError("top/bottom column counts differ")
    nc = c_top.shape[1]
    rt = _lib.runtime()
    ct, cb = _dev(c_top), _dev(c_bot) if k else _buf(1)
    yd = _dev(ref.y) if k else _buf(1)
    ws, per, _ = rt.workspace(max(n, k, 64), max(n, nc), n + k)
    td = _dev(ref.t)
    _lib.check(rt.lib.blrqr_apply_tp(n, k, nc, yd.data_ptr(), td.data_ptr(), ct.data_ptr(),
                                     cb.data_ptr(), int(transpose), ws, per, rt.status.data_ptr(),
                                     rt.flops.data_ptr(), _lib.stream_ptr()), "apply_tp")
    rt.harvest()
    return _host(ct.reshape(-1), n, nc), (_host(cb.reshape(-1), k, nc) if k else np.zeros((0, nc)))


def apply_tp(ref: TPReflector, c_top: np.ndarray, c_bot: np.ndarray):
    return _apply_tp(ref, c_top, c_bot, False)


def apply_tp_transpose(ref: TPReflector, c_top: np.ndarray, c_bot: np.ndarray):
    return _apply_tp(ref, c_top, c_bot, True)


def mgs_panel_qr(a: np.ndarray):
    m, n = a.shape
    if m < n:
        raise ValueError(f"panel must be tall: got {m} x {n}")
    rt = _lib.runtime()
    q, r = _buf(m * n), _buf(n * n)
    ws, per, _ = rt.workspace(max(m, 64), n, m)
    ad = _dev(a)
    _lib.check(rt.lib.blrqr_mgs_panel(m, n, ad.data_ptr(), q.data_ptr(), r.data_ptr(), ws, per,
                                      rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()), "mgs_panel")
    rt.harvest()
    return _host(q, m, n), _host(r, n, n)
