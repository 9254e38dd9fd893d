"""Oracle dense panel kernels (test infrastructure only).

Restates kernels.py: compact-WY Householder QR through LAPACK dgeqrt with
nb = n (kernels.py:87-103), the explicit three-GEMM WY application
(kernels.py:111-128), the triangular-pentagonal update QR through dtpqrt
with l = 0 (kernels.py:131-155) and its application (kernels.py:158-186), and
right-looking-equivalent modified Gram-Schmidt (kernels.py:192-225).
"""

from __future__ import annotations

import warnings

import numpy as np
from scipy.linalg import lapack

from . import flops


class RankDeficiencyWarning(UserWarning):
    """MGS column collapsed (kernels.py:34-35)."""


def geqrt(a: np.ndarray):
    """(y, t, r): Q = I - y t y^T, y unit lower trapezoidal with explicit
    unit diagonal, t upper, r = triu (kernels.py:87-103)."""
    m, n = a.shape
    if m < n:
        raise ValueError(f"panel must be tall: got {m} x {n}")
    packed, t, info = lapack.dgeqrt(n, a)
    if info != 0:
        raise RuntimeError(f"geqrt failed with info={info}")
    r = np.ascontiguousarray(np.triu(packed[:n, :]))
    y = np.tril(packed, -1)
    np.fill_diagonal(y, 1.0)
    flops.add("panel_qr", flops.qr(m, n) + flops.tgen(m, n))
    return np.ascontiguousarray(y), np.ascontiguousarray(np.triu(t)), r


def apply_wy(y: np.ndarray, t: np.ndarray, c: np.ndarray, transpose: bool) -> np.ndarray:
    """c - y (t or t^T) (y^T c)  (kernels.py:111-128)."""
    if c.ndim != 2 or c.shape[0] != y.shape[0]:
        raise ValueError(f"apply_wy: operand rows {c.shape} do not match {y.shape[0]}")
    m, n = y.shape
    nc = c.shape[1]
    w = (t.T if transpose else t) @ (y.T @ c)
    flops.add("apply_wy", flops.mm(n, m, nc) + flops.mm(n, n, nc) + flops.mm(m, n, nc))
    return c - y @ w


def tpqrt(r_top: np.ndarray, a_bot: np.ndarray):
    """(y, t, r_new) for QR of [r_top; a_bot] (kernels.py:131-155)."""
    n = r_top.shape[0]
    if r_top.shape != (n, n):
        raise ValueError("top block must be square upper triangular")
    if a_bot.ndim != 2 or a_bot.shape[1] != n:
        raise ValueError(f"bottom block has {a_bot.shape[1]} cols, expected {n}")
    k = a_bot.shape[0]
    if k == 0:
        return np.zeros((0, n)), np.zeros((n, n)), r_top.copy()
    r_new, y, t, info = lapack.dtpqrt(0, n, r_top, a_bot)
    if info != 0:
        raise RuntimeError(f"tpqrt failed with info={info}")
    flops.add("update_qr", flops.qr(n + k, n) + flops.tgen(n + k, n))
    return (np.ascontiguousarray(y), np.ascontiguousarray(np.triu(t)),
            np.ascontiguousarray(np.triu(r_new)))


def apply_tp(y: np.ndarray, t: np.ndarray, c_top: np.ndarray, c_bot: np.ndarray,
             transpose: bool):
    """(c_top - w, c_bot - y w), w = t(^T) (c_top + y^T c_bot) (kernels.py:158-186)."""
    k, n = y.shape
    if c_top.ndim != 2 or c_top.shape[0] != n:
        raise ValueError("apply_tp top rows mismatch")
    if c_bot.ndim != 2 or c_bot.shape[0] != k:
        raise ValueError("apply_tp bottom rows mismatch")
    if c_top.shape[1] != c_bot.shape[1]:
        raise ValueError("top/bottom column counts differ")
    nc = c_top.shape[1]
    w = (t.T if transpose else t) @ (c_top + y.T @ c_bot)
    flops.add("apply_tp", flops.mm(n, k, nc) + flops.mm(n, n, nc) + flops.mm(k, n, nc))
    return c_top - w, c_bot - y @ w


def mgs(a: np.ndarray):
    """Modified Gram-Schmidt (kernels.py:192-225)."""
    m, n = a.shape
    if m < n:
        raise ValueError(f"panel must be tall: got {m} x {n}")
    q = np.array(a, dtype=float, copy=True)
    r = np.zeros((n, n))
    for j in range(n):
        w = q[:, j]
        for i in range(j):
            rij = q[:, i] @ w
            w -= rij * q[:, i]
            r[i, j] = rij
        rjj = np.linalg.norm(w)
        r[j, j] = rjj
        if rjj < 1e-300:
            warnings.warn(f"panel column {j} collapsed (|r_jj|={rjj:.3e})",
                          RankDeficiencyWarning, stacklevel=2)
            continue
        q[:, j] = w / rjj
    flops.add("panel_qr", flops.mgs(m, n))
    return q, r
