"""Oracle BLR-QR factorizations (test infrastructure only).

Restates factorize.py: kind-dispatched block arithmetic
(factorize.py:68-138), blocked Householder (factorize.py:187-292), tiled
Householder (factorize.py:369-458), blocked MGS (factorize.py:576-671), the
dense apply-Q paths used for Res/Orth (factorize.py:295-352, 461-524) and the
metric formulas (metrics.py:45-109, without the n <= 8192 guard).

Each algorithm is expressed as per-task functions over a ``State`` so the
sequential order, the level-parallel executor and the GPU drivers can be
compared task by task.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import flops
from . import lowrank as lrk
from . import panels
from .blr import LR, Grid, is_lr, to_dense, zero_cell

# ---------------------------------------------------------------------------
# kind dispatch (factorize.py:68-138)
# ---------------------------------------------------------------------------


def mul(x, y):
    """x @ y, no truncation (factorize.py:68-82)."""
    if is_lr(x):
        if is_lr(y):
            core = y.u.T @ x.v
            flops.add("lr_mul", flops.mm(y.rank, x.cols, x.rank))
            flops.add("lr_mul", flops.mm(y.cols, y.rank, x.rank))
            return LR(x.u, y.v @ core)
        flops.add("lr_mul", flops.mm(y.shape[1], x.cols, x.rank))
        return LR(x.u, y.T @ x.v)
    if is_lr(y):
        flops.add("lr_mul", flops.mm(x.shape[0], x.shape[1], y.rank))
        return LR(x @ y.u, y.v)
    flops.add("gemm", flops.mm(x.shape[0], x.shape[1], y.shape[1]))
    return x @ y


def mul_t(x, y):
    """x^T @ y, no truncation (factorize.py:85-99)."""
    if is_lr(x):
        if is_lr(y):
            core = y.u.T @ x.u
            flops.add("lr_mul", flops.mm(y.rank, x.rows, x.rank))
            flops.add("lr_mul", flops.mm(y.cols, y.rank, x.rank))
            return LR(x.v, y.v @ core)
        flops.add("lr_mul", flops.mm(y.shape[1], x.rows, x.rank))
        return LR(x.v, y.T @ x.u)
    if is_lr(y):
        flops.add("lr_mul", flops.mm(x.shape[1], x.shape[0], y.rank))
        return LR(x.T @ y.u, y.v)
    flops.add("gemm", flops.mm(x.shape[1], x.shape[0], y.shape[1]))
    return x.T @ y


def dense_times(t: np.ndarray, s):
    """t @ s keeping s's kind (factorize.py:102-108)."""
    if is_lr(s):
        flops.add("lr_mul", flops.mm(t.shape[0], t.shape[1], s.rank))
        return LR(t @ s.u, s.v)
    flops.add("gemm", flops.mm(t.shape[0], t.shape[1], s.shape[1]))
    return t @ s


def neg(x):  # factorize.py:111-114
    return LR(x.u, -x.v) if is_lr(x) else -x


def acc(s, term, eps: float):
    """s + term (factorize.py:117-125)."""
    if is_lr(s):
        if is_lr(term):
            return lrk.rounded_add(s, term, eps)
        return lrk.add_into_dense(term, s)
    if is_lr(term):
        return lrk.add_into_dense(s, term)
    return s + term


def sub_into(target, term, lowrank_cell: bool, eps: float):
    """target - term coerced to the cell kind (factorize.py:128-138)."""
    if lowrank_cell:
        if is_lr(term):
            return lrk.rounded_add(target, neg(term), eps)
        return lrk.compress_lr(to_dense(target) - term, eps)
    if is_lr(term):
        return lrk.add_into_dense(target, neg(term))
    return target - term


# ---------------------------------------------------------------------------
# blocked Householder (factorize.py:187-292)
# ---------------------------------------------------------------------------


@dataclass
class ColumnReflector:
    """factorize.py:146-156: entries [(i, Y_i)] and the shared T."""

    col: int
    entries: list
    t: np.ndarray


def blocked_panel(g: Grid, k: int) -> ColumnReflector:
    """triangularize_block_column (factorize.py:187-229)."""
    b = g.b
    if is_lr(g[k, k]):
        raise ValueError(f"diagonal block {k} must be dense")
    parts, heights = [g[k, k]], [b]
    for i in range(k + 1, g.p):
        x = g[i, k]
        parts.append(x.v.T if is_lr(x) else x)
        heights.append(x.rank if is_lr(x) else b)
    y, t, r = panels.geqrt(np.vstack(parts))
    entries, off = [], 0
    for idx, i in enumerate(range(k, g.p)):
        h = heights[idx]
        yi = y[off:off + h, :]
        off += h
        src = g[i, k]
        if i != k and is_lr(src):
            entries.append((i, LR(src.u, np.ascontiguousarray(yi.T))))
        else:
            entries.append((i, np.ascontiguousarray(yi)))
    g[k, k] = r
    for i in range(k + 1, g.p):
        g[i, k] = zero_cell(b, g.lowrank[i, k])
    return ColumnReflector(k, entries, t)


def blocked_apply(ref: ColumnReflector, g: Grid, j: int, eps: float,
                  transpose: bool = True) -> None:
    """_refcol_apply_blr (factorize.py:232-249)."""
    s = None
    for i, y in ref.entries:
        term = mul_t(y, g[i, j])
        s = term if s is None else acc(s, term, eps)
    z = dense_times(ref.t.T if transpose else ref.t, s)
    for i, y in ref.entries:
        g[i, j] = sub_into(g[i, j], mul(y, z), g.lowrank[i, j], eps)


@dataclass
class BlockedState:
    """BlockedState (factorize.py:265-282)."""

    g: Grid
    eps: float
    cols: list = field(default_factory=list)

    @classmethod
    def start(cls, a: Grid, eps: float) -> "BlockedState":
        if a.p < a.q:
            raise ValueError("grid must have at least as many block rows as columns")
        return cls(a.clone(), eps)

    def panel(self, k: int) -> None:
        self.cols.append(blocked_panel(self.g, k))

    def apply_column(self, k: int, j: int) -> None:
        if j <= k:
            raise ValueError("update column must lie right of the reflector column")
        blocked_apply(self.cols[k], self.g, j, self.eps, True)


def blocked_hh(a: Grid, eps: float) -> BlockedState:
    """blocked_householder_qr (factorize.py:285-292)."""
    st = BlockedState.start(a, eps)
    for k in range(a.q):
        st.panel(k)
        for j in range(k + 1, a.q):
            st.apply_column(k, j)
    return st


def blocked_q_dense(st: BlockedState, c: np.ndarray, transpose: bool) -> np.ndarray:
    """blocked_apply_q on a dense operand (factorize.py:295-352)."""
    out = c.copy()
    b = st.g.b
    order = range(len(st.cols)) if transpose else range(len(st.cols) - 1, -1, -1)
    for k in order:
        ref = st.cols[k]
        nc = out.shape[1]
        accum = np.zeros((ref.t.shape[0], nc))
        for i, y in ref.entries:
            ci = out[i * b:(i + 1) * b]
            if is_lr(y):
                if y.rank == 0:
                    continue
                accum += y.v @ (y.u.T @ ci)
            else:
                accum += y.T @ ci
        z = (ref.t.T if transpose else ref.t) @ accum
        for i, y in ref.entries:
            sl = slice(i * b, (i + 1) * b)
            if is_lr(y):
                if y.rank == 0:
                    continue
                out[sl] -= y.u @ (y.v.T @ z)
            else:
                out[sl] -= y @ z
    return out


def blocked_q_blr(st: BlockedState, c: Grid, transpose: bool, eps: float) -> Grid:
    """blocked_apply_q on a block low-rank operand (factorize.py:343-350):
    for each reflector column in order, _refcol_apply_blr on every column j."""
    out = c.clone()
    order = range(len(st.cols)) if transpose else range(len(st.cols) - 1, -1, -1)
    for k in order:
        for j in range(out.q):
            blocked_apply(st.cols[k], out, j, eps, transpose)
    return out


# ---------------------------------------------------------------------------
# tiled Householder (factorize.py:369-458)
# ---------------------------------------------------------------------------


@dataclass
class TiledState:
    """TiledState (factorize.py:369-425): diag[k] = (Y, T); upd[(i,k)] = (Ytilde, T)."""

    g: Grid
    eps: float
    diag: dict = field(default_factory=dict)
    upd: dict = field(default_factory=dict)

    @classmethod
    def start(cls, a: Grid, eps: float) -> "TiledState":
        if a.p < a.q:
            raise ValueError("grid must have at least as many block rows as columns")
        return cls(a.clone(), eps)

    def diag_qr(self, k: int) -> None:  # factorize.py:379-385
        x = self.g[k, k]
        if is_lr(x):
            raise ValueError(f"diagonal block {k} must be dense")
        y, t, r = panels.geqrt(x)
        self.diag[k] = (y, t)
        self.g[k, k] = r

    def apply_block(self, k: int, j: int) -> None:  # factorize.py:387-396
        y, t = self.diag[k]
        x = self.g[k, j]
        if is_lr(x):
            if x.rank:
                self.g[k, j] = LR(panels.apply_wy(y, t, x.u, True), x.v)
        else:
            self.g[k, j] = panels.apply_wy(y, t, x, True)

    def update_qr(self, k: int, i: int) -> None:  # factorize.py:398-411
        x = self.g[i, k]
        if is_lr(x):
            yb, t, rn = panels.tpqrt(self.g[k, k], np.ascontiguousarray(x.v.T))
            yt = LR(x.u, np.ascontiguousarray(yb.T))
        else:
            yb, t, rn = panels.tpqrt(self.g[k, k], x)
            yt = yb
        self.upd[(i, k)] = (yt, t)
        self.g[k, k] = rn
        self.g[i, k] = zero_cell(self.g.b, self.g.lowrank[i, k])

    def apply_trap(self, k: int, i: int, j: int) -> None:  # factorize.py:413-422
        yt, t = self.upd[(i, k)]
        top, bot = trap_pair(yt, t, self.g[k, j], self.g[i, j], True,
                             self.g.lowrank[k, j], self.g.lowrank[i, j], self.eps)
        self.g[k, j] = top
        self.g[i, j] = bot


def trap_pair(yt, t, top, bot, transpose, top_lr, bot_lr, eps):
    """_trap_apply_pair (factorize.py:428-444)."""
    prod = mul_t(yt, bot)
    ssum = acc(top, prod, eps)
    w = dense_times(t.T if transpose else t, ssum)
    return (sub_into(top, w, top_lr, eps),
            sub_into(bot, mul(yt, w), bot_lr, eps))


def tiled_q_blr(st: "TiledState", c: Grid, transpose: bool, eps: float) -> Grid:
    """tiled_apply_q on a block low-rank operand (factorize.py:534-567)."""
    out = c.clone()
    p, q = st.g.p, st.g.q
    adm = out.lowrank

    def diag_apply(k):
        y, t = st.diag[k]
        for j in range(out.q):
            x = out[k, j]
            if is_lr(x):
                if x.rank:
                    out[k, j] = LR(panels.apply_wy(y, t, x.u, transpose), x.v)
            else:
                out[k, j] = panels.apply_wy(y, t, x, transpose)

    def trap(k, i):
        yt, t = st.upd[(i, k)]
        for j in range(out.q):
            out[k, j], out[i, j] = trap_pair(yt, t, out[k, j], out[i, j], transpose, adm[k, j], adm[i, j], eps)

    if transpose:
        for k in range(q):
            diag_apply(k)
            for i in range(k + 1, p):
                trap(k, i)
    else:
        for k in range(q - 1, -1, -1):
            for i in range(p - 1, k, -1):
                trap(k, i)
            diag_apply(k)
    return out


def tiled_tasks(p: int, q: int) -> list[tuple]:
    """Canonical sweep order (scheduler.py:127-138): (kind, k, i, j)."""
    out = []
    for k in range(q):
        out.append(("diag", k, -1, -1))
        for j in range(k + 1, q):
            out.append(("block", k, -1, j))
        for i in range(k + 1, p):
            out.append(("update", k, i, -1))
            for j in range(k + 1, q):
                out.append(("trap", k, i, j))
    return out


def run_tiled_task(st: TiledState, task: tuple) -> None:
    kind, k, i, j = task
    if kind == "diag":
        st.diag_qr(k)
    elif kind == "block":
        st.apply_block(k, j)
    elif kind == "update":
        st.update_qr(k, i)
    elif kind == "trap":
        st.apply_trap(k, i, j)
    else:
        raise ValueError(f"not a tiled task: {task}")


def tiled_hh(a: Grid, eps: float) -> TiledState:
    """tiled_householder_qr (factorize.py:447-458)."""
    st = TiledState.start(a, eps)
    for task in tiled_tasks(a.p, a.q):
        run_tiled_task(st, task)
    return st


def tiled_q_dense(st: TiledState, c: np.ndarray, transpose: bool) -> np.ndarray:
    """tiled_apply_q on a dense operand (factorize.py:461-524)."""
    g = st.g
    p, q, b = g.p, g.q, g.b
    out = c.copy()
    rows = [out[i * b:(i + 1) * b] for i in range(p)]

    def trap_dense(yt, t, ct, cb, tr):
        if is_lr(yt):
            ytcb = np.zeros_like(ct) if yt.rank == 0 else yt.v @ (yt.u.T @ cb)
        else:
            ytcb = yt.T @ cb
        w = (t.T if tr else t) @ (ct + ytcb)
        ct -= w
        if is_lr(yt):
            if yt.rank:
                cb -= yt.u @ (yt.v.T @ w)
        else:
            cb -= yt @ w

    if transpose:
        for k in range(q):
            y, t = st.diag[k]
            rows[k][:] = panels.apply_wy(y, t, rows[k], True)
            for i in range(k + 1, p):
                trap_dense(*st.upd[(i, k)], rows[k], rows[i], True)
    else:
        for k in range(q - 1, -1, -1):
            for i in range(p - 1, k, -1):
                trap_dense(*st.upd[(i, k)], rows[k], rows[i], False)
            y, t = st.diag[k]
            rows[k][:] = panels.apply_wy(y, t, rows[k], False)
    return out


# ---------------------------------------------------------------------------
# blocked MGS (factorize.py:576-671)
# ---------------------------------------------------------------------------


class MgsState:
    """MgsState (factorize.py:576-658): explicit Q with A's kind map, R q x q."""

    def __init__(self, a: Grid, eps: float):
        if a.p < a.q:
            raise ValueError("grid must have at least as many block rows as columns")
        self.g = a.clone()
        self.eps = eps
        b = a.b
        self.qg = Grid(a.m, a.n, b, a.lowrank,
                       [[zero_cell(b, a.lowrank[i, j]) for j in range(a.q)] for i in range(a.p)])
        rl = a.lowrank[:a.q, :].copy()
        d = np.arange(a.q)
        rl[d, d] = False
        self.rg = Grid(a.n, a.n, b, rl,
                       [[zero_cell(b, rl[i, j]) for j in range(a.q)] for i in range(a.q)])

    def panel(self, j: int) -> None:  # factorize.py:605-632
        g, b = self.g, self.g.b
        parts, heights = [], []
        for i in range(g.p):
            x = g[i, j]
            parts.append(x.v.T if is_lr(x) else x)
            heights.append(x.rank if is_lr(x) else b)
        qb, rb = panels.mgs(np.vstack(parts))
        off = 0
        for i in range(g.p):
            h = heights[i]
            qi = qb[off:off + h, :]
            off += h
            x = g[i, j]
            self.qg[i, j] = LR(x.u, np.ascontiguousarray(qi.T)) if is_lr(x) else np.ascontiguousarray(qi)
        self.rg[j, j] = rb

    def project(self, j: int, k: int) -> None:  # factorize.py:634-645
        s = None
        for i in range(self.g.p):
            term = mul_t(self.qg[i, j], self.g[i, k])
            s = term if s is None else acc(s, term, self.eps)
        if self.rg.lowrank[j, k] and not is_lr(s):
            s = lrk.compress_lr(s, self.eps)
        elif not self.rg.lowrank[j, k] and is_lr(s):
            s = to_dense(s)
        self.rg[j, k] = s

    def update(self, j: int, i: int, k: int) -> None:  # factorize.py:647-655
        term = mul(self.qg[i, j], self.rg[j, k])
        self.g[i, k] = sub_into(self.g[i, k], term, self.g.lowrank[i, k], self.eps)


def mgs_qr(a: Grid, eps: float) -> MgsState:
    """blocked_mgs_qr (factorize.py:661-671)."""
    st = MgsState(a, eps)
    for j in range(a.q):
        st.panel(j)
        for k in range(j + 1, a.q):
            st.project(j, k)
        for k in range(j + 1, a.q):
            for i in range(a.p):
                st.update(j, i, k)
    return st


# ---------------------------------------------------------------------------
# drivers + metrics
# ---------------------------------------------------------------------------

METHODS = ("mgs", "blocked-hh", "tiled-hh")


def factorize(method: str, a: Grid, eps: float):
    """execute_sequential (scheduler.py:250-276)."""
    if method == "blocked-hh":
        return blocked_hh(a, eps)
    if method == "tiled-hh":
        return tiled_hh(a, eps)
    if method == "mgs":
        return mgs_qr(a, eps)
    raise ValueError(f"unknown algorithm {method!r}")


def r_grid(st) -> Grid:
    return st.rg if isinstance(st, MgsState) else st.g


def q_dense(st) -> np.ndarray:
    """materialize_q (metrics.py:45-56)."""
    if isinstance(st, MgsState):
        return st.qg.dense()
    g = st.g
    n = min(g.n, g.m)
    slab = np.zeros((g.m, n))
    slab[np.arange(n), np.arange(n)] = 1.0
    if isinstance(st, BlockedState):
        return blocked_q_dense(st, slab, False)
    return tiled_q_dense(st, slab, False)


def res_orth(a_dense: np.ndarray, st) -> tuple[float, float]:
    """Res and Orth (metrics.py:84-88), without the n <= 8192 guard."""
    n = a_dense.shape[1]
    qm = q_dense(st)
    rd = r_grid(st).dense()[:n, :]
    res = float(np.linalg.norm(qm @ rd - a_dense) / np.linalg.norm(a_dense))
    gram = qm.T @ qm
    gram[np.arange(n), np.arange(n)] -= 1.0
    return res, float(np.linalg.norm(gram) / np.sqrt(n))
