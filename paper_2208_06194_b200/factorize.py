"""BLR-QR factorizations with the reference API (factorize.py), on the GPU.

Each method replays the reference's task sequence (factorize.py:187-262
blocked, :369-458 tiled, :576-671 MGS) with one CTA per block task; the
parallelism comes only from running independent tasks side by side
(levels of the tiled DAG, the j-loop of a blocked step, the k-loop of an MGS
step), never from re-associating sums (SURVEY §7 guiding constraint).

Device drivers (``DeviceFactorization``) keep everything in HBM; the
reference-compatible entry points (``tiled_householder_qr`` ...) upload a
host ``BlrMatrix``, run, and download a ``FactorizationResult`` holding the
same containers as the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .core import BlrMatrix, LowRankBlock, is_lowrank
from .device import DeviceGrid, DeviceRefl
from .kernels import WYReflector
from .lowrank import ToleranceConfig

__all__ = ["ReflectorColumn", "TileReflectorStore", "FactorizationResult", "DeviceFactorization",
           "blocked_householder_qr", "tiled_householder_qr", "blocked_mgs_qr", "factorize_device",
           "blocked_apply_q", "tiled_apply_q"]

METHODS = ("mgs", "blocked-hh", "tiled-hh")
DAG_TIMEOUT_S = 120.0  # a persistent CTA waiting this long for a ready task aborts the run


@dataclass
class ReflectorColumn:
    """factorize.py:146-156."""

    col: int
    entries: list
    t: np.ndarray


@dataclass
class TileReflectorStore:
    """factorize.py:159-170."""

    diag: dict = field(default_factory=dict)
    updates: dict = field(default_factory=dict)


@dataclass
class FactorizationResult:
    """factorize.py:173-179."""

    algorithm: str
    r: BlrMatrix
    q_columns: list | None = None
    q_tiles: TileReflectorStore | None = None
    q_explicit: BlrMatrix | None = None


@lru_cache(maxsize=16)
def tiled_dag_arrays(p: int, q: int, policy: int = 0):
    """(tasks[n,4], indeg[n], succ_off[n+1], succ[e], prio[n]) of the tiled DAG (policy =
    blrqr_dag_policy(): part of the cache key because prio depends on the knobs)
    (same read/write-set edges as scheduler.py:173-201), from libblrqr."""
    lib = _lib.load()
    ne = C.c_int64(0)
    n = int(lib.blrqr_tiled_dag_size(p, q, C.byref(ne)))
    if n < 0:
        raise ValueError("need p >= q >= 1")
    tasks = np.zeros((n, 4), dtype=np.int32)
    indeg = np.zeros(n, dtype=np.int32)
    off = np.zeros(n + 1, dtype=np.int64)
    succ = np.zeros(max(ne.value, 1), dtype=np.int32)
    prio = np.zeros(n, dtype=np.int32)
    rc = lib.blrqr_tiled_dag(p, q, tasks.ctypes.data, indeg.ctypes.data, off.ctypes.data, succ.ctypes.data,
                             prio.ctypes.data)
    if rc != 0:
        raise RuntimeError("tiled DAG build failed")
    return tasks, indeg, off, succ, prio


SCHEDULERS = ("auto", "dag", "levels")
# "auto": the persistent dynamic-DAG kernel from b = 32 on, the level scheduler
# below.  At b = 16 the DAG kernel produced box-dependent wrong results on
# B200 until the 16-row panel staging was taken out (DESIGN 7); the level
# scheduler never did, and toy block sizes gain nothing from the DAG kernel.
DAG_MIN_B = 32


@lru_cache(maxsize=16)
def tiled_schedule(p: int, q: int):
    """(tasks ndarray[n, 4] int32, level_start ndarray[int64]) from the C++
    level scheduler over the reference DAG's read/write sets."""
    lib = _lib.load()
    n = int(lib.blrqr_tiled_task_count(p, q))
    if n < 0:
        raise ValueError("need p >= q >= 1")
    tasks = (_lib.Task * n)()
    ls = (C.c_int64 * (n + 2))()
    nlev = lib.blrqr_tiled_schedule(p, q, C.addressof(tasks), C.addressof(ls), n + 1)
    if nlev < 0:
        raise RuntimeError("tiled schedule failed")
    arr = np.ctypeslib.as_array(C.cast(tasks, C.POINTER(C.c_int32)), shape=(n, 4)).copy()
    lv = np.ctypeslib.as_array(ls, shape=(n + 2,))[: nlev + 1].copy()
    return arr, lv


class DeviceFactorization:
    """A BLR-QR factorization resident on the GPU (input grid is cloned)."""

    def __init__(self, method: str, a: DeviceGrid, cfg: ToleranceConfig, clone: bool = True,
                 scheduler: str = "auto"):
        if method not in METHODS:
            raise ValueError(f"unknown algorithm {method!r}")
        if a.p < a.q:
            raise ValueError("grid must have at least as many block rows as columns")
        self.method = method
        self.cfg = cfg
        self.rt = _lib.runtime()
        self.g = a.clone() if clone else a
        self.rf = None
        self.qg = None
        self.rg = None
        if method == "tiled-hh":
            self.rf = DeviceRefl(self.g)
            if scheduler not in SCHEDULERS:
                raise ValueError(f"scheduler must be one of {SCHEDULERS}")
            if scheduler == "auto":
                scheduler = "dag" if self.g.b >= DAG_MIN_B else "levels"
            self.scheduler = scheduler
            tasks, self.levels = tiled_schedule(self.g.p, self.g.q)
            self.tasks = torch.from_numpy(tasks).to(self.rt.dev)
            self.nlevels = len(self.levels) - 1
            if scheduler == "dag":
                self.rf.enable_split_traps()
                # prio bakes in the ring / team knobs: key the cache on them too
                key = (self.g.p, self.g.q, int(self.rt.lib.blrqr_dag_policy()))
                dev = self.rt.dev
                if key not in self.rt.dag_cache:  # read-only device copy of the DAG, once per shape
                    dt, ind, off, succ, prio = tiled_dag_arrays(*key)
                    self.rt.dag_cache[key] = {
                        "n": len(dt), "tasks": torch.from_numpy(dt).to(dev), "indeg": torch.from_numpy(ind).to(dev),
                        "off": torch.from_numpy(off).to(dev), "succ": torch.from_numpy(succ).to(dev),
                        "prio": torch.from_numpy(prio).to(dev)}
                self.dag = dict(self.rt.dag_cache[key])
                nwork = int(self.rt.lib.blrqr_dag_work_ints(self.dag["n"]))
                self.dag["work"] = torch.empty(nwork, dtype=torch.int32, device=dev)
        elif method == "blocked-hh":
            g = self.g
            self.rf = DeviceRefl(self.g)
            dev = self.rt.dev
            self.zbuf = torch.empty(g.q * 2 * g.b * g.b, dtype=torch.float64, device=dev)
            self.zrank = torch.zeros(g.q, dtype=torch.int32, device=dev)
            self.panel = torch.empty(2 * g.p * g.b * g.b, dtype=torch.float64, device=dev)
        else:
            g = self.g
            self.qg = DeviceGrid(g.m, g.n, g.b, g.kind_host, g.cap)
            rl = g.kind_host[: g.q, :].copy()
            d = np.arange(g.q)
            rl[d, d] = False
            self.rg = DeviceGrid(g.n, g.n, g.b, rl, g.cap)
            self.panel = torch.empty(g.p * g.b * g.b, dtype=torch.float64, device=self.rt.dev)

    # -- execution ---------------------------------------------------------
    def run(self, nctas: int | None = None) -> "DeviceFactorization":
        """Enqueue the whole factorization on the current stream (no sync)."""
        rt = self.rt
        g = self.g
        ws, per, nct = rt.workspace(g.b, g.cap, 0, nctas)
        if self.method == "tiled-hh" and self.scheduler == "dag":
            gs, rs = g.cstruct(), self.rf.cstruct()
            d = self.dag
            _lib.check(rt.lib.blrqr_tiled_run_dag(
                C.byref(gs), C.byref(rs), d["n"], d["tasks"].data_ptr(), d["indeg"].data_ptr(), d["off"].data_ptr(),
                d["succ"].data_ptr(), d["prio"].data_ptr(), d["work"].data_ptr(), self.cfg.epsilon, ws, per, nct,
                DAG_TIMEOUT_S, rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()), "tiled_run_dag")
        elif self.method == "tiled-hh":
            gs, rs = g.cstruct(), self.rf.cstruct()
            lv = self.levels.ctypes.data_as(C.c_void_p)
            _lib.check(rt.lib.blrqr_tiled_run(C.byref(gs), C.byref(rs), self.tasks.data_ptr(), lv, 0,
                                              self.nlevels, self.cfg.epsilon, ws, per, nct,
                                              rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
                       "tiled_run")
        elif self.method == "blocked-hh":
            gs, rs = g.cstruct(), self.rf.cstruct()
            for k in range(g.q):
                _lib.check(rt.lib.blrqr_blocked_step(C.byref(gs), C.byref(rs), k, self.cfg.epsilon,
                                                     self.zbuf.data_ptr(), self.zrank.data_ptr(),
                                                     self.panel.data_ptr(), self.panel.numel(), ws, per, nct,
                                                     rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
                           "blocked_step")
        else:
            gs, qs, rs = g.cstruct(), self.qg.cstruct(), self.rg.cstruct()
            for j in range(g.q):
                _lib.check(rt.lib.blrqr_mgs_step(C.byref(gs), C.byref(qs), C.byref(rs), j, self.cfg.epsilon,
                                                 self.panel.data_ptr(), self.panel.numel(), ws, per, nct,
                                                 rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
                           "mgs_step")
        return self

    def finish(self) -> dict:
        """Synchronise, raise on device errors, return the model-flop report."""
        _, counts = self.rt.harvest()
        return counts

    # -- results -----------------------------------------------------------
    def r_device(self) -> DeviceGrid:
        return self.rg if self.method == "mgs" else self.g

    def to_host(self) -> FactorizationResult:
        if self.method == "mgs":
            return FactorizationResult("mgs", self.rg.to_host(), q_explicit=self.qg.to_host())
        r = self.g.to_host()
        if self.method == "tiled-hh":
            return FactorizationResult("tiled-hh", r, q_tiles=self._tiles_host())
        return FactorizationResult("blocked-hh", r, q_columns=self._columns_host())

    # -- reflector download: one D2H of the reflector store and one packed D2H
    # of the low-rank Ytilde factors; the returned numpy arrays are views into
    # those (pinned, caching-allocator) host buffers -- no per-tile copies
    def _host_stores(self):
        g, rf = self.g, self.rf
        b = g.b
        pool_h = torch.empty(rf.pool.numel(), dtype=torch.float64, pin_memory=True)
        pool_h.copy_(rf.pool)
        yr = rf.yrank.cpu().numpy()
        sel = (yr >= 0) & g.kind_host.ravel()
        ranks = np.where(sel, yr, 0).astype(np.int32)
        sz = (2 * b * ranks).astype(np.int64)
        off = np.zeros_like(sz)
        off[1:] = np.cumsum(sz)[:-1]
        tot = int(sz.sum())
        off_pack = np.where(sel, off, -1)
        fac_h = torch.empty(max(tot, 1), dtype=torch.float64, pin_memory=True)
        if tot:
            dev = g.pool.device
            stage = torch.empty(tot, dtype=torch.float64, device=dev)
            rank_t = torch.from_numpy(ranks).to(dev)
            od = torch.from_numpy(off_pack).to(dev)
            gs = g.cstruct()
            gs.rank = rank_t.data_ptr()
            _lib.check(_lib.load().blrqr_grid_pack(C.byref(gs), stage.data_ptr(), od.data_ptr(), 0,
                                                   _lib.stream_ptr()), "grid_pack")
            fac_h.copy_(stage)
        self._host_bufs = (pool_h, fac_h)  # the views below keep them alive
        P, F = pool_h.numpy(), fac_h.numpy()

        def mat(o, rows, cols):
            return P[o:o + rows * cols].reshape(cols, rows).T

        def ytilde(c):
            if sel[c]:
                r, o = int(ranks[c]), int(off[c])
                return LowRankBlock(F[o:o + b * r].reshape(r, b).T, F[o + b * r:o + 2 * b * r].reshape(r, b).T)
            return mat(int(rf.y_off_host[c]), b, b)

        return mat, ytilde

    def _columns_host(self) -> list:
        g, rf = self.g, self.rf
        b = g.b
        mat, ytilde = self._host_stores()
        cols = []
        for k in range(g.q):
            c = k * g.q + k
            entries = [(k, mat(int(rf.y_off_host[c]), b, b))]
            entries += [(i, ytilde(i * g.q + k)) for i in range(k + 1, g.p)]
            cols.append(ReflectorColumn(k, entries, mat(int(rf.t_off_host[c]), b, b)))
        return cols

    def _tiles_host(self) -> TileReflectorStore:
        g, rf = self.g, self.rf
        b, p, q = g.b, g.p, g.q
        mat, ytilde = self._host_stores()
        store = TileReflectorStore()
        for k in range(q):
            c = k * q + k
            store.diag[k] = WYReflector(mat(int(rf.y_off_host[c]), b, b), mat(int(rf.t_off_host[c]), b, b))
            for i in range(k + 1, p):
                c = i * q + k
                store.updates[(i, k)] = (ytilde(c), mat(int(rf.t_off_host[c]), b, b))
        return store


def factorize_device(method: str, a: DeviceGrid, cfg: ToleranceConfig, clone: bool = True,
                     scheduler: str = "auto") -> DeviceFactorization:
    f = DeviceFactorization(method, a, cfg, clone, scheduler)
    f.run()
    f.finish()
    return f


def _host_entry(method: str, a: BlrMatrix, cfg: ToleranceConfig) -> FactorizationResult:
    if a.p < a.q:
        raise ValueError("grid must have at least as many block rows as columns")
    g = DeviceGrid.from_host(a)
    return factorize_device(method, g, cfg, clone=False).to_host()


def tiled_householder_qr(a: BlrMatrix, cfg: ToleranceConfig) -> FactorizationResult:
    """factorize.py:447-458."""
    return _host_entry("tiled-hh", a, cfg)


def blocked_householder_qr(a: BlrMatrix, cfg: ToleranceConfig) -> FactorizationResult:
    """factorize.py:285-292."""
    return _host_entry("blocked-hh", a, cfg)


def blocked_mgs_qr(a: BlrMatrix, cfg: ToleranceConfig) -> FactorizationResult:
    """factorize.py:661-671."""
    return _host_entry("mgs", a, cfg)


def _upload_result(result, method: str) -> "DeviceFactorization":
    """A host FactorizationResult's R-tilde grid + reflectors on the device."""
    from .metrics import _upload_reflectors

    rt = _lib.runtime()
    f = DeviceFactorization.__new__(DeviceFactorization)
    f.method, f.rt = method, rt
    f.g = DeviceGrid.from_host(result.r)
    f.rf = DeviceRefl(f.g)
    _upload_reflectors(f, result)
    return f


def _apply_q_dense(result, c: np.ndarray, transpose: bool, method: str) -> np.ndarray:
    """Q (or Q^T) times a dense host operand, on the GPU."""
    rt = _lib.runtime()
    m = result.r.structure.m
    if c.ndim != 2 or c.shape[0] != m:
        raise ValueError(f"operand has {c.shape[0]} rows, expected {m}")
    f = _upload_result(result, method)
    nc = c.shape[1]
    ct = torch.from_numpy(np.ascontiguousarray(np.asarray(c, dtype=np.float64).T)).to(rt.dev)
    ws, per, nct = rt.workspace(f.g.b, f.g.cap)
    gs, rs = f.g.cstruct(), f.rf.cstruct()
    _lib.check(rt.lib.blrqr_apply_q(C.byref(gs), C.byref(rs), 0 if method == "tiled-hh" else 1, ct.data_ptr(), m,
                                    nc, int(transpose), ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(),
                                    _lib.stream_ptr()), "apply_q")
    rt.harvest()
    return np.ascontiguousarray(ct.cpu().numpy().T)


def _apply_q_blr(result, c: BlrMatrix, transpose: bool, cfg: ToleranceConfig, method: str) -> BlrMatrix:
    """Q (or Q^T) times a block low-rank host operand, on the GPU: the
    factorization's kind-aware block updates with rounded additions
    (factorize.py:343-350 blocked, :534-567 tiled); the input is not mutated."""
    rt = _lib.runtime()
    rm = result.r.structure
    if c.structure.m != rm.m:
        raise ValueError("operand row count does not match the factorization")
    if c.structure.b != rm.b:
        raise ValueError("operand block size does not match the factorization")
    f = _upload_result(result, method)
    gc = DeviceGrid.from_host(c)
    b = gc.b
    zbuf = zrank = None
    if method == "blocked-hh":
        zbuf = torch.empty(gc.q * 2 * b * b, dtype=torch.float64, device=rt.dev)
        zrank = torch.zeros(gc.q, dtype=torch.int32, device=rt.dev)
    ws, per, nct = rt.workspace(b, max(f.g.cap, gc.cap))
    gs, rs, cs = f.g.cstruct(), f.rf.cstruct(), gc.cstruct()
    _lib.check(rt.lib.blrqr_apply_q_blr(C.byref(gs), C.byref(rs), 0 if method == "tiled-hh" else 1, C.byref(cs),
                                        int(transpose), cfg.epsilon,
                                        zbuf.data_ptr() if zbuf is not None else None,
                                        zrank.data_ptr() if zrank is not None else None, ws, per, nct,
                                        rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()), "apply_q_blr")
    rt.harvest()
    return gc.to_host()


def blocked_apply_q(result, c, transpose, cfg=None):
    """factorize.py:326-361 on the GPU: dense operands with plain dense
    arithmetic, block low-rank operands with the factorization's kind-aware
    updates (needs a tolerance config)."""
    if result.q_columns is None:
        raise ValueError("result does not carry blocked reflector columns")
    if not isinstance(c, np.ndarray):
        if cfg is None:
            raise ValueError("block low-rank operands need a tolerance config")
        return _apply_q_blr(result, c, transpose, cfg, "blocked-hh")
    return _apply_q_dense(result, c, transpose, "blocked-hh")


def tiled_apply_q(result, c, transpose, cfg=None):
    """factorize.py:495-568 on the GPU (dense and block low-rank operands)."""
    if result.q_tiles is None:
        raise ValueError("result does not carry tiled reflectors")
    if not isinstance(c, np.ndarray):
        if cfg is None:
            raise ValueError("block low-rank operands need a tolerance config")
        return _apply_q_blr(result, c, transpose, cfg, "tiled-hh")
    return _apply_q_dense(result, c, transpose, "tiled-hh")
