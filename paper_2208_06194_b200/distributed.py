"""Multi-GPU tiled Householder BLR-QR: 1-D block-cyclic columns + reflector
broadcast.

Column j (every block row of it, including R-tilde's row blocks) lives on
rank j mod G.  Task ownership follows the written cells
(scheduler.py:109-124): DiagQR(k) and UpdateQR(k, i) write column k, so the
owner of column k runs them (the serial UpdateQR chain of a column stays on
one GPU); ApplyBlockReflector(k, j) and ApplyTrapReflector(k, i, j) write
column j only.  The only data a rank needs from another is the reflectors of
column k: (Y_kk, T_kk) after DiagQR(k) and (Ytilde_ik, T_ik) after
UpdateQR(k, i).  They are broadcast from the owner (NCCL over NVLink on GPUs,
gloo in the CPU tests) in the canonical (k, i) order of the level in which
they are produced, so every rank issues the same collective sequence.

Execution is level-synchronous over the tiled DAG levels of the C++ level
scheduler (the same levels as the single-GPU ``scheduler="levels"`` path):
each rank runs its own tasks of level L as one batched launch, then the
level's reflectors are broadcast, then level L+1 starts.  No reduction is
needed anywhere: R_kj is computed where column j lives.

The driver is written against a small ``Store`` interface so the protocol
(ownership, message order, payload layout) is shared by the GPU store below
and by the oracle-backed store of the gloo tests.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

DIAG, BLOCK, UPDATE, TRAP = 0, 1, 2, 3


def task_owner(task, world: int) -> int:
    kind, k, i, j = (int(x) for x in task)
    return (k if kind in (DIAG, UPDATE) else j) % world


def column_owner(j: int, world: int) -> int:
    return j % world


def level_plan(tasks: np.ndarray, level_start: np.ndarray, world: int, rank: int):
    """Per level: (this rank's tasks, reflector-producing tasks of the level in
    canonical (k, i) order).  ``tasks`` / ``level_start`` are the global
    schedule (factorize.tiled_schedule)."""
    plan = []
    for lv in range(len(level_start) - 1):
        blk = tasks[level_start[lv]:level_start[lv + 1]]
        own = np.array([task_owner(t, world) == rank for t in blk], dtype=bool)
        refl = [tuple(int(x) for x in t) for t in blk if t[0] in (DIAG, UPDATE)]
        refl.sort(key=lambda t: (t[1], t[2]))
        plan.append((blk[own], refl))
    return plan


def run_tiled_distributed(store, plan, world: int, rank: int, broadcast) -> None:
    """Drive the level-synchronous distributed tiled factorization.

    store.run(level, tasks)       -- execute this rank's tasks of one level
    store.reflector_buffers(t)    -- tensors holding reflector t's payload
                                     (filled on the owner, overwritten elsewhere)
    store.received(t, buffers)    -- unpack on non-owners (no-op when in place)
    broadcast(tensor, src)        -- in-place collective broadcast
    """
    for lv, (own, refl) in enumerate(plan):
        if len(own):
            store.run(lv, own)
        if world > 1:
            for t in refl:
                src = task_owner(t, world)
                bufs = store.reflector_buffers(t)
                for buf in bufs:
                    broadcast(buf, src)
                if src != rank:
                    store.received(t, bufs)
    store.finish()


class GpuStore:
    """A rank's device grid + reflector store (full-size layout; only the
    owned columns and the received reflectors are ever touched)."""

    def __init__(self, grid, cfg, world: int, rank: int):
        from . import _lib
        from .device import DeviceRefl
        from .factorize import tiled_schedule

        self.lib = _lib
        self.rt = _lib.runtime()
        self.g = grid
        self.rf = DeviceRefl(grid)
        self.cfg = cfg
        tasks, levels = tiled_schedule(grid.p, grid.q)
        self.plan = level_plan(tasks, levels, world, rank)
        # one device task list for all owned tasks, level by level
        own = [blk for blk, _ in self.plan]
        self.level_start = np.zeros(len(own) + 1, dtype=np.int64)
        for lv, blk in enumerate(own):
            self.level_start[lv + 1] = self.level_start[lv] + len(blk)
        allt = np.concatenate([b for b in own if len(b)] or [np.zeros((0, 4), dtype=np.int32)])
        self.tasks = torch.from_numpy(np.ascontiguousarray(allt, dtype=np.int32)).to(self.rt.dev)
        b, q = grid.b, grid.q
        self.b, self.q = b, q

    def run(self, lv, own):
        rt, g = self.rt, self.g
        ws, per, nct = rt.workspace(g.b, g.cap)
        gs, rs = g.cstruct(), self.rf.cstruct()
        self.lib.check(rt.lib.blrqr_tiled_run(C.byref(gs), C.byref(rs), self.tasks.data_ptr(),
                                              self.level_start.ctypes.data_as(C.c_void_p), lv, lv + 1,
                                              self.cfg.epsilon, ws, per, nct, rt.status.data_ptr(),
                                              rt.flops.data_ptr(), self.lib.stream_ptr()), "tiled_run")

    def received(self, t, bufs):
        pass  # broadcasts land in place

    def reflector_buffers(self, t):
        kind, k, i, _ = t
        g, rf, b = self.g, self.rf, self.b
        if kind == DIAG:
            c = k * self.q + k
            y = int(rf.y_off_host[c])
            return [rf.pool[y:y + 2 * b * b]]  # Y_kk then T_kk (adjacent)
        c = i * self.q + k
        to = int(rf.t_off_host[c])
        bufs = []
        if g.kind_host[i, k]:
            ou = int(g.off_u_host[c])
            bufs.append(g.pool[ou:ou + 2 * b * g.cap])  # U slab then V slab (holds Y^T)
        else:
            y = int(rf.y_off_host[c])
            bufs.append(rf.pool[y:y + b * b])
        bufs.append(rf.pool[to:to + b * b])
        bufs.append(rf.yrank[c:c + 1])
        return bufs

    def finish(self):
        pass


def factorize_distributed(grid, cfg, world: int, rank: int, broadcast=None):
    """Distributed tiled-hh on this rank's GPU.  ``grid`` holds the full input
    (only owned columns are read).  Returns the GpuStore; owned columns of
    store.g hold R-tilde, store.rf the reflectors of every column."""
    if broadcast is None:
        import torch.distributed as dist

        def broadcast(t, src):
            dist.broadcast(t, src)
    st = GpuStore(grid, cfg, world, rank)
    run_tiled_distributed(st, st.plan, world, rank, broadcast)
    return st
