"""Multi-GPU BLR-QR: 1-D block-cyclic columns + panel broadcast.

All three methods.  Tiled Householder is described first; blocked
Householder and blocked MGS (``run_column_distributed``) follow the same
ownership with one broadcast per panel.

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


def run_tiled_distributed(store, plan, world: int, rank: int, broadcast, allreduce=None) -> None:
    """Drive the level-synchronous distributed tiled factorization.

    store.run(level, tasks)       -- execute this rank's tasks of one level
    store.level_ranks(refl)       -- optional: int32 tensor, the Ytilde rank of
                                     each of the level's reflectors this rank
                                     produced (0 elsewhere); summed over ranks
                                     (allreduce) and handed back through
                                     store.set_level_ranks, so every payload
                                     below is sized by its rank (b * r), not by
                                     the slab capacity -- one small collective
                                     and one host read per level
    store.reflector_buffers(t)    -- tensors holding reflector t's payload
                                     (filled on the owner, overwritten elsewhere)
    store.received(t, buffers)    -- unpack on non-owners (no-op when in place)
    broadcast(tensor, src)        -- in-place collective broadcast
    allreduce(tensor)             -- in-place sum over ranks
    """
    for lv, (own, refl) in enumerate(plan):
        if len(own):
            store.run(lv, own)
        if world > 1:
            if refl and hasattr(store, "level_ranks"):
                hdr = store.level_ranks(refl)
                allreduce(hdr)
                store.set_level_ranks(refl, hdr)
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
    owned columns and the received reflectors are ever touched).

    Built once per grid shape (schedule, ownership plan and device task list:
    host work that stays out of any timed region); ``reset`` re-arms it for a
    new input.  Reflector payloads are sized by rank: the Ytilde ranks of a
    level are exchanged first (one all-reduce of an int vector), then only
    b * r columns of U_ik and of Y_i^T travel, not the 2 b cap slabs."""

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
        self.world, self.rank = world, rank
        self._ranks = {}

    def reset(self, grid) -> None:
        """Re-arm for a new input of the same structure (the schedule, plan and
        reflector store are reused; the store's contents are rewritten by the run)."""
        self.g = grid
        self.rf.grid = grid
        self.rf.yrank.fill_(-1)
        self._ranks = {}

    def level_ranks(self, refl):
        dev = self.rf.yrank.device
        rk = torch.zeros(len(refl), dtype=torch.int32, device=dev)
        sel = [(n, t[2] * self.q + t[1]) for n, t in enumerate(refl)
               if t[0] == UPDATE and task_owner(t, self.world) == self.rank]
        if sel:
            pos = torch.tensor([x[0] for x in sel], dtype=torch.int64, device=dev)
            cel = torch.tensor([x[1] for x in sel], dtype=torch.int64, device=dev)
            rk[pos] = self.rf.yrank[cel].clamp(min=0)
        return rk

    def set_level_ranks(self, refl, hdr):
        for t, r in zip(refl, hdr.cpu().tolist()):
            self._ranks[t] = int(r)

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
            r = self._ranks.get(t)
            if r is None:  # no rank exchange (single process / emulation): whole slabs
                bufs.append(g.pool[ou:ou + 2 * b * g.cap])  # U slab then V slab (holds Y^T)
            elif r > 0:  # U_ik (b x r) and Y_i^T (b x r) at the head of the U / V slabs
                bufs.append(g.pool[ou:ou + b * r])
                bufs.append(g.pool[ou + b * g.cap:ou + b * g.cap + b * r])
        else:
            y = int(rf.y_off_host[c])
            bufs.append(rf.pool[y:y + b * b])
        bufs.append(rf.pool[to:to + b * b])
        bufs.append(rf.yrank[c:c + 1])
        return bufs

    def finish(self):
        pass


def factorize_distributed(grid, cfg, world: int, rank: int, broadcast=None, allreduce=None, store=None):
    """Distributed tiled-hh on this rank's GPU.  ``grid`` holds the full input
    (only owned columns are read).  Returns the GpuStore; owned columns of
    store.g hold R-tilde, store.rf the reflectors of every column.  Pass a
    previously built ``store`` to reuse its plan (it is reset to ``grid``)."""
    import torch.distributed as dist
    if broadcast is None:
        def broadcast(t, src):
            dist.broadcast(t, src)
    if allreduce is None:
        def allreduce(t):
            dist.all_reduce(t)
    st = store if store is not None else GpuStore(grid, cfg, world, rank)
    if store is not None:
        st.reset(grid)
    run_tiled_distributed(st, st.plan, world, rank, broadcast, allreduce)
    return st


# ---------------------------------------------------------------------------
# blocked Householder and blocked MGS
# ---------------------------------------------------------------------------
# Both methods are "factor panel c, then update every column right of c
# independently" (factorize.py:285-292, :661-671).  Column c's owner runs the
# panel (triangularize_block_column, factorize.py:187-229 / MgsState.panel,
# :605-632) and broadcasts its payload -- the ReflectorColumn (y_kk, T_k and
# every Ytilde_ik) for blocked HH, the explicit Q column j for MGS -- and then
# every rank applies it to the columns it owns (apply_block_column_reflector,
# :252-262 / project + update, :634-655).  Each column's arithmetic is the
# single-GPU one (same chain order), so the assembled result is bitwise the
# single-GPU factorization.


def run_column_distributed(store, ncols: int, world: int, rank: int, broadcast) -> None:
    """store.panel(c)             -- factor panel c (called on its owner only)
    store.panel_buffers(c)       -- tensors holding panel c's payload
    store.received(c, buffers)   -- unpack on non-owners (no-op when in place)
    store.apply(c)               -- apply panel c to this rank's columns > c
    broadcast(tensor, src)       -- in-place collective broadcast"""
    for c in range(ncols):
        src = column_owner(c, world)
        if src == rank:
            store.panel(c)
        if world > 1:
            bufs = store.panel_buffers(c)
            for buf in bufs:
                broadcast(buf, src)
            if src != rank:
                store.received(c, bufs)
        store.apply(c)
    store.finish()


class _ColumnGpuStore:
    def __init__(self, world: int, rank: int, cfg):
        from . import _lib

        self.lib = _lib
        self.rt = _lib.runtime()
        self.world, self.rank, self.cfg = world, rank, cfg

    def _cell_payload(self, g, i, j):
        """Views of cell (i, j)'s storage: U and V slabs (LR) or the block."""
        c = i * g.q + j
        o = int(g.off_u_host[c])
        if g.kind_host[i, j]:
            return [g.pool[o:o + 2 * g.b * g.cap], g.rank[c:c + 1]]  # U slab then V slab
        return [g.pool[o:o + g.b * g.b]]

    def received(self, c, bufs):
        pass  # broadcasts land in place

    def finish(self):
        pass


class BlockedGpuStore(_ColumnGpuStore):
    """A rank's device grid + reflector store for blocked Householder."""

    def __init__(self, grid, cfg, world: int, rank: int):
        from .device import DeviceRefl

        super().__init__(world, rank, cfg)
        self.g = grid
        self.rf = DeviceRefl(grid)
        dev = self.rt.dev
        self.zbuf = torch.empty(grid.q * 2 * grid.b * grid.b, dtype=torch.float64, device=dev)
        self.zrank = torch.zeros(grid.q, dtype=torch.int32, device=dev)
        self.panel_ws = torch.empty(2 * grid.p * grid.b * grid.b, dtype=torch.float64, device=dev)

    def _step(self, k, phases):
        rt, g = self.rt, self.g
        ws, per, nct = rt.workspace(g.b, g.cap)
        gs, rs = g.cstruct(), self.rf.cstruct()
        self.lib.check(rt.lib.blrqr_blocked_step_dist(
            C.byref(gs), C.byref(rs), k, self.cfg.epsilon, self.zbuf.data_ptr(), self.zrank.data_ptr(),
            self.panel_ws.data_ptr(), self.panel_ws.numel(), ws, per, nct, phases, self.world, self.rank,
            rt.status.data_ptr(), rt.flops.data_ptr(), self.lib.stream_ptr()), "blocked_step_dist")

    def panel(self, k):
        self._step(k, 1)

    def apply(self, k):
        self._step(k, 2)

    def panel_buffers(self, k):
        """ReflectorColumn k (factorize.py:146-156): y_kk and T_k (adjacent in
        the store), then per i > k the Ytilde_ik payload: the LR cell's U / V
        slabs (V holds y_i^T) + yrank, or the dense Y block."""
        g, rf, b, q = self.g, self.rf, self.g.b, self.g.q
        c = k * q + k
        y = int(rf.y_off_host[c])
        bufs = [rf.pool[y:y + 2 * b * b]]
        for i in range(k + 1, g.p):
            c = i * q + k
            if g.kind_host[i, k]:
                o = int(g.off_u_host[c])
                bufs.append(g.pool[o:o + 2 * b * g.cap])
            else:
                y = int(rf.y_off_host[c])
                bufs.append(rf.pool[y:y + b * b])
            bufs.append(rf.yrank[c:c + 1])
        return bufs


class MgsGpuStore(_ColumnGpuStore):
    """A rank's device grids (A, explicit Q, R) for blocked MGS."""

    def __init__(self, grid, cfg, world: int, rank: int):
        from .device import DeviceGrid

        super().__init__(world, rank, cfg)
        g = grid
        self.g = g
        self.qg = DeviceGrid(g.m, g.n, g.b, g.kind_host, g.cap)
        rl = g.kind_host[: g.q, :].copy()
        d = np.arange(g.q)
        rl[d, d] = False
        self.rg = DeviceGrid(g.n, g.n, g.b, rl, g.cap)
        self.panel_ws = torch.empty(g.p * g.b * g.b, dtype=torch.float64, device=self.rt.dev)

    def _step(self, j, phases):
        rt, g = self.rt, self.g
        ws, per, nct = rt.workspace(g.b, g.cap)
        gs, qs, rs = g.cstruct(), self.qg.cstruct(), self.rg.cstruct()
        self.lib.check(rt.lib.blrqr_mgs_step_dist(
            C.byref(gs), C.byref(qs), C.byref(rs), j, self.cfg.epsilon, self.panel_ws.data_ptr(),
            self.panel_ws.numel(), ws, per, nct, phases, self.world, self.rank, rt.status.data_ptr(),
            rt.flops.data_ptr(), self.lib.stream_ptr()), "mgs_step_dist")

    def panel(self, j):
        self._step(j, 1)

    def apply(self, j):
        self._step(j, 2)

    def panel_buffers(self, j):
        """Explicit Q column j: every block of qg's column j."""
        bufs = []
        for i in range(self.g.p):
            bufs += self._cell_payload(self.qg, i, j)
        return bufs


def factorize_columns_distributed(method: str, grid, cfg, world: int, rank: int, broadcast=None):
    """Distributed blocked-hh / mgs on this rank's GPU.  ``grid`` holds the
    full input (only owned columns are read and written).  Returns the store:
    owned columns of store.g (blocked) / store.rg (mgs) hold R-tilde."""
    if broadcast is None:
        import torch.distributed as dist

        def broadcast(t, src):
            dist.broadcast(t, src)
    if method == "blocked-hh":
        st = BlockedGpuStore(grid, cfg, world, rank)
    elif method == "mgs":
        st = MgsGpuStore(grid, cfg, world, rank)
    else:
        raise ValueError(f"column-cyclic driver covers blocked-hh and mgs, not {method!r}")
    run_column_distributed(st, grid.q, world, rank, broadcast)
    return st


# ---------------------------------------------------------------------------
# tiled Householder on per-rank dynamic DAGs with NVLink peer pushes
# ---------------------------------------------------------------------------
# The level-synchronous driver above puts a host-issued collective between
# every pair of DAG levels.  The peer-DAG driver below runs the reference's
# task-graph engine (execute_taskgraph, scheduler.py:335-416) per rank with no
# host in the loop: each rank's persistent k_tiled_dag runs the tasks of its
# columns; a reflector producer (DiagQR(k), UpdateQR(k, i)) is followed by one
# push task per peer that stores the reflector straight into the peer's
# stores over NVLink and releases the peer's dependent ApplyBlock / ApplyTrap
# tasks with system-scope atomics (blrqr_tiled_run_dag_multi).  Ownership is
# the block-cyclic one above; every rank's DAG is derived from the same global
# DAG (blrqr_tiled_dist_dag), so the operation sequence on each cell, and
# hence R-tilde and every reflector, is bitwise the single-GPU result.

PUSH = 8


def dist_dag_arrays(p: int, q: int, world: int, rank: int):
    """Rank's DAG (numpy): tasks[n, 4], indeg, succ_off, succ, prio, rsucc_off, rsucc."""
    from . import _lib
    lib = _lib.load()
    ne, nr = C.c_int64(0), C.c_int64(0)
    n = int(lib.blrqr_tiled_dist_dag_size(p, q, world, rank, C.byref(ne), C.byref(nr)))
    if n < 0:
        raise ValueError(f"bad distributed DAG shape p={p} q={q} world={world} rank={rank} ({n})")
    a = {"tasks": np.zeros((n, 4), dtype=np.int32), "indeg": np.zeros(n, dtype=np.int32),
         "off": np.zeros(n + 1, dtype=np.int64), "succ": np.zeros(max(ne.value, 1), dtype=np.int32),
         "prio": np.zeros(n, dtype=np.int32), "roff": np.zeros(n + 1, dtype=np.int64),
         "rsucc": np.zeros(max(nr.value, 1), dtype=np.int32)}
    rc = lib.blrqr_tiled_dist_dag(p, q, world, rank, *(a[k].ctypes.data for k in
                                                        ("tasks", "indeg", "off", "succ", "prio", "roff", "rsucc")))
    if rc != 0:
        raise RuntimeError(f"distributed DAG build failed ({rc})")
    return a


class PeerDagStore:
    """One rank's device state for the peer-DAG driver: its copy of the grid
    (the full layout, so reflector offsets agree on every rank; only owned
    columns are written by its tasks, remote columns receive the pushed
    reflectors), its reflector store, and its DAG arrays.  Built once per
    shape (host DAG derivation stays out of timed regions); ``reset`` re-arms
    it for a new input."""

    def __init__(self, grid, cfg, world: int, rank: int):
        from . import _lib
        from .device import DeviceRefl

        if world < 1 or world > _lib.MAX_WORLD or not 0 <= rank < world:
            raise ValueError(f"world must be 1..{_lib.MAX_WORLD} and 0 <= rank < world")
        self.lib = _lib
        self.rt = _lib.runtime()
        self.cfg = cfg
        self.world, self.rank = world, rank
        self.g = grid
        self.rf = DeviceRefl(grid)
        self.rf.enable_split_traps()
        a = dist_dag_arrays(grid.p, grid.q, world, rank)
        self.host = a
        dev = self.rt.dev
        self.n = len(a["tasks"])
        self.dev = {k: torch.from_numpy(v).to(dev) for k, v in a.items()}
        self.work = torch.empty(int(self.rt.lib.blrqr_dag_work_ints(self.n)), dtype=torch.int32, device=dev)

    def reset(self, grid) -> None:
        self.g = grid
        self.rf.grid = grid
        self.rf.yrank.fill_(-1)

    def dag_rank(self):
        d = self.dev
        r = self.lib.DagRank()
        r.g, r.rf = self.g.cstruct(), self.rf.cstruct()
        r.ntasks = self.n
        r.tasks, r.indeg0 = d["tasks"].data_ptr(), d["indeg"].data_ptr()
        r.succ_off, r.succ, r.prio = d["off"].data_ptr(), d["succ"].data_ptr(), d["prio"].data_ptr()
        r.rsucc_off, r.rsucc = d["roff"].data_ptr(), d["rsucc"].data_ptr()
        r.work = self.work.data_ptr()
        return r

    def peer_tensors(self):
        """The tensors other ranks write into or read: grid pool, reflector
        pool, yrank, scheduler work area, priorities."""
        return [self.g.pool, self.rf.pool, self.rf.yrank, self.work, self.dev["prio"]]

    def local_peer(self):
        return self._peer([t.data_ptr() for t in self.peer_tensors()], self.n)

    def _peer(self, ptrs, n):
        p = self.lib.Peer()
        p.gpool, p.rpool, p.yrank, p.work, p.prio = ptrs
        p.ntasks = n
        return p


def _launch(stores, peers, rank_ids, world, nctas=None):
    """Reset the hosted ranks' scheduler state, then one persistent launch."""
    from . import _lib
    from .factorize import DAG_TIMEOUT_S
    rt = stores[0].rt
    g = stores[0].g
    nr = len(stores)
    ranks = (_lib.DagRank * nr)(*[s.dag_rank() for s in stores])
    _lib.check(rt.lib.blrqr_tiled_dag_reset(nr, C.addressof(ranks), _lib.stream_ptr()), "tiled_dag_reset")
    return ranks


def _run(stores, ranks, peers, rank_ids, world, nctas=None):
    from . import _lib
    from .factorize import DAG_TIMEOUT_S
    rt = stores[0].rt
    g = stores[0].g
    ws, per, nct = rt.workspace(g.b, g.cap, 0, nctas)
    nr = len(stores)
    ids = (C.c_int * nr)(*rank_ids)
    pa = (_lib.Peer * world)(*peers) if world > 1 else None
    _lib.check(rt.lib.blrqr_tiled_run_dag_multi(
        world, nr, C.addressof(ids), C.addressof(ranks), C.addressof(pa) if pa is not None else None,
        stores[0].cfg.epsilon, ws, per, nct, DAG_TIMEOUT_S, rt.status.data_ptr(), rt.flops.data_ptr(),
        _lib.stream_ptr()), "tiled_run_dag_multi")


def factorize_peer_dag_emulated(grid, cfg, world: int, stores=None):
    """All `world` ranks of the peer-DAG protocol in ONE persistent launch on
    this GPU (CTA block r runs rank r's DAG; pushes go to the other ranks'
    copies on the same device).  Each rank gets its own clone of ``grid``.
    This exercises the exact device protocol -- push tasks, remote releases,
    per-rank DAGs -- without ranks in separate kernels waiting on one another.
    Returns the stores (rank r's owned columns hold R-tilde)."""
    if stores is None:
        stores = [PeerDagStore(grid.clone(), cfg, world, r) for r in range(world)]
    else:
        for s in stores:
            s.reset(grid.clone())
    peers = [s.local_peer() for s in stores]
    ranks = _launch(stores, peers, list(range(world)), world)
    _run(stores, ranks, peers, list(range(world)), world)
    return stores


class PeerDagRank:
    """One process per GPU: this rank's PeerDagStore plus the other ranks'
    memory opened through CUDA IPC (exchanged once with all_gather_object)."""

    def __init__(self, grid, cfg, world: int, rank: int, group=None):
        import torch.distributed as dist
        from . import _lib

        self.store = PeerDagStore(grid, cfg, world, rank)
        self.world, self.rank = world, rank
        self.group = group
        lib = self.store.rt.lib
        _lib.check(lib.blrqr_enable_peer_access(), "enable_peer_access")
        mine = []
        for t in self.store.peer_tensors():
            h = (C.c_char * 64)()
            off = C.c_int64(0)
            _lib.check(lib.blrqr_ipc_handle(t.data_ptr(), C.addressof(h), C.byref(off)), "ipc_handle")
            mine.append((bytes(h), int(off.value)))
        allh = [None] * world
        dist.all_gather_object(allh, (mine, self.store.n), group=group)
        self._opened = []
        self.peers = []
        for r in range(world):
            if r == rank:
                self.peers.append(self.store.local_peer())
                continue
            ptrs = []
            for hb, off in allh[r][0]:
                base = C.c_void_p()
                hbuf = (C.c_char * 64).from_buffer_copy(hb)
                _lib.check(lib.blrqr_ipc_open(C.addressof(hbuf), C.byref(base)), "ipc_open")
                self._opened.append(base.value)
                ptrs.append(base.value + off)
            self.peers.append(self.store._peer(ptrs, allh[r][1]))

    def run(self, grid=None, nctas=None):
        """Reset (every rank, then a barrier: no push may land in a rank that
        has not re-armed), then this rank's persistent launch (no host sync)."""
        import torch.distributed as dist
        if grid is not None:
            self.store.reset(grid)
        ranks = _launch([self.store], self.peers, [self.rank], self.world)
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        _run([self.store], ranks, self.peers, [self.rank], self.world, nctas)
        return self.store

    def close(self):
        lib = self.store.rt.lib
        for b in self._opened:
            lib.blrqr_ipc_close(b)
        self._opened = []
