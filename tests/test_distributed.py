"""Multi-rank (gloo, world_size 2 and 3, CPU) test of the distributed tiled
protocol: block-cyclic ownership, per-level reflector broadcasts in canonical
order.  The per-rank compute here is the CPU oracle (test-only store); the
GPU store shares the driver (paper_2208_06194_b200.distributed).  Every rank's
owned columns of R and every reflector must equal the single-process oracle
bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import algorithms as oalg, blr as oblr, configs, schedule
from paper_2208_06194_b200 import distributed as D


def _tiled_schedule_py(p, q):
    """Level schedule from the oracle DAG (no GPU library needed)."""
    tasks, _ = schedule.tiled_dag(p, q)
    lev = schedule.levels(p, q)
    kinds = {"diag": 0, "block": 1, "update": 2, "trap": 3}
    prio = {0: 0, 2: 1, 1: 2, 3: 2}
    arr = np.array([[kinds[t[0]], t[1], t[2], t[3]] for t in tasks], dtype=np.int32)
    order = sorted(range(len(arr)), key=lambda t: (lev[t], prio[arr[t, 0]], arr[t, 1], arr[t, 2], arr[t, 3]))
    arr = arr[order]
    lv = np.array([lev[t] for t in order])
    starts = np.searchsorted(lv, np.arange(lv.max() + 2))
    return arr, starts


class OracleStore:
    """Test-only store: oracle TiledState + flat payload tensors."""

    def __init__(self, g, eps):
        self.st = oalg.TiledState.start(g, eps)
        self.b = g.b
        self.names = {0: "diag", 1: "block", 2: "update", 3: "trap"}

    def run(self, lv, own):
        for t in own:
            oalg.run_tiled_task(self.st, (self.names[int(t[0])], int(t[1]), int(t[2]), int(t[3])))

    def reflector_buffers(self, t):
        kind, k, i, _ = t
        b = self.b
        if kind == D.DIAG:
            buf = torch.zeros(2 * b * b, dtype=torch.float64)
            if k in self.st.diag:
                y, tt = self.st.diag[k]
                buf[: b * b] = torch.from_numpy(y.ravel())
                buf[b * b:] = torch.from_numpy(tt.ravel())
            return [buf]
        hdr = torch.zeros(2, dtype=torch.float64)
        data = torch.zeros(3 * b * b, dtype=torch.float64)
        if (i, k) in self.st.upd:
            y, tt = self.st.upd[(i, k)]
            if oblr.is_lr(y):
                r = y.rank
                hdr[0], hdr[1] = r, 1
                data[: b * r] = torch.from_numpy(y.u.ravel())
                data[b * b: b * b + b * r] = torch.from_numpy(y.v.ravel())
            else:
                hdr[0], hdr[1] = b, 0
                data[: b * b] = torch.from_numpy(y.ravel())
            data[2 * b * b:] = torch.from_numpy(tt.ravel())
        return [hdr, data]

    def received(self, t, bufs):
        kind, k, i, _ = t
        b = self.b
        if kind == D.DIAG:
            x = bufs[0].numpy()
            self.st.diag[k] = (x[: b * b].reshape(b, b).copy(), x[b * b:].reshape(b, b).copy())
            return
        hdr, data = bufs[0].numpy(), bufs[1].numpy()
        r, lr = int(hdr[0]), int(hdr[1])
        tt = data[2 * b * b:].reshape(b, b).copy()
        if lr:
            y = oblr.LR(data[: b * r].reshape(b, r).copy(), data[b * b: b * b + b * r].reshape(b, r).copy())
        else:
            y = data[: b * b].reshape(b, b).copy()
        self.st.upd[(i, k)] = (y, tt)

    def finish(self):
        pass


def _worker(rank, world, port, out):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n, b, eps = 256, 32, 1e-8
        dense = configs.random16_dense(n, b, 0, rank=8)
        g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
        tasks, starts = _tiled_schedule_py(g.p, g.q)
        plan = D.level_plan(tasks, starts, world, rank)
        store = OracleStore(g, eps)
        D.run_tiled_distributed(store, plan, world, rank, lambda t, src: dist.broadcast(t, src))
        ref = oalg.tiled_hh(g, eps)
        ok = True
        for j in range(g.q):
            if D.column_owner(j, world) != rank:
                continue
            for i in range(g.p):
                a, r = store.st.g[i, j], ref.g[i, j]
                da = a.dense() if oblr.is_lr(a) else a
                dr = r.dense() if oblr.is_lr(r) else r
                ok &= np.array_equal(da, dr)
        for key, (y, t) in ref.upd.items():
            y2, t2 = store.st.upd[key]
            ok &= np.array_equal(t, t2)
            ok &= np.array_equal(y.dense() if oblr.is_lr(y) else y, y2.dense() if oblr.is_lr(y2) else y2)
        out[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_tiled_matches_single_process(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert dict(out) == {r: True for r in range(world)}


def test_ownership_and_plan():
    tasks, starts = _tiled_schedule_py(6, 5)
    for world in (1, 2, 4):
        seen = 0
        for rank in range(world):
            plan = D.level_plan(tasks, starts, world, rank)
            for own, refl in plan:
                seen += len(own)
                for t in own:
                    assert D.task_owner(t, world) == rank
                # reflectors in canonical (k, i) order, same list on every rank
                assert refl == sorted(refl, key=lambda t: (t[1], t[2]))
        assert seen == len(tasks)


# ---------------------------------------------------------------------------
# blocked Householder / blocked MGS: column-cyclic driver with one broadcast
# per panel
# ---------------------------------------------------------------------------

def _encode_blocks(blocks, b):
    """[(rank or -1, block)] -> (hdr int64 tensor, data float64 tensor); a
    low-rank block (u, v) occupies 2 b*b slots, a dense one the first."""
    hdr = torch.full((len(blocks),), -2, dtype=torch.int64)
    data = torch.zeros(len(blocks) * 2 * b * b, dtype=torch.float64)
    for n_, x in enumerate(blocks):
        if x is None:
            continue
        o = n_ * 2 * b * b
        if oblr.is_lr(x):
            r = x.rank
            hdr[n_] = r
            data[o:o + b * r] = torch.from_numpy(np.ascontiguousarray(x.u).ravel())
            data[o + b * b:o + b * b + b * r] = torch.from_numpy(np.ascontiguousarray(x.v).ravel())
        else:
            hdr[n_] = -1
            data[o:o + b * b] = torch.from_numpy(np.ascontiguousarray(x).ravel())
    return [hdr, data]


def _decode_blocks(bufs, b):
    hdr, data = bufs[0].numpy(), bufs[1].numpy()
    out = []
    for n_, r in enumerate(hdr):
        o = n_ * 2 * b * b
        if r == -1:
            out.append(data[o:o + b * b].reshape(b, b).copy())
        else:
            r = int(r)
            out.append(oblr.LR(data[o:o + b * r].reshape(b, r).copy(), data[o + b * b:o + b * b + b * r].reshape(b, r).copy()))
    return out


class OracleBlockedStore:
    """Test-only store: oracle BlockedState; payload = ReflectorColumn k."""

    def __init__(self, g, eps, world, rank):
        self.st = oalg.BlockedState.start(g, eps)
        self.b, self.world, self.rank = g.b, world, rank

    def panel(self, k):
        self.st.panel(k)

    def panel_buffers(self, k):
        g = self.st.g
        if len(self.st.cols) > k:
            col = self.st.cols[k]
            blocks = [col.t] + [y for _, y in col.entries]
        else:
            blocks = [None] * (1 + g.p - k)
        return _encode_blocks(blocks, self.b)

    def received(self, k, bufs):
        blocks = _decode_blocks(bufs, self.b)
        g = self.st.g
        self.st.cols.append(oalg.ColumnReflector(k, list(zip(range(k, g.p), blocks[1:])), blocks[0]))

    def apply(self, k):
        for j in range(k + 1, self.st.g.q):
            if D.column_owner(j, self.world) == self.rank:
                self.st.apply_column(k, j)

    def finish(self):
        pass


class OracleMgsStore:
    """Test-only store: oracle MgsState; payload = explicit Q column j."""

    def __init__(self, g, eps, world, rank):
        self.st = oalg.MgsState(g, eps)
        self.b, self.world, self.rank = g.b, world, rank

    def panel(self, j):
        self.st.panel(j)

    def panel_buffers(self, j):
        qg = self.st.qg
        return _encode_blocks([qg[i, j] for i in range(qg.p)], self.b)

    def received(self, j, bufs):
        for i, x in enumerate(_decode_blocks(bufs, self.b)):
            self.st.qg[i, j] = x

    def apply(self, j):
        st = self.st
        own = [k for k in range(j + 1, st.g.q) if D.column_owner(k, self.world) == self.rank]
        for k in own:
            st.project(j, k)
        for k in own:
            for i in range(st.g.p):
                st.update(j, i, k)

    def finish(self):
        pass


def _same(a, r):
    da = a.dense() if oblr.is_lr(a) else a
    dr = r.dense() if oblr.is_lr(r) else r
    return np.array_equal(da, dr)


def _column_worker(rank, world, port, method, out):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n, b, eps = 256, 32, 1e-8
        dense = configs.random16_dense(n, b, 0, rank=8)
        g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
        store = (OracleBlockedStore if method == "blocked-hh" else OracleMgsStore)(g, eps, world, rank)
        D.run_column_distributed(store, g.q, world, rank, lambda t, src: dist.broadcast(t, src))
        ok = True
        if method == "blocked-hh":
            ref = oalg.blocked_hh(g, eps)
            rg, rg_ref = store.st.g, ref.g
            for k, col in enumerate(ref.cols):
                c2 = store.st.cols[k]
                ok &= np.array_equal(col.t, c2.t)
                ok &= all(_same(y, y2) for (_, y), (_, y2) in zip(col.entries, c2.entries))
        else:
            ref = oalg.mgs_qr(g, eps)
            rg, rg_ref = store.st.rg, ref.rg
            for j in range(g.q):
                ok &= all(_same(store.st.qg[i, j], ref.qg[i, j]) for i in range(g.p))
        for j in range(g.q):
            if D.column_owner(j, world) == rank:
                ok &= all(_same(rg[i, j], rg_ref[i, j]) for i in range(rg_ref.p))
        out[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("method", ["blocked-hh", "mgs"])
def test_distributed_columns_match_single_process(method, world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_column_worker, args=(world, _free_port(), method, out), nprocs=world, join=True)
    assert dict(out) == {r: True for r in range(world)}
