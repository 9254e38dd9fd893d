"""Multi-GPU tiled Householder on per-rank DAGs with peer pushes.

CPU side of blrqr_tiled_dist_dag (the host builder in libblrqr.so; no GPU):
  * structure: the ranks' DAGs partition the single-GPU task set by column
    ownership, each producer has one push task per peer, every global edge
    is a local edge or a producer -> push -> remote release;
  * a deterministic-random event simulation of all ranks (any interleaving
    of ready tasks, remote releases as the device pushes do them) with the
    CPU oracle as the per-rank executor: each rank's state starts WITHOUT any
    reflector, receives them only through its push tasks, and must end with
    R-tilde columns and reflectors bitwise equal to the single-process oracle;
  * the same protocol over gloo, world 2 and 3: one process per rank, each
    running its rank's DAG in canonical order, push tasks as point-to-point
    sends of the reflector payload.
The device protocol itself (one launch hosting every rank on one GPU) is in
tests/test_gpu_factorize.py::test_peer_dag_emulated_bitwise."""

import copy
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import algorithms as oalg, blr as oblr, configs, schedule

D = pytest.importorskip("paper_2208_06194_b200.distributed")
NAMES = {0: "diag", 1: "block", 2: "update"}


def _lib_ok():
    try:
        from paper_2208_06194_b200 import _lib
        _lib.load()
        return True
    except Exception:  # noqa: BLE001
        return False


pytestmark = pytest.mark.skipif(not _lib_ok(), reason="libblrqr.so not built")


def _single(p, q):
    from paper_2208_06194_b200.factorize import tiled_dag_arrays
    tasks, indeg, off, succ, prio = tiled_dag_arrays(p, q)
    return tasks, off, succ


def _owner(t, world):
    kind, k, i, j = (int(x) for x in t)
    return (k if kind in (0, 2) else j) % world


@pytest.mark.parametrize("p,q,world", [(6, 6, 1), (6, 6, 2), (7, 5, 3), (8, 8, 4), (9, 9, 8)])
def test_dist_dag_structure(p, q, world):
    gt, goff, gsucc = _single(p, q)
    key = {tuple(int(x) for x in t): n for n, t in enumerate(gt)}
    dags = [D.dist_dag_arrays(p, q, world, r) for r in range(world)]
    seen = []
    for r, a in enumerate(dags):
        for t in a["tasks"]:
            if t[0] == D.PUSH:
                assert 0 <= t[3] < world and t[3] != r
            else:
                assert _owner(t, world) == r
                seen.append(tuple(int(x) for x in t))
    assert sorted(seen) == sorted(key)  # a partition of the single-GPU task set
    npush = sum(int((a["tasks"][:, 0] == D.PUSH).sum()) for a in dags)
    nprod = int(np.isin(gt[:, 0], (0, 2)).sum())
    assert npush == nprod * (world - 1)
    # every global edge is local, or producer -> push(producer, owner(v)) -> v
    lid = [{tuple(int(x) for x in t): n for n, t in enumerate(a["tasks"])} for a in dags]
    for u in range(len(gt)):
        tu = tuple(int(x) for x in gt[u])
        ru = _owner(tu, world)
        lsu = set(dags[ru]["succ"][dags[ru]["off"][lid[ru][tu]]:dags[ru]["off"][lid[ru][tu] + 1]].tolist())
        for e in range(goff[u], goff[u + 1]):
            tv = tuple(int(x) for x in gt[gsucc[e]])
            rv = _owner(tv, world)
            if rv == ru:
                assert lid[rv][tv] in lsu
                continue
            assert tu[0] in (0, 2)  # only reflector reads cross ranks
            push = (D.PUSH, tu[1], tu[2] if tu[0] == 2 else -1, rv)
            pl = lid[ru][push]
            assert pl in lsu
            a = dags[ru]
            assert lid[rv][tv] in set(a["rsucc"][a["roff"][pl]:a["roff"][pl + 1]].tolist())
    # in-degrees: local edges + one per remote release
    for r, a in enumerate(dags):
        ind = np.zeros(len(a["tasks"]), dtype=np.int64)
        np.add.at(ind, a["succ"][:a["off"][-1]], 1)
        for r2, b in enumerate(dags):
            if r2 != r:
                for t in range(len(b["tasks"])):
                    if b["tasks"][t, 0] == D.PUSH and b["tasks"][t, 3] == r:
                        np.add.at(ind, b["rsucc"][b["roff"][t]:b["roff"][t + 1]], 1)
        assert np.array_equal(ind, a["indeg"])
    if world == 1:
        assert np.array_equal(dags[0]["tasks"], gt)


def _input(n=256, b=32, eps=1e-8):
    dense = configs.random16_dense(n, b, 0, rank=8)
    return schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps), eps


def _exec(st, t):
    """Oracle execution of one device task; the split ApplyTrap runs whole at
    its first part (A1): its predecessors cover those of A2 and B."""
    kind, k, i, j = (int(x) for x in t)
    if kind in (0, 1, 2):
        oalg.run_tiled_task(st, (NAMES[kind], k, i, j))
    elif kind == 4:
        oalg.run_tiled_task(st, ("trap", k, i, j))


def _push_payload(st, t):
    _, k, i, _ = (int(x) for x in t)
    return ("diag", k, copy.deepcopy(st.diag[k])) if i < 0 else ("upd", (i, k), copy.deepcopy(st.upd[(i, k)]))


def _land(st, payload):
    kind, key, val = payload
    (st.diag if kind == "diag" else st.upd)[key] = val


def _check(states, ref, world, g):
    for j in range(g.q):
        st = states[j % world]
        for i in range(g.p):
            a, r = st.g[i, j], ref.g[i, j]
            assert np.array_equal(a.dense() if oblr.is_lr(a) else a, r.dense() if oblr.is_lr(r) else r), (i, j)
    for k, (y, t) in ref.diag.items():
        y2, t2 = states[k % world].diag[k]
        assert np.array_equal(y, y2) and np.array_equal(t, t2)
    for (i, k), (y, t) in ref.upd.items():
        y2, t2 = states[k % world].upd[(i, k)]
        assert np.array_equal(t, t2)
        assert np.array_equal(y.dense() if oblr.is_lr(y) else y, y2.dense() if oblr.is_lr(y2) else y2)


@pytest.mark.parametrize("world,seed", [(2, 0), (3, 1), (4, 2)])
def test_peer_dag_simulated_ranks_bitwise(world, seed):
    g, eps = _input()
    ref = oalg.tiled_hh(g, eps)
    dags = [D.dist_dag_arrays(g.p, g.q, world, r) for r in range(world)]
    states = [oalg.TiledState.start(g, eps) for _ in range(world)]  # no reflectors anywhere yet
    indeg = [a["indeg"].copy() for a in dags]
    ready = [(r, t) for r in range(world) for t in np.flatnonzero(indeg[r] == 0)]
    rng = np.random.default_rng(seed)
    done = 0
    total = sum(len(a["tasks"]) for a in dags)
    while ready:
        r, t = ready.pop(int(rng.integers(len(ready))))
        a, task = dags[r], dags[r]["tasks"][t]
        if task[0] == D.PUSH:
            to = int(task[3])
            _land(states[to], _push_payload(states[r], task))
            for v in a["rsucc"][a["roff"][t]:a["roff"][t + 1]]:
                indeg[to][v] -= 1
                if indeg[to][v] == 0:
                    ready.append((to, int(v)))
        else:
            _exec(states[r], task)
        for v in a["succ"][a["off"][t]:a["off"][t + 1]]:
            indeg[r][v] -= 1
            if indeg[r][v] == 0:
                ready.append((r, int(v)))
        done += 1
    assert done == total, "the ranks' DAGs deadlocked"
    _check(states, ref, world, g)


def _gloo_worker(rank, world, port, out):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import pickle
        g, eps = _input()
        dags = [D.dist_dag_arrays(g.p, g.q, world, r) for r in range(world)]
        a = dags[rank]
        st = oalg.TiledState.start(g, eps)
        # which of this rank's tasks wait on which peer's n-th push to this rank
        need, total = {}, {}
        for P, b in enumerate(dags):
            if P == rank:
                continue
            seq = 0
            for t in range(len(b["tasks"])):
                if b["tasks"][t, 0] == D.PUSH and b["tasks"][t, 3] == rank:
                    for v in b["rsucc"][b["roff"][t]:b["roff"][t + 1]]:
                        need.setdefault(int(v), []).append((P, seq))
                    seq += 1
            total[P] = seq
        got = {P: 0 for P in range(world)}

        def recv_from(P):
            n = torch.zeros(1, dtype=torch.int64)
            dist.recv(n, P)
            buf = torch.zeros(int(n), dtype=torch.uint8)
            dist.recv(buf, P)
            _land(st, pickle.loads(buf.numpy().tobytes()))
            got[P] += 1

        for t in range(len(a["tasks"])):  # canonical order: a topological order of the global DAG
            for P, s in need.get(t, []):
                while got[P] <= s:
                    recv_from(P)
            task = a["tasks"][t]
            if task[0] == D.PUSH:
                raw = np.frombuffer(pickle.dumps(_push_payload(st, task)), dtype=np.uint8).copy()
                dist.send(torch.tensor([raw.size], dtype=torch.int64), int(task[3]))
                dist.send(torch.from_numpy(raw), int(task[3]))
            else:
                _exec(st, task)
        for P, n in total.items():  # pushes nothing here waited on (no dependents on this rank)
            while got[P] < n:
                recv_from(P)
        ref = oalg.tiled_hh(g, eps)
        ok = True
        for j in range(g.q):
            if j % world != rank:
                continue
            for i in range(g.p):
                x, r = st.g[i, j], ref.g[i, j]
                ok &= np.array_equal(x.dense() if oblr.is_lr(x) else x, r.dense() if oblr.is_lr(r) else r)
        for (i, k), (y, t) in ref.upd.items():  # every rank ends with every reflector
            y2, t2 = st.upd[(i, k)]
            ok &= np.array_equal(t, t2)
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
def test_peer_dag_gloo_ranks_bitwise(world):
    out = mp.Manager().dict()
    mp.spawn(_gloo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
