"""Oracle task DAG and executors (test infrastructure only).

Restates scheduler.py: tiled read/write cell sets (scheduler.py:109-124), DAG
edges from last-writer / readers-since conflicts (scheduler.py:173-201) and a
threaded executor in the spirit of execute_taskgraph (scheduler.py:335-416):
ready tasks run on a thread pool ordered by (priority, k, i, j)
(scheduler.py:73-82, 98-99).  Results are bitwise identical to the
sequential order because every task accumulates internally in a fixed order.
Also ``dense_to_blr`` (core.py:227-259).
"""

from __future__ import annotations

import heapq
import threading

import numpy as np

from . import algorithms as alg
from . import lowrank as lrk
from .blr import Grid, is_lr

PRIORITY = {"diag": 0, "update": 1, "block": 2, "trap": 2}  # scheduler.py:73-82


def access(task: tuple):
    """(reads, writes) of one tiled task (scheduler.py:109-124)."""
    kind, k, i, j = task
    if kind == "diag":
        return [("A", k, k)], [("A", k, k), ("D", k, k)]
    if kind == "block":
        return [("D", k, k), ("A", k, j)], [("A", k, j)]
    if kind == "update":
        return [("A", k, k), ("A", i, k)], [("A", k, k), ("A", i, k), ("U", i, k)]
    if kind == "trap":
        return [("U", i, k), ("A", k, j), ("A", i, j)], [("A", k, j), ("A", i, j)]
    raise ValueError(f"not a tiled task: {task}")


def tiled_dag(p: int, q: int):
    """(tasks, edges) with edges as a set of (u, v) index pairs (scheduler.py:173-201)."""
    if not 1 <= q <= p:
        raise ValueError("need p >= q >= 1")
    tasks = alg.tiled_tasks(p, q)
    edges = set()
    writer, readers = {}, {}
    for t, task in enumerate(tasks):
        rd, wr = access(task)
        for cell in set(rd) | set(wr):
            w = writer.get(cell)
            if w is not None and w != t:
                edges.add((w, t))
        for cell in wr:
            for r in readers.get(cell, ()):
                if r != t:
                    edges.add((r, t))
        for cell in wr:
            writer[cell] = t
            readers[cell] = []
        for cell in rd:
            if cell not in wr:
                readers.setdefault(cell, []).append(t)
    return tasks, edges


def levels(p: int, q: int) -> list[int]:
    """Longest-path level of every task in canonical order."""
    tasks, edges = tiled_dag(p, q)
    preds = [[] for _ in tasks]
    for u, v in edges:
        preds[v].append(u)
    lev = [0] * len(tasks)
    for t in range(len(tasks)):  # canonical order is topological
        if preds[t]:
            lev[t] = 1 + max(lev[u] for u in preds[t])
    return lev


def run_taskgraph(a: Grid, eps: float, threads: int):
    """Priority ready-heap thread pool over the tiled DAG (scheduler.py:335-416)."""
    st = alg.TiledState.start(a, eps)
    tasks, edges = tiled_dag(a.p, a.q)
    succ = [[] for _ in tasks]
    indeg = [0] * len(tasks)
    for u, v in sorted(edges):
        succ[u].append(v)
        indeg[v] += 1
    key = lambda t: (PRIORITY[tasks[t][0]], tasks[t][1], tasks[t][2], tasks[t][3], t)
    ready = [key(t) for t in range(len(tasks)) if indeg[t] == 0]
    heapq.heapify(ready)
    cv = threading.Condition()
    state = {"done": 0, "running": 0, "err": None}
    total = len(tasks)

    def worker():
        while True:
            with cv:
                while not ready and state["err"] is None and state["done"] < total:
                    if state["running"] == 0:
                        state["err"] = RuntimeError("scheduler deadlock")
                        cv.notify_all()
                        return
                    cv.wait()
                if state["err"] is not None or state["done"] >= total:
                    return
                t = heapq.heappop(ready)[-1]
                state["running"] += 1
            try:
                alg.run_tiled_task(st, tasks[t])
            except BaseException as e:  # noqa: BLE001
                with cv:
                    state["err"] = e
                    state["running"] -= 1
                    cv.notify_all()
                return
            with cv:
                state["running"] -= 1
                state["done"] += 1
                for s in succ[t]:
                    indeg[s] -= 1
                    if indeg[s] == 0:
                        heapq.heappush(ready, key(s))
                cv.notify_all()

    ws = [threading.Thread(target=worker) for _ in range(max(1, threads))]
    for w in ws:
        w.start()
    for w in ws:
        w.join()
    if state["err"] is not None:
        raise state["err"]
    return st


def run_forkjoin(method: str, a: Grid, eps: float, threads: int):
    """Parallel j/k loops with barriers (scheduler.py:279-332)."""
    from concurrent.futures import ThreadPoolExecutor

    def pfor(pool, fn, args):
        for f in [pool.submit(fn, *x) for x in args]:
            f.result()

    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        if method == "blocked-hh":
            st = alg.BlockedState.start(a, eps)
            for k in range(a.q):
                st.panel(k)
                pfor(pool, st.apply_column, [(k, j) for j in range(k + 1, a.q)])
            return st
        if method == "tiled-hh":
            st = alg.TiledState.start(a, eps)
            for k in range(a.q):
                st.diag_qr(k)
                pfor(pool, st.apply_block, [(k, j) for j in range(k + 1, a.q)])
                for i in range(k + 1, a.p):
                    st.update_qr(k, i)
                    pfor(pool, st.apply_trap, [(k, i, j) for j in range(k + 1, a.q)])
            return st
        if method == "mgs":
            st = alg.MgsState(a, eps)
            for j in range(a.q):
                st.panel(j)
                pfor(pool, st.project, [(j, k) for k in range(j + 1, a.q)])
                pfor(pool, st.update, [(j, i, k) for k in range(j + 1, a.q) for i in range(a.p)])
            return st
    raise ValueError(f"unknown algorithm {method!r}")


def dense_to_blr(dense: np.ndarray, b: int, lowrank: np.ndarray, eps: float,
                 fallback: float = 0.5) -> Grid:
    """core.py:227-259: compress admissible tiles row-major; b/2 fallback."""
    m, n = dense.shape
    g = Grid(m, n, b, lowrank, [])
    lr = g.lowrank
    cells = []
    for i in range(g.p):
        row = []
        for j in range(g.q):
            tile = np.ascontiguousarray(dense[i * b:(i + 1) * b, j * b:(j + 1) * b])
            if lr[i, j]:
                x = lrk.compress(tile, eps, fallback)
                if not is_lr(x):
                    lr[i, j] = False
                row.append(x)
            else:
                row.append(tile)
        cells.append(row)
    g.cells = cells
    return g
