"""Execution engines with the reference API (scheduler.py).

On the GPU the three reference engines collapse onto one device driver per
method: independent tasks of a step / DAG level run as concurrent CTAs of
one launch.  The results are those of the sequential order (every task
accumulates internally in the reference's fixed order), so
``execute_sequential``, ``execute_forkjoin`` and ``execute_taskgraph`` return
identical factorizations, exactly like the reference's bitwise guarantee
(scheduler.py:1-11).  ``threads`` is accepted for API compatibility and
ignored; ``BLRQR_THREADS`` likewise.

The tiled DAG itself (``build_tiled_dag``, scheduler.py:173-201) comes from
libblrqr.so (``blrqr_tiled_ref_dag``): the C++ builder that also derives the
device schedules, run on the reference's task set; this module only wraps
its CSR arrays in the reference's ``Task`` / ``TaskDag`` containers so
callers can inspect it (DOT output, levels, edge sets).
"""

from __future__ import annotations

import enum
import os
from dataclasses import dataclass, field

import numpy as np

from .core import BlrMatrix
from .factorize import FactorizationResult, _host_entry
from .lowrank import ToleranceConfig

__all__ = ["TaskKind", "Task", "TaskDag", "build_tiled_dag", "execute_sequential", "execute_forkjoin",
           "execute_taskgraph", "resolve_threads", "ALGORITHMS", "tiled_sequential_tasks"]

ALGORITHMS = ("mgs", "blocked-hh", "tiled-hh")
THREADS_ENV = "BLRQR_THREADS"


def resolve_threads(requested: int | None) -> int:
    env = os.environ.get(THREADS_ENV)
    if env:
        return max(1, int(env))
    return max(1, requested or 1)


class TaskKind(enum.Enum):
    DIAG_QR = "DiagQR"
    PANEL_QR = "PanelQR"
    UPDATE_QR = "UpdateQR"
    APPLY_BLOCK_REFLECTOR = "ApplyBlockReflector"
    APPLY_TRAP_REFLECTOR = "ApplyTrapReflector"
    APPLY_COLUMN_REFLECTOR = "ApplyColumnReflector"
    MGS_PROJECT = "MgsProject"
    MGS_UPDATE = "MgsUpdate"


_PRIORITY_RANK = {TaskKind.DIAG_QR: 0, TaskKind.PANEL_QR: 0, TaskKind.UPDATE_QR: 1,
                  TaskKind.APPLY_TRAP_REFLECTOR: 2, TaskKind.APPLY_BLOCK_REFLECTOR: 2,
                  TaskKind.APPLY_COLUMN_REFLECTOR: 2, TaskKind.MGS_PROJECT: 1, TaskKind.MGS_UPDATE: 2}


@dataclass(frozen=True)
class Task:
    kind: TaskKind
    k: int = -1
    i: int = -1
    j: int = -1

    @property
    def priority(self) -> int:
        return _PRIORITY_RANK[self.kind]

    def sort_key(self):
        return (self.priority, self.k, self.i, self.j)

    def __str__(self) -> str:
        return f"{self.kind.value}({','.join(str(c) for c in (self.k, self.i, self.j) if c >= 0)})"


_KINDS = (TaskKind.DIAG_QR, TaskKind.APPLY_BLOCK_REFLECTOR, TaskKind.UPDATE_QR, TaskKind.APPLY_TRAP_REFLECTOR)


def _ref_dag_arrays(p: int, q: int):
    """(tasks[n, 4] int32 (kind, k, i, j), succ_off[n + 1], succ[e]) from libblrqr."""
    from . import _lib
    lib = _lib.load()
    n = int(lib.blrqr_tiled_task_count(p, q))
    if n < 0:
        raise ValueError("need p >= q >= 1")
    ne = int(lib.blrqr_tiled_ref_dag(p, q, None, None, None, 0))
    tasks = np.zeros((n, 4), dtype=np.int32)
    off = np.zeros(n + 1, dtype=np.int64)
    succ = np.zeros(max(ne, 1), dtype=np.int32)
    rc = lib.blrqr_tiled_ref_dag(p, q, tasks.ctypes.data, off.ctypes.data, succ.ctypes.data, ne)
    if rc != ne:
        raise RuntimeError("tiled DAG build failed")
    return tasks, off, succ[:ne]


def _task(row) -> Task:
    kind, k, i, j = (int(x) for x in row)
    return Task(_KINDS[kind], k=k, i=i, j=j)


def tiled_sequential_tasks(p: int, q: int) -> list[Task]:
    """Sweep order of the tiled method (scheduler.py:127-138)."""
    return [_task(r) for r in _ref_dag_arrays(p, q)[0]]


@dataclass
class TaskDag:
    nodes: list
    edges: set
    successors: list = field(default_factory=list)
    indegree: list = field(default_factory=list)

    def __post_init__(self):
        if not self.successors:
            self.successors = [[] for _ in self.nodes]
            self.indegree = [0] * len(self.nodes)
            for u, v in sorted(self.edges):
                self.successors[u].append(v)
                self.indegree[v] += 1

    def edge_tasks(self):
        return {(self.nodes[u], self.nodes[v]) for u, v in self.edges}

    def topological_order(self):
        return list(self.nodes)

    def levels(self) -> list[int]:
        lev = [0] * len(self.nodes)
        for u in range(len(self.nodes)):
            for v in self.successors[u]:
                lev[v] = max(lev[v], lev[u] + 1)
        return lev

    def to_dot(self) -> str:
        lines = ["digraph blrqr {"]
        lines += [f'  "{t}" [label="{t}"];' for t in self.nodes]
        lines += [f'  "{self.nodes[u]}" -> "{self.nodes[v]}";' for u, v in sorted(self.edges)]
        lines.append("}")
        return "\n".join(lines)


def build_tiled_dag(p: int, q: int) -> TaskDag:
    """scheduler.py:173-201: edges from last-writer / readers-since conflicts in
    sweep order, built by libblrqr's C++ DAG builder."""
    if not 1 <= q <= p:
        raise ValueError("need p >= q >= 1")
    tasks, off, succ = _ref_dag_arrays(p, q)
    nodes = [_task(r) for r in tasks]
    src = np.repeat(np.arange(len(nodes), dtype=np.int64), np.diff(off))
    edges = set(zip(src.tolist(), succ.astype(np.int64).tolist()))
    return TaskDag(nodes, edges)


def execute_sequential(algorithm: str, a: BlrMatrix, cfg: ToleranceConfig) -> FactorizationResult:
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    return _host_entry(algorithm, a, cfg)


def execute_forkjoin(algorithm: str, a: BlrMatrix, cfg: ToleranceConfig, threads: int) -> FactorizationResult:
    return execute_sequential(algorithm, a, cfg)


def execute_taskgraph(dag: TaskDag, a: BlrMatrix, cfg: ToleranceConfig, threads: int) -> FactorizationResult:
    expected = tiled_sequential_tasks(a.p, a.q)
    if len(expected) != len(dag.nodes) or set(expected) != set(dag.nodes):
        raise ValueError("DAG does not match the operand's grid")
    return _host_entry("tiled-hh", a, cfg)
