"""Execution engines with the reference API (scheduler.py).

On the GPU the three reference engines collapse onto one device driver per
method: independent tasks of a step / DAG level run as concurrent CTAs of
one launch.  The results are those of the sequential order (every task
accumulates internally in the reference's fixed order), so
``execute_sequential``, ``execute_forkjoin`` and ``execute_taskgraph`` return
identical factorizations, exactly like the reference's bitwise guarantee
(scheduler.py:1-11).  ``threads`` is accepted for API compatibility and
ignored; ``BLRQR_THREADS`` likewise.

The tiled DAG itself (``build_tiled_dag``, scheduler.py:173-201) is built
here on the host with the reference's read/write sets so callers can inspect
it; the device path uses the C++ level scheduler of libblrqr.so, which
derives levels from the same sets.
"""

from __future__ import annotations

import enum
import os
from dataclasses import dataclass, field

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


def _access(t: Task):
    k, i, j = t.k, t.i, t.j
    if t.kind is TaskKind.DIAG_QR:
        return [("A", k, k)], [("A", k, k), ("D", k, k)]
    if t.kind is TaskKind.APPLY_BLOCK_REFLECTOR:
        return [("D", k, k), ("A", k, j)], [("A", k, j)]
    if t.kind is TaskKind.UPDATE_QR:
        return [("A", k, k), ("A", i, k)], [("A", k, k), ("A", i, k), ("U", i, k)]
    if t.kind is TaskKind.APPLY_TRAP_REFLECTOR:
        return [("U", i, k), ("A", k, j), ("A", i, j)], [("A", k, j), ("A", i, j)]
    raise ValueError(f"not a tiled task: {t}")


def tiled_sequential_tasks(p: int, q: int) -> list[Task]:
    out = []
    for k in range(q):
        out.append(Task(TaskKind.DIAG_QR, k=k))
        out += [Task(TaskKind.APPLY_BLOCK_REFLECTOR, k=k, j=j) for j in range(k + 1, q)]
        for i in range(k + 1, p):
            out.append(Task(TaskKind.UPDATE_QR, k=k, i=i))
            out += [Task(TaskKind.APPLY_TRAP_REFLECTOR, k=k, i=i, j=j) for j in range(k + 1, q)]
    return out


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
    """Edges from last-writer / readers-since conflicts in sweep order."""
    if not 1 <= q <= p:
        raise ValueError("need p >= q >= 1")
    nodes = tiled_sequential_tasks(p, q)
    edges = set()
    writer, readers = {}, {}
    for t, task in enumerate(nodes):
        rd, wr = _access(task)
        for cell in set(rd) | set(wr):
            w = writer.get(cell)
            if w is not None and w != t:
                edges.add((w, t))
        for cell in wr:
            edges.update((r, t) for r in readers.get(cell, ()) if r != t)
        for cell in wr:
            writer[cell] = t
            readers[cell] = []
        for cell in rd:
            if cell not in wr:
                readers.setdefault(cell, []).append(t)
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
