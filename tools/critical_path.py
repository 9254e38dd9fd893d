"""Trace one dynamic-scheduler C3 run: per-task durations, DAG critical path,
SM utilisation.  python tools/critical_path.py [C3]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
from paper_2208_06194_b200 import _lib, configs
from paper_2208_06194_b200.core import weak_admissibility
from paper_2208_06194_b200.device import DeviceGrid
from paper_2208_06194_b200.factorize import DeviceFactorization, tiled_dag_arrays
from paper_2208_06194_b200.lowrank import ToleranceConfig

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = configs.CONFIGS[name]
dense = configs.dense_device(cfg)
g = DeviceGrid.from_dense(dense, cfg.b, weak_admissibility(cfg.n // cfg.b, cfg.n // cfg.b), cfg.eps, 0.5, cap=cfg.cap, colmajor=True)
del dense
tasks, indeg, off, succ, prio = tiled_dag_arrays(g.p, g.q)
n = len(tasks)
rt = _lib.runtime()
trace = torch.zeros(3 * n, dtype=torch.int64, device=rt.dev)
rt.lib.blrqr_debug_trace(trace.data_ptr())
ptrace = torch.zeros(16 * n, dtype=torch.int64, device=rt.dev)
rt.lib.blrqr_debug_phase_trace(ptrace.data_ptr())
f = DeviceFactorization("tiled-hh", g, ToleranceConfig(cfg.eps))
torch.cuda.synchronize(); t0 = time.perf_counter()
f.run(); f.finish()
torch.cuda.synchronize(); wall = time.perf_counter() - t0
rt.lib.blrqr_debug_trace(None)
rt.lib.blrqr_debug_phase_trace(None)
ph = ptrace.cpu().numpy().reshape(n, 16).astype(np.float64) / 1.965e9
tr = trace.cpu().numpy().reshape(n, 3)
st, en = tr[:, 0].astype(np.float64), tr[:, 1].astype(np.float64)
dur = (en - st) / 1e9
t0g = st.min()
# longest path with measured durations (canonical order is topological)
best = np.zeros(n)
pred = -np.ones(n, dtype=np.int64)
finish = np.zeros(n)
for t in range(n):
    finish[t] = best[t] + dur[t]
    for e in range(off[t], off[t + 1]):
        s = succ[e]
        if finish[t] > best[s]:
            best[s] = finish[t]
            pred[s] = t
end = int(np.argmax(finish))
path = []
t = end
while t >= 0:
    path.append(t)
    t = pred[t]
path = path[::-1]
kinds = ["diag", "block", "update", "trap", "trapA1", "trapB", "trapA2"]
kind_time = {k: float(dur[tasks[:, 0] == i].sum()) for i, k in enumerate(kinds)}
path_kinds = {k: 0.0 for k in kinds}
for t in path:
    path_kinds[kinds[tasks[t, 0]]] += dur[t]
path_phases = {nm: round(float(ph[path, i].sum()), 4) for i, nm in enumerate(_lib.PHASES[:13]) if ph[path, i].sum() > 0}
print(json.dumps({"wall_s": wall, "makespan_s": (en.max() - t0g) / 1e9, "sum_task_s": float(dur.sum()),
                  "sum_task_per_sm_s": float(dur.sum()) / rt.nctas, "critical_path_s": float(finish.max()),
                  "critical_path_tasks": len(path), "time_by_kind_s": kind_time, "critical_path_by_kind_s": path_kinds,
                  "critical_path_by_phase_s": path_phases,
                  "kind_stats_ms": {k: {"n": int((tasks[:, 0] == i).sum()),
                                        "mean": round(float(dur[tasks[:, 0] == i].mean() * 1e3), 3),
                                        "max": round(float(dur[tasks[:, 0] == i].max() * 1e3), 3)}
                                    for i, k in enumerate(kinds) if (tasks[:, 0] == i).any()},
                  "path_update_phases_s": {nm: round(float(ph[[t for t in path if tasks[t, 0] == 2], i].sum()), 4)
                                           for i, nm in enumerate(_lib.PHASES[:13])},
                  "top_tasks": [[kinds[tasks[t, 0]], int(tasks[t, 1]), int(tasks[t, 2]), int(tasks[t, 3]), round(float(dur[t]), 4)]
                                for t in np.argsort(-dur)[:15]],
                  "path_sample": [[kinds[tasks[t, 0]], int(tasks[t, 1]), int(tasks[t, 2]), int(tasks[t, 3]), round(float(dur[t]), 4)]
                                  for t in path[::max(1, len(path) // 25)]]}, indent=1))
if len(sys.argv) > 2:  # full path, one task per line: kind k i j seconds
    with open(sys.argv[2], "w") as fh:
        for t in path:
            extra = f" r={int(ph[t, 15] * 1.965e9)}" if tasks[t, 0] == 2 else ""
            fh.write(f"{kinds[tasks[t, 0]]} {int(tasks[t, 1])} {int(tasks[t, 2])} {int(tasks[t, 3])} {dur[t]:.5f}{extra}\n")
# phase breakdown of the longest tasks (seconds of the leader CTA's SM clock)
top = np.argsort(-dur)[:12]
print(json.dumps({"top_task_phases_ms": [
    [kinds[tasks[t, 0]], int(tasks[t, 1]), int(tasks[t, 2]), int(tasks[t, 3]), round(float(dur[t]) * 1e3, 2),
     {nm: round(float(ph[t, i]) * 1e3, 2) for i, nm in enumerate(_lib.PHASES[:15]) if ph[t, i] > 0 and i not in (13, 14)}]
    for t in top]}, indent=0))
