"""Repro: tiled-hh on the apply-Q golden grid (n = 128, b = 16) under debug knobs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import paper_2208_06194_b200 as pk
from paper_2208_06194_b200 import _lib
from paper_2208_06194_b200.device import DeviceGrid
from paper_2208_06194_b200.factorize import DeviceFactorization

mode = sys.argv[1] if len(sys.argv) > 1 else "default"
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "applyq_blr.npz"))
n, b, eps = int(z["n"]), int(z["b"]), float(z["eps"])
ranks = z["a_ranks"]; p = n // b
blocks = [[pk.LowRankBlock(z[f"a_u_{i}_{j}"], z[f"a_v_{i}_{j}"]) if ranks[i, j] >= 0 else z[f"a_d_{i}_{j}"]
           for j in range(p)] for i in range(p)]
a = pk.BlrMatrix(pk.BlrStructure(n, n, b, z["a_adm"].copy()), blocks)
rt = _lib.runtime()
if int(os.environ.get("BLRQR_STACK", "0")):
    import ctypes
    cr = ctypes.CDLL("libcudart.so.12")
    v = ctypes.c_size_t(0)
    cr.cudaDeviceGetLimit(ctypes.byref(v), 0)
    print("stack limit was", v.value, "set rc", cr.cudaDeviceSetLimit(0, ctypes.c_size_t(int(os.environ["BLRQR_STACK"]))))
if mode == "noteams":
    rt.lib.blrqr_set_teams(0)
if mode == "dfma":
    rt.lib.blrqr_debug_gemm_impl(1)
if mode == "guard":
    rt.set_arena_guard(4096)
g = DeviceGrid.from_host(a)
f = DeviceFactorization("tiled-hh", g, pk.ToleranceConfig(eps), clone=True,
                        scheduler="levels" if mode == "levels" else "dag")
print("cap", g.cap, "p", g.p, flush=True)
from paper_2208_06194_b200.factorize import tiled_dag_arrays
tasks, indeg, off, succ, prio = tiled_dag_arrays(g.p, g.q, int(rt.lib.blrqr_dag_policy()))
nt = len(tasks)
trace = torch.zeros(3 * nt, dtype=torch.int64).pin_memory()
ptrace = torch.zeros(16 * nt, dtype=torch.int64).pin_memory()
rt.lib.blrqr_debug_trace(trace.data_ptr())
rt.lib.blrqr_debug_phase_trace(ptrace.data_ptr())
try:
    f.run(nctas=int(mode[4:]) if mode.startswith("ncta") else None)
    import time
    t0 = time.time()
    while not torch.cuda.current_stream().query():
        if time.time() - t0 > 15:
            raise TimeoutError("kernel still running after 15 s")
        time.sleep(0.2)
    torch.cuda.synchronize()
    print(mode, "ran; counts", f.finish())
except Exception as e:
    print("FAILED", e)
    import struct
    rt.harvest_noraise() if hasattr(rt,'harvest_noraise') else None
    ls = getattr(rt, 'last_stats', [0]*16)
    print("debug stats", ls[9:], [struct.unpack("d", struct.pack("q", int(v)))[0] for v in (ls[12], ls[13], ls[15])])
    tr = trace.numpy().reshape(nt, 3)
    pt = ptrace.numpy().reshape(nt, 16)
    started = np.nonzero(tr[:, 0])[0]
    print("tasks started", len(started), "finished", int((tr[:, 1] != 0).sum()))
    for t in started:
        if tr[t, 1] == 0:
            print("UNFINISHED task", t, "kind,k,i,j =", tasks[t].tolist(), "prio", prio[t], "phases", pt[t].tolist())
    order = started[np.argsort(tr[started, 0])]
    print("last 5 started:", [(int(t), tasks[t].tolist()) for t in order[-5:]])
    sys.stdout.flush()
    os._exit(3)
if mode == "guard":
    print("guards intact:", rt.guards_intact())
