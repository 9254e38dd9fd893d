"""Counts ranking repairs (stats slot 57) over repeated tiled-hh runs of the
b = 16 apply-Q golden grid under the dynamic DAG."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import paper_2208_06194_b200 as pk
from paper_2208_06194_b200 import _lib
from paper_2208_06194_b200.device import DeviceGrid
from paper_2208_06194_b200.factorize import DeviceFactorization

z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "applyq_blr.npz"))
n, b, eps = int(z["n"]), int(z["b"]), float(z["eps"])
ranks = z["a_ranks"]; p = n // b
blocks = [[pk.LowRankBlock(z[f"a_u_{i}_{j}"], z[f"a_v_{i}_{j}"]) if ranks[i, j] >= 0 else z[f"a_d_{i}_{j}"]
           for j in range(p)] for i in range(p)]
a = pk.BlrMatrix(pk.BlrStructure(n, n, b, z["a_adm"].copy()), blocks)
rt = _lib.runtime()
g = DeviceGrid.from_host(a)
rep = []
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    f = DeviceFactorization("tiled-hh", g, pk.ToleranceConfig(eps), clone=True)
    f.run()
    f.finish()
    rep.append(int(rt.last_stats[9]))
print("lib", os.environ.get("BLRQR_LIB", "in-tree"), "repairs per run", rep, "total", sum(rep))
