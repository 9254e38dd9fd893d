"""Barrier-count check (-DBLR_BARCHECK build via BLRQR_LIB) on the b = 16 grid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
nct = int(sys.argv[1]) if len(sys.argv) > 1 else None
for it in range(4):
    f = DeviceFactorization("tiled-hh", g, pk.ToleranceConfig(eps), clone=True, scheduler="dag")
    f.run(nctas=nct)
    try:
        f.finish()
        print("run", it, "ok stats", rt.last_stats[9:14])
    except Exception as e:  # noqa: BLE001
        print("run", it, type(e).__name__, str(e)[:60], "stats[57..61] =", rt.last_stats[9:14])
