"""b = 16 open issue (DESIGN 7): repeat the tiled factorization of the apply-Q
golden grid under the dynamic DAG and compare its stores bitwise with the level
scheduler's.  python tools/repro_cmp.py [reps] [nctas]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import paper_2208_06194_b200 as pk
from paper_2208_06194_b200 import _lib
from paper_2208_06194_b200.device import DeviceGrid
from paper_2208_06194_b200.factorize import DeviceFactorization

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
nctas = int(sys.argv[2]) if len(sys.argv) > 2 else None
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "applyq_blr.npz"))
n, b, eps = int(z["n"]), int(z["b"]), float(z["eps"])
ranks = z["a_ranks"]; p = n // b
blocks = [[pk.LowRankBlock(z[f"a_u_{i}_{j}"], z[f"a_v_{i}_{j}"]) if ranks[i, j] >= 0 else z[f"a_d_{i}_{j}"]
           for j in range(p)] for i in range(p)]
a = pk.BlrMatrix(pk.BlrStructure(n, n, b, z["a_adm"].copy()), blocks)
rt = _lib.runtime()
g = DeviceGrid.from_host(a)
cfg = pk.ToleranceConfig(eps)


ZERO = os.environ.get("ZERO", "").split(",")


def run(sched):
    f = DeviceFactorization("tiled-hh", g, cfg, clone=True, scheduler=sched)
    if sched == "dag":
        if "ws" in ZERO:
            rt.workspace(g.b, g.cap, 0, nctas)
            rt._ws.zero_()
        if "wsnan" in ZERO:
            rt.workspace(g.b, g.cap, 0, nctas)
            rt._ws.fill_(float("nan"))
        if "wpool" in ZERO:
            f.rf.wpool.zero_()
        if "work" in ZERO:
            f.dag["work"].zero_()
    f.run(nctas=nctas if sched == "dag" else None)
    f.finish()
    return f


if os.environ.get("TEAMS") == "0":
    rt.lib.blrqr_set_teams(0)
if os.environ.get("RESERVE"):
    rt.lib.blrqr_set_team_reserve(int(os.environ["RESERVE"]))
if os.environ.get("SLACK"):
    rt.lib.blrqr_set_teams(2 + int(os.environ["SLACK"]))
if os.environ.get("NOSMEM"):
    print("nosmem mask", os.environ["NOSMEM"], "rc", rt.lib.blrqr_debug_nosmem(int(os.environ["NOSMEM"])))
ref = run("dag" if os.environ.get("NOREF") else "levels")
rr = ref.g.rank_map()
bad = []
for it in range(reps):
    try:
        f = run("dag")
    except Exception as e:  # noqa: BLE001
        print("run", it, "raised", type(e).__name__, str(e)[:80]); bad.append((it, "raise")); continue
    rk = f.g.rank_map()
    same_rank = (rk == rr).all()
    same_pool = torch.equal(f.rf.pool, ref.rf.pool)
    dr = np.abs(pk.blr_to_dense(f.g.to_host()) - pk.blr_to_dense(ref.g.to_host())).max()
    if not (same_rank and same_pool and dr == 0.0):
        cells = np.argwhere(rk != rr)[:4].tolist()
        bad.append((it, bool(same_rank), bool(same_pool), float(dr), cells, int(rt.last_stats[9])))
print("nctas", nctas, "reps", reps, "bad runs", len(bad), bad[:6])
