"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
the persistent dynamic-DAG tiled factorization with CTA teams, the blocked
and MGS drivers, a batched rounded addition with large cores (team Jacobi,
team QRCP), and the two-level GEQRT team job.  Prints one line per part.

compute-sanitizer --tool memcheck python tools/sanitize_run.py [parts]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2208_06194_b200 as pk  # noqa: E402
from paper_2208_06194_b200 import _lib, configs  # noqa: E402
from paper_2208_06194_b200.core import weak_admissibility  # noqa: E402
from paper_2208_06194_b200.device import DeviceGrid  # noqa: E402
from paper_2208_06194_b200.factorize import factorize_device  # noqa: E402

parts = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tiled", "blocked", "mgs", "radd", "geqrt"]
rt = _lib.runtime()
cfg = pk.ToleranceConfig(1e-8)
if any(p in parts for p in ("tiled", "blocked", "mgs")):
    c = configs.CONFIGS["C3"]
    n, b = 1024, 128
    dense = configs.dense_device(c, n)
    g = DeviceGrid.from_dense(dense, b, weak_admissibility(n // b, n // b), 1e-8, 0.5, colmajor=True)
    for m in ("tiled", "blocked", "mgs"):
        if m in parts:
            method = {"tiled": "tiled-hh", "blocked": "blocked-hh", "mgs": "mgs"}[m]
            f = factorize_device(method, g, cfg, clone=True)
            torch.cuda.synchronize()
            print(m, "ok, R max rank", int(f.r_device().rank_map().max()), flush=True)
if "radd" in parts:
    rng = np.random.default_rng(0)
    pairs = []
    for t in range(24):
        bb, ra, rbk = 256, 60 + t, 50 + t
        ua = np.linalg.qr(rng.standard_normal((bb, ra)))[0]
        ub = np.linalg.qr(rng.standard_normal((bb, rbk)))[0]
        pairs.append((pk.LowRankBlock(ua, rng.standard_normal((bb, ra)) * 10.0 ** (-np.arange(ra) / 12)),
                      pk.LowRankBlock(ub, rng.standard_normal((bb, rbk)) * 10.0 ** (-np.arange(rbk) / 12))))
    outs = pk.rounded_add_batched(pairs, cfg)
    print("radd ok, ranks", [o.rank for o in outs[:6]], flush=True)
if "geqrt" in parts:
    a = np.random.default_rng(1).standard_normal((1024, 1024))
    ref, r = pk.qr_compact_wy(a)
    print("geqrt ok, |diag R| min", float(np.abs(np.diag(r)).min()), flush=True)
