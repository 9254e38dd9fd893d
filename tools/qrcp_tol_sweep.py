"""Sweep the core-QRCP stopping level (blrqr_set_qrcp_tol) on a full-size
config: factorization time, mean kp of large cores, and parity against the
reference run stored in tests/golden (rank map, R-tilde sketch).

python tools/qrcp_tol_sweep.py C3 1 16 64 256
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import test_gpu_fullsize as tf  # noqa: E402
from conftest import GOLDEN  # noqa: E402
from oracle import blr as oblr  # noqa: E402


def main():
    name = sys.argv[1]
    tols = [float(x) for x in sys.argv[2:]] or [1.0]
    method = {"C2": "blocked-hh", "C3": "tiled-hh", "C4": "tiled-hh"}[name]
    import __graft_entry__ as ge
    ge.build()
    import paper_2208_06194_b200 as pk
    from paper_2208_06194_b200 import _lib
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    z = np.load(os.path.join(GOLDEN, f"fact_{name}.npz"))
    t0 = time.perf_counter()
    c, lr, cells = tf._oracle_blr(name)
    print(f"oracle compression {time.perf_counter() - t0:.1f} s", flush=True)
    b, p = c.b, c.n // c.b
    blocks = [[pk.LowRankBlock(cells[(i, j)].u, cells[(i, j)].v) if oblr.is_lr(cells[(i, j)]) else cells[(i, j)]
               for j in range(p)] for i in range(p)]
    a = pk.BlrMatrix(pk.BlrStructure(c.n, c.n, b, lr), blocks)
    g0 = DeviceGrid.from_host(a)
    rt = _lib.runtime()
    for tol in tols:
        assert rt.lib.blrqr_set_qrcp_tol(tol) == 0
        best = None
        for rep in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g = g0.clone()
            torch.cuda.synchronize()
            e0.record()
            f = factorize_device(method, g, pk.ToleranceConfig(c.eps), clone=False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        st = rt.last_stats
        r = f.r_device().to_host()
        ranks = np.array([[x.rank if pk.is_lowrank(x) else -1 for x in row] for row in r.blocks])
        ref = z[f"{method}_ranks"]
        sk = tf._sketch(pk, r, c.n, b)
        rel = np.linalg.norm(sk - z[f"{method}_sketch"]) / np.linalg.norm(z[f"{method}_sketch"])
        print(json.dumps({"config": name, "tol": tol, "factorize_s": best / 1e3,
                          "mean_k": st[0] / max(1, st[2]), "mean_kp": st[1] / max(1, st[2]),
                          "rank_mismatch": int((ranks != ref).sum()), "max_rank_diff": int(np.abs(ranks - ref).max()),
                          "sketch_rel": float(rel)}), flush=True)
    rt.lib.blrqr_set_qrcp_tol(1.0)


if __name__ == "__main__":
    main()
