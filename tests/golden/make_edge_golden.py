"""Edge-case golden fixtures written by the REAL reference (build container):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_edge_golden.py

Cases (seeded; exact input factors stored so GPU and oracle consume the same
bits), each factorized by all three methods with the reference's own
execute_sequential:
  tall   -- 12 x 6 block grid (m = 2n, b = 16): p > q (factorize.py:269-270)
  zeros  -- 8 x 8 grid whose admissible blocks below the first sub-diagonal
            are exactly zero (rank-0 cells through every rounded addition)
  dense  -- 6 x 6 all-dense admissibility (core.py:131-132)
Stored per case and method: R-tilde dense, its rank map, flops total.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from blrqr import core as rcore, flops as rflops, lowrank as rlr, scheduler as rsch  # noqa: E402


def lr_tile(rng, b, r):
    u = np.linalg.qr(rng.standard_normal((b, r)))[0]
    v = np.linalg.qr(rng.standard_normal((b, r)))[0]
    return (u * 10.0 ** (-np.arange(r) / 2.0)) @ v.T


def make_dense(case, rng):
    if case == "tall":
        p, q, b, r = 12, 6, 16, 4
    elif case == "zeros":
        p, q, b, r = 8, 8, 16, 4
    else:
        p, q, b, r = 6, 6, 16, 4
    a = np.empty((p * b, q * b))
    for i in range(p):
        for j in range(q):
            if i == j:
                t = rng.standard_normal((b, b))
            elif case == "zeros" and i > j + 1:
                t = np.zeros((b, b))
            else:
                t = lr_tile(rng, b, r)
            a[i * b:(i + 1) * b, j * b:(j + 1) * b] = t
    return a, b, p, q


def pack(a, prefix, out):
    s = a.structure
    out[prefix + "adm"] = s.admissible.copy()
    ranks = np.full((s.p, s.q), -1, dtype=np.int64)
    for i in range(s.p):
        for j in range(s.q):
            x = a.blocks[i][j]
            if hasattr(x, "u"):
                ranks[i, j] = x.rank
                out[f"{prefix}u_{i}_{j}"] = x.u
                out[f"{prefix}v_{i}_{j}"] = x.v
            else:
                out[f"{prefix}d_{i}_{j}"] = x
    out[prefix + "ranks"] = ranks


def main():
    eps = 1e-8
    out = {}
    for n_, case in enumerate(("tall", "zeros", "dense")):
        rng = np.random.default_rng(100 + n_)
        dense, b, p, q = make_dense(case, rng)
        adm = rcore.dense_admissibility(p, q) if case == "dense" else rcore.weak_admissibility(p, q)
        a = rcore.dense_to_blr(dense, b, adm, eps)
        pack(a, f"{case}_a_", out)
        out[f"{case}_shape"] = np.array([p * b, q * b, b])
        for method in ("mgs", "blocked-hh", "tiled-hh"):
            rflops.reset()
            res = rsch.execute_sequential(method, a, rlr.ToleranceConfig(eps))
            out[f"{case}_{method}_r"] = rcore.blr_to_dense(res.r)
            out[f"{case}_{method}_ranks"] = np.array([[x.rank if hasattr(x, "u") else -1 for x in row]
                                                      for row in res.r.blocks])
            out[f"{case}_{method}_flops"] = np.array(rflops.total())
            print(case, method, "R max rank", out[f"{case}_{method}_ranks"].max(), "flops", rflops.total())
    out["eps"] = np.array(eps)
    np.savez_compressed(os.path.join(HERE, "edge_cases.npz"), **out)


if __name__ == "__main__":
    main()
