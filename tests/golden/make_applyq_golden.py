"""Golden vectors for apply-Q on BLOCK LOW-RANK operands (blocked_apply_q /
tiled_apply_q with a BlrMatrix, factorize.py:326-350, :495-568), written by
the REAL reference in the build container:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_applyq_golden.py

For each case: the factorization input A and operand C are seeded random16
BLR matrices (n=128, b=16, rank 4) compressed by the reference; the npz holds
A's and C's exact factors (so the GPU and the oracle consume identical bits),
and, per method and direction, the reference's output as a dense matrix plus
its rank map.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from blrqr import core as rcore, factorize as rfac, lowrank as rlr  # noqa: E402

from oracle import configs  # noqa: E402  (input recipe only)


def pack(a, prefix, out):
    """BlrMatrix -> flat arrays: kind map, ranks, and per-cell factors."""
    s = a.structure
    out[prefix + "adm"] = s.admissible.copy()
    ranks = np.full((s.p, s.q), -1, dtype=np.int64)
    for i in range(s.p):
        for j in range(s.q):
            x = a.blocks[i][j]
            if rcore.is_lowrank(x) if hasattr(rcore, "is_lowrank") else hasattr(x, "u"):
                ranks[i, j] = x.rank
                out[f"{prefix}u_{i}_{j}"] = x.u
                out[f"{prefix}v_{i}_{j}"] = x.v
            else:
                out[f"{prefix}d_{i}_{j}"] = x
    out[prefix + "ranks"] = ranks


def main():
    n, b, eps = 128, 16, 1e-8
    p = n // b
    out = {"n": np.array(n), "b": np.array(b), "eps": np.array(eps)}
    adm = rcore.weak_admissibility(p, p)
    a = rcore.dense_to_blr(configs.random16_dense(n, b, 0, rank=4), b, adm, eps)
    # operand: A's own blocks plus a seeded low-rank perturbation of every
    # admissible cell (Q^T C then keeps R-like structure with nonzero ranks)
    c = rcore.dense_to_blr(configs.random16_dense(n, b, 0, rank=4) + 1e-3 * configs.random16_dense(n, b, 7, rank=4),
                           b, adm, eps)
    pack(a, "a_", out)
    pack(c, "c_", out)
    cfg = rlr.ToleranceConfig(eps)
    for method, fn, app in (("blocked-hh", rfac.blocked_householder_qr, rfac.blocked_apply_q),
                            ("tiled-hh", rfac.tiled_householder_qr, rfac.tiled_apply_q)):
        res = fn(a, cfg)
        for tr in (True, False):
            got = app(res, c, tr, cfg)
            key = f"{method}_{'qt' if tr else 'q'}"
            out[key + "_dense"] = rcore.blr_to_dense(got)
            out[key + "_ranks"] = np.array([[x.rank if hasattr(x, "u") else -1 for x in row] for row in got.blocks])
            print(key, "max rank", out[key + "_ranks"].max())
    np.savez_compressed(os.path.join(HERE, "applyq_blr.npz"), **out)


if __name__ == "__main__":
    main()
