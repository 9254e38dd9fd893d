"""BLR1 golden streams written by the REAL reference ``blrqr.serialize``.

Build container only (needs /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_blr1_golden.py

Outputs (committed): tests/golden/blr1_mixed.bin -- a seeded 96 x 64 grid
(b = 16) with dense, low-rank and rank-0 cells; tests/golden/blr1_tiled_r.bin
-- the reference's tiled-hh R-tilde of the Laplace-on-a-circle matrix (n = 128,
b = 32, eps = 1e-8), plus its input as tests/golden/blr1_tiled_a.bin.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from blrqr import core as rcore, factorize as rfac, lowrank as rlr, serialize as rser  # noqa: E402


def mixed():
    rng = np.random.default_rng(77)
    m, n, b = 96, 64, 16
    p, q = m // b, n // b
    adm = rcore.weak_admissibility(p, q)
    blocks = []
    for i in range(p):
        row = []
        for j in range(q):
            if not adm[i, j]:
                row.append(rng.standard_normal((b, b)))
            else:
                r = int(rng.integers(0, 5)) if (i + j) % 3 else 0
                u = np.linalg.qr(rng.standard_normal((b, max(r, 1))))[0][:, :r]
                row.append(rcore.LowRankBlock(u, rng.standard_normal((b, r))))
        blocks.append(row)
    return rcore.BlrMatrix(rcore.BlrStructure(m, n, b, adm), blocks)


def tiled_case():
    # points on the unit circle, log kernel (the C2 Laplace recipe at n = 128)
    n, b = 128, 32
    th = 2.0 * np.pi * np.arange(n) / n
    x = np.stack([np.cos(th), np.sin(th)], 1)
    d = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(d, 1.0)
    dense = -np.log(d) / (2.0 * np.pi)
    np.fill_diagonal(dense, 0.0)
    dense += np.diag(1.0 + np.abs(dense).sum(1) / n)
    a = rcore.dense_to_blr(dense, b, rcore.weak_admissibility(n // b, n // b), 1e-8)
    res = rfac.tiled_householder_qr(a, rlr.ToleranceConfig(1e-8))
    return a, res.r


def main():
    with open(os.path.join(HERE, "blr1_mixed.bin"), "wb") as fh:
        rser.dump_blr1(mixed(), fh)
    a, r = tiled_case()
    with open(os.path.join(HERE, "blr1_tiled_a.bin"), "wb") as fh:
        rser.dump_blr1(a, fh)
    with open(os.path.join(HERE, "blr1_tiled_r.bin"), "wb") as fh:
        rser.dump_blr1(r, fh)
    for f in ("blr1_mixed.bin", "blr1_tiled_a.bin", "blr1_tiled_r.bin"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
