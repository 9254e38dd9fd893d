"""Seeded config-scale kernel inputs (test infrastructure only).

The round-1 unit goldens were toy-sized (rounded additions b <= 64, c <= 26;
RRQR tiles <= 64^2; GEQRT <= 200 x 64).  The factorizations at C2-C5 run the
same operations at b = 256 / 512 / 1024 with cores up to c = 340
(tests/golden/fact_C3.npz ``radd_hist``), which take different device code
paths (shared-memory / blocked / team Jacobi, register TPQRT with two columns
per thread, 1024^2 GEQRT, b = 1024 RRQR).  These recipes regenerate the
inputs of ``tests/golden/make_golden_scale.py`` bit-for-bit from a seed so
the committed fixtures hold only what the UNMODIFIED reference returned
(ranks, singular values, error norms, small sketches), not megabytes of
operands.

Input recipes use numpy's PCG64 generator and ``np.linalg.qr`` (the same
numpy/OpenBLAS build in the build container and on the GPU box); each case
carries an input checksum so recipe drift is detected instead of silently
shifting the comparison.
"""

from __future__ import annotations

import numpy as np

from .configs import ExpCov, Laplace

# ---------------------------------------------------------------------------
# rounded additions (lowrank.py:173-221) at the factorizations' shapes
# ---------------------------------------------------------------------------

RADD_COUNT = 1200
RADD_MODES = ("independent", "cancel", "shared", "raw")


def _spectrum(rng, r, decades):
    if r == 0:
        return np.zeros(0)
    if r == 1:
        return np.ones(1)
    return 10.0 ** (-decades * np.arange(r) / (r - 1))


def _orth(rng, b, r):
    if r == 0:
        return np.zeros((b, 0))
    return np.linalg.qr(rng.standard_normal((b, r)))[0]


def radd_case(t: int):
    """Operands (ua, va, ub, vb), eps and (b, c, mode) of rounded-addition case t.

    b in {256, 512, 1024}; c = r_A + r_B spread over the C3 histogram's range
    (60 % in [2, 64], 30 % in [64, 200], 10 % in [200, 340]).  A is a stored
    factor pair (orthonormal U, spectrum decaying to about eps); B is
    independent, a near-cancellation of A, a term inside A's column space, or
    a raw product with non-orthonormal U (the transient factors of
    factorize.py:92-106).
    """
    rng = np.random.default_rng(7_000_000 + t)
    b = int(rng.choice([256, 512, 1024], p=[0.3, 0.4, 0.3]))
    u = rng.uniform()
    if u < 0.6:
        c = int(rng.integers(2, 65))
    elif u < 0.9:
        c = int(rng.integers(64, 201))
    else:
        c = int(rng.integers(200, 341))
    c = min(c, b)
    mode = RADD_MODES[t % len(RADD_MODES)]
    eps = float(rng.choice([1e-8, 1e-8, 1e-10, 1e-6]))
    ra = int(rng.integers(1, c)) if c > 1 else 1
    rb = c - ra
    sa = _spectrum(rng, ra, float(rng.uniform(2.0, 10.0)))
    ua = _orth(rng, b, ra)
    va = _orth(rng, b, ra) * sa
    scale = float(10.0 ** rng.uniform(-3.0, 1.0))
    if mode == "independent" or rb == 0:
        ub = _orth(rng, b, rb)
        vb = _orth(rng, b, rb) * (scale * _spectrum(rng, rb, float(rng.uniform(2.0, 12.0))))
    elif mode == "cancel":
        # B = -A restricted to rb of A's directions, plus a small new part
        k = min(rb, ra)
        ub = np.hstack([ua[:, :k], _orth(rng, b, rb - k)])
        pert = 10.0 ** rng.uniform(-9.0, -3.0)
        vb = np.hstack([-va[:, :k] * (1.0 + pert * rng.standard_normal(k)),
                        _orth(rng, b, rb - k) * (pert * _spectrum(rng, rb - k, 4.0))])
    elif mode == "shared":
        k = min(rb, ra)
        rot = np.linalg.qr(rng.standard_normal((ra, k)))[0]
        ub = np.hstack([ua @ rot, _orth(rng, b, rb - k)])
        vb = _orth(rng, b, rb) * (scale * _spectrum(rng, rb, float(rng.uniform(1.0, 8.0))))
    else:  # raw: non-orthonormal U (T_ik^T u products), graded columns
        ub = rng.standard_normal((b, rb)) * (10.0 ** rng.uniform(-1.0, 1.0, rb))
        vb = rng.standard_normal((b, rb)) * (scale * _spectrum(rng, rb, float(rng.uniform(2.0, 9.0))))
    return dict(ua=ua, va=va, ub=ub, vb=vb, eps=eps, b=b, c=c, mode=mode)


def checksum(*arrs) -> float:
    """Order-sensitive input fingerprint (detects recipe / BLAS drift)."""
    s = 0.0
    for k, a in enumerate(arrs):
        if a.size:
            w = np.cos(np.arange(a.size, dtype=float) * 0.001 + k)
            s += float(np.dot(a.ravel(order="F"), w))
    return s


def sketch_mats(b: int, seed: int, k: int = 4):
    g = np.random.default_rng(seed)
    return g.standard_normal((b, k)), g.standard_normal((b, k))


# ---------------------------------------------------------------------------
# RRQR compression (lowrank.py:64-158) of config tiles at b = 512 / 1024
# ---------------------------------------------------------------------------

_SOURCES = {}


def _source(name):
    if name not in _SOURCES:
        if name == "C3":
            _SOURCES[name] = ExpCov(32768, 0).tile
        elif name == "C5":
            _SOURCES[name] = Laplace(65536).tile
        else:
            raise ValueError(name)
    return _SOURCES[name]


def rrqr_cases():
    """(tag, b, tile index or synthetic spec) list: 48 C3 tiles (b = 512,
    spread over block distances, so ranks cover ~8..127), 24 C5 tiles
    (b = 1024), 16 synthetic graded tiles at each b (ranks up to ~b/2, and
    above b/2 for the dense fallback)."""
    rng = np.random.default_rng(424242)
    out = []
    for t in range(48):
        i = int(rng.integers(0, 64))
        d = int(rng.choice([1, 1, 2, 3, 5, 9, 17, 33, 63]))
        j = (i + d) % 64 if t % 2 else (i - d) % 64
        if i == j:
            j = (i + 1) % 64
        out.append(("C3", 512, (i, j)))
    for t in range(24):
        i = int(rng.integers(0, 64))
        d = int(rng.choice([1, 2, 3, 7, 15, 31, 63]))
        j = (i + d) % 64
        out.append(("C5", 1024, (i, j)))
    for b in (512, 1024):
        for t in range(16):
            r = int(rng.integers(1, (b * 3) // 5))
            decades = float(rng.uniform(1.0, 14.0))
            out.append(("synthetic", b, (int(rng.integers(0, 2**31)), r, decades)))
    return out


def rrqr_tile(case):
    src, b, spec = case
    if src in ("C3", "C5"):
        i, j = spec
        return np.ascontiguousarray(_source(src)(i * b, j * b, b, b))
    seed, r, decades = spec
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((b, r)))[0]
    v = np.linalg.qr(rng.standard_normal((b, r)))[0]
    s = 10.0 ** (-decades * np.arange(r) / max(r - 1, 1))
    return (u * s) @ v.T


# ---------------------------------------------------------------------------
# dense panels (kernels.py:87-186) at b = 512 / 1024
# ---------------------------------------------------------------------------

# (m, n, kind): kind "gauss" = N(0,1); "graded" = column j scaled 10^(-8 j / n)
GEQRT_CASES = [(512, 512, "gauss"), (512, 512, "graded"), (1024, 1024, "gauss"), (1024, 1024, "graded"),
               (1300, 1024, "gauss"), (768, 512, "graded")]
# (n, k): UpdateQR bottoms (low-rank V_ik^T rows or a dense tile)
TPQRT_CASES = [(512, 8), (512, 16), (512, 17), (512, 31), (512, 32), (512, 33), (512, 64), (512, 135),
               (1024, 3), (1024, 8), (1024, 16), (1024, 17), (1024, 32), (1024, 135)]


def geqrt_input(t):
    m, n, kind = GEQRT_CASES[t]
    rng = np.random.default_rng(31_000 + t)
    a = rng.standard_normal((m, n))
    if kind == "graded":
        a *= 10.0 ** (-8.0 * np.arange(n) / n)
    return a, rng.standard_normal((m, 48))


def tpqrt_input(t):
    n, k = TPQRT_CASES[t]
    rng = np.random.default_rng(32_000 + t)
    top = np.triu(rng.standard_normal((n, n))) + np.diag(np.sqrt(n) * np.sign(rng.standard_normal(n)))
    bot = rng.standard_normal((k, n)) * (10.0 ** -rng.uniform(0.0, 6.0, (k, 1)))
    return top, bot, rng.standard_normal((n, 24)), rng.standard_normal((k, 24))
