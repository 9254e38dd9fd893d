"""Out-of-bounds tripwire (GPU box).  compute-sanitizer is closed on this
GPU pool, so memory safety of the hand-rolled persistent scheduler, the CTA
teams and the arena allocator is checked with canaries instead: every CTA's
workspace stride ends in a guard zone the device arena never allocates
(blrqr_debug_arena_guard), filled with a canary before each launch; after the
dynamic-DAG tiled factorization (with CTA teams and reserved helpers), the
blocked and MGS drivers, a batched rounded addition with large cores (team
Jacobi / QRCP / back-transform), and the two-level 1024^2 GEQRT team job, the
canaries must be intact, no status bit may be raised (arena or rank
overflow, bad argument, non-finite, scheduler timeout), and the results must
still match the unguarded run bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 1 << 14


@pytest.fixture(scope="module")
def pk():
    import __graft_entry__ as ge
    ge.build()
    import paper_2208_06194_b200 as pkg
    return pkg


@pytest.fixture()
def guarded(pk):
    from paper_2208_06194_b200 import _lib
    rt = _lib.runtime()
    rt.set_arena_guard(GUARD)
    yield rt
    rt.set_arena_guard(0)


@pytest.mark.parametrize("method", ["tiled-hh", "blocked-hh", "mgs"])
def test_factorization_stays_in_its_arena(pk, method):
    import torch
    from paper_2208_06194_b200 import _lib, configs
    from paper_2208_06194_b200.core import weak_admissibility
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    rt = _lib.runtime()
    c = configs.CONFIGS["C3"]
    n, b = 2048, 128
    dense = configs.dense_device(c, n)
    g = DeviceGrid.from_dense(dense, b, weak_admissibility(n // b, n // b), 1e-8, 0.5, colmajor=True)
    cfg = pk.ToleranceConfig(1e-8)
    ref = factorize_device(method, g, cfg, clone=True).r_device()
    rt.set_arena_guard(GUARD)
    try:
        f = factorize_device(method, g, cfg, clone=True)  # harvest() inside raises on any status bit
        assert rt.guards_intact()
        out = f.r_device()
        assert torch.equal(out.rank, ref.rank) and torch.equal(out.pool, ref.pool)
    finally:
        rt.set_arena_guard(0)


def test_team_kernels_stay_in_their_arenas(pk, guarded):
    rng = np.random.default_rng(0)
    pairs = []
    for t in range(40):
        bb, ra, rb = 512, 90 + 3 * t, 60 + 2 * t
        ua = np.linalg.qr(rng.standard_normal((bb, ra)))[0]
        ub = np.linalg.qr(rng.standard_normal((bb, rb)))[0]
        pairs.append((pk.LowRankBlock(ua, rng.standard_normal((bb, ra)) * 10.0 ** (-np.arange(ra) / 15)),
                      pk.LowRankBlock(ub, rng.standard_normal((bb, rb)) * 10.0 ** (-np.arange(rb) / 15))))
    outs = pk.rounded_add_batched(pairs, pk.ToleranceConfig(1e-8))
    assert guarded.guards_intact()
    assert all(o.rank > 0 for o in outs)
    a = rng.standard_normal((1024, 1024))
    ref, r = pk.qr_compact_wy(a)
    assert guarded.guards_intact()
    q = np.eye(1024) - ref.y @ ref.t @ ref.y.T
    assert np.linalg.norm(q.T @ q - np.eye(1024)) < 1e-12 * 1024
    assert np.linalg.norm(q @ r - a) < 1e-12 * np.linalg.norm(a)
