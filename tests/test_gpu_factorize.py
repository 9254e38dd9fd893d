"""GPU BLR-QR parity against the oracle (two-stage procedure).

Stage 1 (compression): GPU dense_to_blr vs oracle ranks (ties aside) and
per-tile accuracy.  Stage 2 (factorization): the GPU factorizes the ORACLE's
compressed BLR; R-tilde rank map must match and dense R-tilde agree to 1e-8
relative; Res/Orth within max(10x reference, 10 eps).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import algorithms as oalg, blr as oblr, configs, schedule

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import __graft_entry__ as ge
    ge.build()
    import paper_2208_06194_b200 as pkg
    return pkg


def _input(tag):
    z = np.load(os.path.join(GOLDEN, f"fact_{tag}.npz"))
    meta = json.load(open(os.path.join(GOLDEN, f"fact_{tag}.json")))
    n, b = meta["n"], meta["b"]
    if z["dense"].size:
        dense = z["dense"]
    elif meta["family"] == "random16":
        dense = configs.random16_dense(n, b, 0, rank=min(16, b // 4))
    else:
        dense = configs.dense(configs.Config(tag, meta["family"], n, b, meta["eps"], ()), n)
    return z, meta, dense


def _to_pkg(pk, g):
    blocks = [[pk.LowRankBlock(c.u, c.v) if oblr.is_lr(c) else c for c in row] for row in g.cells]
    return pk.BlrMatrix(pk.BlrStructure(g.m, g.n, g.b, g.lowrank.copy()), blocks)


@pytest.mark.parametrize("tag", ["rand256", "lap512", "exp512", "inv256"])
def test_compression_parity(pk, tag):
    z, meta, dense = _input(tag)
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    a = pk.dense_to_blr(dense, b, pk.weak_admissibility(n // b, n // b), eps)
    ref = z["input_ranks"]
    got = np.array([[x.rank if pk.is_lowrank(x) else -1 for x in row] for row in a.blocks])
    assert (np.abs(got - ref) <= 1).all()
    assert (got != ref).sum() <= max(1, ref.size // 50)
    for i, row in enumerate(a.blocks):
        for j, x in enumerate(row):
            tile = dense[i * b:(i + 1) * b, j * b:(j + 1) * b]
            if pk.is_lowrank(x):
                assert np.linalg.norm(tile - x.to_dense()) <= eps * np.linalg.norm(tile) * (1 + 1e-6)


@pytest.mark.parametrize("tag", ["rand256", "lap512", "exp512", "inv256", "C1"])
@pytest.mark.parametrize("method", ["tiled-hh", "blocked-hh", "mgs"])
def test_factorization_parity(pk, tag, method):
    from paper_2208_06194_b200 import flops as pflops
    from paper_2208_06194_b200.scheduler import execute_sequential

    z, meta, dense = _input(tag)
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    pflops.reset()
    res = execute_sequential(method, _to_pkg(pk, g), pk.ToleranceConfig(eps))
    ranks = np.array([[x.rank if pk.is_lowrank(x) else -1 for x in row] for row in res.r.blocks])
    ref_ranks = z[f"{method}_ranks"]
    assert (np.abs(ranks - ref_ranks) <= 1).all()
    assert (ranks != ref_ranks).sum() <= max(0, ref_ranks.size // 100)
    rd = pk.blr_to_dense(res.r)
    g5 = np.random.default_rng(5).standard_normal((n, 8))
    sk = z[f"{method}_sketch"]
    assert np.linalg.norm(rd @ g5 - sk) <= 1e-8 * np.linalg.norm(sk)
    if f"{method}_r" in z:
        assert np.linalg.norm(rd - z[f"{method}_r"]) <= 1e-8 * np.linalg.norm(z[f"{method}_r"])
    mm = meta["methods"][method]
    # model flops follow the realised ranks of every intermediate; a tie
    # flip inside a chain moves them slightly even when R's ranks agree
    assert abs(pflops.total() - mm["flops_total"]) <= 0.01 * mm["flops_total"]
    # Res / Orth with the oracle's apply-Q on the GPU result's reflectors
    if n <= 2048:
        st = _oracle_state(pk, res, g, eps)
        resid, orth = oalg.res_orth(dense, st)
        assert resid <= max(10 * mm["res"], 10 * eps)
        assert orth <= max(10 * mm["orth"], 10 * eps)


def _ogrid(pk, a):
    s = a.structure
    return oblr.Grid(s.m, s.n, s.b, s.admissible,
                     [[oblr.LR(x.u, x.v) if pk.is_lowrank(x) else x for x in row] for row in a.blocks])


def _oblk(pk, y):
    return oblr.LR(y.u, y.v) if pk.is_lowrank(y) else y


def _oracle_state(pk, res, g, eps):
    """Oracle state objects wrapping the GPU result (for apply-Q / metrics)."""
    if res.algorithm == "tiled-hh":
        st = oalg.TiledState(_ogrid(pk, res.r), eps)
        st.diag = {k: (w.y, w.t) for k, w in res.q_tiles.diag.items()}
        st.upd = {key: (_oblk(pk, y), t) for key, (y, t) in res.q_tiles.updates.items()}
        return st
    if res.algorithm == "blocked-hh":
        cols = [oalg.ColumnReflector(c.col, [(i, _oblk(pk, y)) for i, y in c.entries], c.t) for c in res.q_columns]
        return oalg.BlockedState(_ogrid(pk, res.r), eps, cols)
    st = oalg.MgsState.__new__(oalg.MgsState)
    st.g, st.eps = g, eps
    st.qg = _ogrid(pk, res.q_explicit)
    st.rg = _ogrid(pk, res.r)
    return st


def test_smoke_entry():
    import __graft_entry__ as ge
    ge.smoke()


@pytest.mark.parametrize("tag", ["exp512", "C1"])
def test_dynamic_and_level_schedulers_bitwise_equal(pk, tag):
    """Acceptance #5 analogue: every schedule respecting the DAG gives
    bit-identical R and reflectors (scheduler.py:1-11)."""
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    z, meta, dense = _input(tag)
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    dg = DeviceGrid.from_host(_to_pkg(pk, g))
    fa = factorize_device("tiled-hh", dg, pk.ToleranceConfig(eps), clone=True, scheduler="dag")
    fb = factorize_device("tiled-hh", dg, pk.ToleranceConfig(eps), clone=True, scheduler="levels")
    import torch
    assert torch.equal(fa.g.rank, fb.g.rank)
    assert torch.equal(fa.g.pool, fb.g.pool)
    assert torch.equal(fa.rf.pool, fb.rf.pool)


def test_cta_teams_bitwise_equal_to_single_cta(pk):
    """CTA teams (team.cuh) replay jacobi_blocked's rotation sequence: an
    expcov problem whose rounded additions have large cores gives the same
    bits with teams (dynamic scheduler), without teams, and under the level
    scheduler (no teams)."""
    import torch
    from paper_2208_06194_b200 import _lib, configs
    from paper_2208_06194_b200.core import weak_admissibility
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    cfg = configs.CONFIGS["C3"]
    n = 8192
    dense = configs.dense_device(cfg, n)
    dg = DeviceGrid.from_dense(dense, cfg.b, weak_admissibility(n // cfg.b, n // cfg.b), cfg.eps, colmajor=True)
    del dense
    tol = pk.ToleranceConfig(cfg.eps)
    rt = _lib.runtime()
    fa = factorize_device("tiled-hh", dg, tol, clone=True, scheduler="dag")
    jobs = rt.last_stats[5]
    try:
        rt.lib.blrqr_set_teams(0)
        fb = factorize_device("tiled-hh", dg, tol, clone=True, scheduler="dag")
        assert rt.last_stats[5] == 0
    finally:
        rt.lib.blrqr_set_teams(1)
    fc = factorize_device("tiled-hh", dg, tol, clone=True, scheduler="levels")
    assert jobs > 0, "no team job formed: the test no longer exercises teams"
    for f in (fb, fc):
        assert torch.equal(fa.g.rank, f.g.rank)
        assert torch.equal(fa.g.pool, f.g.pool)
        assert torch.equal(fa.rf.pool, f.rf.pool)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_distributed_gpu_store_emulated_ranks(pk, world):
    """The GPU store of the block-cyclic driver, with `world` ranks emulated
    on one GPU level by level (no rank ever waits on another; the per-level
    rank exchange is summed on the host and broadcasts are device copies of
    the owner's rank-sized payloads): the assembled R-tilde and every
    reflector must equal the single-GPU run bit for bit."""
    import torch
    from paper_2208_06194_b200 import distributed as D
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    z, meta, dense = _input("exp512")
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    dg = DeviceGrid.from_host(_to_pkg(pk, g))
    cfg = pk.ToleranceConfig(eps)
    ref = factorize_device("tiled-hh", dg, cfg, clone=True, scheduler="levels")
    stores = [D.GpuStore(dg.clone(), cfg, world, r) for r in range(world)]
    for lv in range(len(stores[0].plan)):
        for r, st in enumerate(stores):
            own = st.plan[lv][0]
            if len(own):
                st.run(lv, own)
        refl = stores[0].plan[lv][1]
        if world > 1 and refl:  # the rank exchange (all-reduce of the level's Ytilde ranks)
            hdr = sum(st.level_ranks(refl) for st in stores)
            for st in stores:
                st.set_level_ranks(refl, hdr)
        for t in stores[0].plan[lv][1]:
            src = D.task_owner(t, world)
            sb = stores[src].reflector_buffers(t)
            for r in range(world):
                if r != src:
                    for dst, s_ in zip(stores[r].reflector_buffers(t), sb):
                        dst.copy_(s_)
    torch.cuda.synchronize()
    q = ref.g.q
    for j in range(q):
        st = stores[D.column_owner(j, world)]
        for i in range(ref.g.p):
            c = i * q + j
            assert int(st.g.rank[c]) == int(ref.g.rank[c])
            o = int(ref.g.off_u_host[c])
            sz = 2 * b * ref.g.cap if ref.g.kind_host[i, j] else b * b
            if ref.g.kind_host[i, j]:
                r_ = int(ref.g.rank[c])
                assert torch.equal(st.g.pool[o:o + b * r_], ref.g.pool[o:o + b * r_])
            else:
                assert torch.equal(st.g.pool[o:o + sz], ref.g.pool[o:o + sz])
    for st in stores:  # every rank ends with every column's T factors
        for c in np.nonzero(ref.rf.t_off_host >= 0)[0]:
            t0 = int(ref.rf.t_off_host[c])
            assert torch.equal(st.rf.pool[t0:t0 + b * b], ref.rf.pool[t0:t0 + b * b])


@pytest.mark.parametrize("tag,world", [("exp512", 1), ("exp512", 2), ("exp512", 3), ("C1", 4), ("C1", 8)])
def test_peer_dag_emulated_bitwise(pk, tag, world):
    """Peer-DAG multi-GPU protocol (per-rank dynamic DAGs, reflector pushes
    into the peers' stores, remote releases by system-scope atomics) with
    every rank hosted by ONE cooperative launch on this GPU: the owners'
    R-tilde columns and reflectors, and the pushed copies on every other
    rank, equal the single-GPU dynamic run bit for bit."""
    import torch
    from paper_2208_06194_b200 import distributed as D
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    z, meta, dense = _input(tag)
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    dg = DeviceGrid.from_host(_to_pkg(pk, g))
    cfg = pk.ToleranceConfig(eps)
    ref = factorize_device("tiled-hh", dg, cfg, clone=True, scheduler="dag")
    stores = D.factorize_peer_dag_emulated(dg, cfg, world)
    torch.cuda.synchronize()
    pk._lib.runtime().harvest()
    q, p = ref.g.q, ref.g.p
    for j in range(q):
        st = stores[D.column_owner(j, world)]
        for i in range(p):
            c = i * q + j
            o = int(ref.g.off_u_host[c])
            if ref.g.kind_host[i, j]:
                r_ = int(ref.g.rank[c])
                assert int(st.g.rank[c]) == r_, (i, j)
                assert torch.equal(st.g.pool[o:o + b * r_], ref.g.pool[o:o + b * r_]), (i, j)
                o2 = int(ref.g.off_v_host[c])
                assert torch.equal(st.g.pool[o2:o2 + b * r_], ref.g.pool[o2:o2 + b * r_]), (i, j)
            else:
                assert torch.equal(st.g.pool[o:o + b * b], ref.g.pool[o:o + b * b]), (i, j)
    for st in stores:  # every rank holds every column's reflectors (owned or pushed)
        assert torch.equal(st.rf.yrank, ref.rf.yrank)
        for c in np.nonzero(ref.rf.t_off_host >= 0)[0]:
            t0 = int(ref.rf.t_off_host[c])
            assert torch.equal(st.rf.pool[t0:t0 + b * b], ref.rf.pool[t0:t0 + b * b])
        for c in np.nonzero(ref.rf.y_off_host >= 0)[0]:
            if int(ref.rf.yrank[c]) < 0:
                y0 = int(ref.rf.y_off_host[c])
                assert torch.equal(st.rf.pool[y0:y0 + b * b], ref.rf.pool[y0:y0 + b * b])


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("method", ["blocked-hh", "mgs"])
def test_distributed_column_stores_emulated_ranks(pk, method, world):
    """Blocked HH / MGS GPU stores of the column-cyclic driver with `world`
    ranks emulated on one GPU (panel on the owner, payload copied to the
    others, each rank applies to its own columns): owned R-tilde columns and
    every panel payload equal the single-GPU run bit for bit."""
    import torch
    from paper_2208_06194_b200 import distributed as D
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    z, meta, dense = _input("lap512")
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    dg = DeviceGrid.from_host(_to_pkg(pk, g))
    cfg = pk.ToleranceConfig(eps)
    ref = factorize_device(method, dg, cfg, clone=True)
    cls = D.BlockedGpuStore if method == "blocked-hh" else D.MgsGpuStore
    stores = [cls(dg.clone(), cfg, world, r) for r in range(world)]
    for c in range(dg.q):
        src = D.column_owner(c, world)
        stores[src].panel(c)
        sb = stores[src].panel_buffers(c)
        for r in range(world):
            if r != src:
                for dst, s_ in zip(stores[r].panel_buffers(c), sb):
                    dst.copy_(s_)
        for st in stores:
            st.apply(c)
    torch.cuda.synchronize()
    rgrid = (lambda st: st.g) if method == "blocked-hh" else (lambda st: st.rg)
    rr = ref.r_device()
    for j in range(rr.q):
        got = rgrid(stores[D.column_owner(j, world)])
        for i in range(rr.p):
            c = i * rr.q + j
            o = int(rr.off_u_host[c])
            if rr.kind_host[i, j]:
                r_ = int(rr.rank[c])
                assert int(got.rank[c]) == r_
                assert torch.equal(got.pool[o:o + b * r_], rr.pool[o:o + b * r_])
                ov = int(rr.off_v_host[c])
                assert torch.equal(got.pool[ov:ov + b * r_], rr.pool[ov:ov + b * r_])
            else:
                assert torch.equal(got.pool[o:o + b * b], rr.pool[o:o + b * b])
    for c in range(dg.q):  # every rank holds every panel payload
        ref_st = stores[D.column_owner(c, world)]
        for st in stores:
            for x, y in zip(st.panel_buffers(c), ref_st.panel_buffers(c)):
                assert torch.equal(x, y)
    if method == "blocked-hh":  # y_kk and T_k equal the single-GPU reflector store
        for k in range(dg.q):
            y = int(ref.rf.y_off_host[k * dg.q + k])
            for st in stores:
                assert torch.equal(st.rf.pool[y:y + 2 * b * b], ref.rf.pool[y:y + 2 * b * b])


@pytest.mark.parametrize("tag", ["rand256", "lap512", "C1"])
@pytest.mark.parametrize("method", ["tiled-hh", "blocked-hh", "mgs"])
def test_gpu_metrics_match_oracle(pk, tag, method):
    """GPU apply-Q + Res/Orth (no n <= 8192 guard) against the oracle's
    materialize_q / metrics on the same factorization result."""
    from paper_2208_06194_b200 import metrics as pm
    from paper_2208_06194_b200.scheduler import execute_sequential
    z, meta, dense = _input(tag)
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    res = execute_sequential(method, _to_pkg(pk, g), pk.ToleranceConfig(eps))
    rep = pm.compute_metrics(dense, res, eps)
    ores, oorth = oalg.res_orth(dense, _oracle_state(pk, res, g, eps))
    assert abs(rep.res - ores) <= 1e-3 * ores + 1e-15, (rep.res, ores)
    assert abs(rep.orth - oorth) <= 1e-3 * oorth + 1e-15, (rep.orth, oorth)
    mm = meta["methods"][method]
    assert rep.res <= max(10 * mm["res"], 10 * eps) and rep.orth <= max(10 * mm["orth"], 10 * eps)
    if method != "mgs":  # Q^T (Q c) == c through the drop-in apply-Q API
        cmat = np.random.default_rng(1).standard_normal((n, 5))
        fn = pk.factorize.tiled_apply_q if method == "tiled-hh" else pk.factorize.blocked_apply_q
        back = fn(res, fn(res, cmat, False), True)
        assert np.linalg.norm(back - cmat) <= 1e-12 * np.linalg.norm(cmat)


@pytest.mark.parametrize("method", ["blocked-hh", "tiled-hh"])
@pytest.mark.parametrize("transpose", [True, False])
def test_apply_q_blr_operand_matches_reference(pk, method, transpose):
    """blocked_apply_q / tiled_apply_q with a BlrMatrix operand on the GPU
    (kind-aware updates with rounded additions) against the reference-written
    golden output: ranks equal except ties, dense result to 1e-8 relative."""
    from paper_2208_06194_b200.scheduler import execute_sequential
    z = np.load(os.path.join(GOLDEN, "applyq_blr.npz"))
    n, b, eps = int(z["n"]), int(z["b"]), float(z["eps"])

    def grid(prefix):
        ranks = z[prefix + "ranks"]
        p = n // b
        blocks = [[pk.LowRankBlock(z[f"{prefix}u_{i}_{j}"], z[f"{prefix}v_{i}_{j}"]) if ranks[i, j] >= 0
                   else z[f"{prefix}d_{i}_{j}"] for j in range(p)] for i in range(p)]
        return pk.BlrMatrix(pk.BlrStructure(n, n, b, z[prefix + "adm"].copy()), blocks)

    cfg = pk.ToleranceConfig(eps)
    res = execute_sequential(method, grid("a_"), cfg)
    fn = pk.factorize.blocked_apply_q if method == "blocked-hh" else pk.factorize.tiled_apply_q
    c = grid("c_")
    before = pk.blr_to_dense(c)
    out = fn(res, c, transpose, cfg)
    assert np.array_equal(pk.blr_to_dense(c), before)  # operand not mutated
    key = f"{method}_{'qt' if transpose else 'q'}"
    got = pk.blr_to_dense(out)
    ref = z[key + "_dense"]
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-8, rel
    ranks = np.array([[x.rank if pk.is_lowrank(x) else -1 for x in row] for row in out.blocks])
    assert np.abs(ranks - z[key + "_ranks"]).max() <= 1
    with pytest.raises(ValueError):
        fn(res, c, transpose, None)  # BLR operands need a tolerance config


@pytest.mark.parametrize("case", ["tall", "zeros", "dense"])
@pytest.mark.parametrize("method", ["mgs", "blocked-hh", "tiled-hh"])
def test_edge_cases_match_reference(pk, case, method):
    """GPU factorization of tall grids (p > q), exact-zero low-rank blocks and
    all-dense admissibility against the reference-written R-tilde
    (tests/golden/make_edge_golden.py): ranks equal except ties, R-tilde to
    1e-8 relative, model flops within 1 %; the input is not mutated."""
    from paper_2208_06194_b200 import flops as pflops
    from paper_2208_06194_b200.scheduler import execute_sequential
    z = np.load(os.path.join(GOLDEN, "edge_cases.npz"))
    eps = float(z["eps"])
    m, n, b = (int(x) for x in z[f"{case}_shape"])
    pre = f"{case}_a_"
    ranks = z[pre + "ranks"]
    blocks = [[pk.LowRankBlock(z[f"{pre}u_{i}_{j}"], z[f"{pre}v_{i}_{j}"]) if ranks[i, j] >= 0
               else z[f"{pre}d_{i}_{j}"] for j in range(n // b)] for i in range(m // b)]
    a = pk.BlrMatrix(pk.BlrStructure(m, n, b, z[pre + "adm"].copy()), blocks)
    before = pk.blr_to_dense(a)
    pflops.reset()
    res = execute_sequential(method, a, pk.ToleranceConfig(eps))
    assert np.array_equal(pk.blr_to_dense(a), before)
    got = pk.blr_to_dense(res.r)
    ref = z[f"{case}_{method}_r"]
    assert got.shape == ref.shape
    assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)
    gr = np.array([[x.rank if pk.is_lowrank(x) else -1 for x in row] for row in res.r.blocks])
    assert np.abs(gr - z[f"{case}_{method}_ranks"]).max() <= 1
    ft = int(z[f"{case}_{method}_flops"])
    assert abs(pflops.total() - ft) <= 0.01 * ft


@pytest.mark.parametrize("method", ["mgs", "blocked-hh", "tiled-hh"])
def test_metrics_tall_grid(pk, method):
    """compute_metrics on a tall grid (p > q): the GPU Res/Orth equal a host
    evaluation of the reference formulas (metrics.py:69-109 uses
    blr_to_dense(result.r)[:n, :]) on the same factorization."""
    from paper_2208_06194_b200 import metrics as pm
    from paper_2208_06194_b200.scheduler import execute_sequential
    z = np.load(os.path.join(GOLDEN, "edge_cases.npz"))
    eps = float(z["eps"])
    m, n, b = (int(x) for x in z["tall_shape"])
    pre = "tall_a_"
    ranks = z[pre + "ranks"]
    blocks = [[pk.LowRankBlock(z[f"{pre}u_{i}_{j}"], z[f"{pre}v_{i}_{j}"]) if ranks[i, j] >= 0
               else z[f"{pre}d_{i}_{j}"] for j in range(n // b)] for i in range(m // b)]
    a = pk.BlrMatrix(pk.BlrStructure(m, n, b, z[pre + "adm"].copy()), blocks)
    dense = pk.blr_to_dense(a)
    res = execute_sequential(method, a, pk.ToleranceConfig(eps))
    rep = pm.compute_metrics(dense, res, eps)
    r = pk.blr_to_dense(res.r)[:n, :]
    if method == "mgs":
        q = pk.blr_to_dense(res.q_explicit)[:, :n]
    else:
        fn = pk.factorize.tiled_apply_q if method == "tiled-hh" else pk.factorize.blocked_apply_q
        q = fn(res, np.eye(m)[:, :n], False)
    hres = np.linalg.norm(q @ r - dense) / np.linalg.norm(dense)
    horth = np.linalg.norm(q.T @ q - np.eye(n)) / np.sqrt(n)
    assert abs(rep.res - hres) <= 1e-3 * hres + 1e-15, (rep.res, hres)
    assert abs(rep.orth - horth) <= 1e-3 * horth + 1e-15, (rep.orth, horth)
    assert rep.res <= 10 * eps


def test_foreign_containers_duck_typed(pk):
    """A BlrMatrix built from another package's block class (the reference's
    LowRankBlock is such a class: core.py:31-66; is_lowrank there is an
    isinstance check) factorizes unchanged: DeviceGrid.from_host duck-types
    u / v factors, and the result is bitwise the one from this package's
    containers."""
    from dataclasses import dataclass
    from paper_2208_06194_b200.scheduler import execute_sequential

    @dataclass
    class ForeignLR:
        u: np.ndarray
        v: np.ndarray

        @property
        def rank(self):
            return self.u.shape[1]

        @property
        def rows(self):
            return self.u.shape[0]

        @property
        def cols(self):
            return self.v.shape[0]

    @dataclass
    class ForeignMatrix:
        structure: object
        blocks: list

        @property
        def p(self):
            return self.structure.p

        @property
        def q(self):
            return self.structure.q

    z, meta, dense = _input("lap512")
    n, b, eps = meta["n"], meta["b"], meta["eps"]
    g = schedule.dense_to_blr(dense, b, oblr.weak_map(n // b, n // b), eps)
    ours = _to_pkg(pk, g)
    foreign = ForeignMatrix(ours.structure, [[ForeignLR(x.u, x.v) if pk.is_lowrank(x) else x for x in row]
                                             for row in ours.blocks])
    cfg = pk.ToleranceConfig(eps)
    r1 = pk.blr_to_dense(execute_sequential("tiled-hh", ours, cfg).r)
    r2 = pk.blr_to_dense(execute_sequential("tiled-hh", foreign, cfg).r)
    assert np.array_equal(r1, r2)
