"""Generate the golden fixtures by running the REAL reference ``blrqr`` package.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--full]

Outputs (committed, small): tests/golden/*.npz / *.json.  Inputs are stored
explicitly (or regenerated from the oracle's seeded config recipes), outputs
are what the reference returned.  ``--full`` additionally runs the reference
on the full-size C1 config for all three methods (a few seconds each) and on
C2/C4 (minutes) and stores rank maps, R sketches and Res/Orth.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import blrqr  # noqa: E402
from blrqr import core as rcore, factorize as rfac, flops as rflops  # noqa: E402
from blrqr import kernels as rker, lowrank as rlr, metrics as rmet  # noqa: E402
from blrqr import scheduler as rsch  # noqa: E402

from oracle import configs  # noqa: E402  (input recipes only)


def _lr_pair(rng, b, r, scale=1.0, orth=True):
    u = rng.standard_normal((b, r))
    if orth and r:
        u = np.linalg.qr(u)[0]
    v = scale * rng.standard_normal((b, r)) * (10.0 ** (-np.arange(r) / 3.0))
    return u, v


def gen_rounded_add(path):
    """Seeded operand pairs spanning ranks, cancellation and rank-0 edges."""
    rng = np.random.default_rng(1234)
    cases = []
    for t in range(150):
        b = int(rng.choice([16, 32, 64]))
        ra = int(rng.integers(0, 14))
        rb = int(rng.integers(0, 14))
        eps = float(rng.choice([1e-4, 1e-8, 1e-10]))
        ua, va = _lr_pair(rng, b, ra, orth=bool(rng.integers(0, 2)) or True)
        mode = t % 6
        if mode == 0 and ra:  # exact cancellation
            ub, vb = ua.copy(), -va.copy()
        elif mode == 1 and ra:  # shared column space, graded coefficients
            ub = ua @ np.linalg.qr(rng.standard_normal((ra, ra)))[0]
            vb = rng.standard_normal((b, ra)) * 1e-6
        else:
            ub, vb = _lr_pair(rng, b, rb, scale=float(10.0 ** rng.integers(-3, 2)),
                              orth=bool(rng.integers(0, 2)))
        a = rcore.LowRankBlock(ua, va)
        bk = rcore.LowRankBlock(ub, vb)
        out = rlr.rounded_add(a, bk, rlr.ToleranceConfig(eps))
        cases.append(dict(ua=ua, va=va, ub=ub, vb=vb, eps=eps, uo=out.u, vo=out.v))
    flat = {}
    for t, c in enumerate(cases):
        for k, v in c.items():
            flat[f"{t}_{k}"] = np.asarray(v)
    flat["count"] = np.array(len(cases))
    np.savez_compressed(path, **flat)


def gen_rrqr(path):
    rng = np.random.default_rng(99)
    flat = {}
    tiles = []
    for t in range(80):
        b = int(rng.choice([16, 32, 48, 64]))
        kind = t % 8
        if kind == 0:
            a = np.eye(b)  # SPEC KAT: identity -> dense fallback
        elif kind == 1:
            a = np.zeros((b, b))
        elif kind == 2:
            x = rng.standard_normal(b)
            a = np.outer(x, rng.standard_normal(b))
        elif kind == 3:  # pivot ties: repeated equal-norm columns
            x = rng.standard_normal((b, 3))
            a = np.hstack([x] * (b // 3 + 1))[:, :b]
        else:
            r = int(rng.integers(1, b))
            u = np.linalg.qr(rng.standard_normal((b, r)))[0]
            v = np.linalg.qr(rng.standard_normal((b, r)))[0]
            s = 10.0 ** (-float(rng.uniform(0.2, 2.0)) * np.arange(r))
            a = (u * s) @ v.T
        eps = float(rng.choice([1e-4, 1e-8, 1e-10]))
        frac = float(rng.choice([0.5, 1.0]))
        out = rlr.compress_rrqr(a, rlr.ToleranceConfig(eps, frac))
        flat[f"{t}_a"] = a
        flat[f"{t}_eps"] = np.array(eps)
        flat[f"{t}_frac"] = np.array(frac)
        if rcore.is_lowrank(out):
            flat[f"{t}_u"] = out.u
            flat[f"{t}_v"] = out.v
        tiles.append(t)
    flat["count"] = np.array(len(tiles))
    np.savez_compressed(path, **flat)


def gen_panels(path):
    rng = np.random.default_rng(7)
    flat = {}
    for t, (m, n) in enumerate([(1, 1), (2, 1), (8, 8), (40, 16), (96, 32), (64, 64), (200, 64)]):
        a = rng.standard_normal((m, n))
        if t == 1:
            a = np.array([[3.0], [4.0]])
        ref, r = rker.qr_compact_wy(a)
        c = rng.standard_normal((m, 5))
        flat[f"geqrt{t}_a"] = a
        flat[f"geqrt{t}_y"] = ref.y
        flat[f"geqrt{t}_t"] = ref.t
        flat[f"geqrt{t}_r"] = r
        flat[f"geqrt{t}_c"] = c
        flat[f"geqrt{t}_qc"] = rker.apply_wy(ref, c)
        flat[f"geqrt{t}_qtc"] = rker.apply_wy_transpose(ref, c)
        q, rr = rker.mgs_panel_qr(a)
        flat[f"mgs{t}_q"] = q
        flat[f"mgs{t}_r"] = rr
    for t, (n, k) in enumerate([(1, 1), (8, 0), (8, 3), (32, 7), (64, 64), (48, 100)]):
        top = np.triu(rng.standard_normal((n, n)))
        bot = rng.standard_normal((k, n))
        if t == 0:
            top, bot = np.array([[1.0]]), np.array([[1.0]])
        ref, rn = rker.tp_qr(top, bot)
        ct = rng.standard_normal((n, 4))
        cb = rng.standard_normal((k, 4))
        flat[f"tp{t}_top"] = top
        flat[f"tp{t}_bot"] = bot
        flat[f"tp{t}_y"] = ref.y
        flat[f"tp{t}_t"] = ref.t
        flat[f"tp{t}_r"] = rn
        flat[f"tp{t}_ct"] = ct
        flat[f"tp{t}_cb"] = cb
        a1, a2 = rker.apply_tp(ref, ct, cb)
        t1, t2 = rker.apply_tp_transpose(ref, ct, cb)
        flat[f"tp{t}_q1"], flat[f"tp{t}_q2"] = a1, a2
        flat[f"tp{t}_qt1"], flat[f"tp{t}_qt2"] = t1, t2
    np.savez_compressed(path, **flat)


def _sketch(dense, seed=5, k=8):
    g = np.random.default_rng(seed).standard_normal((dense.shape[1], k))
    return dense @ g


SMALL = [
    # (tag, family, n, b, eps)
    ("rand256", "random16", 256, 32, 1e-8),
    ("lap512", "laplace", 512, 64, 1e-8),
    ("exp512", "expcov", 512, 64, 1e-8),
    ("inv256", "invpoisson", 256, 32, 1e-10),
]


def run_case(tag, family, n, b, eps, methods, store_full):
    cfg = configs.Config(tag, family, n, b, eps, methods)
    if family == "random16":
        dense = configs.random16_dense(n, b, 0, rank=min(16, b // 4))
    else:
        dense = configs.dense(cfg, n)
    t0 = time.perf_counter()
    a = rcore.dense_to_blr(dense, b, rcore.weak_admissibility(n // b, n // b), eps)
    tc = time.perf_counter() - t0
    out = {}
    summary = {"tag": tag, "family": family, "n": n, "b": b, "eps": eps,
               "compress_s": tc, "methods": {}}
    out["input_ranks"] = np.array([[blk.rank if rcore.is_lowrank(blk) else -1
                                    for blk in row] for row in a.blocks])
    out["dense"] = dense if store_full else np.zeros(0)
    for m in methods:
        rflops.reset()
        t0 = time.perf_counter()
        res = rsch.execute_sequential(m, a, rlr.ToleranceConfig(eps))
        tf = time.perf_counter() - t0
        fl = rflops.report()
        rdense = rcore.blr_to_dense(res.r)
        q = rmet.materialize_q(res)
        n_ = dense.shape[1]
        resid = float(np.linalg.norm(q @ rdense[:n_] - dense) / np.linalg.norm(dense))
        gram = q.T @ q - np.eye(n_)
        orth = float(np.linalg.norm(gram) / np.sqrt(n_))
        out[f"{m}_ranks"] = np.array([[blk.rank if rcore.is_lowrank(blk) else -1
                                       for blk in row] for row in res.r.blocks])
        out[f"{m}_sketch"] = _sketch(rdense)
        out[f"{m}_fro"] = np.array([[np.linalg.norm(rcore.block_to_dense(blk))
                                     for blk in row] for row in res.r.blocks])
        if store_full:
            out[f"{m}_r"] = rdense
        summary["methods"][m] = {"factorize_s": tf, "res": resid, "orth": orth,
                                 "flops": fl, "flops_total": int(sum(fl.values()))}
        print(tag, m, f"{tf:.2f}s res={resid:.3e} orth={orth:.3e} F={sum(fl.values()):.4e}",
              flush=True)
    np.savez_compressed(os.path.join(HERE, f"fact_{tag}.npz"), **out)
    with open(os.path.join(HERE, f"fact_{tag}.json"), "w") as fh:
        json.dump(summary, fh, indent=1, sort_keys=True)


def gen_kat(path):
    cfg8 = rlr.ToleranceConfig(1e-8)
    kat = {}
    kat["compress_identity8_dense"] = not rcore.is_lowrank(rlr.compress_rrqr(np.eye(8), cfg8))
    z = rlr.compress_rrqr(np.zeros((8, 8)), cfg8)
    kat["compress_zero8_rank"] = z.rank
    x = np.arange(1.0, 9.0)
    o = rlr.compress_rrqr(np.outer(x, x), cfg8)
    kat["compress_outer_rank"] = o.rank
    u = np.linalg.qr(np.random.default_rng(0).standard_normal((8, 2)))[0]
    a = rcore.LowRankBlock(u, np.ones((8, 2)))
    kat["rounded_add_cancel_rank"] = rlr.rounded_add(a, rcore.LowRankBlock(u, -np.ones((8, 2))), cfg8).rank
    _, r = rker.qr_compact_wy(np.array([[3.0], [4.0]]))
    kat["geqrt_34_r11"] = float(r[0, 0])
    _, r = rker.tp_qr(np.array([[1.0]]), np.array([[1.0]]))
    kat["tpqrt_11_r"] = float(r[0, 0])
    q, r = rker.mgs_panel_qr(np.array([[3.0], [4.0]]))
    kat["mgs_34"] = {"r": float(r[0, 0]), "q": q[:, 0].tolist()}
    for p, q_ in [(1, 1), (2, 2), (3, 3), (4, 4), (6, 4)]:
        dag = rsch.build_tiled_dag(p, q_)
        kat[f"dag_{p}x{q_}"] = {"nodes": [str(t) for t in dag.nodes],
                                "edges": sorted([list(e) for e in dag.edges])}
    mat = rcore.BlrMatrix(rcore.BlrStructure(64, 64, 16, rcore.weak_admissibility(4, 4)),
                          [[rcore.LowRankBlock(np.zeros((16, 3)), np.zeros((16, 3)))
                            if i != j else np.zeros((16, 16)) for j in range(4)] for i in range(4)])
    kat["memory_footprint_4x4_b16_r3"] = rcore.memory_footprint(mat)
    kat["flops_qr_64_64"] = rflops.qr_cost(64, 64)
    kat["flops_geqrt_64_64"] = rflops.qr_cost(64, 64) + rflops.tgen_cost(64, 64)
    with open(path, "w") as fh:
        json.dump(kat, fh, indent=1, sort_keys=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None

    def want(x):
        return only is None or x in only

    if want("kat"):
        gen_kat(os.path.join(HERE, "kat.json"))
    if want("rounded_add"):
        gen_rounded_add(os.path.join(HERE, "rounded_add.npz"))
    if want("rrqr"):
        gen_rrqr(os.path.join(HERE, "rrqr.npz"))
    if want("panels"):
        gen_panels(os.path.join(HERE, "panels.npz"))
    if want("small"):
        for tag, fam, n, b, eps in SMALL:
            run_case(tag, fam, n, b, eps, ("mgs", "blocked-hh", "tiled-hh"), store_full=(n <= 256))
    if args.full or want("C1"):
        c = configs.CONFIGS["C1"]
        run_case("C1", c.family, c.n, c.b, c.eps, c.methods, store_full=False)


if __name__ == "__main__" and not os.environ.get("GOLDEN_FULL"):
    main()


# ---------------------------------------------------------------------------
# full-size configs (background job; minutes to tens of minutes)
# ---------------------------------------------------------------------------


def run_full(name, methods=None):
    """Full-size config: store rank maps, R sketches, Frobenius norms, flop
    totals and the reference's rounded-add operand-rank histogram."""
    from threadpoolctl import threadpool_limits

    c = configs.CONFIGS[name]
    methods = methods or c.methods
    with threadpool_limits(8):
        tile, n = configs.tile_source(c)
    b, eps = c.b, c.eps
    p = n // b
    adm = rcore.weak_admissibility(p, p)
    t0 = time.perf_counter()
    with threadpool_limits(1):
        blocks = []
        for i in range(p):
            row = []
            for j in range(p):
                t = np.ascontiguousarray(tile(i * b, j * b, b, b))
                if adm[i, j]:
                    blk = rlr.compress_rrqr(t, rlr.ToleranceConfig(eps))
                    if not rcore.is_lowrank(blk):
                        adm[i, j] = False
                    row.append(blk)
                else:
                    row.append(t)
            blocks.append(row)
    a = rcore.BlrMatrix(rcore.BlrStructure(n, n, b, adm), blocks)
    tc = time.perf_counter() - t0
    out = {"input_ranks": np.array([[blk.rank if rcore.is_lowrank(blk) else -1
                                     for blk in row] for row in a.blocks])}
    summary = {"tag": name, "family": c.family, "n": n, "b": b, "eps": eps,
               "compress_s": tc, "methods": {}}
    print(name, "compressed", f"{tc:.1f}s", flush=True)
    orig = rlr.rounded_add
    for m in methods:
        hist = {}

        def counting(x, y, cfg, _orig=orig, _h=hist):
            o = _orig(x, y, cfg)
            key = (x.rank + y.rank, o.rank)
            _h[key] = _h.get(key, 0) + 1
            return o

        rfac.rounded_add = counting
        rflops.reset()
        t0 = time.perf_counter()
        with threadpool_limits(1):
            res = rsch.execute_sequential(m, a, rlr.ToleranceConfig(eps))
        tf = time.perf_counter() - t0
        rfac.rounded_add = orig
        fl = rflops.report()
        g = np.random.default_rng(5).standard_normal((n, 8))
        sk = np.zeros((n, 8))
        fro = np.zeros((p, p))
        sig3 = np.full((p, p, 3), np.nan)  # smallest 3 singular values of each LR block (tie proofs)
        for i in range(p):
            for j in range(p):
                blk = res.r.blocks[i][j]
                d = rcore.block_to_dense(blk)
                sk[i * b:(i + 1) * b] += d @ g[j * b:(j + 1) * b]
                fro[i, j] = np.linalg.norm(d)
                if rcore.is_lowrank(blk) and blk.rank:
                    ru = np.linalg.qr(blk.u)[1]
                    rv = np.linalg.qr(blk.v)[1]
                    s = np.linalg.svd(ru @ rv.T, compute_uv=False)[::-1][:3]
                    sig3[i, j, :len(s)] = s
        out[f"{m}_ranks"] = np.array([[blk.rank if rcore.is_lowrank(blk) else -1
                                       for blk in row] for row in res.r.blocks])
        out[f"{m}_sketch"] = sk
        out[f"{m}_fro"] = fro
        out[f"{m}_sig3"] = sig3
        out[f"{m}_radd_hist"] = np.array([[k[0], k[1], v] for k, v in sorted(hist.items())])
        summary["methods"][m] = {"factorize_s": tf, "flops": fl,
                                 "flops_total": int(sum(fl.values()))}
        print(name, m, f"{tf:.1f}s F={sum(fl.values()):.4e}", flush=True)
        np.savez_compressed(os.path.join(HERE, f"fact_{name}.npz"), **out)
        with open(os.path.join(HERE, f"fact_{name}.json"), "w") as fh:
            json.dump(summary, fh, indent=1, sort_keys=True)


if __name__ == "__main__" and os.environ.get("GOLDEN_FULL"):
    for nm in os.environ["GOLDEN_FULL"].split(","):
        run_full(nm)
