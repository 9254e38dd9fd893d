"""Config-scale kernel goldens from the UNMODIFIED reference ``blrqr`` package.

Run in the build container only (needs /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_scale.py [radd|rrqr|panels ...]

Inputs are regenerated bit-for-bit from ``oracle/scale_cases.py`` (seeded
numpy recipes); only what the reference returned is stored:

* ``radd_scale.npz``  -- 1200 rounded additions (lowrank.py:173-221) at
  b in {256, 512, 1024}, c up to 340: output rank, the SVD's singular values
  (captured from the reference's own ``np.linalg.svd`` call), the noise
  floor, ||C_ref - (A + B)||_F, ||A + B||_F and a 4 x 4 two-sided sketch.
* ``rrqr_scale.npz``  -- compress_rrqr (lowrank.py:138-150) of 48 C3 tiles
  (b = 512), 24 C5 tiles (b = 1024) and 32 synthetic graded tiles: rank
  (-1 = dense fallback), ||a - U V^T||_F, ||a||_F, sketch of U V^T.
* ``panels_scale.npz`` -- qr_compact_wy / apply_wy(_transpose)
  (kernels.py:87-128) at 512^2, 1024^2, 1300 x 1024, 768 x 512 and tp_qr /
  apply_tp(_transpose) (kernels.py:131-186) with n = 512 / 1024 tops over
  3..135-row bottoms: diag(R), row sketches of R, T, Y and the applications.
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from blrqr import core as rcore, kernels as rker, lowrank as rlr  # noqa: E402

from oracle import scale_cases as sc  # noqa: E402  (input recipes only)


def gen_radd(path):
    t0 = time.perf_counter()
    captured = []
    orig_svd = np.linalg.svd

    def svd_capture(x, *a, **k):
        out = orig_svd(x, *a, **k)
        captured.append(np.array(out[1]))
        return out

    ranks, floors, errs, nabs, cks, sks, sig, off, eps_, bs, cs, modes = ([] for _ in range(12))
    for t in range(sc.RADD_COUNT):
        d = sc.radd_case(t)
        a = rcore.LowRankBlock(d["ua"], d["va"])
        bk = rcore.LowRankBlock(d["ub"], d["vb"])
        captured.clear()
        np.linalg.svd = svd_capture
        try:
            out = rlr.rounded_add(a, bk, rlr.ToleranceConfig(d["eps"]))
        finally:
            np.linalg.svd = orig_svd
        s = captured[0] if captured else np.zeros(0)
        exact = d["ua"] @ d["va"].T + d["ub"] @ d["vb"].T
        cref = out.u @ out.v.T
        h, g = sc.sketch_mats(d["b"], 77 + t)
        ranks.append(out.rank)
        floors.append(rlr.NOISE_FLOOR * np.hypot(rlr._lr_norm(a), rlr._lr_norm(bk)))
        errs.append(np.linalg.norm(cref - exact))
        nabs.append(np.linalg.norm(exact))
        cks.append(sc.checksum(d["ua"], d["va"], d["ub"], d["vb"]))
        sks.append(h.T @ cref @ g)
        off.append(len(sig))
        sig.extend(s.tolist())
        eps_.append(d["eps"])
        bs.append(d["b"])
        cs.append(d["c"])
        modes.append(sc.RADD_MODES.index(d["mode"]))
    off.append(len(sig))
    np.savez_compressed(path, rank=np.array(ranks), floor=np.array(floors), err=np.array(errs),
                        nab=np.array(nabs), checksum=np.array(cks), sketch=np.array(sks),
                        sigma=np.array(sig), sigma_off=np.array(off), eps=np.array(eps_), b=np.array(bs),
                        c=np.array(cs), mode=np.array(modes))
    r = np.array(ranks)
    print(f"radd: {len(ranks)} cases, c max {max(cs)}, rank max {r.max()}, "
          f"{time.perf_counter() - t0:.1f}s", flush=True)


def gen_rrqr(path):
    t0 = time.perf_counter()
    cases = sc.rrqr_cases()
    ranks, errs, nrms, cks, sks, eps_ = [], [], [], [], [], []
    for t, case in enumerate(cases):
        a = sc.rrqr_tile(case)
        eps = 1e-8 if t % 3 else 1e-10
        out = rlr.compress_rrqr(a, rlr.ToleranceConfig(eps))
        b = a.shape[0]
        h, g = sc.sketch_mats(b, 99 + t)
        cks.append(sc.checksum(a))
        nrms.append(np.linalg.norm(a))
        eps_.append(eps)
        if rcore.is_lowrank(out):
            ranks.append(out.rank)
            d = out.u @ out.v.T
            errs.append(np.linalg.norm(a - d))
            sks.append(h.T @ d @ g)
        else:
            ranks.append(-1)
            errs.append(0.0)
            sks.append(np.zeros((4, 4)))
    np.savez_compressed(path, rank=np.array(ranks), err=np.array(errs), nrm=np.array(nrms),
                        checksum=np.array(cks), sketch=np.array(sks), eps=np.array(eps_))
    print(f"rrqr: {len(cases)} tiles, ranks {sorted(set(ranks))[:5]}..{max(ranks)}, "
          f"{time.perf_counter() - t0:.1f}s", flush=True)


def _hs(rows, seed, k=8):
    return np.random.default_rng(seed).standard_normal((rows, k))


def gen_panels(path):
    t0 = time.perf_counter()
    flat = {}
    for t in range(len(sc.GEQRT_CASES)):
        a, c = sc.geqrt_input(t)
        m, n = a.shape
        ref, r = rker.qr_compact_wy(a)
        flat[f"geqrt{t}_ck"] = np.array(sc.checksum(a, c))
        flat[f"geqrt{t}_diag"] = np.diag(r).copy()
        flat[f"geqrt{t}_r"] = _hs(n, 1000 + t).T @ r          # 8 x n
        flat[f"geqrt{t}_t"] = _hs(n, 2000 + t).T @ ref.t      # 8 x n
        flat[f"geqrt{t}_y"] = ref.y.T @ _hs(m, 3000 + t)      # n x 8
        flat[f"geqrt{t}_qc"] = rker.apply_wy(ref, c)[:, :8].copy()
        flat[f"geqrt{t}_qtc"] = rker.apply_wy_transpose(ref, c)[:, :8].copy()
        print(f"  geqrt {m}x{n}", flush=True)
    for t in range(len(sc.TPQRT_CASES)):
        top, bot, ct, cb = sc.tpqrt_input(t)
        n, k = bot.shape[1], bot.shape[0]
        ref, rn = rker.tp_qr(top, bot)
        flat[f"tp{t}_ck"] = np.array(sc.checksum(top, bot, ct, cb))
        flat[f"tp{t}_diag"] = np.diag(rn).copy()
        flat[f"tp{t}_r"] = _hs(n, 4000 + t).T @ rn
        flat[f"tp{t}_t"] = _hs(n, 5000 + t).T @ ref.t
        flat[f"tp{t}_y"] = _hs(k, 6000 + t).T @ ref.y       # 8 x n
        a1, a2 = rker.apply_tp(ref, ct, cb)
        b1, b2 = rker.apply_tp_transpose(ref, ct, cb)
        flat[f"tp{t}_q1"], flat[f"tp{t}_q2"] = _hs(n, 7000 + t).T @ a1, a2
        flat[f"tp{t}_qt1"], flat[f"tp{t}_qt2"] = _hs(n, 8000 + t).T @ b1, b2
        print(f"  tpqrt n={n} k={k}", flush=True)
    np.savez_compressed(path, **flat)
    print(f"panels: {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    want = set(sys.argv[1:]) or {"radd", "rrqr", "panels"}
    if "radd" in want:
        gen_radd(os.path.join(HERE, "radd_scale.npz"))
    if "rrqr" in want:
        gen_rrqr(os.path.join(HERE, "rrqr_scale.npz"))
    if "panels" in want:
        gen_panels(os.path.join(HERE, "panels_scale.npz"))
