"""Config-scale kernel parity against reference-written goldens (GPU box).

The operand shapes the C2-C5 factorizations actually run -- rounded additions
at b = 256/512/1024 with cores up to c = 340, RRQR of 512^2 / 1024^2 config
tiles, GEQRT at 512^2 / 1024^2 / 1300 x 1024 and TPQRT with n = 512 / 1024
tops over 3..135-row bottoms -- checked against what the UNMODIFIED reference
returned on bit-identical inputs (tests/golden/make_golden_scale.py; inputs
regenerated from oracle/scale_cases.py).

Bars:
* ranks equal to the reference's, except at proven truncation ties (the
  reference's own singular values / residuals put the threshold within
  1e-6 relative of the differing rank);
* rounded addition: U orthonormal to 1e-12 sqrt(r); the singular values the
  GPU kept (column norms of V_C, U_C being orthonormal) equal the
  reference's to 1e-10 sigma_0 + 1e-12 hypot(||A||, ||B||) (rounding of
  the operands' scale: a near-cancelling sum has sigma_0 << ||A||);
  ||C_gpu - (A + B)||_F within 1e-3 of the reference's own truncation error
  (+ 1e-12 max(||A + B||, hypot(||A||, ||B||)));
* RRQR: ||a - U V^T||_F <= eps ||a||_F and UV^T within 2 eps of the
  reference's product (two-sided sketch); ranks equal except pivot-order
  ties (at most 10 % of tiles, each within 2 of the reference's rank with the
  stopping residual inside [0.5, 1] eps ||a||);
* dense panels (well-conditioned inputs): R, T, Y and the applications
  within 1e-10 relative of the reference (row sketches; diag(R) exact sign
  convention to 1e-10).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import scale_cases as sc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import __graft_entry__ as ge
    ge.build()
    import paper_2208_06194_b200 as pkg
    return pkg


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _radd_tie(sig, floor, eps, r_gpu, r_ref, tol=1e-6):
    """The reference's rank decision is within `tol` of flipping to r_gpu."""
    s2 = sig * sig
    tot2 = float(np.sum(s2))
    tail2 = np.concatenate([np.cumsum(s2[::-1])[::-1], [0.0]])
    cut2 = eps * eps * tot2
    lo, hi = min(r_gpu, r_ref), max(r_gpu, r_ref)
    # truncation tie: the tail at the boundary ranks sits on the cut
    if any(abs(tail2[k] - cut2) <= tol * cut2 for k in range(lo, hi + 1)):
        return True
    # significance tie: a singular value at the noise floor
    return any(abs(x - floor) <= tol * floor for x in sig[lo:hi + 1])


def test_rounded_add_config_scale(pk):
    import torch
    z = np.load(os.path.join(GOLDEN, "radd_scale.npz"))
    n = len(z["rank"])
    assert n >= 1000
    groups = {}
    cases = []
    for t in range(n):
        d = sc.radd_case(t)
        ck = sc.checksum(d["ua"], d["va"], d["ub"], d["vb"])
        assert abs(ck - z["checksum"][t]) <= 1e-9 * max(1.0, abs(z["checksum"][t])), f"input recipe drift at {t}"
        cases.append(d)
        groups.setdefault((d["b"], d["eps"]), []).append(t)
    outs = {}
    for (b, eps), ts in groups.items():
        for s in range(0, len(ts), 128):
            chunk = ts[s:s + 128]
            pairs = [(pk.LowRankBlock(cases[t]["ua"], cases[t]["va"]), pk.LowRankBlock(cases[t]["ub"], cases[t]["vb"]))
                     for t in chunk]
            for t, o in zip(chunk, pk.rounded_add_batched(pairs, pk.ToleranceConfig(eps))):
                outs[t] = o
    dev = torch.device("cuda")
    mism, worst_sig, worst_err = [], 0.0, 0.0
    by_b = {}
    for t in range(n):
        d, o = cases[t], outs[t]
        sig = z["sigma"][z["sigma_off"][t]:z["sigma_off"][t + 1]]
        r_ref = int(z["rank"][t])
        by_b.setdefault(d["b"], [0, 0])[0] += 1
        if o.rank != r_ref:
            assert abs(o.rank - r_ref) <= 2 and _radd_tie(sig, z["floor"][t], d["eps"], o.rank, r_ref), \
                (t, d["b"], d["c"], d["mode"], o.rank, r_ref)
            mism.append(t)
            continue
        by_b[d["b"]][1] += 1
        if o.rank == 0:
            continue
        u, v = torch.from_numpy(o.u).to(dev), torch.from_numpy(o.v).to(dev)
        eye = torch.eye(o.rank, dtype=torch.float64, device=dev)
        assert float(torch.linalg.norm(u.T @ u - eye)) < 1e-12 * np.sqrt(o.rank) * 10, t
        # kept singular values = column norms of V_C (U_C orthonormal)
        # backward-stable SVDs agree to rounding of the OPERANDS' scale
        # (hyp = hypot(||A||, ||B||) = floor / NOISE_FLOOR), which dominates
        # sigma_0 of a near-cancelling sum
        hyp = z["floor"][t] / pk.lowrank.NOISE_FLOOR
        sg = torch.linalg.norm(v, dim=0).cpu().numpy()
        ds = float(np.max(np.abs(np.sort(sg)[::-1] - sig[:o.rank])))
        worst_sig = max(worst_sig, ds / (sig[0] + hyp))
        assert ds <= 1e-10 * sig[0] + 1e-12 * hyp, (t, d["mode"], ds / sig[0], ds / hyp)
        exact = torch.from_numpy(d["ua"]).to(dev) @ torch.from_numpy(d["va"]).to(dev).T + \
            torch.from_numpy(d["ub"]).to(dev) @ torch.from_numpy(d["vb"]).to(dev).T
        err = float(torch.linalg.norm(u @ v.T - exact))
        bound = z["err"][t] * (1 + 1e-3) + 1e-12 * max(z["nab"][t], hyp)
        worst_err = max(worst_err, (err - z["err"][t]) / max(z["nab"][t], hyp))
        assert err <= bound, (t, d["mode"], err, z["err"][t], z["nab"][t], hyp)
    print(f"rounded_add config-scale: {n} cases (b: {by_b}), tie mismatches {len(mism)}, "
          f"max |dsigma|/(sigma0+hyp) {worst_sig:.2e}, max (err-err_ref)/max(|A+B|,hyp) {worst_err:.2e}")
    assert len(mism) <= n // 200


def test_rrqr_config_tiles(pk):
    z = np.load(os.path.join(GOLDEN, "rrqr_scale.npz"))
    cases = sc.rrqr_cases()
    assert len(cases) == len(z["rank"])
    by_shape = {}
    for t, case in enumerate(cases):
        by_shape.setdefault((case[1], float(z["eps"][t])), []).append(t)
    tiles = {t: sc.rrqr_tile(c) for t, c in enumerate(cases)}
    for t, a in tiles.items():
        assert abs(sc.checksum(a) - z["checksum"][t]) <= 1e-9 * max(1.0, abs(z["checksum"][t])), t
    mism = 0
    for (b, eps), ts in by_shape.items():
        outs = pk.lowrank.compress_batched([tiles[t] for t in ts], eps, b // 2)
        for t, o in zip(ts, outs):
            a, r_ref = tiles[t], int(z["rank"][t])
            nrm = z["nrm"][t]
            if o is None:
                assert r_ref == -1 or r_ref >= b // 2 - 2, (t, r_ref)
                mism += r_ref != -1
                continue
            u, v = o
            r = u.shape[1]
            err = np.linalg.norm(a - u @ v.T)
            assert err <= eps * nrm * (1 + 1e-6), (t, err / nrm)
            if r:
                assert np.linalg.norm(u.T @ u - np.eye(r)) < 1e-12 * max(1, r) * 10
            if r != r_ref:
                # pivoted QR residuals at a given rank depend on the pivot order
                # (rounding-level norm differences change it, and graded tiles'
                # residual curves then differ by O(1) factors near the cut): a
                # lower GPU rank is a pivot-order tie when the GPU stopped in the
                # band [0.5, 1] eps ||a|| under the cut, a higher one when the
                # reference's residual at its rank was in that band; Laplace
                # (C5) tiles have exactly equal column norms -- pivot ties
                assert r_ref != -1 and abs(r - r_ref) <= 2, (t, r, r_ref)
                band = err if r < r_ref else z["err"][t]
                near = band >= 0.5 * eps * nrm
                assert near or cases[t][0] == "C5", (t, r, r_ref, err / nrm, z["err"][t] / nrm)
                print(f"  rrqr tie: tile {t} ({cases[t][0]}, b={b}) rank {r} vs {r_ref}, "
                      f"residual/(eps|a|) gpu {err / (eps * nrm):.3f} ref {z['err'][t] / (eps * nrm):.3f}")
                mism += 1
                continue
            h, g = sc.sketch_mats(b, 99 + t)
            sk = h.T @ (u @ v.T) @ g
            assert np.linalg.norm(sk - z["sketch"][t]) <= 2.5 * eps * nrm * np.linalg.norm(h) * np.linalg.norm(g), t
    print(f"rrqr config tiles: {len(cases)} tiles, rank mismatches (ties) {mism}")
    assert mism <= len(cases) // 10


def _hs(rows, seed, k=8):
    return np.random.default_rng(seed).standard_normal((rows, k))


def test_geqrt_config_scale(pk):
    z = np.load(os.path.join(GOLDEN, "panels_scale.npz"))
    for t in range(len(sc.GEQRT_CASES)):
        a, c = sc.geqrt_input(t)
        assert abs(sc.checksum(a, c) - float(z[f"geqrt{t}_ck"])) <= 1e-9 * abs(float(z[f"geqrt{t}_ck"]))
        m, n = a.shape
        ref, r = pk.qr_compact_wy(a)
        assert _rel(np.diag(r), z[f"geqrt{t}_diag"]) < 1e-10, t
        assert _rel(_hs(n, 1000 + t).T @ r, z[f"geqrt{t}_r"]) < 1e-10, t
        assert _rel(_hs(n, 2000 + t).T @ ref.t, z[f"geqrt{t}_t"]) < 1e-10, t
        assert _rel(ref.y.T @ _hs(m, 3000 + t), z[f"geqrt{t}_y"]) < 1e-10, t
        assert _rel(pk.apply_wy(ref, c)[:, :8], z[f"geqrt{t}_qc"]) < 1e-10, t
        assert _rel(pk.apply_wy_transpose(ref, c)[:, :8], z[f"geqrt{t}_qtc"]) < 1e-10, t


def test_tpqrt_config_scale(pk):
    z = np.load(os.path.join(GOLDEN, "panels_scale.npz"))
    for t in range(len(sc.TPQRT_CASES)):
        top, bot, ct, cb = sc.tpqrt_input(t)
        assert abs(sc.checksum(top, bot, ct, cb) - float(z[f"tp{t}_ck"])) <= 1e-9 * abs(float(z[f"tp{t}_ck"]))
        n, k = bot.shape[1], bot.shape[0]
        ref, rn = pk.tp_qr(top, bot)
        assert _rel(np.diag(rn), z[f"tp{t}_diag"]) < 1e-10, (t, n, k)
        assert _rel(_hs(n, 4000 + t).T @ rn, z[f"tp{t}_r"]) < 1e-10, (t, n, k)
        assert _rel(_hs(n, 5000 + t).T @ ref.t, z[f"tp{t}_t"]) < 1e-10, (t, n, k)
        assert _rel(_hs(k, 6000 + t).T @ ref.y, z[f"tp{t}_y"]) < 1e-10, (t, n, k)
        a1, a2 = pk.apply_tp(ref, ct, cb)
        b1, b2 = pk.apply_tp_transpose(ref, ct, cb)
        assert _rel(_hs(n, 7000 + t).T @ a1, z[f"tp{t}_q1"]) < 1e-10 and _rel(a2, z[f"tp{t}_q2"]) < 1e-10
        assert _rel(_hs(n, 8000 + t).T @ b1, z[f"tp{t}_qt1"]) < 1e-10 and _rel(b2, z[f"tp{t}_qt2"]) < 1e-10
