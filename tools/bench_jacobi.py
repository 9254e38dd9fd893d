"""Micro-benchmark of the rounded addition's one-sided Jacobi stage.

The input is what rounded_add hands to Jacobi: R2 of the QR of P R1^T, with
R1 from the column-pivoted QR of a k x k core with a graded spectrum
(sigma_i = 10^(-16 i / k)).  Modes: 0 jacobi_blocked (1 CTA), 1 jacobi_cols
(1 CTA), 2 CTA team over all SMs.

python tools/bench_jacobi.py [kp ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sl  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
from paper_2208_06194_b200 import _lib  # noqa: E402

rt = _lib.runtime()
dev = rt.dev


def make_r2(k, seed=0):
    g = np.random.default_rng(seed)
    u = np.linalg.qr(g.standard_normal((k, k)))[0]
    v = np.linalg.qr(g.standard_normal((k, k)))[0]
    s = 10.0 ** (-16.0 * np.arange(k) / k)
    core = (u * s) @ v.T
    q1, r1, piv = sl.qr(core, pivoting=True)
    d = np.abs(np.diag(r1))
    kp = int(np.sum(d > 2.2e-16 * d[0])) or 1
    x = np.zeros((k, kp))
    x[piv, :] = r1[:kp, :].T
    r2 = np.linalg.qr(x)[1]
    return r2, s


sizes = [int(a) for a in sys.argv[1:]] or [128, 200, 260, 320]
for k in sizes:
    r2, s = make_r2(k)
    kp = r2.shape[0]
    ref = np.linalg.svd(r2, compute_uv=False)
    for mode in (int(m) for m in os.environ.get("MODES", "0,2,1,3").split(",")):
        if mode == 1 and kp > 160:
            continue
        x = torch.from_numpy(np.asfortranarray(r2).ravel(order="F").copy()).to(dev)
        jm = torch.empty(kp * kp, dtype=torch.float64, device=dev)
        sig = torch.empty(kp, dtype=torch.float64, device=dev)
        perm = torch.empty(kp, dtype=torch.int32, device=dev)
        ws, per, nct = rt.workspace(512, 512)
        x0 = x.clone()
        times = []
        for rep in range(3):
            x.copy_(x0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(rt.lib.blrqr_debug_jacobi(kp, kp, x.data_ptr(), jm.data_ptr(), sig.data_ptr(), perm.data_ptr(),
                                                 mode, ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(),
                                                 _lib.stream_ptr()), "jacobi")
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            rt.harvest()
        ph = rt.last_phases
        got = np.sort(sig.cpu().numpy())[::-1]
        err = float(np.max(np.abs(got - ref)) / ref[0])
        print(json.dumps({"k": k, "kp": kp, "mode": {0: "blocked", 1: "cols", 2: "team", 3: "pair_sweep_x1", 4: "pair_sweep_x50"}[mode], "ms": round(min(times), 3),
                          "sweeps": ph.get("jacobi_sweeps", 0), "team_members": rt.last_stats[6],
                          "svd_phase_ms": round(ph.get("svd", 0) / 1.965e6, 3),
                          "max_sigma_err_rel": err}), flush=True)
