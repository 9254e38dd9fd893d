"""Isolated dense-class kernels: GEQRT (DiagQR) at b = 512 /
1024 and TPQRT (UpdateQR) with n = 512 / 1024 tops, through
blrqr_panel_team -- the tiled factorization's own device routines on a CTA
team of `nctas` CTAs (1 = a lone CTA, 17 = the team size the critical chain
gets, 148 = the whole GPU).  CUDA-event time per call; GFLOP/s on the
reference flop model of the call (flops.py: qr_cost + tgen_cost) and on the
executed dense-contraction count.

python tools/bench_panels.py [--reps R] [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

FP64_PEAK = 37.07


def qr_cost(h, w):
    return 2 * h * w * w - (2 * w * w * w) // 3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default=None)
    ap.add_argument("--ctas", default="1,17,148")
    args = ap.parse_args()
    ge.build()
    from paper_2208_06194_b200 import _lib
    rt = _lib.runtime()
    dev = rt.dev
    out = []
    cases = [("geqrt", 512, 512), ("geqrt", 1024, 1024), ("tpqrt", 8, 512), ("tpqrt", 64, 512), ("tpqrt", 135, 512),
             ("tpqrt", 8, 1024), ("tpqrt", 16, 1024), ("tpqrt", 64, 1024)]
    g = torch.Generator(device="cpu").manual_seed(0)
    for op, m, n in cases:
        if op == "geqrt":
            a = torch.randn(m * n, dtype=torch.float64, generator=g).to(dev)
            a2 = None
            o1, o2, o3 = (torch.empty(x, dtype=torch.float64, device=dev) for x in (m * n, n * n, n * n))
            model = qr_cost(m, n) + m * n * n
        else:
            top = torch.triu(torch.randn(n, n, dtype=torch.float64, generator=g)) + n ** 0.5 * torch.eye(n, dtype=torch.float64)
            a = top.T.contiguous().reshape(-1).to(dev)  # column-major upper triangle
            a2 = torch.randn(m * n, dtype=torch.float64, generator=g).to(dev)
            o1, o2, o3 = (torch.empty(x, dtype=torch.float64, device=dev) for x in (n * n, m * n, n * n))
            model = qr_cost(n + m, n) + (n + m) * n * n
        for nct in [int(x) for x in args.ctas.split(",")]:
            ws, per, _ = rt.workspace(max(m, n, 64), n, m + n, nctas=nct)

            def call():
                _lib.check(rt.lib.blrqr_panel_team(0 if op == "geqrt" else 1, m, n, a.data_ptr(),
                                                   a2.data_ptr() if a2 is not None else None, o1.data_ptr(),
                                                   o2.data_ptr(), o3.data_ptr(), ws, per, nct, rt.status.data_ptr(),
                                                   rt.flops.data_ptr(), _lib.stream_ptr()), op)

            call()
            rt.harvest()
            phases = {k: round(v / 1.965e6 / 1, 3) for k, v in rt.last_phases.items()}  # ms (SM clock)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            rt.harvest()
            ms = e0.elapsed_time(e1) / args.reps
            rec = {"op": op, "rows": m, "n": n, "nctas": nct, "ms": round(ms, 4),
                   "model_gflops": round(model / ms / 1e6, 1),
                   "frac_fp64_peak": round(model / ms / 1e9 / FP64_PEAK, 4), "phases_ms": phases}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
