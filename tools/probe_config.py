"""Probe one config end to end on the GPU: generate, compress, factorize.

python tools/probe_config.py C3 [--method tiled-hh] [--n N] [--cap CAP]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--method", default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--cap", type=int, default=None)
    ap.add_argument("--levels", type=int, default=None, help="only run the first L levels")
    ap.add_argument("--profile-levels", action="store_true")
    ap.add_argument("--sched", default="dag")
    ap.add_argument("--no-teams", action="store_true")
    ap.add_argument("--team-slack", type=int, default=None)
    ap.add_argument("--rings", type=int, default=None)
    ap.add_argument("--reserve", type=int, default=None, help="reserved team-helper CTAs of the DAG kernel")
    args = ap.parse_args()
    ge.build()
    from paper_2208_06194_b200 import _lib, configs, flops
    from paper_2208_06194_b200.core import weak_admissibility
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import DeviceFactorization
    from paper_2208_06194_b200.lowrank import ToleranceConfig

    if args.no_teams:
        _lib.runtime().lib.blrqr_set_teams(0)
    elif args.team_slack is not None:
        _lib.runtime().lib.blrqr_set_teams(2 + args.team_slack)
    if args.reserve is not None:
        _lib.runtime().lib.blrqr_set_team_reserve(args.reserve)
    if args.rings is not None:
        _lib.runtime().lib.blrqr_set_dag_rings(args.rings)
    cfg = configs.CONFIGS[args.config]
    n = args.n or cfg.n
    method = args.method or cfg.method
    t0 = time.perf_counter()
    dense = configs.dense_device(cfg, n)
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    g = DeviceGrid.from_dense(dense, cfg.b, weak_admissibility(n // cfg.b, n // cfg.b), cfg.eps, 0.5,
                              cap=args.cap or cfg.cap, colmajor=True)
    torch.cuda.synchronize()
    tc = time.perf_counter() - t0
    del dense
    rk = g.rank_map()
    lr = rk[rk >= 0]
    print(json.dumps({"gen_s": tg, "compress_s": tc, "in_rank_min": int(lr.min()), "in_rank_med": float(np.median(lr)),
                      "in_rank_max": int(lr.max())}), flush=True)
    flops.reset()
    f = DeviceFactorization(method, g, ToleranceConfig(cfg.eps), scheduler=args.sched if method == "tiled-hh" else "dag")
    rt = _lib.runtime()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    if method == "tiled-hh" and (args.levels or args.profile_levels) and args.sched == "levels":
        import ctypes as C
        ws, per, nct = rt.workspace(g.b, g.cap)
        gs, rs = f.g.cstruct(), f.rf.cstruct()
        L = args.levels or f.nlevels
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
        evs[0].record()
        for lv in range(L):
            _lib.check(rt.lib.blrqr_tiled_run(C.byref(gs), C.byref(rs), f.tasks.data_ptr(),
                                              f.levels.ctypes.data_as(C.c_void_p), lv, lv + 1, cfg.eps, ws, per,
                                              nct, rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()),
                       "run")
            evs[lv + 1].record()
        torch.cuda.synchronize()
        tasks = f.tasks.cpu().numpy()
        rows = []
        for lv in range(L):
            t0_, t1_ = f.levels[lv], f.levels[lv + 1]
            kinds = np.bincount(tasks[t0_:t1_, 0], minlength=4).tolist()
            rows.append((evs[lv].elapsed_time(evs[lv + 1]), lv, kinds))
        rows.sort(reverse=True)
        tot_ms = sum(r[0] for r in rows)
        print("levels total ms", tot_ms, "top levels:")
        for r in rows[:25]:
            print(f"  lv {r[1]:4d} {r[0]:9.2f} ms kinds(diag,block,update,trap)={r[2]}")
        acc = np.cumsum(sorted([r[0] for r in rows], reverse=True))
        print("share of top 10/50/100 levels:", [float(acc[min(k, len(acc)) - 1] / tot_ms) for k in (10, 50, 100)])
    else:
        f.run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rep = f.finish()
    ph = dict(_lib.runtime().last_phases)
    clk = 1.965e9
    print(json.dumps({"phase_seconds_summed_over_ctas": {k: v / clk for k, v in ph.items()
                                                         if not k.startswith("jacobi")},
                      "task_seconds_per_sm": ph.get("task", 0) / clk / _lib.runtime().nctas,
                      "jacobi_sweeps_per_call": ph.get("jacobi_sweeps", 0) / max(1, ph.get("jacobi_calls", 1)),
                      "big_core_stats(k>=64)": {"count": _lib.runtime().last_stats[2], "mean_k": _lib.runtime().last_stats[0] / max(1, _lib.runtime().last_stats[2]), "mean_kp": _lib.runtime().last_stats[1] / max(1, _lib.runtime().last_stats[2]), "sum_k3_over_sum_kp3": _lib.runtime().last_stats[3] / max(1, _lib.runtime().last_stats[4])},
                      "team_jobs": _lib.runtime().last_stats[5], "team_members": _lib.runtime().last_stats[6]}))
    tot = sum(rep.values())
    rr = f.g.rank_map()
    rl = rr[rr >= 0]
    print(json.dumps({"config": args.config, "n": n, "method": method, "factorize_s": ms / 1e3,
                      "F_model": tot, "gflops": tot / ms / 1e6, "flops": rep,
                      "r_rank_med": float(np.median(rl)) if rl.size else 0, "r_rank_max": int(rl.max()) if rl.size else 0,
                      "mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)


if __name__ == "__main__":
    main()
