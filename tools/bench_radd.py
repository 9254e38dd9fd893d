"""Micro-benchmark: one wave of batched rounded additions at given (b, c)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
from paper_2208_06194_b200 import _lib
from paper_2208_06194_b200.lowrank import _ptrs

rt = _lib.runtime()
dev = rt.dev
if os.environ.get("TEAMS", "1") == "0":
    rt.lib.blrqr_set_teams(0)
rng = np.random.default_rng(0)
CASES = [(512, 16, 16), (512, 32, 32), (512, 64, 64), (512, 100, 100), (512, 150, 150), (256, 4, 8), (1024, 8, 8)]
if len(sys.argv) > 1:
    CASES = [tuple(int(x) for x in a.split(',')) for a in sys.argv[1:]]
for b, ra, rb in CASES:
    nb = int(os.environ.get('BATCH', rt.nctas))
    # operands with geometric spectra, shared column space partly (typical sums)
    def lr(r, seed):
        g = np.random.default_rng(seed)
        u = np.linalg.qr(g.standard_normal((b, r)))[0]
        v = g.standard_normal((b, r)) * (10.0 ** (-np.arange(r) * 12.0 / max(r, 1)))
        return torch.from_numpy(u.T.copy()).to(dev).reshape(-1), torch.from_numpy(v.T.copy()).to(dev).reshape(-1)
    A = [lr(ra, 1) for _ in range(1)] * nb
    B = [lr(rb, 2) for _ in range(1)] * nb
    cap = min(b, ra + rb)
    uo = [torch.empty(b * cap, dtype=torch.float64, device=dev) for _ in range(nb)]
    vo = [torch.empty(b * cap, dtype=torch.float64, device=dev) for _ in range(nb)]
    ro = torch.zeros(nb, dtype=torch.int32, device=dev)
    ra_t = torch.full((nb,), ra, dtype=torch.int32, device=dev)
    rb_t = torch.full((nb,), rb, dtype=torch.int32, device=dev)
    pa = [_ptrs([x[0] for x in A]), _ptrs([x[1] for x in A]), _ptrs([x[0] for x in B]), _ptrs([x[1] for x in B]), _ptrs(uo), _ptrs(vo)]
    ws, per, nct = rt.workspace(b, cap)
    nct = nct if os.environ.get("TEAMS", "1") != "0" else min(nct, nb)
    def run():
        _lib.check(rt.lib.blrqr_rounded_add_batched(nb, b, b, pa[0].data_ptr(), pa[1].data_ptr(), ra_t.data_ptr(), pa[2].data_ptr(), pa[3].data_ptr(), rb_t.data_ptr(), pa[4].data_ptr(), pa[5].data_ptr(), ro.data_ptr(), cap, 1e-8, ws, per, nct, rt.status.data_ptr(), rt.flops.data_ptr(), _lib.stream_ptr()), "radd")
    run(); torch.cuda.synchronize(); rt.harvest()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    _, fl = rt.harvest()
    ph = rt.last_phases
    tot = ph.get("task", 0) or sum(v for k, v in ph.items() if k in ("qr", "core", "svd", "back"))
    print(json.dumps({"b": b, "c": ra + rb, "rank_out": int(ro[0].item()), "ms_per_wave": round(ms, 3), "batch": nb,
                      "phase_ms_per_radd": {k: round(v / 1.965e6 / nb, 3) for k, v in ph.items() if not k.startswith("jacobi")}, "sweeps_per_call": ph.get("jacobi_sweeps", 0) / max(1, ph.get("jacobi_calls", 1)),
                      "us_per_radd_per_cta": round(ms * 1e3, 1), "team_jobs": rt.last_stats[5], "team_members": rt.last_stats[6]}), flush=True)
