"""Time the phases of bench.py's e2e path (host BlrMatrix -> GPU -> R to host) at C3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__ as ge
ge.build()
from paper_2208_06194_b200 import configs
from paper_2208_06194_b200.core import weak_admissibility
from paper_2208_06194_b200.device import DeviceGrid
from paper_2208_06194_b200.factorize import DeviceFactorization
from paper_2208_06194_b200.lowrank import ToleranceConfig

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
dense = configs.dense_device(cfg)
g0 = DeviceGrid.from_dense(dense, cfg.b, weak_admissibility(cfg.n // cfg.b, cfg.n // cfg.b), cfg.eps, 0.5, cap=cfg.cap,
                           colmajor=True)
del dense
host = g0.to_host()
tol = ToleranceConfig(cfg.eps)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gd = DeviceGrid.from_host(host, pinned=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    fe = DeviceFactorization(cfg.method, gd, tol, clone=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    fe.run(); torch.cuda.synchronize(); t3 = time.perf_counter()
    r = fe.g.to_host()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    fe.finish()
    print(f"from_host {t1-t0:.3f}s  setup {t2-t1:.3f}s  run {t3-t2:.3f}s  to_host {t4-t3:.3f}s  total {t4-t0:.3f}s", flush=True)
