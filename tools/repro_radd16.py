"""Repro: rounded additions at b = 16 with c = ra + rb above and below b."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__ as ge
ge.build()
import paper_2208_06194_b200 as pk
from oracle import lowrank as olr, blr as oblr
b = int(sys.argv[1]); ra = int(sys.argv[2]); rb = int(sys.argv[3])
rng = np.random.default_rng(0)
def lr(r):
    u = np.linalg.qr(rng.standard_normal((b, r)))[0]
    return pk.LowRankBlock(u, rng.standard_normal((b, r)) * 10.0 ** -np.arange(r))
a, c = lr(ra), lr(rb)
o = pk.rounded_add(a, c, pk.ToleranceConfig(1e-8))
ref = olr.rounded_add(oblr.LR(a.u, a.v), oblr.LR(c.u, c.v), 1e-8)
print("b", b, "ra", ra, "rb", rb, "rank", o.rank, ref.rank, "err", np.linalg.norm(o.to_dense() - ref.dense()))
