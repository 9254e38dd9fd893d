"""Is the reference arm's bounded sample representative of the full run?

Compresses C3 with the oracle (threaded), then times on ONE core (single-
threaded BLAS, no pool): (1) bench.py's sample (k = 0 sweep, block rows
1..R) and (2) the oracle's whole tiled-hh factorization of the same grid.
Prints both GFLOP/s and their ratio as one JSON line (profiles/)."""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from concurrent.futures import ThreadPoolExecutor  # noqa: E402

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle import algorithms as oalg, blr as oblr, configs as ocfg, flops as ofl, lowrank as olr  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    rows_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "12,24").split(",")]
    c = ocfg.CONFIGS[name]
    b, p = c.b, c.n // c.b
    tile, _ = ocfg.tile_source(c)

    def comp(ij):
        i, j = ij
        t = np.ascontiguousarray(tile(i * b, j * b, b, b))
        return ij, (t if i == j else olr.compress(t, c.eps))

    t0 = time.perf_counter()
    cells = {}
    with threadpool_limits(1), ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
        for ij, x in pool.map(comp, [(i, j) for i in range(p) for j in range(p)]):
            cells[ij] = x
    t_comp = time.perf_counter() - t0
    out = {"config": name, "compress_s_threads": t_comp, "cores": 1}
    import copy

    def grid():
        lowrank = oblr.weak_map(p, p)
        return oblr.Grid(c.n, c.n, b, lowrank, [[copy.deepcopy(cells[(i, j)]) for j in range(p)] for i in range(p)])

    with threadpool_limits(1):
        for rows in rows_list:
            st = oalg.TiledState(grid(), c.eps)
            ofl.reset()
            t0 = time.perf_counter()
            st.diag_qr(0)
            for j in range(1, p):
                st.apply_block(0, j)
            for i in range(1, rows + 1):
                st.update_qr(0, i)
                for j in range(1, p):
                    st.apply_trap(0, i, j)
            dt = time.perf_counter() - t0
            out[f"sample_rows{rows}"] = {"s": dt, "flops": ofl.total(), "gflops": ofl.total() / dt / 1e9}
        ofl.reset()
        t0 = time.perf_counter()
        oalg.tiled_hh(grid(), c.eps)
        dt = time.perf_counter() - t0
        out["full"] = {"s": dt, "flops": ofl.total(), "gflops": ofl.total() / dt / 1e9}
    for rows in rows_list:
        out[f"sample_rows{rows}"]["rate_vs_full"] = out[f"sample_rows{rows}"]["gflops"] / out["full"]["gflops"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
