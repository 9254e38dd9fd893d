"""CTA-level FP64 GEMM on the shapes of the hot path: DFMA tiles (impl 1)
against DMMA tensor-core tiles (impl 2) and the default dispatch (impl 0).

One CTA (latency of a single task's GEMM) and 148 CTAs (throughput, one per
SM); correctness of every impl against torch float64.  Prints one JSON line
per (shape, impl, ctas)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
from paper_2208_06194_b200 import _lib  # noqa: E402

rt = _lib.runtime()
SHAPES = [  # (ta, tb, M, N, K, what)
    (0, 0, 512, 200, 16, "QR trailing / back: Z -= Y W (K=panel)"),
    (0, 0, 1024, 960, 16, "GEQRT 1024 trailing, K=16"),
    (0, 0, 1024, 960, 64, "GEQRT 1024 trailing, K=64"),
    (1, 0, 64, 960, 1024, "W = Y^T A2 (K=1024, 64 rows)"),
    (1, 0, 16, 200, 512, "W = Y^T Z (long K)"),
    (1, 0, 512, 30, 512, "T^T u products (dense_times)"),
    (0, 0, 512, 30, 512, "T u"),
    (0, 1, 300, 300, 150, "core R_U R_V^T"),
    (1, 0, 30, 30, 512, "small cores y.u^T x.u"),
    (0, 0, 512, 512, 16, "geqrt trailing"),
    (1, 0, 128, 128, 512, "S = Y^T Y"),
    (0, 0, 512, 512, 512, "square 512"),
    (0, 0, 1024, 64, 1024, "T(1024) x 64 cols"),
]


def run(ta, tb, M, N, K, reps, ctas, impl):
    _lib.check(rt.lib.blrqr_debug_gemm_impl(impl), "impl")
    lda = K if ta else M
    ldb = N if tb else K
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(lda * (M if ta else K), dtype=torch.float64, generator=g).to(rt.dev)
    B = torch.randn(ldb * (K if tb else N), dtype=torch.float64, generator=g).to(rt.dev)
    C = torch.zeros(M * N, dtype=torch.float64, device=rt.dev)
    rt.lib.blrqr_debug_gemm(ta, tb, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), M, 1, 1,
                            _lib.stream_ptr())
    torch.cuda.synchronize()
    Am = A.view(M if ta else K, lda).T if True else None  # column-major view: (lda x cols)
    Am = A.view(-1, lda).T[: (K if ta else M)]
    opA = Am.T if ta else Am
    Bm = B.view(-1, ldb).T[: (N if tb else K)]
    opB = Bm.T if tb else Bm
    ref = opA @ opB
    got = C.view(N, M).T
    err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rt.lib.blrqr_debug_gemm(ta, tb, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), M, 2, ctas,
                            _lib.stream_ptr())
    torch.cuda.synchronize()
    e0.record()
    rt.lib.blrqr_debug_gemm(ta, tb, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), M, reps, ctas,
                            _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fl = 2.0 * M * N * K * reps * ctas
    return err, ms * 1e3 / reps, fl / ms / 1e9


if __name__ == "__main__":
    for ta, tb, M, N, K, what in SHAPES:
        for impl in (1, 2, 0):
            for ctas in (1, 148):
                err, us, tf = run(ta, tb, M, N, K, 10, ctas, impl)
                print(json.dumps({"shape": [ta, tb, M, N, K], "what": what, "impl": ["default", "dfma", "dmma"][impl],
                                  "ctas": ctas, "rel_err": err, "us_per_gemm": round(us, 2),
                                  "total_tflops": round(tf, 3)}), flush=True)
    rt.lib.blrqr_debug_gemm_impl(0)
