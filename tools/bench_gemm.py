"""Single-CTA GEMM throughput of the device gemm() for shapes on the hot path."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__ as ge
ge.build()
from paper_2208_06194_b200 import _lib
rt = _lib.runtime()
SHAPES = [  # (ta, tb, M, N, K, what)
    (0, 0, 512, 200, 16, "QR trailing / back: Z -= Y W (K=panel)"),
    (1, 0, 16, 200, 512, "W = Y^T Z (long K)"),
    (1, 0, 512, 30, 512, "T^T u products (dense_times)"),
    (0, 0, 512, 30, 512, "T u"),
    (0, 1, 300, 300, 150, "core R_U R_V^T"),
    (1, 0, 30, 30, 512, "small cores y.u^T x.u"),
    (0, 0, 512, 512, 16, "geqrt trailing"),
    (1, 0, 128, 128, 512, "S = Y^T Y"),
]
for ta, tb, M, N, K, what in SHAPES:
    A = torch.randn(max(M, K) * max(M, K), dtype=torch.float64, device=rt.dev)
    B = torch.randn(max(N, K) * max(N, K), dtype=torch.float64, device=rt.dev)
    C = torch.zeros(M * N, dtype=torch.float64, device=rt.dev)
    lda = K if ta else M
    ldb = N if tb else K
    reps = 20
    for ctas in (1, 148):
        Cc = torch.zeros(M * N * ctas, dtype=torch.float64, device=rt.dev) if ctas > 1 else C
        rt.lib.blrqr_debug_gemm(ta, tb, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), M, 2, ctas, _lib.stream_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rt.lib.blrqr_debug_gemm(ta, tb, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), M, reps, ctas, _lib.stream_ptr())
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        fl = 2.0 * M * N * K * reps * ctas
        print(json.dumps({"shape": [ta, tb, M, N, K], "what": what, "ctas": ctas, "us_per_gemm": ms * 1e3 / reps,
                          "gflops_per_cta": fl / ms / 1e6 / ctas, "total_tflops": fl / ms / 1e9}))
