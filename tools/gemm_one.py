"""One DMMA CTA-GEMM probe launch (for ncu): M N K ta tb impl ctas reps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__ as ge
ge.build()
from paper_2208_06194_b200 import _lib
rt = _lib.runtime()
M, N, K, ta, tb, impl, ctas, reps = (int(x) for x in sys.argv[1:9])
lda = K if ta else M
ldb = N if tb else K
A = torch.randn(lda * (M if ta else K), dtype=torch.float64, device=rt.dev)
B = torch.randn(ldb * (K if tb else N), dtype=torch.float64, device=rt.dev)
C = torch.zeros(M * N, dtype=torch.float64, device=rt.dev)
rt.lib.blrqr_debug_gemm_impl(impl)
rt.lib.blrqr_debug_gemm(ta, tb, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), M, reps, ctas, _lib.stream_ptr())
torch.cuda.synchronize()
