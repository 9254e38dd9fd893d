import os
import sys

# Single-threaded BLAS for the oracle so it replays the reference's arithmetic
# (the golden fixtures were generated with OPENBLAS_NUM_THREADS=1).
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
