"""ctypes binding of libblrqr.so (include/blrqr.h) plus device plumbing.

The CUDA library is the only compute path: importing this module on a
machine without the built library raises, and every entry point raises if no
CUDA device is present.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BLRQR_LIB") or os.path.join(_HERE, "lib", "libblrqr.so")

FLOP_KINDS = ("compress", "rounded_add", "expand", "lr_mul", "gemm", "panel_qr",
              "apply_wy", "update_qr", "apply_tp")
PHASES = ("norm", "qr", "core", "svd", "back", "product", "tpqrt", "geqrt", "apply_wy", "rrqr", "expand", "task",
          "qrcp", "jacobi_sweeps", "jacobi_calls", "tbuild")
ST_RANK_OVERFLOW, ST_ARENA_OVERFLOW, ST_NONFINITE, ST_MGS_COLLAPSE, ST_BAD_KIND, ST_BAD_ARG = (
    1, 2, 4, 8, 16, 32)
ST_SCHED_TIMEOUT = 64

_lib = None
_lock = threading.Lock()


class Grid(C.Structure):
    _fields_ = [("p", C.c_int), ("q", C.c_int), ("b", C.c_int), ("cap", C.c_int),
                ("lowrank", C.c_void_p), ("rank", C.c_void_p), ("pool", C.c_void_p),
                ("off_u", C.c_void_p), ("off_v", C.c_void_p)]


class Refl(C.Structure):
    _fields_ = [("pool", C.c_void_p), ("y_off", C.c_void_p), ("t_off", C.c_void_p),
                ("yrank", C.c_void_p), ("wpool", C.c_void_p), ("wrank", C.c_void_p), ("wslot", C.c_int64)]


class Task(C.Structure):
    _fields_ = [("kind", C.c_int), ("k", C.c_int), ("i", C.c_int), ("j", C.c_int)]


class DagRank(C.Structure):
    """blrqr_dag_rank: one rank's DAG as device arrays."""
    _fields_ = [("g", Grid), ("rf", Refl), ("ntasks", C.c_int), ("tasks", C.c_void_p), ("indeg0", C.c_void_p),
                ("succ_off", C.c_void_p), ("succ", C.c_void_p), ("prio", C.c_void_p), ("rsucc_off", C.c_void_p),
                ("rsucc", C.c_void_p), ("work", C.c_void_p)]


class Peer(C.Structure):
    """blrqr_peer: another rank's memory as addressed from this device."""
    _fields_ = [("gpool", C.c_void_p), ("rpool", C.c_void_p), ("yrank", C.c_void_p), ("work", C.c_void_p),
                ("prio", C.c_void_p), ("ntasks", C.c_int)]


MAX_WORLD = 8


_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_D = C.c_double

_SIGS = {
    "blrqr_version": ([], _I),
    "blrqr_workspace_doubles": ([_I, _I, _I], _L),
    "blrqr_default_ctas": ([], _I),
    "blrqr_rounded_add_batched": ([_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _D, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_compress_batched": ([_I, _I, _I, _P, _P, _P, _P, _I, _D, _I, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_lr_product": ([_I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _I, _P, _P, _P, _P, _L, _P, _P, _P], _I),
    "blrqr_geqrt": ([_I, _I, _P, _P, _P, _P, _P, _L, _P, _P, _P], _I),
    "blrqr_apply_wy": ([_I, _I, _I, _P, _P, _P, _I, _P, _L, _P, _P, _P], _I),
    "blrqr_tpqrt": ([_I, _I, _P, _P, _P, _P, _P, _P, _L, _P, _P, _P], _I),
    "blrqr_apply_tp": ([_I, _I, _I, _P, _P, _P, _P, _I, _P, _L, _P, _P, _P], _I),
    "blrqr_mgs_panel": ([_I, _I, _P, _P, _P, _P, _L, _P, _P, _P], _I),
    "blrqr_dense_to_blr": ([_P, _L, C.POINTER(Grid), _P, _D, _D, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_grid_pack": ([C.POINTER(Grid), _P, _P, _I, _P], _I),
    "blrqr_tiled_task_count": ([_I, _I], _L),
    "blrqr_tiled_schedule": ([_I, _I, _P, _P, _L], _I),
    "blrqr_tiled_run": ([C.POINTER(Grid), C.POINTER(Refl), _P, _P, _I, _I, _D, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_tiled_dag_size": ([_I, _I, _P], _L),
    "blrqr_debug_trace": ([_P], None),
    "blrqr_set_teams": ([_I], None),
    "blrqr_set_dag_rings": ([_I], None),
    "blrqr_set_qrcp_tol": ([_D], _I),
    "blrqr_set_team_reserve": ([_I], None),
    "blrqr_dag_work_ints": ([_I], _L),
    "blrqr_debug_phase_trace": ([_P], None),
    "blrqr_apply_q": ([C.POINTER(Grid), C.POINTER(Refl), _I, _P, _L, _I, _I, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_blr_to_dense": ([C.POINTER(Grid), _P, _L, _P], _I),
    "blrqr_apply_q_blr": ([C.POINTER(Grid), C.POINTER(Refl), _I, C.POINTER(Grid), _I, _D, _P, _P, _P, _L, _I, _P,
                           _P, _P], _I),
    "blrqr_debug_jacobi": ([_I, _I, _P, _P, _P, _P, _I, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_debug_gemm": ([_I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _I, _I, _P], _I),
    "blrqr_debug_gemm_impl": ([_I], _I),
    "blrqr_debug_arena_guard": ([_L], _I),
    "blrqr_set_arena_hot": ([_L], _I),
    "blrqr_arena_hot": ([], _L),
    "blrqr_panel_team": ([_I, _I, _I, _P, _P, _P, _P, _P, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_tiled_dag": ([_I, _I, _P, _P, _P, _P, _P], _I),
    "blrqr_tiled_ref_dag": ([_I, _I, _P, _P, _P, _L], _L),
    "blrqr_dag_policy": ([], _L),
    "blrqr_tiled_run_dag": ([C.POINTER(Grid), C.POINTER(Refl), _I, _P, _P, _P, _P, _P, _P, _D, _P, _L, _I, _D, _P,
                             _P, _P], _I),
    "blrqr_tiled_dist_dag_size": ([_I, _I, _I, _I, _P, _P], _L),
    "blrqr_tiled_dist_dag": ([_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "blrqr_tiled_dag_reset": ([_I, _P, _P], _I),
    "blrqr_tiled_run_dag_multi": ([_I, _I, _P, _P, _P, _D, _P, _L, _I, _D, _P, _P, _P], _I),
    "blrqr_ipc_handle": ([_P, _P, _P], _I),
    "blrqr_ipc_open": ([_P, _P], _I),
    "blrqr_ipc_close": ([_P], _I),
    "blrqr_enable_peer_access": ([], _I),
    "blrqr_blocked_step": ([C.POINTER(Grid), C.POINTER(Refl), _I, _D, _P, _P, _P, _L, _P, _L, _I, _P, _P, _P], _I),
    "blrqr_blocked_step_dist": ([C.POINTER(Grid), C.POINTER(Refl), _I, _D, _P, _P, _P, _L, _P, _L, _I, _I, _I, _I,
                                 _P, _P, _P], _I),
    "blrqr_mgs_step_dist": ([C.POINTER(Grid), C.POINTER(Grid), C.POINTER(Grid), _I, _D, _P, _L, _P, _L, _I, _I, _I,
                             _I, _P, _P, _P], _I),
    "blrqr_mgs_step": ([C.POINTER(Grid), C.POINTER(Grid), C.POINTER(Grid), _I, _D, _P, _L, _P, _L, _I, _P, _P, _P],
                       _I),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load (once) and type the C ABI.  Raises if the library is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"libblrqr.so not built at {path}; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(path)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc < 0:
        raise ValueError(f"{what}: invalid argument (code {rc})")
    raise RuntimeError(f"{what}: CUDA error {rc - 1000 if rc >= 1000 else rc}")


ARENA_HOT_DEFAULT = 0  # doubles per CTA pinned in L2 (0: plain per-CTA strides); see DESIGN 5d


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2208_06194_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


class Runtime:
    """Per-process device state: workspace arena, status word, flop counters.

    One stream at a time: the per-CTA workspace, the status word and the flop
    counters are process-wide, so two factorizations must not run
    concurrently on different streams (the CTA-team tables inside libblrqr
    are per (device, stream), but these buffers are not)."""

    def __init__(self):
        self.dev = require_cuda()
        self.lib = load()
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # [0:9] model flops per kind, [16:32] per-phase SM cycles (see PHASES)
        self.flops = torch.zeros(64, dtype=torch.int64, device=self.dev)
        self.last_phases = {}
        self.nctas = int(self.lib.blrqr_default_ctas())
        self._ws = None
        self._ws_per_cta = 0
        self.arena_guard = 0
        self._guard = (0, 0)
        # split arena + L2 persistence of the hot scratch (blrqr_set_arena_hot), doubles per CTA
        self.arena_hot = int(os.environ.get("BLRQR_ARENA_HOT", ARENA_HOT_DEFAULT))
        check(self.lib.blrqr_set_arena_hot(self.arena_hot), "arena_hot")
        self._pinned = None
        self._pinned_ev = None
        self.dag_cache = {}

    def pinned(self, ndoubles: int) -> torch.Tensor:
        """Persistent pinned host staging buffer (float64, >= ndoubles), reused
        by the host <-> device BLR transfers; waits for the previous transfer
        that used it before handing it out again."""
        if self._pinned_ev is not None:
            self._pinned_ev.synchronize()
        if self._pinned is None or self._pinned.numel() < ndoubles:
            self._pinned = None
            self._pinned = torch.empty(max(ndoubles, 1), dtype=torch.float64, pin_memory=True)
        return self._pinned

    def pinned_in_flight(self) -> None:
        """Mark the pinned buffer busy until the work queued so far completes."""
        ev = torch.cuda.Event()
        ev.record()
        self._pinned_ev = ev

    CANARY = -1.2345678901234567e300

    def workspace(self, b: int, cap: int, panel_rows: int = 0, nctas: int | None = None):
        """(ptr, doubles_per_cta, nctas) — grows the shared arena on demand.
        With an arena guard set (set_arena_guard), every CTA stride ends in a
        canary-filled zone the device arena never allocates."""
        nctas = nctas or self.nctas
        per = int(self.lib.blrqr_workspace_doubles(b, cap, panel_rows)) + self.arena_guard
        need = per * nctas
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            torch.cuda.synchronize()
            self._ws = torch.empty(need, dtype=torch.float64, device=self.dev)
        if self.arena_guard:
            self._ws[:need].view(nctas, per)[:, per - self.arena_guard:] = self.CANARY
            self._guard = (per, nctas)
        return self._ws.data_ptr(), per, nctas

    def set_arena_guard(self, doubles: int) -> None:
        """Debug tripwire for out-of-arena writes (blrqr_debug_arena_guard)."""
        torch.cuda.synchronize()
        self.arena_guard = int(doubles)
        check(self.lib.blrqr_debug_arena_guard(self.arena_guard), "arena_guard")
        # the canary zones assume one plain stride per CTA: no split while guarded
        check(self.lib.blrqr_set_arena_hot(0 if self.arena_guard else self.arena_hot), "arena_hot")

    def guards_intact(self) -> bool:
        """True when every CTA's guard zone of the last workspace still holds the canary."""
        per, nct = self._guard
        torch.cuda.synchronize()
        z = self._ws[:per * nct].view(nct, per)[:, per - self.arena_guard:]
        return bool((z == self.CANARY).all())

    def reset_counters(self):
        self.status.zero_()
        self.flops.zero_()

    def harvest(self, warn_mgs: bool = True) -> tuple[int, dict]:
        """Synchronise, read and clear status + flop counters; raise on errors."""
        st = int(self.status.item())
        fl = self.flops.cpu().numpy().astype(np.int64)
        self.status.zero_()
        self.flops.zero_()
        counts = {k: int(v) for k, v in zip(FLOP_KINDS, fl) if v}
        self.last_phases = {k: int(v) for k, v in zip(PHASES, fl[16:32]) if v}
        self.last_stats = fl[48:64].tolist()  # [8]: low-rank-class bytes of the rounded additions
        from . import flops as _fl
        for k, v in counts.items():
            _fl.add(k, v)
        if st & ST_ARENA_OVERFLOW:
            raise RuntimeError("per-CTA workspace overflow (blrqr_workspace_doubles too small)")
        if st & ST_RANK_OVERFLOW:
            raise RuntimeError("a low-rank result exceeded the slab capacity (raise cap)")
        if st & ST_SCHED_TIMEOUT:
            raise RuntimeError("dynamic scheduler timed out (no ready task); results are invalid")
        if st & ST_BAD_KIND:
            raise ValueError("diagonal blocks must be dense")
        if st & ST_BAD_ARG:
            raise RuntimeError("device invariant check failed (ST_BAD_ARG); results are invalid")
        if st & ST_NONFINITE:
            raise FloatingPointError("non-finite value produced on the device")
        if st & ST_MGS_COLLAPSE and warn_mgs:
            import warnings
            from .kernels import RankDeficiencyWarning
            warnings.warn("MGS panel column collapsed below 1e-300", RankDeficiencyWarning, stacklevel=3)
        return st, counts


_rt = None


def runtime() -> Runtime:
    global _rt
    if _rt is None:
        _rt = Runtime()
    return _rt
