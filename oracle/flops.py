"""Closed-form model-flop counts (oracle copy; test infrastructure only).

Restates flops.py:28-55 (qr/tgen/mm/svd/mgs/rrqr costs) and the global
accumulator flops.py:58-98.  Integer arithmetic, order independent.
"""

from __future__ import annotations

import threading
from collections import Counter

_lock = threading.Lock()
_tally: Counter = Counter()


def qr(h: int, w: int) -> int:  # flops.py:28-30
    return 2 * h * w * w - (2 * w * w * w) // 3


def tgen(h: int, w: int) -> int:  # flops.py:33-35
    return h * w * w


def mm(m: int, k: int, n: int) -> int:  # flops.py:38-40
    return 2 * m * k * n


def svd(c: int) -> int:  # flops.py:43-45
    return 12 * c * c * c


def mgs(h: int, w: int) -> int:  # flops.py:48-50
    return 2 * h * w * w


def rrqr(rows: int, cols: int, rank: int) -> int:  # flops.py:53-55
    return 4 * rows * cols * rank + 2 * rows * cols


def add(kind: str, n: int) -> None:
    with _lock:
        _tally[kind] += n


def reset() -> None:
    with _lock:
        _tally.clear()


def report() -> dict[str, int]:
    with _lock:
        return dict(_tally)


def total() -> int:
    with _lock:
        return sum(_tally.values())
