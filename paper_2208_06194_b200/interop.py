"""Conversions between the reference ``blrqr`` containers and this package's.

The reference recognises a low-rank block by ``isinstance(block,
blrqr.core.LowRankBlock)`` (core.py:73-74), so its ``metrics.materialize_q``,
``factorize.blocked_apply_q`` / ``tiled_apply_q`` and ``serialize.dump_blr1``
need its own classes.  In the other direction this package duck-types
(``core.is_lowrank``: anything with ``u`` / ``v`` factors that is not an
ndarray), so a reference-built ``BlrMatrix`` can be passed straight to
``DeviceGrid.from_host`` / ``execute_sequential``; ``from_reference`` makes
an explicit copy into this package's classes when one is wanted.

Field-for-field: LowRankBlock(u, v), BlrStructure(m, n, b, admissible),
BlrMatrix(structure, blocks), WYReflector(y, t) (kernels.py:38-59),
ReflectorColumn(col, entries, t), TileReflectorStore(diag, updates),
FactorizationResult(algorithm, r, q_columns, q_tiles, q_explicit)
(factorize.py:146-179).
"""

from __future__ import annotations

import importlib

import numpy as np

from . import core
from .factorize import FactorizationResult, ReflectorColumn, TileReflectorStore
from .kernels import WYReflector

__all__ = ["from_reference", "to_reference"]


def _ref_modules(blrqr=None):
    """(core, kernels, factorize) modules of the reference package."""
    if blrqr is None:
        blrqr = importlib.import_module("blrqr")
    name = blrqr.__name__
    return (importlib.import_module(name + ".core"), importlib.import_module(name + ".kernels"),
            importlib.import_module(name + ".factorize"))


def _block(x, lr_cls):
    if core.is_lowrank(x):
        return lr_cls(np.array(x.u, dtype=np.float64), np.array(x.v, dtype=np.float64))
    return np.array(x, dtype=np.float64)


def _matrix(a, structure_cls, matrix_cls, lr_cls):
    s = a.structure
    st = structure_cls(s.m, s.n, s.b, np.array(s.admissible, dtype=bool))
    return matrix_cls(st, [[_block(x, lr_cls) for x in row] for row in a.blocks])


def _convert(obj, lr_cls, structure_cls, matrix_cls, wy_cls, col_cls, store_cls, result_cls):
    if obj is None:
        return None
    if hasattr(obj, "structure") and hasattr(obj, "blocks"):
        return _matrix(obj, structure_cls, matrix_cls, lr_cls)
    if hasattr(obj, "algorithm") and hasattr(obj, "r"):
        conv = lambda x: _convert(x, lr_cls, structure_cls, matrix_cls, wy_cls, col_cls, store_cls,  # noqa: E731
                                  result_cls)
        qc = None if obj.q_columns is None else [conv(c) for c in obj.q_columns]
        return result_cls(obj.algorithm, conv(obj.r), q_columns=qc, q_tiles=conv(obj.q_tiles),
                          q_explicit=conv(obj.q_explicit))
    if hasattr(obj, "col") and hasattr(obj, "entries"):
        return col_cls(obj.col, [(i, _block(y, lr_cls)) for i, y in obj.entries], np.array(obj.t))
    if hasattr(obj, "diag") and hasattr(obj, "updates"):
        return store_cls({k: wy_cls(np.array(w.y), np.array(w.t)) for k, w in obj.diag.items()},
                         {ik: (_block(y, lr_cls), np.array(t)) for ik, (y, t) in obj.updates.items()})
    if hasattr(obj, "y") and hasattr(obj, "t"):
        return wy_cls(np.array(obj.y), np.array(obj.t))
    if core.is_lowrank(obj) or isinstance(obj, np.ndarray):
        return _block(obj, lr_cls)
    raise TypeError(f"cannot convert {type(obj).__name__}")


def from_reference(obj):
    """Reference container (BlrMatrix, block, FactorizationResult, ...) -> this package's."""
    return _convert(obj, core.LowRankBlock, core.BlrStructure, core.BlrMatrix, WYReflector, ReflectorColumn,
                    TileReflectorStore, FactorizationResult)


def to_reference(obj, blrqr=None):
    """This package's container -> the reference's classes (``blrqr`` must be
    importable, or pass the imported package as ``blrqr``), so the
    reference's metrics / apply-Q / serialisation accept it."""
    rcore, rker, rfac = _ref_modules(blrqr)
    return _convert(obj, rcore.LowRankBlock, rcore.BlrStructure, rcore.BlrMatrix, rker.WYReflector,
                    rfac.ReflectorColumn, rfac.TileReflectorStore, rfac.FactorizationResult)
