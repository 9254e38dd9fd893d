"""BLR1 format (serialize.py:1-89) against streams written by the reference
(tests/golden/make_blr1_golden.py)."""

import io
import os
import struct

import numpy as np
import pytest

from paper_2208_06194_b200 import serialize as S
from paper_2208_06194_b200.core import blr_to_dense, is_lowrank

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FILES = ["blr1_mixed.bin", "blr1_tiled_a.bin", "blr1_tiled_r.bin"]


def _bytes(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def _ranks(a):
    return [[x.rank if is_lowrank(x) else -1 for x in row] for row in a.blocks]


@pytest.mark.parametrize("name", FILES)
def test_reference_stream_round_trips_byte_exact(name):
    raw = _bytes(name)
    a = S.loads_blr1(raw)
    assert S.dumps_blr1(a) == raw
    buf = io.BytesIO()
    S.dump_blr1(a, buf)
    assert buf.getvalue() == raw


def test_reference_stream_contents():
    a = S.loads_blr1(_bytes("blr1_mixed.bin"))
    s = a.structure
    assert (s.m, s.n, s.b) == (96, 64, 16)
    r = np.array(_ranks(a))
    assert r.shape == (6, 4)
    assert (np.diag(r[:4]) == -1).all() and (r == 0).any() and (r > 0).any()
    rt = np.array(_ranks(S.loads_blr1(_bytes("blr1_tiled_r.bin"))))
    assert (rt[np.tril_indices(4, -1)] == 0).all()  # R-tilde: strictly-lower cells rank 0


def test_reader_errors():
    raw = _bytes("blr1_mixed.bin")
    with pytest.raises(ValueError, match="not a BLR1"):
        S.loads_blr1(b"BLR0" + raw[4:])
    with pytest.raises(ValueError, match="truncated"):
        S.loads_blr1(raw[:-3])
    bad = bytearray(raw)
    bad[28] = 7  # first record's tag
    with pytest.raises(ValueError, match="bad block tag"):
        S.loads_blr1(bytes(bad))
    # a low-rank diagonal cell is rejected
    m = n = b = 1
    stream = struct.pack("<4sQQQ", b"BLR1", m, n, b) + b"\x01" + struct.pack("<Q", 0)
    with pytest.raises(ValueError, match="diagonal"):
        S.loads_blr1(stream)


@pytest.mark.gpu
def test_device_grid_dump_equals_reference_bytes():
    from paper_2208_06194_b200.device import DeviceGrid
    raw = _bytes("blr1_tiled_a.bin")
    g = DeviceGrid.from_host(S.loads_blr1(raw))
    assert S.dumps_blr1(g) == raw


@pytest.mark.gpu
def test_gpu_tiled_r_matches_reference_blr1():
    """GPU tiled-hh on the reference's input stream vs the reference's R-tilde
    stream: same rank map, R-tilde within 1e-8 relative (row signs are fixed
    by the Householder convention, so no normalisation is needed)."""
    from paper_2208_06194_b200.device import DeviceGrid
    from paper_2208_06194_b200.factorize import factorize_device
    from paper_2208_06194_b200.lowrank import ToleranceConfig
    a = S.loads_blr1(_bytes("blr1_tiled_a.bin"))
    ref = S.loads_blr1(_bytes("blr1_tiled_r.bin"))
    f = factorize_device("tiled-hh", DeviceGrid.from_host(a), ToleranceConfig(1e-8))
    got = S.loads_blr1(S.dumps_blr1(f.g))
    assert _ranks(got) == _ranks(ref)
    rg, rr = blr_to_dense(got), blr_to_dense(ref)
    assert np.linalg.norm(rg - rr) <= 1e-8 * np.linalg.norm(rr)
