"""Interop with the reference's own containers (build container: needs
/root/reference; skipped where it is absent, e.g. on the GPU box).

* a reference-built BlrMatrix converts (``interop.from_reference``) and is
  recognised as-is (duck-typed ``core.is_lowrank``);
* this package's result containers convert back (``interop.to_reference``)
  into objects the UNMODIFIED reference's ``metrics.materialize_q`` and
  ``serialize.dump_blr1`` accept, reproducing the reference's own outputs
  bit-for-bit after a reference -> package -> reference round trip.
"""

import io
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import blrqr
    from blrqr import core, factorize, lowrank, metrics, scheduler, serialize
    return dict(pkg=blrqr, core=core, factorize=factorize, lowrank=lowrank, metrics=metrics, scheduler=scheduler,
                serialize=serialize)


def _ref_input(ref):
    from oracle import configs
    n, b = 256, 32
    dense = configs.random16_dense(n, b, 0, rank=6)
    return dense, ref["core"].dense_to_blr(dense, b, ref["core"].weak_admissibility(n // b, n // b), 1e-8)


def test_reference_blrmatrix_in(ref):
    from paper_2208_06194_b200 import core, interop
    _, a = _ref_input(ref)
    assert all(core.is_lowrank(x) == ref["core"].is_lowrank(x) for row in a.blocks for x in row)
    ours = interop.from_reference(a)
    assert isinstance(ours, core.BlrMatrix)
    assert np.array_equal(core.blr_to_dense(ours), ref["core"].blr_to_dense(a))
    assert core.memory_footprint(ours) == ref["core"].memory_footprint(a)
    assert core.max_rank(ours) == ref["core"].max_rank(a)


@pytest.mark.parametrize("method", ["tiled-hh", "blocked-hh", "mgs"])
def test_results_out_to_reference(ref, method):
    from paper_2208_06194_b200 import interop
    from paper_2208_06194_b200.factorize import FactorizationResult
    from paper_2208_06194_b200.serialize import dumps_blr1
    _, a = _ref_input(ref)
    res_ref = ref["scheduler"].execute_sequential(method, a, ref["lowrank"].ToleranceConfig(1e-8))
    ours = interop.from_reference(res_ref)
    assert isinstance(ours, FactorizationResult)
    back = interop.to_reference(ours)
    q0 = ref["metrics"].materialize_q(res_ref)
    q1 = ref["metrics"].materialize_q(back)
    assert np.array_equal(q0, q1)
    buf0, buf1 = io.BytesIO(), io.BytesIO()
    ref["serialize"].dump_blr1(res_ref.r, buf0)
    ref["serialize"].dump_blr1(back.r, buf1)
    assert buf0.getvalue() == buf1.getvalue()
    assert dumps_blr1(ours.r) == buf0.getvalue()  # this package's writer agrees byte-for-byte
