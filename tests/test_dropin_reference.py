"""Drop-in proof: the UNMODIFIED reference pipelines (slotrank, imported from
/root/reference when present -- this container only) run on the product's
engine bookkeeping over the CPU CKKS oracle, and agree with the reference's
own simulator within the CKKS tolerance, with identical CostReports."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def slotrank():
    sys.path.insert(0, REF)
    import slotrank as R

    return R


def test_reference_rank_runs_on_ckks_engine(slotrank):
    from oracle.oracle import oracle_engine
    from paper_2412_15126_b200.params import preset

    R = slotrank
    p = preset("toy_deep")
    eng = oracle_engine(p)
    sim = R.HESimulator(R.HEParams(slot_count=p.slot_count, max_level=p.max_level))
    v = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    cfg = R.KernelConfig(mode="chebyshev", degree=64)
    got = R.read_row(eng, R.rank(eng, eng.encrypt(v), 8, cfg).ranks, 8)
    want = R.read_row(sim, R.rank(sim, sim.encrypt(v), 8, cfg).ranks, 8)
    assert np.abs(got - want).max() < 1e-4
    from slotrank import reference

    assert np.array_equal(np.rint(got), reference.fractional_ranks(v))
    a, b = eng.cost_snapshot(), sim.cost_snapshot()
    assert tuple(a.__dict__.values()) == tuple(b.__dict__.values())
    assert eng.rotation_offsets() == sim.rotation_offsets()
