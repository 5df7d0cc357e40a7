"""sweep.py (the degree study, reference cli.py:269-326) on the CPU oracle engine:
one record per kernel configuration, errors against the plaintext truth, the
monotone-trend flag, and the reference workload generator's ties."""

import numpy as np

import paper_2412_15126_b200 as M
from oracle.oracle import oracle_engine
from oracle.plain import fractional_ranks
from paper_2412_15126_b200.params import preset
from paper_2412_15126_b200.sweep import _fractional_ranks, degree_sweep, generate_values


def test_generator_and_ranks():
    v = generate_values(64, 3, tie_fraction=0.25)
    assert v.shape == (64,) and len(np.unique(v)) < 64
    assert np.array_equal(_fractional_ranks(v), fractional_ranks(v))


def test_rank_degree_sweep_on_oracle():
    eng = oracle_engine(preset("toy"))
    cfgs = [M.KernelConfig(mode="chebyshev", degree=d) for d in (16, 64)]
    cfgs.append(M.KernelConfig(mode="composite", composite=(2, 1)))
    recs, monotone = degree_sweep(eng, "rank", 8, cfgs, seeds=2)
    assert len(recs) == 3
    assert recs[1]["avg_err"] <= recs[0]["avg_err"] * 1.1  # higher degree, lower error
    assert all(r["report"]["cmp_evals"] == 1 for r in recs)
    assert isinstance(monotone, bool)
