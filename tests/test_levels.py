"""levels.py: the level tracer applies the engine's own level rules without data
-- a whole rank / sort traced on it ends at the levels the real engine reaches,
with the same CostReport (the multi-GPU level plans rest on this)."""

import numpy as np

import paper_2412_15126_b200 as M
from oracle.oracle import oracle_engine
from paper_2412_15126_b200.levels import level_tracer
from paper_2412_15126_b200.params import preset


def test_tracer_matches_engine_levels_and_costs():
    p = preset("toy_sort")
    eng = oracle_engine(p)
    tr = level_tracer(eng)
    assert level_tracer(eng) is tr  # cached per engine
    v = np.random.default_rng(3).choice(128, 40, replace=False) / 128
    kcfg = M.KernelConfig(mode="composite", composite=(3, 2), indicator_composite=(4, 2))
    bv = M.block_split(eng, v)
    tbv = M.BlockVector(blocks=tuple(tr.token(b.level) for b in bv.blocks), block_size=bv.block_size,
                        total_len=bv.total_len)
    eng.cost_reset()
    tr.cost_reset()
    real = M.multi_sort(eng, bv, M.SortConfig(kernel=kcfg, tie_correction=False))
    traced = M.multi_sort(tr, tbv, M.SortConfig(kernel=kcfg, tie_correction=False))
    assert [b.level for b in traced.blocks] == [b.level for b in real.blocks]
    assert tr.cost_snapshot() == eng.cost_snapshot()
    assert tr.rotation_offsets() == eng.rotation_offsets()
