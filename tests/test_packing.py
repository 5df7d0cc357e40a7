"""Two blocks per ciphertext (packing.py, the opt-in layout of BASELINE config
5's "32 ciphertexts") on the slot oracle: the decrypted sort equals the
reference layout's, with half the comparison / indicator evaluations and no
extra level (reference sorting.py:106-142, ranking.py:307-392)."""

import numpy as np
import pytest

import paper_2412_15126_b200 as M
from oracle.slotsim import SimParams, SlotSim

KCFG = M.KernelConfig(mode="composite", composite=(6, 2), indicator_composite=(6, 2))


def _run(n, span, packed, levels):
    v = np.random.default_rng(0).choice(span, n, replace=False) / span
    sim = SlotSim(SimParams(32768, levels))
    res = M.multi_sort(sim, M.block_split(sim, v),
                       M.SortConfig(kernel=KCFG, tie_correction=False, packed=packed))
    return v, M.block_merge(sim, res), sim.cost_snapshot(), [b.level for b in res.blocks]


@pytest.mark.parametrize("n,span,levels", [(1024, 8192, 56), (300, 2048, 58), (640, 8192, 56)])
def test_packed_sort_equals_reference_layout(n, span, levels):
    v, ref, c_ref, lv_ref = _run(n, span, False, levels)
    _, got, c_pk, lv_pk = _run(n, span, True, levels)
    assert np.abs(got - ref).max() < 1e-12
    assert np.abs(got - np.sort(v)).max() < 1e-6
    assert lv_pk == lv_ref and c_pk.levels_consumed == c_ref.levels_consumed
    count = -(-n // 128)
    assert c_ref.cmp_evals == count * (count + 1) // 2 and c_pk.cmp_evals == -(-c_ref.cmp_evals // 2)
    assert c_ref.ind_evals == count * count and c_pk.ind_evals == count * (-(-count // 2))
    assert c_pk.ctct_mults < (0.62 if count % 2 == 0 else 0.7) * c_ref.ctct_mults


def test_packed_requires_untied_and_room():
    sim = SlotSim(SimParams(32768, 56))
    bv = M.block_split(sim, np.arange(256) / 256)
    with pytest.raises(ValueError):
        M.multi_sort(sim, bv, M.SortConfig(kernel=KCFG, tie_correction=True, packed=True))
    from paper_2412_15126_b200.packing import can_pack

    assert can_pack(sim, 128) and not can_pack(sim, 256)


def test_packed_multi_rank_equals_reference_layout():
    from oracle.plain import fractional_ranks

    v = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    sim = SlotSim(SimParams(32768, 56))
    bv = M.block_split(sim, v)
    ref = M.block_merge(sim, M.multi_rank(sim, bv, KCFG))
    got = M.block_merge(sim, M.multi_rank(sim, bv, KCFG, packed=True))
    assert np.abs(got - ref).max() < 1e-9
    assert np.array_equal(np.rint(got), fractional_ranks(v))
