"""The product's pipeline mirror, run on the slot-level oracle, reproduces the
reference's own circuits bit for bit: decrypted slots, CostReport and rotation
trace (fixtures: tests/golden/circuits.json, made by oracle/gen_golden.py from
the real slotrank package)."""

import json
import os

import numpy as np
import pytest

import paper_2412_15126_b200 as M
from oracle.circuits import circuits
from oracle.slotsim import SlotSim, SimParams

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "circuits.json")))
BY_NAME = {c["name"]: c for c in GOLDEN["cases"]}
CIRCUITS = {c["name"]: c for c in circuits()}


def test_golden_covers_every_circuit():
    assert set(BY_NAME) == set(CIRCUITS)


@pytest.mark.parametrize("name", sorted(CIRCUITS))
def test_mirror_matches_reference(name):
    c, g = CIRCUITS[name], BY_NAME[name]
    eng = SlotSim(SimParams(c["slot_count"], c["max_level"]))
    out = np.asarray(c["fn"](eng, M, c["kernel"]))[: c["keep"]]
    assert np.array_equal(out, np.array(g["output"])), (out, g["output"])
    assert eng.cost_snapshot().__dict__ == g["cost"]
    assert eng.rotation_offsets() == g["trace"]


def test_known_answers_present():
    # the reference's pinned fixtures
    assert BY_NAME["fig3_rank"]["output"] == [2.0, 3.0, 1.0, 4.0]
    assert BY_NAME["sec31_rank_ties"]["output"] == [5.0, 1.0, 2.5, 2.5, 4.0]
    assert BY_NAME["sec4_ties_corrected"]["output"] == [1.0, 2.0, 3.0, 4.0]
    assert BY_NAME["fig5_sort"]["output"] == [10.0, 20.0, 30.0, 40.0]
    assert BY_NAME["fig2_transpose_n8"]["trace"][:3] == [64 - 28, 64 - 14, 64 - 7]
    assert BY_NAME["rotate_left_1"]["output"] == [2.0, 3.0, 4.0, 1.0]
    assert BY_NAME["rotate_right_1"]["output"] == [4.0, 1.0, 2.0, 3.0]
    sel = np.array(BY_NAME["fig5_selection_matrix"]["output"]).reshape(4, 4)
    assert np.array_equal(sel, [[0, 0, 1, 0], [1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1]])
