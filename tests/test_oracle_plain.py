"""oracle/plain.py pinned against the reference's own plaintext functions."""

import json
import os

import numpy as np
import pytest

from oracle import plain

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plain.json")))


@pytest.mark.parametrize("case", FIX, ids=lambda c: str(len(c["values"])))
def test_plain_oracle(case):
    v = case["values"]
    assert np.array_equal(plain.fractional_ranks(v), case["fractional"])
    assert np.array_equal(plain.corrected_ranks(v), case["corrected"])
    assert np.array_equal(plain.tie_offsets(v), case["offsets"])
    assert np.array_equal(plain.sorted_values(v), case["sorted"])
    assert plain.median_value(v) == case["median"]
    assert plain.percentile_value(v, 25.0) == case["p25"]
    assert plain.percentile_value(v, 90.0) == case["p90"]
    assert plain.kth_smallest(v, 2) == case["k2"]
