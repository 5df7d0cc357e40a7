"""The product's engine bookkeeping over the CPU oracle backend (toy rings):
CKKS semantics against numpy, and the reference simulator's method contract
(levels, counters, trace, errors; reference engine.py:133-328)."""

import numpy as np
import pytest

import paper_2412_15126_b200 as M
from oracle.oracle import oracle_engine
from oracle.plain import fractional_ranks
from oracle.slotsim import SimParams, SlotSim
from paper_2412_15126_b200.engine import CapacityError, DepthBudgetError, EngineError, IncompatibleParamsError
from paper_2412_15126_b200.params import preset

TOL = 1e-7


@pytest.fixture(scope="module")
def eng():
    return oracle_engine(preset("toy"))


@pytest.fixture(scope="module")
def x(eng):
    return np.linspace(-1, 1, eng.params.slot_count)


def test_roundtrip_and_capacity(eng, x):
    ct = eng.encrypt(x)
    assert ct.level == eng.params.max_level
    assert np.abs(eng.decrypt(ct) - x).max() < TOL
    short = eng.decrypt(eng.encrypt([1.0, 2.0]))
    assert np.abs(short[:2] - [1, 2]).max() < TOL and np.abs(short[2:]).max() < TOL
    with pytest.raises(CapacityError):
        eng.encrypt(np.zeros(eng.params.slot_count + 1))
    with pytest.raises(ValueError):
        eng.plain(np.zeros(3))


def test_arithmetic(eng, x):
    a, b = eng.encrypt(x), eng.encrypt(x[::-1])
    y = x[::-1]
    checks = [
        (eng.add(a, b), x + y), (eng.sub(a, b), x - y), (eng.negate(a), -x),
        (eng.add_plain(a, 0.25), x + 0.25), (eng.add_plain(a, y), x + y),
        (eng.mul(a, b), x * y), (eng.mul_plain(a, -3.5), -3.5 * x), (eng.mul_plain(a, y), x * y),
    ]
    for ct, want in checks:
        assert np.abs(eng.decrypt(ct) - want).max() < TOL
    assert eng.mul(a, b).level == a.level - 1 and eng.mul_plain(a, y).level == a.level - 1
    assert eng.add(a, b).level == a.level and eng.negate(a).level == a.level


def test_mixed_levels_take_min(eng, x):
    a = eng.encrypt(x)
    sq = eng.mul(a, a)
    cube = eng.mul(sq, a)
    s = eng.add(cube, a)
    assert s.level == a.level - 2
    assert np.abs(eng.decrypt(s) - (x ** 3 + x)).max() < TOL
    m = eng.mul_plain(a, 2.0, level=a.level - 3)
    assert m.level == a.level - 3 and np.abs(eng.decrypt(m) - 2 * x).max() < TOL


def test_rotation_direction_and_trace(eng, x):
    n = eng.params.slot_count
    a = eng.encrypt(x)
    eng.cost_reset()
    assert eng.rotate(a, 0) is a and eng.rotate(a, n) is a
    assert np.abs(eng.decrypt(eng.rotate(a, 1)) - np.roll(x, -1)).max() < TOL
    assert np.abs(eng.decrypt(eng.rotate(a, -3)) - np.roll(x, 3)).max() < TOL
    assert eng.rotation_offsets() == [1, n - 3]
    rep = eng.cost_snapshot()
    assert rep.rotations == 2 and rep.critical_rotations == 1


def test_depth_budget_error(eng):
    a = eng.encrypt([0.5])
    while a.level > 0:
        a = eng.mul_plain(a, 1.0)
    with pytest.raises(DepthBudgetError) as ei:
        eng.mul(a, a, site="here")
    assert ei.value.site == "here" and ei.value.available == 0
    with pytest.raises(DepthBudgetError):
        eng.mul_plain(a, 2.0)


def test_incompatible_params(eng):
    other = oracle_engine(preset("toy", seed=7))
    with pytest.raises(IncompatibleParamsError):
        eng.add(eng.encrypt([1.0]), other.encrypt([1.0]))


def test_ideal_map_constant_only(eng, x):
    a = eng.encrypt(x)
    c = eng.ideal_map(lambda s: np.full_like(s, 0.75), a, levels=2)
    assert c.level == a.level - 2 and np.abs(eng.decrypt(c) - 0.75).max() < TOL
    with pytest.raises(EngineError):
        eng.ideal_map(lambda s: s * 2, a)


def test_composite_rank_matches_simulator_and_plaintext():
    p = preset("toy_deep")
    eng = oracle_engine(p)
    sim = SlotSim(SimParams(p.slot_count, p.max_level))
    v = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    cfg = M.KernelConfig(mode="composite", composite=(3, 2))
    got = M.read_row(eng, M.rank(eng, eng.encrypt(v), 8, cfg).ranks, 8)
    ref = M.read_row(sim, M.rank(sim, sim.encrypt(v), 8, cfg).ranks, 8)
    assert np.abs(got - ref).max() < 1e-5
    assert np.array_equal(np.rint(got), fractional_ranks(v))
    assert eng.cost_snapshot() == sim.cost_snapshot()


def test_batched_pipeline_equals_loop():
    """Lock-step batched multi_sort (B200 path) == the per-unit loop, limb for limb,
    with identical CostReports (counters count every batch element)."""
    p = preset("toy_sort")
    v = np.random.default_rng(5).choice(256, 40, replace=False) / 256
    kc = M.KernelConfig(mode="composite", composite=(3, 2), indicator_composite=(4, 2))
    e1 = oracle_engine(p)
    r1 = M.multi_sort(e1, M.block_split(e1, v), M.SortConfig(kernel=kc, tie_correction=False))
    e2 = oracle_engine(p)
    e2.stack = e2.concat = None  # force the sequential reference structure
    r2 = M.multi_sort(e2, M.block_split(e2, v), M.SortConfig(kernel=kc, tie_correction=False))
    assert all(np.array_equal(a.data, b.data) for a, b in zip(r1.blocks, r2.blocks))
    assert e1.cost_snapshot() == e2.cost_snapshot()
    assert sorted(e1.rotation_offsets()) == sorted(e2.rotation_offsets())
    assert np.abs(M.block_merge(e1, r1) - np.sort(v)).max() < 5e-3


def test_batched_ops_match_single(eng, x):
    a, b = eng.encrypt(x), eng.encrypt(x[::-1])
    xb = eng.stack([a, b])
    yb = eng.stack([b, a])
    pairs = [
        (eng.mul(xb, yb), [eng.mul(a, b), eng.mul(b, a)]),
        (eng.rotate(xb, 3), [eng.rotate(a, 3), eng.rotate(b, 3)]),
        (eng.mul_plain(xb, 0.5), [eng.mul_plain(a, 0.5), eng.mul_plain(b, 0.5)]),
        (eng.add_plain(xb, np.stack([x, -x])), [eng.add_plain(a, x), eng.add_plain(b, -x)]),
        (eng.mul_plain(xb, np.stack([x, x * 2])), [eng.mul_plain(a, x), eng.mul_plain(b, x * 2)]),
        (eng.sub(xb, yb), [eng.sub(a, b), eng.sub(b, a)]),
    ]
    for got, want in pairs:
        for g, w in zip(eng.unstack(got), want):
            assert g.level == w.level and np.array_equal(g.data, w.data)


def test_hoisted_rotations_equal_single_rotations():
    """orc_rotate_hoisted (the CPU baseline's rotations: one base extension for
    all of them) is bit-identical to orc_rotate, at a full and at a lower level."""
    p = preset("toy_deep")
    eng = oracle_engine(p)
    be = eng.backend
    ct = eng.encrypt(np.linspace(-0.9, 0.9, 16))
    two_n = 2 * p.ring_degree
    galois = [pow(5, k, two_n) for k in (1, 2, 5)] + [two_n - 1]
    for level in (ct.level, 2):
        a = np.ascontiguousarray(ct.data[:, : level + 1])
        keys = [be.galois_key(g) for g in galois]
        outs = be.o.rotate_hoisted_raw(a, keys, galois, level)
        for g, k, out in zip(galois, keys, outs):
            assert np.array_equal(out, be.o.rotate_raw(a, k, g, level))


def test_depth_fitted_encryption():
    """engine.encrypt(level=d) with d = circuit_depth(circuit): the circuit ends at
    level 0 with the same decrypted result as from the top of the chain; the depth
    comes from the level tracer (no ciphertext data) and equals the levels consumed."""
    eng = oracle_engine(preset("toy_deep"))
    cfg = M.KernelConfig(mode="composite", composite=(3, 2))
    v = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    depth = eng.circuit_depth(lambda e, c: M.rank(e, c, 8, cfg).ranks)
    full = M.rank(eng, eng.encrypt(v), 8, cfg).ranks
    assert depth == eng.params.max_level - full.level
    fit = M.rank(eng, eng.encrypt(v, level=depth), 8, cfg).ranks
    assert fit.level == 0
    assert np.array_equal(np.rint(M.read_row(eng, fit, 8)), fractional_ranks(v))
    assert np.abs(M.read_row(eng, fit, 8) - M.read_row(eng, full, 8)).max() < 1e-4
    dropped = eng.fit_depth(eng.encrypt(v), lambda e, c: M.rank(e, c, 8, cfg).ranks)
    assert dropped.level == depth and eng.fit_depth(dropped, depth) is dropped
    assert np.abs(eng.decrypt(dropped)[:8] - v).max() < TOL
    assert np.array_equal(np.rint(M.read_row(eng, M.rank(eng, dropped, 8, cfg).ranks, 8)), fractional_ranks(v))
    with pytest.raises(DepthBudgetError):
        M.rank(eng, eng.encrypt(v, level=depth - 1), 8, cfg)
    with pytest.raises(EngineError):
        eng.encrypt(v, level=eng.params.max_level + 1)


def test_levelwise_bsgs_equals_recursive_bsgs():
    """chebyshev._bsgs_levelwise (giant-step products of one tree depth in one
    engine.mul_pairs call; the GPU engine's path) yields the ciphertext, level and
    counters of the recursive _bsgs, limb for limb, on the CPU oracle engine."""
    import math

    from paper_2412_15126_b200 import chebyshev as C

    eng = oracle_engine(preset("toy_deep"))
    x = eng.encrypt(np.linspace(-0.9, 0.9, 32))
    for degree in (37, 64, 127):
        poly = C._step_poly(degree)
        coeffs = C._strip(np.asarray(poly.coeffs, dtype=np.float64))
        m = max(1, math.ceil(math.log2(len(coeffs))))
        bs = 1 << max(1, m // 2)
        eng.cost_reset()
        a_ct, a_c = C._bsgs(eng, coeffs, C._ChebPowers(eng, x), bs)
        cost_a = eng.cost_snapshot()
        eng.cost_reset()
        b_ct, b_c = C._bsgs_levelwise(eng, coeffs, C._ChebPowers(eng, x), bs)
        assert eng.cost_snapshot() == cost_a
        assert a_c == b_c and a_ct.level == b_ct.level
        assert np.array_equal(a_ct.data, b_ct.data)


def test_paired_goldschmidt_equals_sequential():
    """goldschmidt_inverse's paired schedule (y_k and e_{k+1} in one engine.mul_pairs call,
    taken when the backend has batched products) gives the sequential loop's ciphertext
    limb for limb, with the same counters."""
    from paper_2412_15126_b200 import chebyshev as C

    eng = oracle_engine(preset("toy_deep"))
    x = eng.encrypt(np.linspace(1.0, 7.5, 16))
    eng.cost_reset()
    par = C.goldschmidt_inverse(eng, x, (0.5, 8.5), 5)
    cost = eng.cost_snapshot()
    eng.backend.mul_relin_rescale_pairs = None  # hides the batched product: the sequential loop runs
    try:
        eng.cost_reset()
        seq = C.goldschmidt_inverse(eng, x, (0.5, 8.5), 5)
        assert eng.cost_snapshot() == cost
    finally:
        del eng.backend.mul_relin_rescale_pairs
    assert par.level == seq.level and np.array_equal(par.data, seq.data)
    assert np.abs(eng.decrypt(par)[:16] - 1.0 / np.linspace(1.0, 7.5, 16)).max() < 1e-3
