"""Pipelines on the B200 engine: full-pipeline bit-exactness against the CPU
oracle, the reference's golden circuits after decryption, and the BASELINE
configurations' results (ranks / argmin / argmax / k-th / sort order)."""

import json
import os

import numpy as np
import pytest

import paper_2412_15126_b200 as M
from oracle.circuits import circuits
from oracle.plain import fractional_ranks
from oracle.slotsim import SimParams, SlotSim
from paper_2412_15126_b200.params import preset

pytestmark = pytest.mark.gpu

GOLDEN = {c["name"]: c for c in json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                                             "circuits.json")))["cases"]}
# slot-level tolerance vs the reference simulator on the same circuit (CKKS noise
# amplified by the degree-d Chebyshev recursion), checked per circuit
CHEB_TOL = 1e-4


@pytest.fixture(scope="module")
def eng12(require_cuda):
    return M.B200Engine(preset("ring12"))


def test_full_pipeline_limbs_bit_exact_vs_oracle(require_cuda):
    """Every op of a composite-mode rank (rotations, products, plaintext masks,
    level alignments) yields the same limbs on the GPU as on the CPU oracle."""
    from oracle.oracle import oracle_engine

    p = preset("toy_deep")
    gpu, cpu = M.B200Engine(p), oracle_engine(p)
    v = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    cfg = M.KernelConfig(mode="composite", composite=(3, 2))
    rg = M.rank(gpu, gpu.encrypt(v), 8, cfg).ranks
    rc = M.rank(cpu, cpu.encrypt(v), 8, cfg).ranks
    assert rg.level == rc.level
    assert np.array_equal(gpu.backend.to_host(rg.data), rc.data)
    assert gpu.cost_snapshot() == cpu.cost_snapshot()


@pytest.mark.parametrize("name", sorted(c["name"] for c in circuits() if c["gpu"]))
def test_golden_circuit_on_gpu(eng12, name):
    c = next(c for c in circuits() if c["name"] == name)
    g = GOLDEN[name]
    assert eng12.params.slot_count == c["slot_count"]
    eng12.cost_reset()
    out = np.asarray(c["fn"](eng12, M, c["kernel"]))[: c["keep"]]
    want = np.array(g["output"])
    assert np.abs(out - want).max() < CHEB_TOL, np.abs(out - want).max()
    rep = eng12.cost_snapshot().__dict__
    assert {k: v for k, v in rep.items() if k != "levels_consumed"} == \
        {k: v for k, v in g["cost"].items() if k != "levels_consumed"}
    assert eng12.rotation_offsets() == g["trace"]


def test_cfg1_rank_n16(require_cuda):
    """BASELINE config 1: 16 grid values k/64 on ring 2^12 (2048 slots), composite sign."""
    v = np.random.default_rng(0).choice(64, 16, replace=False) / 64
    eng = M.B200Engine(preset("cfg1"))
    cfg = M.KernelConfig(mode="composite", composite=(3, 2))
    r = M.read_row(eng, M.rank(eng, eng.encrypt(v), 16, cfg).ranks, 16)
    assert np.array_equal(np.rint(r), fractional_ranks(v))
    sim = SlotSim(SimParams(2048, 22))
    rs = M.read_row(sim, M.rank(sim, sim.encrypt(v), 16, cfg).ranks, 16)
    assert np.abs(r - rs).max() < 1e-4
    assert eng.cost_snapshot().rotations == 16  # log2(16) x 4 (ReplR, TransR, ReplC, SumR)


def test_cfg3_rank_n128(require_cuda):
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    eng = M.B200Engine(preset("cfg3"))
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))
    r = M.read_row(eng, M.rank(eng, eng.encrypt(v), 128, cfg).ranks, 128)
    assert np.array_equal(np.rint(r), fractional_ranks(v))
    sim = SlotSim(SimParams(32768, 29))
    rs = M.read_row(sim, M.rank(sim, sim.encrypt(v), 128, cfg).ranks, 128)
    assert np.abs(r - rs).max() < 1e-3
    assert eng.cost_snapshot().rotations == 28


@pytest.fixture(scope="module")
def eng_long(require_cuda):
    return M.B200Engine(preset("long"))


def test_cfg4_order_statistic_masks(eng_long):
    v = np.random.default_rng(1).choice(1024, 128, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(4, 2), tie_margin=2.0 ** -11)
    ct = eng_long.encrypt(v)
    order = np.argsort(v)
    for q, idx in ((M.StatisticQuery("min"), order[0]), (M.StatisticQuery("max"), order[-1]),
                   (M.StatisticQuery("kth", k=64), order[63])):
        m = M.read_row(eng_long, M.order_statistic_mask(eng_long, ct, 128, q, cfg), 128)
        assert int(np.argmax(m)) == int(idx)
        assert np.abs(m - np.eye(128)[idx]).max() < 0.05


def test_cfg4_min_value(eng_long):
    v = np.random.default_rng(2).choice(1024, 16, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(3, 2), tie_margin=2.0 ** -9,
                         goldschmidt_iters=4)
    val = eng_long.decrypt(M.order_statistic_value(eng_long, eng_long.encrypt(v), 16,
                                                    M.StatisticQuery("min"), cfg))[0]
    assert abs(val - v.min()) < 1e-3


def test_multi_sort_n256(eng_long):
    v = np.random.default_rng(3).choice(2048, 256, replace=False) / 2048
    cfg = M.SortConfig(kernel=M.KernelConfig(mode="composite", composite=(5, 2),
                                             indicator_composite=(5, 2)), tie_correction=False)
    out = M.block_merge(eng_long, M.multi_sort(eng_long, M.block_split(eng_long, v), cfg))
    assert np.array_equal(np.argsort(out), np.arange(256))
    assert np.abs(out - np.sort(v)).max() < 1e-3


def test_tie_corrected_rank_and_sort(eng12, eng_long):
    """Ties: corrected ranks are a permutation (reference ranking.py:203-232), and
    the tie-corrected sort returns the sorted multiset (composite kernels; the
    sort needs ~38 levels, so it runs on the long chain)."""
    from oracle.plain import corrected_ranks

    v = np.array([0.5, 0.25, 0.5, 0.75, 0.25, 0.5, 0.125, 1.0,
                  0.375, 0.625, 0.375, 0.875, 0.0625, 0.5, 0.9375, 0.25])
    cfg = M.KernelConfig(mode="composite", composite=(3, 2), indicator_composite=(3, 2))
    r = M.read_row(eng12, M.rank_corrected(eng12, eng12.encrypt(v), 16, cfg).ranks, 16)
    assert np.array_equal(np.rint(r), corrected_ranks(v))
    out = M.read_row(eng_long, M.sort(eng_long, eng_long.encrypt(v), 16, M.SortConfig(kernel=cfg)), 16)
    assert np.abs(out - np.sort(v)).max() < 1e-3


def test_chebyshev_sort_matches_reference_simulator(eng12):
    """The reference's own Chebyshev sort circuit on the GPU vs the slot oracle."""
    v = np.array([0.15, 0.55, 0.35, 0.95, 0.05, 0.75, 0.25, 0.85])
    cfg = M.SortConfig(kernel=M.KernelConfig(mode="chebyshev", degree=512), tie_correction=False)
    out = M.read_row(eng12, M.sort(eng12, eng12.encrypt(v), 8, cfg), 8)
    sim = SlotSim(SimParams(eng12.params.slot_count, eng12.params.max_level))
    ref = M.read_row(sim, M.sort(sim, sim.encrypt(v), 8, cfg), 8)
    assert np.abs(out - ref).max() < 1e-4
    assert np.abs(out - np.sort(v)).max() < 1e-3


@pytest.mark.gpu
def test_captured_pipeline_replay_new_inputs(require_cuda):
    """graphs.CapturedPipeline: a rank captured once replays bit-identically to the
    eager pipeline, including on new input ciphertexts copied into its buffers."""
    import torch

    from paper_2412_15126_b200.graphs import CapturedPipeline

    eng = M.B200Engine(preset("toy_deep"))
    cfg = M.KernelConfig(mode="composite", composite=(3, 2))
    v1 = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    v2 = np.array([0.70, 0.15, 0.05, 0.90, 0.35, 0.60, 0.25, 0.45])
    x1, x2 = eng.encrypt(v1), eng.encrypt(v2)
    fn = lambda c: M.rank(eng, c, 8, cfg).ranks  # noqa: E731
    cap = CapturedPipeline(eng, fn, x1)
    e1 = fn(x1).data.clone()
    assert torch.equal(cap.replay().data, e1)
    e2 = fn(x2).data.clone()
    out = cap.replay(x2)
    torch.cuda.synchronize()
    assert torch.equal(out.data, e2)
    assert np.array_equal(np.rint(M.read_row(eng, out, 8)), fractional_ranks(v2))


def test_cfg4_median_and_percentile_values(eng_long):
    """Value retrieval (select.py median / percentile: window mask, SumC, Goldschmidt
    inverse) on the GPU against the plaintext oracle (reference.py:27-87)."""
    from oracle.plain import kth_smallest, median_value, nearest_rank

    v = np.random.default_rng(4).choice(1024, 16, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(3, 2), indicator_composite=(3, 2),
                         tie_margin=2.0 ** -9, goldschmidt_iters=4)
    ct = eng_long.encrypt(v)
    med = eng_long.decrypt(M.median(eng_long, ct, 16, cfg))[0]
    assert abs(med - median_value(v)) < 2e-3
    p90 = eng_long.decrypt(M.percentile(eng_long, ct, 16, 90.0, cfg))[0]
    assert abs(p90 - kth_smallest(v, nearest_rank(16, 90.0))) < 2e-3


def test_ragged_inputs_and_capacity(require_cuda, eng_long):
    """Edge cases of the reference's tests: a length that is not a power of two
    (pad mask), a ragged last sort block, and the capacity error."""
    eng = M.B200Engine(preset("cfg3"))
    v = np.random.default_rng(5).choice(1024, 100, replace=False) / 1024
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))
    r = M.read_row(eng, M.rank(eng, eng.encrypt(v), 100, cfg).ranks, 100)
    assert np.array_equal(np.rint(r), fractional_ranks(v))
    with pytest.raises(M.CapacityError):
        M.rank(eng, eng.encrypt(np.zeros(256)), 256, cfg)
    w = np.random.default_rng(6).choice(2048, 200, replace=False) / 2048
    scfg = M.SortConfig(kernel=M.KernelConfig(mode="composite", composite=(5, 2),
                                              indicator_composite=(5, 2)), tie_correction=False)
    out = M.block_merge(eng_long, M.multi_sort(eng_long, M.block_split(eng_long, w), scfg))
    assert out.shape == (200,)
    assert np.array_equal(np.argsort(out), np.arange(200))
    assert np.abs(out - np.sort(w)).max() < 1e-3


def test_concurrent_ops_from_host_threads(eng12):
    """Ops on distinct inputs from 8 host threads (reference SPEC.md:121; the
    reference's thread-pool multi_rank, ranking.py:345-347): every result equals
    the single-threaded one limb for limb and the counters add up exactly."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    xs = [eng12.encrypt(np.linspace(-1, 1, 64) * (i + 1) / 9) for i in range(8)]

    def work(i):
        x = xs[i]
        return eng12.mul(eng12.rotate(x, i + 1), eng12.add(x, x))

    seq = [work(i).data.clone() for i in range(8)]
    torch.cuda.synchronize()
    eng12.cost_reset()
    with ThreadPoolExecutor(8) as pool:
        par = list(pool.map(work, range(8)))
    torch.cuda.synchronize()
    for a, b in zip(seq, par):
        assert torch.equal(a, b.data)
    rep = eng12.cost_snapshot()
    assert rep.rotations == 8 and rep.ctct_mults == 8 and rep.additions == 8


def test_depth_fitted_rank_bit_exact_and_cfg4_masks(require_cuda, eng_long):
    """Inputs encrypted at the level the circuit's depth needs (engine.encrypt(level=...)):
    the toy rank's limbs stay bit-equal to the CPU oracle's down to level 0, and the
    cfg 4 argmin mask from level 39 of the long chain still selects the right index."""
    from oracle.oracle import oracle_engine

    p = preset("toy_deep")
    gpu, cpu = M.B200Engine(p), oracle_engine(p)
    v = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    cfg = M.KernelConfig(mode="composite", composite=(3, 2))
    d = gpu.circuit_depth(lambda e, c: M.rank(e, c, 8, cfg).ranks)
    assert d == cpu.circuit_depth(lambda e, c: M.rank(e, c, 8, cfg).ranks)
    rg = M.rank(gpu, gpu.encrypt(v, level=d), 8, cfg).ranks
    rc = M.rank(cpu, cpu.encrypt(v, level=d), 8, cfg).ranks
    assert rg.level == rc.level == 0
    assert np.array_equal(gpu.backend.to_host(rg.data), rc.data)
    assert np.array_equal(np.rint(M.read_row(gpu, rg, 8)), fractional_ranks(v))
    # the same from a full-chain ciphertext: fit_depth drops the unused limbs first
    circ = lambda e, c: M.rank(e, c, 8, cfg).ranks  # noqa: E731
    fg, fc = gpu.fit_depth(gpu.encrypt(v), circ), cpu.fit_depth(cpu.encrypt(v), circ)
    assert fg.level == fc.level == d
    assert np.array_equal(gpu.backend.to_host(fg.data), fc.data)
    rg = M.rank(gpu, fg, 8, cfg).ranks
    assert rg.level == 0 and np.array_equal(gpu.backend.to_host(rg.data), M.rank(cpu, fc, 8, cfg).ranks.data)

    v128 = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    cfg4 = M.KernelConfig(mode="composite", composite=(4, 2), indicator_composite=(4, 2),
                          tie_margin=2.0 ** -11)
    q = M.StatisticQuery("min")
    need = eng_long.circuit_depth(lambda e, c: M.order_statistic_mask(e, c, 128, q, cfg4))
    assert need < eng_long.params.max_level
    mask = M.order_statistic_mask(eng_long, eng_long.fit_depth(eng_long.encrypt(v128), need), 128, q, cfg4)
    assert mask.level == 0
    m = M.read_row(eng_long, mask, 128)
    assert int(np.argmax(m)) == int(np.argmin(v128))
    assert np.abs(m - np.eye(128)[int(np.argmin(v128))]).max() < 1e-6


@pytest.mark.parametrize("n_rows", [2, 3, 8, 11])
def test_linear_combinations_equal_single_sums(eng12, n_rows):
    """engine.linear_combinations (srk_lincomb_multi: every term read once per eight
    sums) gives limb for limb the ciphertexts of one linear_combination per row --
    terms at different levels, a batched stack, every output-group size."""
    rng = np.random.default_rng(n_rows)
    x = eng12.encrypt(rng.uniform(-1, 1, 64))
    t2 = eng12.mul(x, x)
    t3 = eng12.mul(t2, x)
    cts = [x, t2, t3, eng12.add(t2, t3), eng12.mul_plain(t3, 0.5)]
    rows = rng.uniform(-2, 2, (n_rows, len(cts))).tolist()
    eng12.cost_reset()
    many = eng12.linear_combinations(cts, rows)
    cost_many = eng12.cost_snapshot()
    eng12.cost_reset()
    single = [eng12.linear_combination(list(zip(cts, row))) for row in rows]
    assert eng12.cost_snapshot() == cost_many
    for a, b in zip(many, single):
        assert a.level == b.level
        assert np.array_equal(eng12.backend.to_host(a.data), eng12.backend.to_host(b.data))
    # lock-step batch of two ciphertexts per term
    st = [eng12.stack([c, c]) for c in cts]
    many_b = eng12.linear_combinations(st, rows)
    for a, b in zip(many_b, single):
        got = eng12.backend.to_host(eng12.unstack(a)[1].data)
        assert np.array_equal(got, eng12.backend.to_host(b.data))


@pytest.mark.parametrize("repeat", [6, 7])
def test_linear_combinations_many_terms(eng12, repeat):
    """30 terms (the FP64-quotient sums of the limbs under 40-bit primes, at their
    32-term limit's side) and 35 terms (128-bit sums everywhere): same limbs as the
    single sums."""
    rng = np.random.default_rng(repeat)
    x = eng12.encrypt(rng.uniform(-1, 1, 64))
    t2 = eng12.mul(x, x)
    base = [x, t2, eng12.mul(t2, x), eng12.add(t2, x), eng12.mul_plain(t2, 0.25)]
    cts = base * repeat
    rows = rng.uniform(-3, 3, (5, len(cts))).tolist()
    many = eng12.linear_combinations(cts, rows)
    for a, row in zip(many, rows):
        b = eng12.linear_combination(list(zip(cts, row)))
        assert np.array_equal(eng12.backend.to_host(a.data), eng12.backend.to_host(b.data))
