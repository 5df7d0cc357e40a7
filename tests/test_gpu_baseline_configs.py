"""Parity at the BASELINE configurations themselves (BASELINE.json configs 1-5).

* config 1: the whole N=16 rank on ring 2^12 is bit-exact, limb for limb,
  against the CPU oracle engine (same circuit, same keys, same randomness);
* config 2: the batched C-ABI primitives at the bench's own batch of 64
  ciphertexts (two internal chunks of 32) are bit-exact against the oracle for
  ciphertexts 0, 31, 32 and 63 -- both sides of the chunk boundary;
* configs 3-5: the decrypted GPU pipelines against the slot oracle (the
  reference simulator restated, ``oracle/slotsim.py``) on the SAME circuit,
  with the measured CKKS error bound asserted per config (``BOUNDS``), plus
  the reference-level result (ranks / indices / order / selected values).

Reference behaviour matched: ``ranking.py:145-187`` (rank), ``select.py:78-130``
(masks and values), ``sorting.py:106-142`` (multi_sort); the reference's own
accuracy test uses 1e-6 (``tests/test_sorting.py:127-133``).
"""

import ctypes

import numpy as np
import pytest

import paper_2412_15126_b200 as M
from oracle.plain import fractional_ranks
from oracle.slotsim import SimParams, SlotSim
from paper_2412_15126_b200.params import preset

pytestmark = pytest.mark.gpu

# max |decrypt(GPU) - SlotSim(same circuit)| per config, Delta = 2^40 (DESIGN.md
# "Slot-level parity"); the reference's own tolerance is 1e-6.  The ranks miss
# it: their diagonal comparisons evaluate the sign composite at 0, where its
# slope (~1900 for g3^4 o f3^2) amplifies the CKKS noise; measured 1.6e-5
# (cfg1) and 5.4e-5 (cfg3), asserted at ~2x.  Delta = 2^47 (preset cfg3_hp)
# reaches 1e-6 on the rank (test_cfg3_hp_rank_reaches_1e6; tools/delta_study.py,
# profiles/r02/delta_study_*.json: 2^46 8.7e-7, 2^47 4.1e-7, 2^48 2.5e-7).
BOUNDS = {
    "cfg1_rank": 4e-5,
    "cfg3_rank": 1.2e-4,
    "cfg4_mask": 1e-6,
    "cfg4_value": 1e-6,
    "cfg5_sort": 1e-6,
    "cfg5_sort_tc": 1e-6,
}


def _sim(eng):
    return SlotSim(SimParams(eng.params.slot_count, eng.params.max_level))


# ---------------------------------------------------------------------------
# config 1: limb-exact full pipeline
# ---------------------------------------------------------------------------
def test_cfg1_rank_n16_limbs_bit_exact_vs_oracle(require_cuda):
    from oracle.oracle import oracle_engine

    p = preset("cfg1")
    v = np.random.default_rng(0).choice(64, 16, replace=False) / 64
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))  # BASELINE: g3^4 o f3^2
    gpu, cpu = M.B200Engine(p), oracle_engine(p)
    rg = M.rank(gpu, gpu.encrypt(v), 16, cfg).ranks
    rc = M.rank(cpu, cpu.encrypt(v), 16, cfg).ranks
    assert rg.level == rc.level
    assert np.array_equal(gpu.backend.to_host(rg.data), rc.data)
    assert gpu.cost_snapshot() == cpu.cost_snapshot()
    assert gpu.rotation_offsets() == cpu.rotation_offsets()
    r = M.read_row(gpu, rg, 16)
    assert np.array_equal(np.rint(r), fractional_ranks(v))
    sim = _sim(gpu)
    rs = M.read_row(sim, M.rank(sim, sim.encrypt(v), 16, cfg).ranks, 16)
    err = float(np.abs(r - rs).max())
    assert err < BOUNDS["cfg1_rank"], err


# ---------------------------------------------------------------------------
# config 2: the bench batch (64 ciphertexts, two internal chunks)
# ---------------------------------------------------------------------------
CHECK = (0, 31, 32, 63)


def _rand_cts(torch, p, n_ct, seed, device):
    nl = len(p.q_primes)
    out = torch.empty((n_ct, 2, nl, p.ring_degree), dtype=torch.int64, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    for i, q in enumerate(p.q_primes):
        out[:, :, i, :] = torch.randint(0, q, (n_ct, 2, p.ring_degree), generator=g, device=device,
                                        dtype=torch.int64)
    return out


@pytest.fixture(scope="module")
def cfg2_batch(require_cuda):
    import torch

    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.backend_cuda import CudaBackend

    p = preset("cfg2")
    gb, orc = CudaBackend(p), OracleCKKS(p)
    x = _rand_cts(torch, p, 64, 1, gb.device)
    y = _rand_cts(torch, p, 64, 2, gb.device)
    hx = {i: gb.to_host(x[i]) for i in CHECK}
    hy = {i: gb.to_host(y[i]) for i in CHECK}
    rng = np.random.default_rng(3)
    n_all = len(p.all_primes)
    key = np.empty((p.dnum, 2, n_all, p.ring_degree), dtype=np.uint64)
    for i, q in enumerate(p.all_primes):
        key[:, :, i, :] = rng.integers(0, q, (p.dnum, 2, p.ring_degree), dtype=np.uint64)
    yield p, gb, orc, x, y, hx, hy, key
    del x, y
    torch.cuda.empty_cache()


def _call(gb, name, *args):
    from paper_2412_15126_b200 import _lib

    _lib.check(getattr(gb.lib, name)(gb.ctx, *args))


def test_cfg2_b64_rotate_hoisted_15(cfg2_batch):
    """All 15 power-of-two rotations of 64 ciphertexts through one hoisted call."""
    p, gb, orc, x, _, hx, _, key = cfg2_batch
    n, L = p.ring_degree, p.max_level
    ct = 2 * (L + 1) * n
    gal = [pow(5, 1 << k, 2 * n) for k in range(15)]
    keys = []
    for g in gal:
        k = gb.from_host(key)
        _call(gb, "srk_permute_key", k.data_ptr(), g, gb.workspace(), gb.stream())
        keys.append(k)
    outs = [gb.empty_ct(L, polys=2 * 64) for _ in gal]
    _call(gb, "srk_rotate_hoisted", x.data_ptr(), ct, 64, 15,
          (ctypes.c_void_p * 15)(*[k.data_ptr() for k in keys]), (ctypes.c_uint64 * 15)(*gal),
          (ctypes.c_void_p * 15)(*[o.data_ptr() for o in outs]), ct, L, gb.workspace(), gb.stream())
    for r, g in enumerate(gal):
        # every rotation on the chunk-boundary ciphertexts, a spread on the others
        for i in (CHECK if r in (0, 7, 14) else (31, 32)):
            got = gb.to_host(outs[r].view(64, 2, L + 1, n)[i])
            assert np.array_equal(got, orc.rotate_raw(hx[i], key, g, L)), (r, i)


@pytest.mark.parametrize("rescale", [0, 1])
def test_cfg2_b64_mul_relin_batch(cfg2_batch, rescale):
    p, gb, orc, x, y, hx, hy, key = cfg2_batch
    n, L = p.ring_degree, p.max_level
    ct = 2 * (L + 1) * n
    ol = L - rescale
    kd = gb.from_host(key)
    out = gb.empty_ct(ol, polys=2 * 64)
    _call(gb, "srk_mul_relin_batch", x.data_ptr(), y.data_ptr(), ct, kd.data_ptr(), out.data_ptr(),
          2 * (ol + 1) * n, 64, L, rescale, gb.workspace(), gb.stream())
    for i in CHECK:
        want = orc.mul_relin(hx[i], hy[i], key, L)
        if rescale:
            want = orc.rescale(want, L)
        assert np.array_equal(gb.to_host(out.view(64, 2, ol + 1, n)[i]), want), i


def test_cfg2_b64_rescale_and_ntt(cfg2_batch):
    p, gb, orc, x, _, hx, _, _ = cfg2_batch
    n, L = p.ring_degree, p.max_level
    ct = 2 * (L + 1) * n
    out = gb.empty_ct(L - 1, polys=2 * 64)
    _call(gb, "srk_rescale_batch", x.data_ptr(), ct, out.data_ptr(), 2 * L * n, 64, L,
          gb.workspace(), gb.stream())
    for i in CHECK:
        assert np.array_equal(gb.to_host(out.view(64, 2, L, n)[i]), orc.rescale(hx[i], L)), i
    t = x.clone()
    _call(gb, "srk_ntt", t.data_ptr(), 128, (L + 1) * n, L + 1, 0, 0, gb.stream())
    for i in (0, 63):
        for r in range(2):
            assert np.array_equal(gb.to_host(t[i, r]), orc.ntt(hx[i][r], range(L + 1))), (i, r)
    _call(gb, "srk_ntt", t.data_ptr(), 128, (L + 1) * n, L + 1, 0, 1, gb.stream())
    assert bool((t == x).all())


# ---------------------------------------------------------------------------
# configs 3-5: decrypted pipelines vs the slot oracle on the same circuit
# ---------------------------------------------------------------------------
def test_cfg3_rank_n128_vs_slotsim(require_cuda):
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    eng = M.B200Engine(preset("cfg3"))
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))
    r = M.read_row(eng, M.rank(eng, eng.encrypt(v), 128, cfg).ranks, 128)
    assert np.array_equal(np.rint(r), fractional_ranks(v))
    sim = _sim(eng)
    rs = M.read_row(sim, M.rank(sim, sim.encrypt(v), 128, cfg).ranks, 128)
    err = float(np.abs(r - rs).max())
    assert err < BOUNDS["cfg3_rank"], err
    assert eng.cost_snapshot() == sim.cost_snapshot()


def test_cfg3_hp_rank_reaches_1e6(require_cuda):
    """The reference's 1e-6 slot tolerance (tests/test_sorting.py:127-133) on the
    N=128 rank: Delta = 2^47 with 10 special primes (integer kernels)."""
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    eng = M.B200Engine(preset("cfg3_hp"))
    cfg = M.KernelConfig(mode="composite", composite=(4, 2))
    r = M.read_row(eng, M.rank(eng, eng.encrypt(v), 128, cfg).ranks, 128)
    assert np.array_equal(np.rint(r), fractional_ranks(v))
    sim = _sim(eng)
    rs = M.read_row(sim, M.rank(sim, sim.encrypt(v), 128, cfg).ranks, 128)
    err = float(np.abs(r - rs).max())
    assert err < 1e-6, err


@pytest.fixture(scope="module")
def eng_long(require_cuda):
    return M.B200Engine(preset("long"))


CFG4 = dict(mode="composite", composite=(4, 2), indicator_composite=(4, 2), tie_margin=2.0 ** -11,
            goldschmidt_iters=8)


@pytest.mark.parametrize("kind", ["min", "max", "kth64"])
def test_cfg4_masks_and_values_n128_vs_slotsim(eng_long, kind):
    """One-hot mask AND selected value at N=128 (BASELINE config 4's outputs)."""
    v = np.random.default_rng(0).choice(1024, 128, replace=False) / 1024
    q = {"min": M.StatisticQuery("min"), "max": M.StatisticQuery("max"),
         "kth64": M.StatisticQuery("kth", k=64)}[kind]
    idx = {"min": 0, "max": 127, "kth64": 63}[kind]
    cfg = M.KernelConfig(**CFG4)
    sim = _sim(eng_long)
    ct, cs = eng_long.encrypt(v), sim.encrypt(v)
    m = M.read_row(eng_long, M.order_statistic_mask(eng_long, ct, 128, q, cfg), 128)
    ms = M.read_row(sim, M.order_statistic_mask(sim, cs, 128, q, cfg), 128)
    want = int(np.argsort(v)[idx])
    assert int(np.argmax(m)) == want
    merr = float(np.abs(m - ms).max())
    assert merr < BOUNDS["cfg4_mask"], merr
    val = eng_long.decrypt(M.order_statistic_value(eng_long, ct, 128, q, cfg))[0]
    vs = sim.decrypt(M.order_statistic_value(sim, cs, 128, q, cfg))[0]
    assert abs(val - np.sort(v)[idx]) < 1e-6, (val, np.sort(v)[idx])
    verr = abs(val - vs)
    assert verr < BOUNDS["cfg4_value"], verr


def _multi_sort_check(eng, v, tie_correction, bound, packed=False, composite=(6, 2), fit=False):
    scfg = M.SortConfig(kernel=M.KernelConfig(mode="composite", composite=composite,
                                              indicator_composite=(6, 2)), tie_correction=tie_correction,
                        packed=packed)
    bv = M.block_split(eng, v)
    if fit:  # blocks dropped to the circuit's depth first (engine.fit_depth; not a counted op)
        depth = eng.circuit_depth(lambda e, c: list(M.multi_sort(
            e, type(bv)(blocks=tuple(c for _ in bv.blocks), block_size=bv.block_size, total_len=bv.total_len),
            scfg).blocks))
        assert depth < eng.params.max_level
        bv = type(bv)(blocks=tuple(eng.fit_depth(b, depth) for b in bv.blocks), block_size=bv.block_size,
                      total_len=bv.total_len)
    eng.cost_reset()
    res = M.multi_sort(eng, bv, scfg)
    if fit:
        assert all(b.level == 0 for b in res.blocks)
    out = M.block_merge(eng, res)
    sim = _sim(eng)
    ref = M.block_merge(sim, M.multi_sort(sim, M.block_split(sim, v), scfg))
    assert np.array_equal(np.argsort(out, kind="stable"), np.argsort(np.sort(v), kind="stable"))
    assert np.abs(out - np.sort(v)).max() < 1e-6
    err = float(np.abs(out - ref).max())
    assert err < bound, err
    got, want = eng.cost_snapshot().__dict__, sim.cost_snapshot().__dict__
    if fit:  # the drop is not an op, but the levels it skips are not "consumed" by the simulator
        got.pop("levels_consumed"), want.pop("levels_consumed")
    assert got == want


@pytest.mark.parametrize("packed", [False, True])
def test_cfg5_multi_sort_n1024_shallower_comparison_depth_fitted(eng_long, packed):
    """bench.py's ``sort_n1024_cmp52*``: comparison g3^5 o f3^2 under the (6,2) indicator,
    52 levels, blocks dropped to level 52 first: order exact, 1e-6 against the slot
    oracle on the same circuit and against np.sort."""
    v = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    _multi_sort_check(eng_long, v, False, BOUNDS["cfg5_sort"], packed=packed, composite=(5, 2), fit=True)


def test_cfg5_multi_sort_n1024_vs_slotsim(eng_long):
    v = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    _multi_sort_check(eng_long, v, False, BOUNDS["cfg5_sort"])


def test_cfg5_multi_sort_n1024_tie_corrected(require_cuda):
    """The tie-corrected N=1024 sort (block tie offsets, ranking.py:395-423) needs
    58 levels: the ``long58`` chain."""
    eng = M.B200Engine(preset("long58"))
    v = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    _multi_sort_check(eng, v, True, BOUNDS["cfg5_sort_tc"])


def test_cfg5_multi_sort_n1024_packed(eng_long):
    """Two blocks per ciphertext (packing.py: 18 comparison + 32 indicator
    evaluations, BASELINE's 32 ciphertexts): same circuit on the slot oracle
    within 1e-6, order exact."""
    v = np.random.default_rng(0).choice(8192, 1024, replace=False) / 8192
    _multi_sort_check(eng_long, v, False, BOUNDS["cfg5_sort"], packed=True)
    rep = eng_long.cost_snapshot()
    assert rep.cmp_evals == 18 and rep.ind_evals == 32
