"""Bit-exact parity of every CUDA primitive against the CPU oracle
(oracle/ckks_oracle.c) on seeded uniform limbs, through the C-ABI."""

import ctypes

import numpy as np
import pytest

from paper_2412_15126_b200.params import preset

pytestmark = pytest.mark.gpu

PARAMS = ["toy", "cfg1", "toy_deep", "cfg2"]


@pytest.fixture(scope="module", params=PARAMS)
def pair(request, require_cuda):
    import torch

    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.backend_cuda import CudaBackend

    p = preset(request.param)
    return p, CudaBackend(p), OracleCKKS(p)


def rand_limbs(p, shape_prefix, level, seed, extended=False):
    rng = np.random.default_rng(seed)
    primes = list(p.q_primes[: level + 1]) + (list(p.p_primes) if extended else [])
    out = np.empty(shape_prefix + (len(primes), p.ring_degree), dtype=np.uint64)
    for i, q in enumerate(primes):
        out[..., i, :] = rng.integers(0, q, size=shape_prefix + (p.ring_degree,), dtype=np.uint64)
    return out


def dev(gb, arr):
    return gb.from_host(arr)


def host(gb, t):
    return gb.to_host(t)


def call(gb, name, *args):
    from paper_2412_15126_b200 import _lib

    _lib.check(getattr(gb.lib, name)(gb.ctx, *args))


def ptr(t):
    return t.data_ptr()


def rot_layout(gb, key, galois):
    """Device copy of a standard-layout switching key in rotation layout."""
    k = dev(gb, key)
    call(gb, "srk_permute_key", ptr(k), galois, gb.workspace(), gb.stream())
    return k


def levels_for(p):
    return sorted({p.max_level, max(1, p.max_level // 2), 1})


def test_ntt_roundtrip_bit_exact(pair):
    p, gb, orc = pair
    L = p.max_level
    a = rand_limbs(p, (2,), L, 1)
    t = dev(gb, a)
    call(gb, "srk_ntt", ptr(t), 2, (L + 1) * p.ring_degree, L + 1, 0, 0, gb.stream())
    want = np.stack([orc.ntt(a[k], range(L + 1)) for k in range(2)])
    assert np.array_equal(host(gb, t), want)
    call(gb, "srk_ntt", ptr(t), 2, (L + 1) * p.ring_degree, L + 1, 0, 1, gb.stream())
    assert np.array_equal(host(gb, t), a)


def test_ntt_special_primes(pair):
    p, gb, orc = pair
    K = len(p.p_primes)
    first = len(p.q_primes)
    rng = np.random.default_rng(2)
    a = np.stack([rng.integers(0, q, p.ring_degree, dtype=np.uint64) for q in p.p_primes])
    t = dev(gb, a)
    call(gb, "srk_ntt", ptr(t), 1, 0, K, first, 0, gb.stream())
    assert np.array_equal(host(gb, t), orc.ntt(a, range(first, first + K)))


@pytest.mark.parametrize("op", [0, 1, 2])
def test_addsub(pair, op):
    p, gb, orc = pair
    lvl = p.max_level // 2
    a, b = rand_limbs(p, (2,), lvl, 3), rand_limbs(p, (2,), lvl, 4)
    out = gb.addsub(dev(gb, a), dev(gb, b), lvl, op)
    want = np.empty_like(a)
    orc.L.orc_addsub(orc.ctx, a.ctypes.data, b.ctypes.data, want.ctypes.data, lvl, op)
    assert np.array_equal(host(gb, out), want)


def test_tensor(pair):
    p, gb, orc = pair
    for lvl in levels_for(p):
        a, b = rand_limbs(p, (2,), lvl, 5), rand_limbs(p, (2,), lvl, 6)
        d = gb.empty_ct(lvl, polys=3)
        ta, tb = dev(gb, a), dev(gb, b)
        call(gb, "srk_tensor", ptr(ta), ptr(tb), ptr(d), lvl, gb.stream())
        assert np.array_equal(host(gb, d), orc.tensor(a, b, lvl))


def test_rescale(pair):
    p, gb, orc = pair
    for lvl in levels_for(p):
        a = rand_limbs(p, (2,), lvl, 7 + lvl)
        out = gb.empty_ct(lvl - 1)
        ta = dev(gb, a)
        call(gb, "srk_rescale", ptr(ta), ptr(out), lvl, gb.workspace(), gb.stream())
        assert np.array_equal(host(gb, out), orc.rescale(a, lvl)), lvl


def test_mul_const_and_plain_rescale(pair):
    p, gb, orc = pair
    lvl = p.max_level
    a = rand_limbs(p, (2,), lvl, 11)
    pt = rand_limbs(p, (), lvl, 12)
    k = [int(x) for x in np.random.default_rng(13).integers(0, 2**40, lvl + 1)]
    out = gb.mul_plain_rescale(dev(gb, a), dev(gb, pt), lvl)
    tmp = np.empty_like(a)
    orc.L.orc_mul_plain(orc.ctx, a.ctypes.data, pt.ctypes.data, tmp.ctypes.data, lvl)
    assert np.array_equal(host(gb, out), orc.rescale(tmp, lvl))
    # constant multiply of a modulus-dropped view (alignment path)
    tgt = lvl - 2
    out = gb.mul_const_rescale(dev(gb, a), lvl, k[: tgt + 1], tgt)
    kk = np.array([x % q for x, q in zip(k, p.q_primes)], dtype=np.uint64)
    tmp = np.empty((2, tgt + 1, p.ring_degree), dtype=np.uint64)
    orc.L.orc_mul_const(orc.ctx, a.ctypes.data, lvl + 1, kk.ctypes.data, tmp.ctypes.data, tgt)
    assert np.array_equal(host(gb, out), orc.rescale(tmp, tgt))


def test_automorph(pair):
    p, gb, orc = pair
    lvl = p.max_level // 2
    a = rand_limbs(p, (2,), lvl, 14)
    ta = dev(gb, a)
    for g in (5, pow(5, 7, 2 * p.ring_degree), 2 * p.ring_degree - 1):
        out = gb.empty_ct(lvl)
        call(gb, "srk_automorph", ptr(ta), ptr(out), 2 * (lvl + 1), g, gb.stream())
        assert np.array_equal(host(gb, out), orc.automorph(a, g))


def test_keyswitch_and_relin(pair):
    p, gb, orc = pair
    n_all = len(p.all_primes)
    rng = np.random.default_rng(15)
    key = np.empty((p.dnum, 2, n_all, p.ring_degree), dtype=np.uint64)
    for i, q in enumerate(p.all_primes):
        key[:, :, i, :] = rng.integers(0, q, (p.dnum, 2, p.ring_degree), dtype=np.uint64)
    kd = dev(gb, key)
    lvls = levels_for(p) if p.log_n < 16 else [p.max_level]
    for lvl in lvls:
        d = rand_limbs(p, (), lvl, 16 + lvl)
        out = gb.empty_ct(lvl)
        ps = (lvl + 1) * p.ring_degree
        td = dev(gb, d)
        call(gb, "srk_keyswitch", ptr(td), ptr(kd), ptr(out), ptr(out) + 8 * ps, lvl,
             gb.workspace(), gb.stream())
        assert np.array_equal(host(gb, out), orc.keyswitch(d, key, lvl)), lvl
    lvl = lvls[-1]
    a, b = rand_limbs(p, (2,), lvl, 17), rand_limbs(p, (2,), lvl, 18)
    out = gb.empty_ct(lvl)
    ta, tb = dev(gb, a), dev(gb, b)
    call(gb, "srk_mul_relin", ptr(ta), ptr(tb), ptr(kd), ptr(out), lvl,
         gb.workspace(), gb.stream())
    assert np.array_equal(host(gb, out), orc.mul_relin(a, b, key, lvl))
    g = pow(5, 3, 2 * p.ring_degree)
    out = gb.empty_ct(lvl)
    kr = rot_layout(gb, key, g)
    call(gb, "srk_rotate", ptr(ta), ptr(kr), ptr(out), lvl, g, gb.workspace(), gb.stream())
    assert np.array_equal(host(gb, out), orc.rotate_raw(a, key, g, lvl))


def test_sampling_and_keygen(pair):
    import torch

    from paper_2412_15126_b200.keys import sample_error, sample_secret

    p, gb, orc = pair
    n_all = len(p.all_primes)
    u = torch.empty((n_all, p.ring_degree), dtype=torch.int64, device=gb.device)
    call(gb, "srk_uniform", ptr(u), n_all, 0, 1234, 77 << 8, gb.stream())
    assert np.array_equal(host(gb, u), orc.uniform(n_all, range(n_all), 1234, 77 << 8))
    s = sample_secret(p)
    gb.set_secret(s)
    sk = orc.small_to_ntt(s, range(n_all))
    assert np.array_equal(host(gb, gb._sk_ntt), sk)
    e = sample_error(p, (2, 9), p.dnum)
    sg = orc.automorph(sk, 5)
    key = torch.empty((p.dnum, 2, n_all, p.ring_degree), dtype=torch.int64, device=gb.device)
    tsg, te = dev(gb, sg), torch.from_numpy(e).to(gb.device)
    call(gb, "srk_keygen", ptr(gb._sk_ntt), ptr(tsg), ptr(te),
         p.seed, 9, ptr(key), gb.workspace(), gb.stream())
    assert np.array_equal(host(gb, key), orc.keygen(sk, sg, e, p.seed, 9))


def _key(p, seed):
    rng = np.random.default_rng(seed)
    n_all = len(p.all_primes)
    key = np.empty((p.dnum, 2, n_all, p.ring_degree), dtype=np.uint64)
    for i, q in enumerate(p.all_primes):
        key[:, :, i, :] = rng.integers(0, q, (p.dnum, 2, p.ring_degree), dtype=np.uint64)
    return key


def test_batched_ops_match_oracle(pair):
    """Batched C-ABI forms (chunked internally by 8) == per-ciphertext oracle."""
    import ctypes

    p, gb, orc = pair
    B = 10 if p.log_n < 16 else 3
    lvl = p.max_level
    n = p.ring_degree
    ps = (lvl + 1) * n
    a = rand_limbs(p, (B, 2), lvl, 40)
    b = rand_limbs(p, (B, 2), lvl, 41)
    key = _key(p, 42)
    ta, tb, tk = dev(gb, a), dev(gb, b), dev(gb, key)
    g = pow(5, 5, 2 * n)
    out = gb.empty_ct(lvl, polys=2 * B)
    tr = rot_layout(gb, key, g)
    call(gb, "srk_rotate_batch", ptr(ta), 2 * ps, ptr(tr), ptr(out), 2 * ps, B, lvl, g,
         gb.workspace(), gb.stream())
    got = host(gb, out).reshape(B, 2, lvl + 1, n)
    for i in range(B):
        assert np.array_equal(got[i], orc.rotate_raw(a[i], key, g, lvl)), i
    # hoisted: two rotations per ciphertext share the base extension and equal single rotations
    g2 = pow(5, 9, 2 * n)
    o1, o2 = gb.empty_ct(lvl, polys=2 * B), gb.empty_ct(lvl, polys=2 * B)
    tr2 = rot_layout(gb, key, g2)
    keys = (ctypes.c_void_p * 2)(ptr(tr), ptr(tr2))
    gal = (ctypes.c_uint64 * 2)(g, g2)
    outs = (ctypes.c_void_p * 2)(ptr(o1), ptr(o2))
    call(gb, "srk_rotate_hoisted", ptr(ta), 2 * ps, B, 2, keys, gal, outs, 2 * ps, lvl,
         gb.workspace(), gb.stream())
    h1 = host(gb, o1).reshape(B, 2, lvl + 1, n)
    h2 = host(gb, o2).reshape(B, 2, lvl + 1, n)
    assert np.array_equal(h1, got)
    for i in range(B):
        assert np.array_equal(h2[i], orc.rotate_raw(a[i], key, g2, lvl)), i
    # relinearised products, with and without the rescale
    for resc in (0, 1):
        ol = lvl - resc
        out = gb.empty_ct(ol, polys=2 * B)
        call(gb, "srk_mul_relin_batch", ptr(ta), ptr(tb), 2 * ps, ptr(tk), ptr(out), 2 * (ol + 1) * n, B,
             lvl, resc, gb.workspace(), gb.stream())
        got = host(gb, out).reshape(B, 2, ol + 1, n)
        for i in range(B):
            want = orc.mul_relin(a[i], b[i], key, lvl)
            if resc:
                want = orc.rescale(want, lvl)
            assert np.array_equal(got[i], want), (resc, i)
    out = gb.empty_ct(lvl - 1, polys=2 * B)
    call(gb, "srk_rescale_batch", ptr(ta), 2 * ps, ptr(out), 2 * lvl * n, B, lvl, gb.workspace(),
         gb.stream())
    got = host(gb, out).reshape(B, 2, lvl, n)
    for i in range(B):
        assert np.array_equal(got[i], orc.rescale(a[i], lvl)), i


@pytest.mark.parametrize("chunk", ["4", "1000"])
@pytest.mark.parametrize("name", ["toy", "cfg1"])
def test_ntt_chunking_and_kernel_variants(name, chunk, require_cuda, monkeypatch):
    """Force multi-chunk NTT launches: limbs must not change."""
    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.backend_cuda import CudaBackend

    monkeypatch.setenv("SRK_NTT_CHUNK", chunk)
    p = preset(name)
    gb, orc = CudaBackend(p), OracleCKKS(p)
    B, lvl, n = 9, p.max_level, p.ring_degree
    ps = (lvl + 1) * n
    a = rand_limbs(p, (B, 2), lvl, 50)
    key = _key(p, 51)
    g = pow(5, 7, 2 * n)
    ta, tr = dev(gb, a), rot_layout(gb, key, g)
    out = gb.empty_ct(lvl, polys=2 * B)
    call(gb, "srk_rotate_batch", ptr(ta), 2 * ps, ptr(tr), ptr(out), 2 * ps, B, lvl, g,
         gb.workspace(), gb.stream())
    got = host(gb, out).reshape(B, 2, lvl + 1, n)
    for i in (0, B - 1):
        assert np.array_equal(got[i], orc.rotate_raw(a[i], key, g, lvl)), i
    t = dev(gb, a)
    call(gb, "srk_ntt", ptr(t), 2 * B, ps, lvl + 1, 0, 0, gb.stream())
    call(gb, "srk_ntt", ptr(t), 2 * B, ps, lvl + 1, 0, 1, gb.stream())
    assert np.array_equal(host(gb, t), a)
    out = gb.empty_ct(lvl - 1, polys=2 * B)
    call(gb, "srk_rescale_batch", ptr(ta), 2 * ps, ptr(out), 2 * lvl * n, B, lvl, gb.workspace(),
         gb.stream())
    got = host(gb, out).reshape(B, 2, lvl, n)
    assert np.array_equal(got[B - 1], orc.rescale(a[B - 1], lvl))


@pytest.mark.parametrize("name", ["toy", "cfg1"])
def test_keyswitch_fused_combine_paths(name, require_cuda):
    """The ciphertext-modulus inner product fused into the ModDown NTT's store
    (ST_KSC) gives the oracle's limbs for rotate, hoisted rotate and relinearise
    (odd batch; ring 2^12 with 23 digits: the runtime digit loop)."""
    import ctypes

    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.backend_cuda import CudaBackend

    p = preset(name)
    gb, orc = CudaBackend(p), OracleCKKS(p)
    B, lvl, n = 3, p.max_level - 1, p.ring_degree
    ps = (lvl + 1) * n
    a = rand_limbs(p, (B, 2), lvl, 60)
    b = rand_limbs(p, (B, 2), lvl, 61)
    key = _key(p, 62)
    ta, tb, tk = dev(gb, a), dev(gb, b), dev(gb, key)
    g1, g2 = pow(5, 3, 2 * n), pow(5, 2 * n // 4 - 1, 2 * n)
    r1, r2 = rot_layout(gb, key, g1), rot_layout(gb, key, g2)
    o1, o2 = gb.empty_ct(lvl, polys=2 * B), gb.empty_ct(lvl, polys=2 * B)
    keys = (ctypes.c_void_p * 2)(ptr(r1), ptr(r2))
    gal = (ctypes.c_uint64 * 2)(g1, g2)
    outs = (ctypes.c_void_p * 2)(ptr(o1), ptr(o2))
    call(gb, "srk_rotate_hoisted", ptr(ta), 2 * ps, B, 2, keys, gal, outs, 2 * ps, lvl,
         gb.workspace(), gb.stream())
    for o, g in ((o1, g1), (o2, g2)):
        got = host(gb, o).reshape(B, 2, lvl + 1, n)
        for i in (0, B - 1):
            assert np.array_equal(got[i], orc.rotate_raw(a[i], key, g, lvl)), (g, i)
    out = gb.empty_ct(lvl, polys=2 * B)
    call(gb, "srk_mul_relin_batch", ptr(ta), ptr(tb), 2 * ps, ptr(tk), ptr(out), 2 * ps, B, lvl, 0,
         gb.workspace(), gb.stream())
    got = host(gb, out).reshape(B, 2, lvl + 1, n)
    for i in range(B):
        assert np.array_equal(got[i], orc.mul_relin(a[i], b[i], key, lvl)), i


@pytest.mark.parametrize("env", [
    {"SRK_NTT_CHUNK": "8"},   # many small NTT chunks on both stream lanes
    {"SRK_WS_BATCH": "1"},    # one ciphertext per internal key-switch chunk
])
def test_kernel_switches_ring16(env, require_cuda, monkeypatch):
    """The run-time settings at ring 2^16 (config 2) give the oracle's limbs."""
    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.backend_cuda import CudaBackend

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    p = preset("cfg2")
    gb, orc = CudaBackend(p), OracleCKKS(p)
    B, lvl, n = 2, p.max_level, p.ring_degree
    ps = (lvl + 1) * n
    a = rand_limbs(p, (B, 2), lvl, 70)
    t = dev(gb, a)
    call(gb, "srk_ntt", ptr(t), 2 * B, ps, lvl + 1, 0, 0, gb.stream())
    fwd = host(gb, t).reshape(B, 2, lvl + 1, n)
    assert np.array_equal(fwd[1, 1], orc.ntt(a[1, 1], range(lvl + 1))), "forward NTT"
    call(gb, "srk_ntt", ptr(t), 2 * B, ps, lvl + 1, 0, 1, gb.stream())
    assert np.array_equal(host(gb, t), a), "inverse NTT"
    key = _key(p, 71)
    g = pow(5, 9, 2 * n)
    ta, tr = dev(gb, a), rot_layout(gb, key, g)
    out = gb.empty_ct(lvl, polys=2 * B)
    call(gb, "srk_rotate_batch", ptr(ta), 2 * ps, ptr(tr), ptr(out), 2 * ps, B, lvl, g,
         gb.workspace(), gb.stream())
    got = host(gb, out).reshape(B, 2, lvl + 1, n)
    assert np.array_equal(got[B - 1], orc.rotate_raw(a[B - 1], key, g, lvl)), "rotation"
    out = gb.empty_ct(lvl - 1, polys=2 * B)
    call(gb, "srk_rescale_batch", ptr(ta), 2 * ps, ptr(out), 2 * lvl * n, B, lvl, gb.workspace(),
         gb.stream())
    got = host(gb, out).reshape(B, 2, lvl, n)
    assert np.array_equal(got[0], orc.rescale(a[0], lvl)), "rescale"


@pytest.mark.parametrize("name", ["toy", "cfg1"])
def test_mul_relin_pointer_table(name, require_cuda):
    """srk_mul_relin_ptrs: pairs sharing operands (the composite polynomials'
    (y y, u y, v y)), more pairs than one internal chunk, rescaled -- each output
    equals the oracle's relinearised, rescaled product of its own pair."""
    import ctypes

    from oracle.oracle import OracleCKKS
    from paper_2412_15126_b200.backend_cuda import CudaBackend

    p = preset(name)
    gb, orc = CudaBackend(p), OracleCKKS(p)
    lvl, n = p.max_level, p.ring_degree
    cts = rand_limbs(p, (5, 2), lvl, 80)
    key = _key(p, 81)
    tc, tk = [dev(gb, c) for c in cts], dev(gb, key)
    pairs = [(i % 5, (3 * i + 1) % 5) for i in range(37)]  # 37 > 32: two chunks
    ta = (ctypes.c_void_p * 37)(*[ptr(tc[i]) for i, _ in pairs])
    tb = (ctypes.c_void_p * 37)(*[ptr(tc[j]) for _, j in pairs])
    out = gb.empty_ct(lvl - 1, polys=2 * 37)
    call(gb, "srk_mul_relin_ptrs", ta, tb, 37, ptr(tk), ptr(out), 2 * lvl * n, lvl, 1, gb.workspace(),
         gb.stream())
    got = host(gb, out).reshape(37, 2, lvl, n)
    for k in (0, 1, 31, 32, 36):
        i, j = pairs[k]
        assert np.array_equal(got[k], orc.rescale(orc.mul_relin(cts[i], cts[j], key, lvl), lvl)), k
