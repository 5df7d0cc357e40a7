import numpy as np
import pytest

from paper_2412_15126_b200.params import PRESETS, is_prime, preset, root_of_unity


@pytest.mark.parametrize("name", sorted(PRESETS))
def test_presets_are_ntt_friendly(name):
    p = preset(name)
    two_n = 2 * p.ring_degree
    assert len(set(p.all_primes)) == len(p.all_primes)
    for q, psi in zip(p.all_primes, p.roots):
        assert is_prime(q) and q % two_n == 1 and q < 2 ** 62
        assert pow(psi, p.ring_degree, q) == q - 1
    # nominal scales stay within 1e-4 of 2^40 over the whole chain
    s = np.array(p.scales) / 2.0 ** p.log_scale
    assert np.abs(s - 1).max() < 1e-4
    assert p.q_primes[0].bit_length() == 60


def test_baseline_shapes():
    c1, c2 = preset("cfg1"), preset("cfg2")
    assert (c1.log_n, len(c1.q_primes), len(c1.p_primes), c1.p_primes[0].bit_length()) == (12, 23, 1, 61)
    assert (c2.log_n, len(c2.q_primes), len(c2.p_primes), c2.dnum) == (16, 30, 3, 3)
    assert all(abs(np.log2(q) - 40) < 1e-3 for q in c2.q_primes[1:])  # "40-bit": ~2^40
    # end-to-end presets: special primes cover the largest digit
    for name in ("cfg3", "long", "toy", "toy_deep"):
        p = preset(name)
        digit = sum(q.bit_length() for q in p.q_primes[: p.alpha])
        assert sum(q.bit_length() for q in p.p_primes) >= digit


def test_root_is_deterministic():
    assert root_of_unity(97, 8) == root_of_unity(97, 8)
    assert pow(root_of_unity(97, 8), 8, 97) == 96
