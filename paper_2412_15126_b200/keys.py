"""Host-side sampling of the small secret/error polynomials.

Only the *small* randomness lives here (ternary secret of fixed Hamming
weight, rounded Gaussian errors); the uniform ring elements ``a`` are drawn
on the device by a counter-based generator (``csrc/kernels.cuh:k_uniform``).
Everything is a deterministic function of ``params.seed`` and a tag, so two
engines with equal parameters hold the same keys -- the analogue of the
reference's seeded simulator (reference ``engine.py:139-141``) -- and any
backend (GPU or the CPU oracle) can be fed identical randomness.
"""

from __future__ import annotations

import numpy as np

from .params import CKKSParams

__all__ = ["sample_secret", "sample_error", "KEY_RELIN", "galois_key_id"]

KEY_RELIN = 1


def galois_key_id(galois: int) -> int:
    return 2 + int(galois)


def sample_secret(params: CKKSParams) -> np.ndarray:
    """Ternary secret with exactly ``hamming_weight`` nonzero coefficients."""
    n = params.ring_degree
    rng = np.random.default_rng([params.seed, 0x5EC7])
    h = min(params.hamming_weight, n)
    idx = rng.choice(n, size=h, replace=False)
    sign = rng.integers(0, 2, size=h) * 2 - 1
    s = np.zeros(n, dtype=np.int64)
    s[idx] = sign
    return s


def sample_error(params: CKKSParams, tag: tuple[int, ...], count: int = 1) -> np.ndarray:
    """``count`` rounded-Gaussian polynomials (sigma = params.sigma, cut at 6 sigma)."""
    n = params.ring_degree
    rng = np.random.default_rng([params.seed, 0xE770, *tag])
    bound = 6.0 * params.sigma
    e = np.clip(rng.normal(0.0, params.sigma, size=(count, n)), -bound, bound)
    return np.rint(e).astype(np.int64)
