"""CKKS canonical-embedding encoder (host side, float64 numpy FFT).

Slot j of a plaintext polynomial m(X) in Z[X]/(X^N + 1) is its value at the
primitive 2N-th root zeta^(5^j); the conjugate slots sit at zeta^(-5^j).  The
Galois automorphism X -> X^(5^k) therefore moves slot j+k into slot j, i.e.
it is a cyclic LEFT rotation by k -- the direction the reference simulator
defines for ``rotate`` (reference ``engine.py:234-251``, ``np.roll(x, -k)``).

Evaluating m at all N odd powers zeta^(2t+1) is one length-N FFT of the
twisted coefficients m_k zeta^k, so both directions cost O(N log N):

    values[t] = sum_k (m_k zeta^k) e^{2 pi i t k / N}  =  N * ifft(m * zeta^k)[t]

The encoder only produces and consumes integer/real coefficient vectors; it
never touches RNS limbs, so the GPU and any CPU restatement share identical
plaintext integers (this is what makes ciphertext limbs bit-comparable).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

__all__ = ["Encoder", "get_encoder"]

# Largest |coefficient| we let round() produce: integer coefficients are
# reduced per prime from int64, and lazy kernels assume < 2^62.
_COEFF_LIMIT = float(1 << 62)


class Encoder:
    def __init__(self, log_n: int):
        self.log_n = log_n
        self.n = 1 << log_n
        self.slots = self.n // 2
        two_n = 2 * self.n
        # 5^j mod 2N for j < N/2: the rotation group generator orbit
        pos = np.empty(self.slots, dtype=np.int64)
        g = 1
        for j in range(self.slots):
            pos[j] = g
            g = (g * 5) % two_n
        self.slot_index = (pos - 1) // 2  # t with 2t+1 = 5^j
        self.conj_index = (two_n - pos - 1) // 2  # t with 2t+1 = -5^j mod 2N
        k = np.arange(self.n)
        self.twist = np.exp(1j * np.pi * k / self.n)  # zeta^k
        self.untwist = np.conj(self.twist)

    def embed(self, values) -> np.ndarray:
        """Real coefficients (unscaled) of the polynomial whose slots are ``values``."""
        z = np.zeros(self.slots, dtype=np.complex128)
        v = np.asarray(values, dtype=np.float64).ravel()
        z[: v.size] = v
        full = np.empty(self.n, dtype=np.complex128)
        full[self.slot_index] = z
        full[self.conj_index] = np.conj(z)
        coeffs = np.fft.fft(full) / self.n * self.untwist
        return coeffs.real

    def encode(self, values, scale: float) -> np.ndarray:
        """Integer coefficients round(scale * m(X)) as int64."""
        c = np.rint(self.embed(values) * scale)
        if np.any(np.abs(c) >= _COEFF_LIMIT):
            raise OverflowError("encoded coefficient exceeds 2^62; lower the scale or values")
        return c.astype(np.int64)

    def decode(self, coeffs) -> np.ndarray:
        """Real slot values of a (real, already unscaled) coefficient vector."""
        c = np.asarray(coeffs, dtype=np.float64)
        vals = np.fft.ifft(c * self.twist) * self.n
        return vals[self.slot_index].real.copy()


@lru_cache(maxsize=None)
def get_encoder(log_n: int) -> Encoder:
    return Encoder(log_n)
