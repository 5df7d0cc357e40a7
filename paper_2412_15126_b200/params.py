"""RNS-CKKS parameter sets for the ranking / order-statistics / sorting path.

The reference engine (`slotrank.engine.HEParams`, reference
``pkg/src/slotrank/engine.py:72-94``) only knows ``slot_count`` and
``max_level``.  Here a parameter set is a concrete RNS-CKKS modulus chain:

* ``q_primes[0]`` is the 60-bit base prime, ``q_primes[1..L]`` the scaling
  primes (one per multiplicative level), ``p_primes`` the special primes
  used by hybrid key switching with ``dnum`` digits;
* every prime is NTT-friendly (``q = 1 mod 2N``) and below 2^62 so the lazy
  butterflies in ``csrc/ntt.cuh`` keep values in [0, 4q) without overflow;
* level ``l`` means the ciphertext lives modulo ``q_0 * ... * q_l``, which
  is exactly the simulator's "remaining level" counter: every ct x ct and
  ct x pt multiplication rescales by one prime and drops one level
  (reference ``engine.py:215-232``).

Scale policy (the FLEXIBLE rule): the nominal scale of a level-l
ciphertext is ``scales[l]`` with ``scales[L] = 2^log_scale`` and
``scales[l-1] = scales[l]^2 / q_l``.  Scaling primes are picked one at a time
as the unused NTT prime nearest the running scale, which keeps every
``scales[l]`` within a few ppm of 2^log_scale.  Products of two level-l
ciphertexts therefore land exactly on ``scales[l-1]`` after rescaling; plaintext
constants are encoded at whatever real scale makes their product land there.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

__all__ = [
    "CKKSParams",
    "is_prime",
    "ntt_prime_candidates",
    "make_params",
    "root_of_unity",
    "PRESETS",
    "preset",
]

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (covers every 64-bit prime)."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_prime_candidates(two_n: int, start: int, direction: int):
    """Yield primes q = 1 (mod two_n) walking from ``start`` in ``direction``."""
    q = start - ((start - 1) % two_n)  # q = 1 mod two_n, q <= start
    if direction > 0 and q < start:
        q += two_n
    while q > two_n:
        if is_prime(q):
            yield q
        q += two_n if direction > 0 else -two_n


@lru_cache(maxsize=None)
def root_of_unity(q: int, n: int) -> int:
    """Canonical primitive 2n-th root of unity mod q.

    psi = x^((q-1)/2n) for the first x = 2, 3, ... with psi^n = -1 (mod q).
    Every implementation of the NTT in this repo (CUDA tables, CPU oracle)
    takes psi from here, so NTT-domain limbs are comparable bit for bit.
    """
    if (q - 1) % (2 * n):
        raise ValueError(f"{q} is not 1 mod {2 * n}")
    e = (q - 1) // (2 * n)
    x = 2
    while True:
        psi = pow(x, e, q)
        if pow(psi, n, q) == q - 1:
            return psi
        x += 1


def _nearest_unused_prime(two_n: int, target: float, used: set[int]) -> int:
    t = int(round(target))
    down = ntt_prime_candidates(two_n, t, -1)
    up = ntt_prime_candidates(two_n, t + 1, +1)
    lo = next(p for p in down if p not in used)
    hi = next(p for p in up if p not in used)
    return lo if (t - lo) <= (hi - t) else hi


@dataclass(frozen=True)
class CKKSParams:
    """A full RNS-CKKS parameter set; equality is by value (reference ``engine.py:309``)."""

    name: str
    log_n: int
    q_primes: tuple[int, ...]
    p_primes: tuple[int, ...]
    dnum: int
    log_scale: int
    hamming_weight: int
    sigma: float = 3.2
    seed: int = 0
    secure: bool = False
    scales: tuple[float, ...] = field(default=(), compare=False)

    @property
    def ring_degree(self) -> int:
        return 1 << self.log_n

    @property
    def slot_count(self) -> int:
        return 1 << (self.log_n - 1)

    @property
    def max_level(self) -> int:
        return len(self.q_primes) - 1

    @property
    def n_special(self) -> int:
        return len(self.p_primes)

    @property
    def alpha(self) -> int:
        """Q-limbs per key-switching digit."""
        return -(-len(self.q_primes) // self.dnum)

    @property
    def all_primes(self) -> tuple[int, ...]:
        """Prime table order used everywhere: Q primes then P primes."""
        return self.q_primes + self.p_primes

    @property
    def roots(self) -> tuple[int, ...]:
        """Primitive 2N-th root psi per prime (Q then P), fixed by ``root_of_unity``."""
        return tuple(root_of_unity(p, self.ring_degree) for p in self.all_primes)

    def digits_at(self, level: int) -> int:
        return -(-(level + 1) // self.alpha)

    def scale_at(self, level: int) -> float:
        return self.scales[level]

    def log_qp(self) -> float:
        return sum(math.log2(p) for p in self.all_primes)

    def ciphertext_bytes(self, level: int | None = None) -> int:
        lvl = self.max_level if level is None else level
        return 2 * (lvl + 1) * self.ring_degree * 8

    def describe(self) -> dict:
        return {
            "name": self.name,
            "log_n": self.log_n,
            "slots": self.slot_count,
            "q_limbs": len(self.q_primes),
            "q_bits": [p.bit_length() for p in self.q_primes[:2]] + ["..."],
            "p_limbs": len(self.p_primes),
            "p_bits": self.p_primes[0].bit_length() if self.p_primes else 0,
            "dnum": self.dnum,
            "log_scale": self.log_scale,
            "log_qp": round(self.log_qp(), 1),
            "hamming_weight": self.hamming_weight,
            "secure": self.secure,
        }


@lru_cache(maxsize=None)
def make_params(
    name: str,
    log_n: int,
    levels: int,
    *,
    base_bits: int = 60,
    scale_bits: int = 40,
    special: int = 3,
    special_bits: int = 60,
    dnum: int = 3,
    hamming_weight: int = 192,
    sigma: float = 3.2,
    seed: int = 0,
    secure: bool = False,
) -> CKKSParams:
    """Deterministic prime chain: base prime, ``levels`` scaling primes, specials."""
    two_n = 2 << log_n
    used: set[int] = set()
    base = next(ntt_prime_candidates(two_n, (1 << base_bits) - 1, -1))
    used.add(base)
    scales = [0.0] * (levels + 1)
    scales[levels] = float(1 << scale_bits)
    chain = [0] * (levels + 1)
    chain[0] = base
    for lvl in range(levels, 0, -1):
        q = _nearest_unused_prime(two_n, scales[lvl], used)
        used.add(q)
        chain[lvl] = q
        scales[lvl - 1] = scales[lvl] * scales[lvl] / q
    specials = []
    gen = ntt_prime_candidates(two_n, (1 << special_bits) - 1, -1)
    while len(specials) < special:
        p = next(gen)
        if p not in used:
            used.add(p)
            specials.append(p)
    for p in chain + specials:
        if p >= 1 << 62:
            raise ValueError("primes must stay below 2^62 for lazy NTT butterflies")
    if dnum < 1 or dnum > levels + 1:
        raise ValueError(f"dnum must lie in [1, {levels + 1}]")
    return CKKSParams(
        name=name,
        log_n=log_n,
        q_primes=tuple(chain),
        p_primes=tuple(specials),
        dnum=dnum,
        log_scale=scale_bits,
        hamming_weight=hamming_weight,
        sigma=sigma,
        seed=seed,
        secure=secure,
        scales=tuple(scales),
    )


# BASELINE.json configs.  Key-switch noise needs P >= the largest digit
# (SURVEY F4d): "cfg2" keeps the microbenchmark's dnum=3 / K=3 exactly (it is
# only checked for bit-exactness on uniform limbs); the end-to-end presets
# size K to the digit.  "long" is the non-secure long chain that fits the
# order-statistic and N=1024 sort circuits without bootstrapping (F4c).
PRESETS = {
    # config 1: ring 2^12, 60 + 22x40 bits, one 61-bit special prime (dnum = 23)
    "cfg1": dict(log_n=12, levels=22, special=1, special_bits=61, dnum=23, hamming_weight=64),
    # config 2: ring 2^16, 60 + 29x40, 3x60 special, dnum = 3 (primitive microbenchmark)
    "cfg2": dict(log_n=16, levels=29, special=3, special_bits=60, dnum=3, hamming_weight=192),
    # config 3: same chain, special primes sized to the 420-bit digit
    "cfg3": dict(log_n=16, levels=29, special=8, special_bits=60, dnum=3, hamming_weight=192),
    # config 3 at the reference's 1e-6 slot tolerance for ranks: Delta = 2^47 (the
    # diagonal comparisons amplify CKKS noise ~1900x; tools/delta_study.py), integer
    # kernels (scaling primes >= 2^41), 10 special primes for the 480-bit digits
    "cfg3_hp": dict(log_n=16, levels=29, special=10, special_bits=60, dnum=3, hamming_weight=192,
                    scale_bits=47),
    # configs 4/5: long non-secure chain for masks + values and the N=1024 sort
    "long": dict(log_n=16, levels=56, special=11, special_bits=60, dnum=4, hamming_weight=192),
    # the tie-corrected N=1024 sort (block tie offsets) needs two more levels
    "long58": dict(log_n=16, levels=58, special=11, special_bits=60, dnum=4, hamming_weight=192),
    # small rings for CPU tests
    "toy": dict(log_n=10, levels=12, special=4, special_bits=60, dnum=4, hamming_weight=32),
    "toy_deep": dict(log_n=11, levels=40, special=6, special_bits=60, dnum=6, hamming_weight=32),
    # ring 2^12 with room for the golden Chebyshev circuits (2048 slots)
    "ring12": dict(log_n=12, levels=34, special=6, special_bits=60, dnum=5, hamming_weight=64),
    "toy_sort": dict(log_n=11, levels=48, special=7, special_bits=60, dnum=6, hamming_weight=32),
}


def preset(name: str, **overrides) -> CKKSParams:
    kw = dict(PRESETS[name])
    kw.update(overrides)
    return make_params(name, **kw)
