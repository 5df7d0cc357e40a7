// modarith.cuh -- 64-bit modular arithmetic for RNS-CKKS limbs on sm_100a.
//
// All primes are < 2^62 (params.py enforces it), so:
//   * Shoup multiplication by a constant w (w' = floor(w 2^64 / q)) leaves
//     a result in [0, 2q) for ANY 64-bit input -- used for twiddles and
//     base-conversion constants;
//   * Harvey's lazy butterflies keep NTT values in [0, 4q) < 2^64;
//   * a 128-bit accumulator of up to 16 products of residues < 2^62 fits,
//     and is reduced once with a two-word Barrett constant floor(2^128 / q).
// sm_100 has no 64x64->128 multiplier: __umul64hi and a*b lower to IMAD.WIDE
// chains, which is why every inner loop tries to pay for one reduction per
// output rather than per product.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define SRK_HD __host__ __device__ __forceinline__
#else
#define SRK_HD static inline
#endif

struct PrimeConst {
    uint64_t q;       // modulus
    uint64_t two_q;   // 2q (lazy ranges)
    uint64_t ratio_hi, ratio_lo;  // floor(2^128 / q)
    uint64_t ninv, ninv_shoup;    // N^-1 mod q and its Shoup constant
    uint64_t qd_bits, qinv_bits;  // (double) q and 1.0 / (double) q as bit patterns
};

SRK_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Shoup: a * w mod q in [0, 2q), for any a < 2^64, w < q, ws = floor(w 2^64/q)
SRK_HD uint64_t mul_shoup_lazy(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t qh = mulhi64(a, ws);
    return a * w - qh * q;
}
SRK_HD uint64_t mul_shoup(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t r = mul_shoup_lazy(a, w, ws, q);
    return r >= q ? r - q : r;
}

SRK_HD uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
SRK_HD uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}
SRK_HD uint64_t neg_mod(uint64_t a, uint64_t q) { return a ? q - a : 0; }

// 128-bit value as (hi, lo)
struct U128 {
    uint64_t hi, lo;
};

SRK_HD U128 mul_wide(uint64_t a, uint64_t b) {
    U128 r;
    r.lo = a * b;
    r.hi = mulhi64(a, b);
    return r;
}
SRK_HD void add_to(U128 &acc, U128 x) {
    uint64_t lo = acc.lo + x.lo;
    acc.hi += x.hi + (lo < x.lo ? 1u : 0u);
    acc.lo = lo;
}
SRK_HD void mac(U128 &acc, uint64_t a, uint64_t b) { add_to(acc, mul_wide(a, b)); }

// Barrett reduction of a 128-bit x mod q with ratio = floor(2^128 / q).
// q_est = floor(x * ratio / 2^128) is computed exactly (all partial-product
// carries kept), so q_est in {floor(x/q) - 1, floor(x/q)} and one
// conditional subtraction finishes.  Valid for every x < 2^128.
SRK_HD uint64_t reduce128(U128 x, uint64_t ratio_hi, uint64_t ratio_lo, uint64_t q) {
    // x*R = x1R1 2^128 + (x1R0 + x0R1) 2^64 + x0R0
    uint64_t c0 = mulhi64(x.lo, ratio_lo);           // floor(x0R0 / 2^64)
    U128 m1 = mul_wide(x.hi, ratio_lo);              // x1R0
    U128 m2 = mul_wide(x.lo, ratio_hi);              // x0R1
    // middle = m1 + m2 + c0 ; carry into the 2^128 word
    uint64_t lo = m1.lo + m2.lo;
    uint64_t carry = lo < m1.lo ? 1u : 0u;
    uint64_t lo2 = lo + c0;
    carry += lo2 < lo ? 1u : 0u;
    uint64_t qest = x.hi * ratio_hi + m1.hi + m2.hi + carry;
    uint64_t r = x.lo - qest * q;
    return r >= q ? r - q : r;
}

SRK_HD uint64_t mul_mod(uint64_t a, uint64_t b, const PrimeConst &p) {
    return reduce128(mul_wide(a, b), p.ratio_hi, p.ratio_lo, p.q);
}
SRK_HD uint64_t reduce_u128(U128 x, const PrimeConst &p) {
    return reduce128(x, p.ratio_hi, p.ratio_lo, p.q);
}
// reduce an arbitrary 64-bit word mod q
SRK_HD uint64_t reduce64(uint64_t x, const PrimeConst &p) {
    U128 v;
    v.hi = 0;
    v.lo = x;
    return reduce128(v, p.ratio_hi, p.ratio_lo, p.q);
}

// Division of small row indices by a runtime divisor without the 64-bit
// division subroutine: q = (r * m) >> 32 with m = floor(2^32 / d) + 1 is exact
// for r * d < 2^32 (row counts here are < 2^16, divisors < 2^8).
struct Div32 {
    uint64_t m;
};
// (floor((2^32 - 1) / d) + 1 == floor(2^32 / d) + 1, or 2^32 / d for d a power of
// two, which is exact too; a 32-bit division, once per thread)
SRK_HD Div32 mk_div32(uint32_t d) { return Div32{(uint64_t)(0xFFFFFFFFu / d) + 1}; }
SRK_HD uint32_t div32(uint32_t r, Div32 d) { return (uint32_t)(((uint64_t)r * d.m) >> 32); }
