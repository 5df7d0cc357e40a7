// ntt.cuh -- merged-radix negacyclic NTT / INTT over batches of RNS limbs.
//
// Convention (shared with oracle/ckks_oracle.c): forward = Cooley-Tukey on
// natural-order coefficients, output slot k holds the evaluation at
// psi^(2 brv(k) + 1); inverse = Gentleman-Sande, then * N^-1.
//
// An N-point limb is viewed as R rows x C columns (N = R*C, R = 2^ceil(logN/2)):
//   * column pass  = global stages 0..logR-1: R-point sub-transforms over
//     {c + C r}; twiddle index 2^s + (r >> (logR - s));
//   * row pass     = global stages logR..logN-1: C-point sub-transforms over
//     contiguous chunks b; twiddle index 2^s' (R + b) + (c >> (logC - s')).
// Forward runs column then row pass, inverse row then column.  Each pass is
// one kernel: a thread owns E = 2^ceil(logT/2) elements of a T-point
// sub-transform, does ceil(logT/2) radix-2 stages in registers, swaps
// through shared memory, and does the remaining stages in registers.
// Values stay lazily reduced (Harvey): [0,4q) forward, [0,2q) inverse, and
// are canonical [0,q) only at the end of the last pass.
//
// With N = 2^16 a pass reads and writes the limb once (1 MiB of traffic per
// limb per pass); launching both passes over one chunk of limbs at a time
// keeps the intermediate in L2, so HBM sees ~one read + one write per limb.
#pragma once
#include <cstdint>

#include "modarith.cuh"

#define SRK_MAXP 128

// per-limb constant with Shoup companion, passed by value (<= 2 KiB)
struct LimbConsts {
    uint64_t w[SRK_MAXP];
    uint64_t ws[SRK_MAXP];
};

// A batch of limbs.  Poly p of the batch belongs to ciphertext b = p / ppc
// (component r = p % ppc) and its limb slot t lives at
//   ptr + b * ct_stride + r * poly_stride + t * N.
// Limb i of a poly maps to slot t and prime pid:
//   mode 0: t = i, pid = i + (i < split ? off_a : off_b);
//   mode 1: ModUp targets of digit j = r at `level`: the ext slots outside
//           [j alpha, j alpha + |G_j|), t >= ne skipped; pid = ext prime of t.
struct LimbBatch {
    uint64_t *ptr;
    long long ct_stride, poly_stride;
    int ppc, n_polys, n_limbs;
    int mode, split, off_a, off_b;
    int alpha, nl, level, L, ne;
    int cls;  // prime-class filter: 0 all limbs, 1 only q < 2^41 (FP64), 2 only q >= 2^41
};

__device__ __forceinline__ int batch_pid(const LimbBatch &b, int i) {
    return i + (i < b.split ? b.off_a : b.off_b);
}

// limb i of poly r -> (slot t, prime pid); false if this (r, i) is skipped
__device__ __forceinline__ bool limb_map(const LimbBatch &b, int r, int i, int &t, int &pid) {
    if (b.mode == 0) {
        t = i;
        pid = batch_pid(b, i);
        return true;
    }
    const int g0 = r * b.alpha;
    const int gsz = min(b.alpha, b.nl - g0);
    t = i < g0 ? i : i + gsz;
    if (t >= b.ne) return false;
    pid = t <= b.level ? t : t + (b.L - b.level);
    return true;
}

// NTT-domain index of X -> X^g: slot k holds the evaluation at psi^(2 brv(k)+1)
__device__ __forceinline__ uint32_t auto_index(uint32_t k, uint64_t g, int log_n) {
    const uint64_t mask = (2ull << log_n) - 1;
    uint32_t r = __brev(k) >> (32 - log_n);
    uint64_t e = ((uint64_t)r * 2 + 1) * g & mask;
    return __brev((uint32_t)((e - 1) >> 1)) >> (32 - log_n);
}

// Fused first-pass loads / last-pass stores (see ntt_pass_kernel).
enum { LD_PLAIN = 0, LD_BCONV = 1, LD_SPREAD = 2, LD_AUTO = 3, LD_BCONV8 = 4, LD_BCONV16 = 5 };
// ModDown conversion load, bucketed by the number of special primes it reads
__host__ __device__ constexpr bool is_bconv(int ld) {
    return ld == LD_BCONV || ld == LD_BCONV8 || ld == LD_BCONV16;
}
__host__ __device__ constexpr int bconv_maxk(int ld) {
    return ld == LD_BCONV ? 4 : (ld == LD_BCONV8 ? 8 : 16);
}
enum { ST_PLAIN = 0, ST_MODDOWN = 1, ST_RESCALE = 2, ST_SCALE = 3 };

struct FuseArgs {
    // loads: source poly (b, r) at src + b*src_ct + r*src_ps (+ slot t * N for
    // LD_PLAIN / LD_AUTO; LD_BCONV reads n_src limbs, LD_SPREAD one limb)
    const uint64_t *src;
    long long src_ct, src_ps;
    uint64_t galois;         // LD_AUTO: X -> X^galois gather
    int n_src, src_pid0;     // LD_BCONV: z limbs under primes src_pid0 ..
    const uint64_t *mat;     // LD_BCONV: [n_src][mat_ld] conversion constants
    const ulonglong2 *mat2;  // the same with Shoup companions (streaming conversion)
    const ulonglong2 *mhl;   // {m, m 2^32 mod q_t} and {m/q_t, (m 2^32 mod q_t)/q_t}:
    const double2 *fhl;      //   FP64-pipe conversion (k_moddown_conv_f64)
    int mat_ld;
    const uint64_t *corr;    // LD_BCONV: [v * prod src primes]_{q_t}, table [v][corr_ld]
    int corr_ld;
    const uint8_t *vround;   // LD_BCONV: v = round(sum z_k / p_k) per (b, r, n), k_moddown_v
    uint64_t top_q;          // LD_SPREAD: modulus of the limb being spread
    // stores: out(b, r, t) from the transform result x and
    //   ST_MODDOWN: add_r + (acc - x) * mulc          (add0 gathered if add_galois != 1)
    //   ST_RESCALE: (acc * pre - x) * mulc            (pre: const pre_k or plaintext pt)
    //   ST_SCALE  : x * mulc   (replaces N^-1 in the inverse transform)
    uint64_t *out;
    long long out_ct, out_ps;
    const uint64_t *acc;
    long long acc_ct, acc_ps;
    uint64_t acc_galois;     // ST_MODDOWN: read acc through X -> X^acc_galois (1 = none)
    const uint64_t *add0, *add1;
    long long add_ct;
    uint64_t add_galois;
    uint64_t out_galois;     // ST_MODDOWN: write sigma_{out_galois}(result) (1 = identity);
    uint64_t out_galois_inv; //   rows of T elements map to rows, staged through smem
    int pre_mode;            // 0 none, 1 per-limb constant, 2 plaintext
    const uint64_t *pt;      // [limbs][N] per ciphertext at stride pt_ct (0 = shared)
    long long pt_ct;
    LimbConsts mulc;
    LimbConsts pre;
    LimbConsts addc;         // ST_MODDOWN: add_r scaled by addc (when add_scaled)
    int add_scaled;
};

struct NttTables {
    const PrimeConst *pc;
    const ulonglong2 *tw;   // [n_primes][N] {psi^brv(k), Shoup}: one 16-B load per twiddle
    const ulonglong2 *itw;  // [n_primes][N] {psi^-brv(k), Shoup}
    const double *twd;      // [n_primes][N] psi^brv(k) as an exact double (FP64 limbs:
    const double *itwd;     //   one 8-B load, no u64 -> f64 conversion per twiddle)
};

template <int LOG_T>
struct NttShape {
    static constexpr int T = 1 << LOG_T;
    static constexpr int LE1 = (LOG_T + 1) / 2;  // stages in round 1
    static constexpr int LE2 = LOG_T - LE1;      // stages in round 2
    static constexpr int E = 1 << LE1;           // elements per thread
    static constexpr int TPS = T / E;            // threads per sub-transform
};

// Forward Harvey butterfly on [0,4q) inputs.
__device__ __forceinline__ void ct_bfly(uint64_t &x, uint64_t &y, uint64_t w, uint64_t ws,
                                        uint64_t q, uint64_t two_q) {
    uint64_t X = x >= two_q ? x - two_q : x;
    uint64_t T = mul_shoup_lazy(y, w, ws, q);
    x = X + T;
    y = X - T + two_q;
}

// Inverse Gentleman-Sande butterfly on [0,2q) inputs.
__device__ __forceinline__ void gs_bfly(uint64_t &x, uint64_t &y, uint64_t w, uint64_t ws,
                                        uint64_t q, uint64_t two_q) {
    uint64_t S = x + y;
    S = S >= two_q ? S - two_q : S;
    uint64_t D = x - y + two_q;
    x = S;
    y = mul_shoup_lazy(D, w, ws, q);
}

// smem index of element c of sub-transform sb in a row-pass tile (pad one
// word every E words so stride-E reads are bank-conflict free)
template <int LOG_T>
__device__ __forceinline__ int row_sidx(int sb, int c) {
    using S = NttShape<LOG_T>;
    return sb * (S::T + S::T / S::E) + c + (c >> S::LE1);
}

// Reduction-free butterflies for primes below 2^46 (all scaling primes):
// forward outputs grow by at most 2q per stage (T in [0, 2q)), so 16 stages
// stay below 34q; inverse sums at most double per stage, and the difference
// is offset by M = q << k (a multiple of q above any operand at step k), so
// 16 steps stay below 2^16 q < 2^62.  Only the final pass reduces.
#define SRK_SMALL_Q (1ull << 46)
#ifndef SRK_NTT_MINB
#define SRK_NTT_MINB 3  // CTAs per SM the register budget is sized for
#endif

__device__ __forceinline__ void ct_bfly_small(uint64_t &x, uint64_t &y, uint64_t w, uint64_t ws,
                                              uint64_t q, uint64_t two_q) {
    uint64_t T = mul_shoup_lazy(y, w, ws, q);
    y = x - T + two_q;
    x = x + T;
}

__device__ __forceinline__ void gs_bfly_small(uint64_t &x, uint64_t &y, uint64_t w, uint64_t ws,
                                              uint64_t q, uint64_t m) {
    uint64_t D = x - y + m;
    x = x + y;
    y = mul_shoup_lazy(D, w, ws, q);
}

// ---------------------------------------------------------------------------
// FP64 path for primes below 2^41 (every scaling prime).  B200's FP64 pipe is
// full rate and independent of the IMAD pipe the integer butterflies saturate;
// a 64-bit Shoup product costs ~17 IMAD slots, the FP64 one 6 full-rate ops:
//   hi = y w;  lo = fma(y, w, -hi)            (y w == hi + lo exactly)
//   t  = fma(hi, 1/q, 1.5*2^52) - 1.5*2^52   (nearest integer, no FRND)
//   r  = fma(-t, q, hi) + lo                  (exact: y w - t q, |r| < q)
// valid while |y| < 2^51 (so hi/q < 2^51) and w < q < 2^41.  Values live as
// signed integer-valued doubles in the same 64-bit registers/smem words:
// forward outputs grow by < q per stage (16 stages < 17 q); inverse sums
// double per stage, so the second pass starts with a centred reduction.
// u64 <-> f64 conversions use the 2^52 magic-number trick (LOP + DADD).
// ---------------------------------------------------------------------------
#define SRK_F64_Q (1ull << 41)
#define SRK_F64_MAGIC 6755399441055744.0  // 1.5 * 2^52
#define SRK_F64_TWO52 4503599627370496.0  // 2^52

__device__ __forceinline__ double f64_of_u64(uint64_t v) {  // v < 2^52
    return __longlong_as_double((long long)(v | 0x4330000000000000ull)) - SRK_F64_TWO52;
}
__device__ __forceinline__ uint64_t u64_of_f64(double d) {  // 0 <= d < 2^52, integral
    return (uint64_t)__double_as_longlong(d + SRK_F64_TWO52) & 0xFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double modmul_f64(double y, double w, double q, double qinv) {
    const double hi = y * w;
    const double lo = fma(y, w, -hi);
    const double t = fma(hi, qinv, SRK_F64_MAGIC) - SRK_F64_MAGIC;
    return fma(-t, q, hi) + lo;
}
// centred representative in [-q/2, q/2] of an integer-valued |v| < 2^51
__device__ __forceinline__ double centre_f64(double v, double q, double qinv) {
    const double t = fma(v, qinv, SRK_F64_MAGIC) - SRK_F64_MAGIC;
    return fma(-t, q, v);
}
// signed integer of an integer-valued double |r| < 2^51: r + 1.5*2^52 keeps
// exponent 52, so its bit pattern is 0x4338000000000000 + r (one DADD + IADD)
__device__ __forceinline__ long long i64_of_f64(double r) {
    return __double_as_longlong(r + SRK_F64_MAGIC) - 0x4338000000000000ll;
}
// canonical [0, q) of an integer-valued double already in (-q, q)
__device__ __forceinline__ uint64_t canon_u64_of_small_f64(double r, uint64_t q) {
    const long long i = i64_of_f64(r);
    return (uint64_t)(i < 0 ? i + (long long)q : i);
}
__device__ __forceinline__ uint64_t canon_u64_of_f64(double v, double q, double qinv) {
    // centred r in [-q/2, q/2] (|r| < q with rounding slack); sign fix-up on the integer pipes
    const long long i = i64_of_f64(centre_f64(v, q, qinv));
    return (uint64_t)(i < 0 ? i + (long long)q : i);
}
__device__ __forceinline__ void ct_bfly_f64(uint64_t &xb, uint64_t &yb, double w, double q,
                                            double qinv) {
    const double x = __longlong_as_double((long long)xb), y = __longlong_as_double((long long)yb);
    const double t = modmul_f64(y, w, q, qinv);
    xb = (uint64_t)__double_as_longlong(x + t);
    yb = (uint64_t)__double_as_longlong(x - t);
}
__device__ __forceinline__ void gs_bfly_f64(uint64_t &xb, uint64_t &yb, double w, double q,
                                            double qinv) {
    const double x = __longlong_as_double((long long)xb), y = __longlong_as_double((long long)yb);
    xb = (uint64_t)__double_as_longlong(x + y);
    yb = (uint64_t)__double_as_longlong(modmul_f64(x - y, w, q, qinv));
}

// Register-resident radix-2 stages, unrolled at compile time through
// template recursion so x[] never spills to local memory.
//   tw_group(g) -> twiddle for butterfly group g of the stage;
//   group g covers x[g*2*HALF .. g*2*HALF + 2*HALF), pairs (e, e + HALF).
// SM: 0 = Harvey lazy (any prime < 2^62), 1 = reduction-free integer (q < 2^46),
// 2 = FP64 (q < 2^41); m = inverse difference offset (q << step) for SM 1
struct F64Q {
    double q, qinv;
};
struct TwPtr {
    const ulonglong2 *w;  // {w, Shoup(w)} (integer modes)
    const double *wd;     // w as double (FP64 mode)
};
template <int E, int HALF, int NG, bool GS, int SM, typename TwFn>
__device__ __forceinline__ void reg_stage(uint64_t (&x)[E], TwPtr tp, TwFn tw_idx, uint64_t q,
                                          uint64_t two_q, uint64_t m, F64Q fq) {
#pragma unroll
    for (int g = 0; g < NG; g++) {
        ulonglong2 w = {0, 0};
        double wf = 0.0;
        if constexpr (SM == 2)
            wf = __ldg(tp.wd + tw_idx(g));
        else
            w = __ldg(tp.w + tw_idx(g));
#pragma unroll
        for (int k = 0; k < HALF; k++) {
            uint64_t &a = x[g * 2 * HALF + k];
            uint64_t &b = x[g * 2 * HALF + k + HALF];
            if (GS) {
                if (SM == 2)
                    gs_bfly_f64(a, b, wf, fq.q, fq.qinv);
                else if (SM == 1)
                    gs_bfly_small(a, b, w.x, w.y, q, m);
                else
                    gs_bfly(a, b, w.x, w.y, q, two_q);
            } else {
                if (SM == 2)
                    ct_bfly_f64(a, b, wf, fq.q, fq.qinv);
                else if (SM == 1)
                    ct_bfly_small(a, b, w.x, w.y, q, two_q);
                else
                    ct_bfly(a, b, w.x, w.y, q, two_q);
            }
        }
    }
}

// forward round 1: stages s = 0..LE1-1, half = E >> (s+1), 2^s groups,
// twiddle (base << s) + g
template <int E, int LE1, int SM, int S = 0>
struct FwdR1 {
    static __device__ __forceinline__ void run(uint64_t (&x)[E], TwPtr tw, int base,
                                               uint64_t q, uint64_t two_q, F64Q fq = {}) {
        if constexpr (S < LE1) {
            reg_stage<E, (E >> (S + 1)), (1 << S), false, SM>(
                x, tw, [&](int g) { return (base << S) + g; }, q, two_q, 0, fq);
            FwdR1<E, LE1, SM, S + 1>::run(x, tw, base, q, two_q, fq);
        }
    }
};
// forward round 2: stages LE1+s, half = TPS >> (s+1), ng = E/(2 half),
// twiddle (base << (LE1+s)) + u ng + g
template <int E, int TPS, int LE1, int LE2, int SM, int S = 0>
struct FwdR2 {
    static __device__ __forceinline__ void run(uint64_t (&x)[E], TwPtr tw, int base,
                                               int u, uint64_t q, uint64_t two_q, F64Q fq = {}) {
        if constexpr (S < LE2) {
            constexpr int half = TPS >> (S + 1), ng = E / (2 * half);
            reg_stage<E, half, ng, false, SM>(
                x, tw, [&](int g) { return (base << (LE1 + S)) + u * ng + g; }, q, two_q, 0,
                fq);
            FwdR2<E, TPS, LE1, LE2, SM, S + 1>::run(x, tw, base, u, q, two_q, fq);
        }
    }
};
// inverse round 1: register stride half = 2^s, stage LOG_T-1-s, ng = E/(2 half),
// twiddle (base << stage) + u ng + g
template <int E, int LOG_T, int LE1, int SM, int S = 0>
struct InvR1 {
    static __device__ __forceinline__ void run(uint64_t (&x)[E], TwPtr tw, int base,
                                               int u, uint64_t q, uint64_t two_q, int k0,
                                               F64Q fq = {}) {
        if constexpr (S < LE1) {
            constexpr int half = 1 << S, ng = E / (2 * half), stage = LOG_T - 1 - S;
            reg_stage<E, half, ng, true, SM>(
                x, tw, [&](int g) { return (base << stage) + u * ng + g; }, q, two_q,
                q << (k0 + S), fq);
            InvR1<E, LOG_T, LE1, SM, S + 1>::run(x, tw, base, u, q, two_q, k0, fq);
        }
    }
};
// inverse round 2: register stride half = (E/TPS) << s, stage LE2-1-s,
// 2^stage groups, twiddle (base << stage) + g
template <int E, int TPS, int LE2, int SM, int S = 0>
struct InvR2 {
    static __device__ __forceinline__ void run(uint64_t (&x)[E], TwPtr tw, int base,
                                               uint64_t q, uint64_t two_q, int k0, F64Q fq = {}) {
        if constexpr (S < LE2) {
            constexpr int half = (E / TPS) << S, stage = LE2 - 1 - S;
            reg_stage<E, half, (1 << stage), true, SM>(
                x, tw, [&](int g) { return (base << stage) + g; }, q, two_q,
                q << (k0 + S), fq);
            InvR2<E, TPS, LE2, SM, S + 1>::run(x, tw, base, q, two_q, k0, fq);
        }
    }
};

// first-pass element load (coefficient / evaluation index n of limb slot t)
template <int LD>
__device__ __forceinline__ uint64_t fused_load(const FuseArgs &f, const PrimeConst *pcs, int bi,
                                               int r, int t, const PrimeConst &P, long long n,
                                               int log_n, const uint64_t *plain_src) {
    if constexpr (LD == LD_PLAIN) {
        return plain_src[n];
    } else if constexpr (LD == LD_AUTO) {
        return __ldg(plain_src + auto_index((uint32_t)n, f.galois, log_n));
    } else if constexpr (LD == LD_SPREAD) {
        const uint64_t v = f.src[bi * f.src_ct + r * f.src_ps + n];
        // centred representative of v mod top_q, reduced mod this prime
        return v > (f.top_q >> 1) ? sub_mod(reduce64(v, P), reduce64(f.top_q, P), P.q)
                                  : reduce64(v, P);
    } else {  // ModDown conversion: handled by bconv_load (per-thread hoisted constants)
        return 0;
    }
}

// ModDown conversion with exact rounding (v precomputed once per coefficient):
//   sum_k z_k[n] * mat[k][t] - corr[v(n)][t]   mod q_t
// mat column / corr table for this limb are hoisted into registers by the caller.
template <int MAXK>
__device__ __forceinline__ uint64_t bconv_load(const FuseArgs &f, const uint64_t *z,
                                               const uint8_t *vr, const uint64_t (&m)[MAXK],
                                               const PrimeConst &P, long long n, int log_n, int t) {
    const long long nn = 1ll << log_n;
    U128 acc = {0, 0};
#pragma unroll
    for (int k = 0; k < MAXK; k++)
        if (k < f.n_src) mac(acc, z[k * nn + n], m[k]);
    const int v = vr[n];
    return sub_mod(reduce_u128(acc, P), __ldg(f.corr + v * f.corr_ld + t), P.q);
}

// last-pass element store; x canonical in [0, q)
template <int ST>
__device__ __forceinline__ void fused_store(const FuseArgs &f, int bi, int r, int t, int limb,
                                            const PrimeConst &P, long long n, int log_n,
                                            uint64_t x, uint64_t *plain_dst) {
    if constexpr (ST == ST_PLAIN || ST == ST_SCALE) {
        plain_dst[n] = x;
    } else {
        const long long nn = 1ll << log_n;
        const long long off = (long long)t * nn + n;
        const long long aoff = (ST == ST_MODDOWN && f.acc_galois != 1)
                                   ? (long long)t * nn + auto_index((uint32_t)n, f.acc_galois, log_n)
                                   : off;
        uint64_t a = f.acc[bi * f.acc_ct + r * f.acc_ps + aoff];
        uint64_t v;
        if constexpr (ST == ST_RESCALE) {
            if (f.pre_mode == 1) a = mul_shoup(a, f.pre.w[limb], f.pre.ws[limb], P.q);
            if (f.pre_mode == 2) a = mul_mod(a, __ldg(f.pt + bi * f.pt_ct + off), P);
            v = mul_shoup(sub_mod(a, x, P.q), f.mulc.w[limb], f.mulc.ws[limb], P.q);
        } else {
            v = mul_shoup(sub_mod(a, x, P.q), f.mulc.w[limb], f.mulc.ws[limb], P.q);
            const uint64_t *ad = r == 0 ? f.add0 : f.add1;
            if (ad) {
                const uint64_t *base = ad + bi * f.add_ct + (long long)t * nn;
                const long long src = (r == 0 && f.add_galois != 1)
                                          ? (long long)auto_index((uint32_t)n, f.add_galois, log_n)
                                          : n;
                uint64_t av = base[src];
                if (f.add_scaled) av = mul_shoup(av, f.addc.w[limb], f.addc.ws[limb], P.q);
                v = add_mod(v, av, P.q);
            }
        }
        f.out[bi * f.out_ct + r * f.out_ps + off] = v;
    }
}

// Final phase of a forward row pass whose canonical results sit in smem
// (sidx layout).  Plain/fused stores write each element in place; with
// ST_MODDOWN and out_galois != 1 the combined values are first written back
// to smem, then every row (chunk) is emitted permuted:
//   out[m] = w[pi(m)],  pi = X -> X^out_galois on NTT slots,
// which maps chunk sub to chunk d = pi^-1(sub*T) / T as a whole, so both the
// reads (acc, add) and the writes stay coalesced.
template <int LOG_T, int ST, typename SIdx>
__device__ __forceinline__ void row_final_store(const FuseArgs &f, uint64_t *sm, SIdx sidx, int bi,
                                                int r, int t, int limb, const PrimeConst &pc,
                                                int sub, int u, int log_n, uint64_t *data) {
    using S = NttShape<LOG_T>;
    constexpr int T = S::T, E = S::E, TPS = S::TPS;
    if constexpr (ST == ST_MODDOWN) {
        if (f.out_galois != 1) {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const int c = u + TPS * e;
                const long long n = (long long)sub * T + c;
                const long long nn = 1ll << log_n;
                const long long off = (long long)t * nn + n;
                uint64_t v = mul_shoup(sub_mod(f.acc[bi * f.acc_ct + r * f.acc_ps + off], sm[sidx(c)], pc.q),
                                       f.mulc.w[limb], f.mulc.ws[limb], pc.q);
                const uint64_t *ad = r == 0 ? f.add0 : f.add1;
                if (ad) {
                    uint64_t av = ad[bi * f.add_ct + off];
                    if (f.add_scaled) av = mul_shoup(av, f.addc.w[limb], f.addc.ws[limb], pc.q);
                    v = add_mod(v, av, pc.q);
                }
                sm[sidx(c)] = v;
            }
            __syncthreads();
            const long long nn = 1ll << log_n;
            const int d = (int)(auto_index((uint32_t)((long long)sub * T), f.out_galois_inv, log_n) >> LOG_T);
            uint64_t *o = f.out + bi * f.out_ct + r * f.out_ps + (long long)t * nn + (long long)d * T;
#pragma unroll
            for (int e = 0; e < E; e++) {
                const int c = u + TPS * e;
                const int p = (int)(auto_index((uint32_t)((long long)d * T + c), f.out_galois, log_n) -
                                    (uint32_t)sub * T);
                o[c] = sm[sidx(p)];
            }
            return;
        }
    }
    if constexpr (ST == ST_RESCALE) {
        // integer rescale combine with every load issued before the first store
        // (the out pointer may alias acc / pt as far as the compiler knows)
        const long long nn = 1ll << log_n;
        const long long off0 = (long long)t * nn + (long long)sub * T + u;
        uint64_t av[E], pv[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            av[e] = __ldg(f.acc + bi * f.acc_ct + r * f.acc_ps + off0 + TPS * e);
            pv[e] = f.pre_mode == 2 ? __ldg(f.pt + bi * f.pt_ct + off0 + TPS * e) : 0;
        }
#pragma unroll
        for (int e = 0; e < E; e++) {
            uint64_t a = av[e];
            if (f.pre_mode == 1) a = mul_shoup(a, f.pre.w[limb], f.pre.ws[limb], pc.q);
            if (f.pre_mode == 2) a = mul_mod(a, pv[e], pc);
            f.out[bi * f.out_ct + r * f.out_ps + off0 + TPS * e] =
                mul_shoup(sub_mod(a, sm[sidx(u + TPS * e)], pc.q), f.mulc.w[limb], f.mulc.ws[limb], pc.q);
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int c = u + TPS * e;
        fused_store<ST>(f, bi, r, t, limb, pc, (long long)sub * T + c, log_n, sm[sidx(c)], data);
    }
}

// One pass of the NTT.  COL = column pass (sub-transforms strided by C),
// else row pass (contiguous chunks).  Grid: x = sub-transform groups of
// one limb, y = (limb, poly) of the batch (poly fastest, so one prime's
// twiddles are reused across consecutive CTAs).  Butterflies sharing a
// twiddle are grouped so each distinct twiddle is one 16-byte load.
// IO selects the fused load of the FIRST pass (forward: column pass,
// inverse: row pass) or the fused store of the LAST pass (forward: row pass,
// inverse: column pass); the intermediate always lives at the batch's own
// limb storage (b.ptr).
// KM 1: every limb of the launch is under a prime < 2^41, so only the FP64
// arithmetic mode is compiled in (no integer-mode code, no register spills).
// LOGN: compile-time log2 ring degree (0 = runtime log_n_arg), so the strided
// element addresses of the 2^16 passes fold into immediate offsets.
// Grid: x = sub-transform groups, y = poly, z = limb.
#ifndef SRK_NTT_MINB_F64
#define SRK_NTT_MINB_F64 3
#endif
#ifndef SRK_NTT_MINB_INT
#define SRK_NTT_MINB_INT 3
#endif
// KM: 0 = arithmetic mode chosen per limb at run time (fused-IO variants),
//     1 = FP64 only (limbs under q < 2^41; others skipped),
//     2 = Harvey lazy integer only (any q < 2^62; with cls 2 the FP64 limbs are skipped)
template <int LOG_T, bool INV, bool COL, int IO, int KM = 0, int LOGN = 0>
__global__ void __launch_bounds__(256, KM == 1 ? SRK_NTT_MINB_F64 : (KM == 2 ? SRK_NTT_MINB_INT : SRK_NTT_MINB))
    ntt_pass_kernel(LimbBatch b, NttTables tb, int log_n_arg, const __grid_constant__ FuseArgs f) {
    const int log_n = LOGN ? LOGN : log_n_arg;
    using S = NttShape<LOG_T>;
    constexpr int T = S::T, E = S::E, TPS = S::TPS, LE1 = S::LE1, LE2 = S::LE2;
    constexpr bool FIRST = (COL != INV);  // forward column / inverse row pass
    constexpr int LD = FIRST ? IO : LD_PLAIN;
    constexpr int ST = FIRST ? ST_PLAIN : IO;
    extern __shared__ uint64_t smem[];

    const int n = 1 << log_n;
    const int CB = blockDim.x / TPS;  // sub-transforms per CTA
    const int limb = blockIdx.z, poly = blockIdx.y;
    const int bi = b.ppc == 2 ? poly >> 1 : (b.ppc == 1 ? poly : poly / b.ppc);
    const int r = poly - bi * b.ppc;
    int t, pid;
    if (!limb_map(b, r, limb, t, pid)) return;
    uint64_t *data =
        b.ptr + (long long)bi * b.ct_stride + (long long)r * b.poly_stride + (long long)t * n;
    const PrimeConst pc = tb.pc[pid];
    const uint64_t q = pc.q, two_q = pc.two_q;
    // prime-class split of mixed batches (uniform per CTA): the FP64 kernel never
    // touches a limb >= 2^41; the integer kernel skips FP64 limbs when filtered
    if ((KM == 1 || b.cls == 1) ? q >= SRK_F64_Q : (b.cls == 2 && q < SRK_F64_Q)) return;
    const bool small = q < SRK_SMALL_Q;  // uniform per CTA (one limb per CTA)
    const TwPtr tw = {(INV ? tb.itw : tb.tw) + (long long)pid * n, (INV ? tb.itwd : tb.twd) + (long long)pid * n};
    const uint64_t *lsrc = data;  // LD_PLAIN / LD_AUTO source limb
    if constexpr (FIRST && (LD == LD_PLAIN || LD == LD_AUTO)) {
        if (f.src) lsrc = f.src + (long long)bi * f.src_ct + (long long)r * f.src_ps + (long long)t * n;
    }

    const int tid = threadIdx.x;
    int sb, u;  // local sub-transform and thread-within-sub-transform
    if (COL) {
        sb = tid % CB;
        u = tid / CB;
    } else {
        sb = tid / TPS;
        u = tid % TPS;
    }
    const int sub = blockIdx.x * CB + sb;  // column index (COL) or chunk index
    const int C = n >> LOG_T;               // COL: #columns ; ROW: #rows (chunks)
    auto gaddr = [&](int c) -> long long {
        return COL ? (long long)c * C + sub : (long long)sub * T + c;
    };
    const int base = COL ? 1 : (C + sub);
    auto sidx = [&](int c) -> int {
        return COL ? c * CB + sb : row_sidx<LOG_T>(sb, c);
    };
    constexpr int MAXK = bconv_maxk(LD);
    uint64_t bm[MAXK];
    const uint64_t *bz = nullptr;
    const uint8_t *bvr = nullptr;
    if constexpr (FIRST && is_bconv(LD)) {
#pragma unroll
        for (int k = 0; k < MAXK; k++)
            bm[k] = k < f.n_src ? __ldg(f.mat + (long long)k * f.mat_ld + t) : 0;
        bz = f.src + (long long)bi * f.src_ct + (long long)r * f.src_ps;
        bvr = f.vround + ((long long)bi * 2 + r) * n;
    }
    auto load = [&](int c) -> uint64_t {
        if constexpr (FIRST && is_bconv(LD)) return bconv_load<MAXK>(f, bz, bvr, bm, pc, gaddr(c), log_n, t);
        else if constexpr (FIRST) return fused_load<LD>(f, tb.pc, bi, r, t, pc, gaddr(c), log_n, lsrc);
        else return data[gaddr(c)];
    };

    // arithmetic mode, uniform per CTA: 2 = FP64 (q < 2^41), 1 = reduction-free
    // integer (q < 2^46), 0 = Harvey lazy integer
    const int mode = KM == 1 ? 2 : (KM == 2 ? 0 : (q < SRK_F64_Q ? 2 : (small ? 1 : 0)));
    // (double) q and 1 / (double) q precomputed per prime (no per-CTA division)
    const F64Q fq = {__longlong_as_double((long long)pc.qd_bits), __longlong_as_double((long long)pc.qinv_bits)};
    // first-pass loads are canonical u64; FP64 limbs convert on load
    auto load_m = [&](int c) -> uint64_t {
        if constexpr (FIRST && LD == LD_SPREAD && KM == 1) {
            // rescale spread on the FP64 path: the centred top-limb value is already a
            // valid FP64-mode operand for every target prime (|v| < 2^61 would not be:
            // the top prime is a scaling prime < 2^41 whenever this kernel runs)
            const long long v = (long long)f.src[bi * f.src_ct + r * f.src_ps + gaddr(c)];
            const long long vc = v > (long long)(f.top_q >> 1) ? v - (long long)f.top_q : v;
            return (uint64_t)__double_as_longlong((double)vc);
        }
        const uint64_t v = load(c);
        return mode == 2 ? (uint64_t)__double_as_longlong(f64_of_u64(v)) : v;
    };
    uint64_t x[E];
    if (!INV) {
        // ---- round 1: strided ownership c = u + TPS e, strides T/2 .. TPS
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = FIRST ? load_m(u + TPS * e) : data[gaddr(u + TPS * e)];
        if (mode == 2)
            FwdR1<E, LE1, 2>::run(x, tw, base, q, two_q, fq);
        else if (mode == 1)
            FwdR1<E, LE1, 1>::run(x, tw, base, q, two_q);
        else
            FwdR1<E, LE1, 0>::run(x, tw, base, q, two_q);
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = x[e];
        __syncthreads();
        // ---- round 2: contiguous ownership c = u E + e, strides TPS/2 .. 1
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
        if (mode == 2)
            FwdR2<E, TPS, LE1, LE2, 2>::run(x, tw, base, u, q, two_q, fq);
        else if (mode == 1)
            FwdR2<E, TPS, LE1, LE2, 1>::run(x, tw, base, u, q, two_q);
        else
            FwdR2<E, TPS, LE1, LE2, 0>::run(x, tw, base, u, q, two_q);
        if (COL) {
#pragma unroll
            for (int e = 0; e < E; e++) data[gaddr(u * E + e)] = x[e];  // lazy / FP64 bits
        } else {
            if constexpr (ST == ST_RESCALE && KM == 1) {
                // FP64 rescale combine: out = ((acc * pre) - x) * q_l^-1 with the raw
                // FP64 transform output x (|x| < 17 q, no canonicalisation first)
                __syncthreads();
#pragma unroll
                for (int e = 0; e < E; e++) smem[sidx(u * E + e)] = x[e];
                __syncthreads();
                const long long nn = 1ll << log_n;
                const double fm = f64_of_u64(f.mulc.w[limb]);
                const double fp = f64_of_u64(f.pre.w[limb]);
                const long long off0 = (long long)t * nn + (long long)sub * T + u;
                // all loads first: the stores below may alias them as far as the
                // compiler knows, which otherwise serialises load -> store per element
                uint64_t av[E], pv[E];
#pragma unroll
                for (int e = 0; e < E; e++) {
                    av[e] = __ldg(f.acc + bi * f.acc_ct + r * f.acc_ps + off0 + TPS * e);
                    pv[e] = f.pre_mode == 2 ? __ldg(f.pt + bi * f.pt_ct + off0 + TPS * e) : 0;
                }
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int c = u + TPS * e;
                    double a = f64_of_u64(av[e]);
                    if (f.pre_mode == 1) a = modmul_f64(a, fp, fq.q, fq.qinv);
                    if (f.pre_mode == 2) a = modmul_f64(a, f64_of_u64(pv[e]), fq.q, fq.qinv);
                    const double d = a - __longlong_as_double((long long)smem[sidx(c)]);
                    f.out[bi * f.out_ct + r * f.out_ps + off0 + TPS * e] =
                        canon_u64_of_small_f64(modmul_f64(d, fm, fq.q, fq.qinv), q);
                }
                return;
            }
            // final pass: each thread owns 16 contiguous outputs; a shared-memory
            // transpose gives fully coalesced 8-byte stores (16-byte vector stores
            // straight from registers were slower: DESIGN.md)
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) {
                uint64_t v = x[e];
                if (mode == 2) {
                    v = canon_u64_of_f64(__longlong_as_double((long long)v), fq.q, fq.qinv);
                } else {
                    if (mode == 1) {  // v < 34 q: one Barrett step (floor(2^64/q)) then one subtraction
                        v -= mulhi64(v, pc.ratio_hi) * q;
                    } else {
                        v = v >= two_q ? v - two_q : v;
                    }
                    v = v >= q ? v - q : v;
                }
                smem[sidx(u * E + e)] = v;
            }
            __syncthreads();
            row_final_store<LOG_T, ST>(f, smem, sidx, bi, r, t, limb, pc, sub, u, log_n, data);
        }
    } else {
        // ---- round 1: contiguous ownership, strides 1 .. E/2
        if (COL) {
            // second pass: FP64 sums doubled every stage of the first -> re-centre
#pragma unroll
            for (int e = 0; e < E; e++) {
                uint64_t v = data[gaddr(u * E + e)];
                if (mode == 2)
                    v = (uint64_t)__double_as_longlong(
                        centre_f64(__longlong_as_double((long long)v), fq.q, fq.qinv));
                x[e] = v;
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = load_m(u + TPS * e);
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
        }
        // step numbers of the inverse: row pass 0.., column pass log_n - LOG_T ..
        const int k0 = COL ? log_n - LOG_T : 0;
        if (mode == 2)
            InvR1<E, LOG_T, LE1, 2>::run(x, tw, base, u, q, two_q, k0, fq);
        else if (mode == 1)
            InvR1<E, LOG_T, LE1, 1>::run(x, tw, base, u, q, two_q, k0);
        else
            InvR1<E, LOG_T, LE1, 0>::run(x, tw, base, u, q, two_q, k0);
        if (!COL) __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u * E + e)] = x[e];
        __syncthreads();
        // ---- round 2: strided ownership c = u + TPS e, strides E .. T/2
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u + TPS * e)];
        if (mode == 2)
            InvR2<E, TPS, LE2, 2>::run(x, tw, base, q, two_q, k0 + LE1, fq);
        else if (mode == 1)
            InvR2<E, TPS, LE2, 1>::run(x, tw, base, q, two_q, k0 + LE1);
        else
            InvR2<E, TPS, LE2, 0>::run(x, tw, base, q, two_q, k0 + LE1);
        if (COL) {
            // last pass of the inverse: * N^-1 (or the fused per-limb scale), canonical
            uint64_t m = pc.ninv, ms = pc.ninv_shoup;
            if constexpr (ST == ST_SCALE) {
                m = f.mulc.w[limb];
                ms = f.mulc.ws[limb];
            }
            if (mode == 2) {
                const double mf = f64_of_u64(m);
#pragma unroll
                for (int e = 0; e < E; e++)  // modmul_f64 output is already in (-q, q)
                    data[gaddr(u + TPS * e)] = canon_u64_of_small_f64(
                        modmul_f64(__longlong_as_double((long long)x[e]), mf, fq.q, fq.qinv), q);
            } else {
#pragma unroll
                for (int e = 0; e < E; e++) data[gaddr(u + TPS * e)] = mul_shoup(x[e], m, ms, q);
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) data[gaddr(u + TPS * e)] = x[e];  // lazy / FP64 bits
        }
    }
}
