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
enum { LD_PLAIN = 0, LD_SPREAD = 2, LD_AUTO = 3 };
enum { ST_PLAIN = 0, ST_KSC = 1, ST_RESCALE = 2, ST_SCALE = 3 };

struct FuseArgs {
    // loads: source poly (b, r) at src + b*src_ct + r*src_ps (+ slot t * N for
    // LD_PLAIN / LD_AUTO; LD_SPREAD reads one limb)
    const uint64_t *src;
    long long src_ct, src_ps;
    uint64_t galois;         // LD_AUTO: X -> X^galois gather
    uint64_t top_q;          // LD_SPREAD: modulus of the limb being spread
    // stores: out(b, r, t) from the transform result x and
    //   ST_KSC    : sigma_{out_galois}(add_r + (sum_j e_j key_j - x) * mulc)   (key switch)
    //   ST_RESCALE: (acc * pre - x) * mulc            (pre: const pre_k or plaintext pt)
    //   ST_SCALE  : x * mulc   (replaces N^-1 in the inverse transform)
    uint64_t *out;
    long long out_ct, out_ps;
    const uint64_t *acc;
    long long acc_ct, acc_ps;
    // ST_KSC addends (c0 of a rotation, d0 / d1 of a product): valid pointers always
    // (a dummy when has_add* is 0, so no load can ever be speculated from null)
    const uint64_t *add0, *add1;
    long long add_ct;
    int has_add0, has_add1;
    uint64_t out_galois;     // ST_KSC: write sigma_{out_galois}(result) (1 = identity);
    uint64_t out_galois_inv; //   rows of T elements map to rows, staged through smem
    // ST_KSC inner product sum_j e_j key_j over the ciphertext-modulus limbs:
    // e_j = the key-switched poly d itself for the digit holding the limb, else
    // the ModUp digit ext[j]; key[j][r] in device layout (rotation-permuted)
    const uint64_t *ks_d;
    long long ks_d_ct;
    const uint64_t *ks_ext;
    long long ks_ext_ct, ks_ext_dig;
    const uint64_t *ks_key;
    long long ks_key_j, ks_key_r;  // key strides: digit, poly (words)
    int ks_alpha, ks_beta;
    int pre_mode;            // 0 none, 1 per-limb constant, 2 plaintext
    const uint64_t *pt;      // [limbs][N] per ciphertext at stride pt_ct (0 = shared); never
    long long pt_ct;         //   null (points at acc when pre_mode != 2)
    LimbConsts mulc;
    LimbConsts pre;
    LimbConsts addc;         // ST_KSC: add_r scaled by addc (when add_scaled)
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
// SM: 0 = Harvey lazy (any prime < 2^62), 2 = FP64 (q < 2^41)
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
                if constexpr (SM == 2)
                    gs_bfly_f64(a, b, wf, fq.q, fq.qinv);
                else
                    gs_bfly(a, b, w.x, w.y, q, two_q);
            } else {
                if constexpr (SM == 2)
                    ct_bfly_f64(a, b, wf, fq.q, fq.qinv);
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
    }
}

// last-pass element store (ST_PLAIN / ST_SCALE); x canonical in [0, q)
template <int ST>
__device__ __forceinline__ void fused_store(const FuseArgs &f, int bi, int r, int t, int limb,
                                            const PrimeConst &P, long long n, int log_n,
                                            uint64_t x, uint64_t *plain_dst) {
    static_assert(ST == ST_PLAIN || ST == ST_SCALE, "other stores run in row_final_store");
    plain_dst[n] = x;
}

#define SRK_KSC_G 8  // elements per digit step of the ST_KSC epilogue (2G loads in flight)

// ST_KSC epilogue of the forward row pass (the ModDown NTT of a key switch):
// the ciphertext-modulus limbs' key-switch inner product and the ModDown combine
//     v = (sum_j e_j[n] key_j[r][t][n] - x[n]) * mulc[t]  +  add_r[n] (* addc[t])
// at every element n = sub*T + c of this thread's strided slots c = u + TPS e, in
// place in smem (sidx layout).  x[n] is the transform output: raw FP64 bits
// (|x| < 17 q) in FP64 mode, canonical in integer mode.  Elements are processed
// in groups of G so that 2G independent digit / key loads are in flight per
// digit step (the loads are L2/HBM-latency bound otherwise).
template <int LOG_T, int KM, typename SIdx>
__device__ __forceinline__ void ksc_epilogue(const FuseArgs &f, uint64_t *sm, SIdx sidx, int bi, int r,
                                             int t, int pid, int limb, const PrimeConst &pc, F64Q fq,
                                             int sub, int u, int log_n) {
    using S = NttShape<LOG_T>;
    constexpr int T = S::T, E = S::E, TPS = S::TPS;
    constexpr int G = E < SRK_KSC_G ? E : SRK_KSC_G;
    const long long nn = 1ll << log_n;
    const long long off0 = (long long)t * nn + (long long)sub * T + u;  // element e at + TPS e
    const int jt = pid / f.ks_alpha;  // the digit that holds this limb
    const uint64_t *dsrc = f.ks_d + bi * f.ks_d_ct + off0;
    const uint64_t *esrc = f.ks_ext + bi * f.ks_ext_ct + off0;
    const uint64_t *ksrc = f.ks_key + r * f.ks_key_r + off0;
    const int has_add = r == 0 ? f.has_add0 : f.has_add1;
    const uint64_t *asrc = (r == 0 ? f.add0 : f.add1) + bi * f.add_ct + off0;
#pragma unroll
    for (int g0 = 0; g0 < E; g0 += G) {
        if constexpr (KM == 1) {
            double s[G];
#pragma unroll
            for (int e = 0; e < G; e++) s[e] = -__longlong_as_double((long long)sm[sidx(u + TPS * (g0 + e))]);
            for (int j = 0; j < f.ks_beta; j++) {
                const uint64_t *ej = (j == jt ? dsrc : esrc + j * f.ks_ext_dig) + TPS * g0;
                const uint64_t *kj = ksrc + j * f.ks_key_j + TPS * g0;
                uint64_t ev[G], kv[G];
#pragma unroll
                for (int e = 0; e < G; e++) {
                    ev[e] = __ldg(ej + TPS * e);
                    kv[e] = __ldg(kj + TPS * e);
                }
#pragma unroll
                for (int e = 0; e < G; e++)
                    s[e] += modmul_f64(f64_of_u64(ev[e]), f64_of_u64(kv[e]), fq.q, fq.qinv);
            }
            const double wf = f64_of_u64(f.mulc.w[limb]);
            uint64_t av[G];
#pragma unroll
            for (int e = 0; e < G; e++) av[e] = has_add ? __ldg(asrc + TPS * (g0 + e)) : 0;
            const double af = f.add_scaled ? f64_of_u64(f.addc.w[limb]) : 1.0;
#pragma unroll
            for (int e = 0; e < G; e++) {
                double v = modmul_f64(s[e], wf, fq.q, fq.qinv);
                double a = f64_of_u64(av[e]);
                if (f.add_scaled) a = modmul_f64(a, af, fq.q, fq.qinv);
                sm[sidx(u + TPS * (g0 + e))] = canon_u64_of_f64(v + a, fq.q, fq.qinv);
            }
        } else {
            // integer limbs (q >= 2^41): 128-bit accumulation, one Barrett reduction
            // per 16 products (products < 2^124)
            U128 s[G];
#pragma unroll
            for (int e = 0; e < G; e++) s[e] = {0, 0};
            for (int j = 0; j < f.ks_beta; j++) {
                const uint64_t *ej = (j == jt ? dsrc : esrc + j * f.ks_ext_dig) + TPS * g0;
                const uint64_t *kj = ksrc + j * f.ks_key_j + TPS * g0;
                uint64_t ev[G], kv[G];
#pragma unroll
                for (int e = 0; e < G; e++) {
                    ev[e] = __ldg(ej + TPS * e);
                    kv[e] = __ldg(kj + TPS * e);
                }
#pragma unroll
                for (int e = 0; e < G; e++) mac(s[e], ev[e], kv[e]);
                if ((j & 15) == 15) {
#pragma unroll
                    for (int e = 0; e < G; e++) s[e] = {0, reduce_u128(s[e], pc)};
                }
            }
            uint64_t av[G];
#pragma unroll
            for (int e = 0; e < G; e++) av[e] = has_add ? __ldg(asrc + TPS * (g0 + e)) : 0;
#pragma unroll
            for (int e = 0; e < G; e++) {
                const int c = u + TPS * (g0 + e);
                uint64_t v = mul_shoup(sub_mod(reduce_u128(s[e], pc), sm[sidx(c)], pc.q), f.mulc.w[limb],
                                       f.mulc.ws[limb], pc.q);
                uint64_t a = av[e];
                if (f.add_scaled) a = mul_shoup(a, f.addc.w[limb], f.addc.ws[limb], pc.q);
                sm[sidx(c)] = add_mod(v, a, pc.q);
            }
        }
    }
}

// Final phase of a forward row pass whose results sit in smem (sidx layout).
// Plain stores write each element in place.  ST_KSC combines in place
// (ksc_epilogue) and, with out_galois != 1, then emits every row (chunk)
// permuted:  out[m] = w[pi(m)],  pi = X -> X^out_galois on NTT slots, which maps
// chunk sub to chunk d = pi^-1(sub*T) / T as a whole, so both the reads (digits,
// keys, addends) and the writes stay coalesced.
template <int LOG_T, int ST, int KM, typename SIdx>
__device__ __forceinline__ void row_final_store(const FuseArgs &f, uint64_t *sm, SIdx sidx, int bi,
                                                int r, int t, int pid, int limb, const PrimeConst &pc,
                                                F64Q fq, int sub, int u, int log_n, uint64_t *data) {
    using S = NttShape<LOG_T>;
    constexpr int T = S::T, E = S::E, TPS = S::TPS;
    if constexpr (ST == ST_KSC) {
        ksc_epilogue<LOG_T, KM>(f, sm, sidx, bi, r, t, pid, limb, pc, fq, sub, u, log_n);
        const long long nn = 1ll << log_n;
        if (f.out_galois != 1) {
            __syncthreads();
            const int d = (int)(auto_index((uint32_t)((long long)sub * T), f.out_galois_inv, log_n) >> LOG_T);
            uint64_t *o = f.out + bi * f.out_ct + r * f.out_ps + (long long)t * nn + (long long)d * T;
#pragma unroll
            for (int e = 0; e < E; e++) {
                const int c = u + TPS * e;
                const int p = (int)(auto_index((uint32_t)((long long)d * T + c), f.out_galois, log_n) -
                                    (uint32_t)sub * T);
                o[c] = sm[sidx(p)];
            }
        } else {
            uint64_t *o = f.out + bi * f.out_ct + r * f.out_ps + (long long)t * nn + (long long)sub * T;
#pragma unroll
            for (int e = 0; e < E; e++) o[u + TPS * e] = sm[sidx(u + TPS * e)];
        }
        return;
    }
    if constexpr (ST == ST_RESCALE) {
        // integer rescale combine with every load issued before the first store
        // (the out pointer may alias acc / pt as far as the compiler knows);
        // f.pt is never null (host points it at acc when there is no plaintext)
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
    if constexpr (ST == ST_PLAIN || ST == ST_SCALE) {
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int c = u + TPS * e;
            fused_store<ST>(f, bi, r, t, limb, pc, (long long)sub * T + c, log_n, sm[sidx(c)], data);
        }
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
// KM: 1 = FP64 only (limbs under q < 2^41; others skipped),
//     2 = Harvey lazy integer only (any q < 2^62; with cls 2 the FP64 limbs are skipped)
template <int LOG_T, bool INV, bool COL, int IO, int KM, int LOGN = 0>
__global__ void __launch_bounds__(256, KM == 1 ? SRK_NTT_MINB_F64 : SRK_NTT_MINB_INT)
    ntt_pass_kernel(LimbBatch b, NttTables tb, int log_n_arg, const __grid_constant__ FuseArgs f) {
    static_assert(KM == 1 || KM == 2, "FP64 or Harvey pass kernels only");
    const int log_n = LOGN ? LOGN : log_n_arg;
    using S = NttShape<LOG_T>;
    constexpr int T = S::T, E = S::E, TPS = S::TPS, LE1 = S::LE1, LE2 = S::LE2;
    constexpr bool FIRST = (COL != INV);  // forward column / inverse row pass
    constexpr int LD = FIRST ? IO : LD_PLAIN;
    constexpr int ST = FIRST ? ST_PLAIN : IO;
    extern __shared__ uint64_t smem[];

    const int n = 1 << log_n;
    // sub-transforms per CTA (a power of two): shifts and masks, no division subroutine
    constexpr int LTPS = LOG_T - LE1;
    const int lcb = (31 - __clz((int)blockDim.x)) - LTPS;
    const int CB = 1 << lcb;
    const int limb = blockIdx.z, poly = blockIdx.y;
    const int bi = b.ppc == 2 ? poly >> 1 : (b.ppc == 1 ? poly : poly / b.ppc);
    const int r = poly - bi * b.ppc;
    int t, pid;
    if (!limb_map(b, r, limb, t, pid)) return;
    uint64_t *data =
        b.ptr + (long long)bi * b.ct_stride + (long long)r * b.poly_stride + (long long)t * n;
    const uint64_t *lsrc = data;  // LD_PLAIN / LD_AUTO source limb
    if constexpr (FIRST && (LD == LD_PLAIN || LD == LD_AUTO)) {
        if (f.src) lsrc = f.src + (long long)bi * f.src_ct + (long long)r * f.src_ps + (long long)t * n;
    }
    const int tid = threadIdx.x;
    int sb, u;  // local sub-transform and thread-within-sub-transform
    if (COL) {
        sb = tid & (CB - 1);
        u = tid >> lcb;
    } else {
        sb = tid >> LTPS;
        u = tid & (TPS - 1);
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
    const TwPtr tw = {(INV ? tb.itw : tb.tw) + (long long)pid * n, (INV ? tb.itwd : tb.twd) + (long long)pid * n};
    // arithmetic mode, uniform per launch: 2 = FP64 (q < 2^41), 0 = Harvey lazy integer
    constexpr int mode = KM == 1 ? 2 : 0;
    // the first loads need no prime constant: issue them before its (dependent) load
    uint64_t x[E];
    constexpr bool RAW = !(FIRST && LD == LD_SPREAD);
    auto raw = [&](int c) -> uint64_t {
        if constexpr (FIRST && LD == LD_AUTO) return __ldg(lsrc + auto_index((uint32_t)gaddr(c), f.galois, log_n));
        else if constexpr (FIRST) return lsrc[gaddr(c)];
        else return data[gaddr(c)];
    };
    if constexpr (RAW) {
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = raw((INV && COL) ? u * E + e : u + TPS * e);
    }
    const PrimeConst pc = tb.pc[pid];
    const uint64_t q = pc.q, two_q = pc.two_q;
    // prime-class split of mixed batches (uniform per CTA): the FP64 kernel never
    // touches a limb >= 2^41; the integer kernel skips FP64 limbs when filtered
    if ((KM == 1 || b.cls == 1) ? q >= SRK_F64_Q : (b.cls == 2 && q < SRK_F64_Q)) return;
    auto load = [&](int c) -> uint64_t {
        if constexpr (FIRST) return fused_load<LD>(f, tb.pc, bi, r, t, pc, gaddr(c), log_n, lsrc);
        else return data[gaddr(c)];
    };
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
        if constexpr (mode == 2) return (uint64_t)__double_as_longlong(f64_of_u64(v));
        else return v;
    };
    // first-pass conversion of the raw loads (canonical u64 -> FP64 operand)
    auto cvt = [&](uint64_t v) -> uint64_t {
        if constexpr (mode == 2 && FIRST) return (uint64_t)__double_as_longlong(f64_of_u64(v));
        else return v;
    };
    if (!INV) {
        // ---- round 1: strided ownership c = u + TPS e, strides T/2 .. TPS
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = RAW ? cvt(x[e]) : load_m(u + TPS * e);
        if constexpr (mode == 2)
            FwdR1<E, LE1, 2>::run(x, tw, base, q, two_q, fq);
        else
            FwdR1<E, LE1, 0>::run(x, tw, base, q, two_q);
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = x[e];
        __syncthreads();
        // ---- round 2: contiguous ownership c = u E + e, strides TPS/2 .. 1
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
        if constexpr (mode == 2)
            FwdR2<E, TPS, LE1, LE2, 2>::run(x, tw, base, u, q, two_q, fq);
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
                if constexpr (mode == 2) {
                    // ST_KSC consumes the raw FP64 value (|x| < 17 q) in its own reduction
                    if constexpr (ST != ST_KSC)
                        v = canon_u64_of_f64(__longlong_as_double((long long)v), fq.q, fq.qinv);
                } else {
                    v = v >= two_q ? v - two_q : v;
                    v = v >= q ? v - q : v;
                }
                smem[sidx(u * E + e)] = v;
            }
            __syncthreads();
            row_final_store<LOG_T, ST, KM>(f, smem, sidx, bi, r, t, pid, limb, pc, fq, sub, u, log_n, data);
        }
    } else {
        // ---- round 1: contiguous ownership, strides 1 .. E/2
        if (COL) {
            // second pass: FP64 sums doubled every stage of the first -> re-centre
#pragma unroll
            for (int e = 0; e < E; e++) {
                uint64_t v = x[e];  // data[gaddr(u * E + e)], loaded above
                if constexpr (mode == 2)
                    v = (uint64_t)__double_as_longlong(
                        centre_f64(__longlong_as_double((long long)v), fq.q, fq.qinv));
                x[e] = v;
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = RAW ? cvt(x[e]) : load_m(u + TPS * e);
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
        }
        // step numbers of the inverse: row pass 0.., column pass log_n - LOG_T ..
        const int k0 = COL ? log_n - LOG_T : 0;
        if constexpr (mode == 2)
            InvR1<E, LOG_T, LE1, 2>::run(x, tw, base, u, q, two_q, k0, fq);
        else
            InvR1<E, LOG_T, LE1, 0>::run(x, tw, base, u, q, two_q, k0);
        if (!COL) __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u * E + e)] = x[e];
        __syncthreads();
        // ---- round 2: strided ownership c = u + TPS e, strides E .. T/2
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u + TPS * e)];
        if constexpr (mode == 2)
            InvR2<E, TPS, LE2, 2>::run(x, tw, base, q, two_q, k0 + LE1, fq);
        else
            InvR2<E, TPS, LE2, 0>::run(x, tw, base, q, two_q, k0 + LE1);
        if (COL) {
            // last pass of the inverse: * N^-1 (or the fused per-limb scale), canonical
            uint64_t m = pc.ninv, ms = pc.ninv_shoup;
            if constexpr (ST == ST_SCALE) {
                m = f.mulc.w[limb];
                ms = f.mulc.ws[limb];
            }
            if constexpr (mode == 2) {
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
