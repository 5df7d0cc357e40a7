// kernels.cuh -- elementwise / base-conversion / key-switching / sampling
// kernels for the RNS-CKKS engine.  Every kernel is a grid-stride loop over
// (limb, coefficient) with 16-byte (2 x uint64) vectorised accesses where
// the layout allows; all of them are HBM-streaming kernels whose roofline is
// the copy bandwidth ("kernels and their roofs").
#pragma once
#include <cstdint>

#include "modarith.cuh"
#include "ntt.cuh"
#include "bconv.cuh"


// ---------------------------------------------------------------------
// elementwise on ciphertexts [2][nl][N] (poly stride may differ per operand)
// ---------------------------------------------------------------------

// op 0: a+b, 1: a-b, 2: -a
__global__ void k_addsub(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                         uint64_t *__restrict__ out, const PrimeConst *__restrict__ pc, int log_n,
                         int nl, int op, long long total) {
    const Div32 dv = mk_div32(nl);
    for (long long x = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; x < total;
         x += (long long)gridDim.x * blockDim.x * 2) {
        const uint32_t row = (uint32_t)(x >> log_n);
        const int limb = (int)(row - div32(row, dv) * nl);
        const uint64_t q = pc[limb].q;
        ulonglong2 va = *reinterpret_cast<const ulonglong2 *>(a + x);
        ulonglong2 r;
        if (op == 2) {
            r.x = neg_mod(va.x, q);
            r.y = neg_mod(va.y, q);
        } else {
            ulonglong2 vb = *reinterpret_cast<const ulonglong2 *>(b + x);
            if (op == 0) {
                r.x = add_mod(va.x, vb.x, q);
                r.y = add_mod(va.y, vb.y, q);
            } else {
                r.x = sub_mod(va.x, vb.x, q);
                r.y = sub_mod(va.y, vb.y, q);
            }
        }
        *reinterpret_cast<ulonglong2 *>(out + x) = r;
    }
}

// out = a + (poly0: pt or const k[limb]); poly1 copied.  pt == nullptr -> const.
// a/out: [batch][2][nl][N]; pt: [nl][N] per ciphertext at stride pt_ct (0 = shared)
__global__ void k_add_plain(const uint64_t *__restrict__ a, const uint64_t *__restrict__ pt,
                            long long pt_ct, LimbConsts k, uint64_t *__restrict__ out,
                            const PrimeConst *__restrict__ pc, int log_n, int nl, int batch) {
    const long long n = 1ll << log_n;
    const long long per = 2ll * nl * n;
    const long long total = per * batch;
    const Div32 dv = mk_div32(2 * nl);
    for (long long x = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; x < total;
         x += (long long)gridDim.x * blockDim.x * 2) {
        const long long b = div32((uint32_t)(x >> log_n), dv), xi = x - b * per;
        const long long limb_all = xi >> log_n;
        ulonglong2 va = *reinterpret_cast<const ulonglong2 *>(a + x);
        if (limb_all < nl) {
            const int limb = (int)limb_all;
            const uint64_t q = pc[limb].q;
            ulonglong2 vb;
            if (pt) {
                vb = *reinterpret_cast<const ulonglong2 *>(pt + b * pt_ct + xi);
            } else {
                vb.x = vb.y = k.w[limb];
            }
            va.x = add_mod(va.x, vb.x, q);
            va.y = add_mod(va.y, vb.y, q);
        }
        *reinterpret_cast<ulonglong2 *>(out + x) = va;
    }
}

// out[p][i] = a[p][i] * (pt ? pt[i] : k[i]); a read with poly stride src_nl*N
__global__ void k_mul_pt(const uint64_t *__restrict__ a, int src_nl,
                         const uint64_t *__restrict__ pt, LimbConsts k, uint64_t *__restrict__ out,
                         const PrimeConst *__restrict__ pc, int log_n, int nl) {
    const long long n = 1ll << log_n;
    const long long total = 2ll * nl * n;
    const Div32 dv = mk_div32(nl);
    for (long long x = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; x < total;
         x += (long long)gridDim.x * blockDim.x * 2) {
        const long long la = x >> log_n;
        const int p = (int)div32((uint32_t)la, dv), limb = (int)(la - (long long)p * nl);
        const long long off = x & (n - 1);
        const long long src = ((long long)p * src_nl + limb) * n + off;
        ulonglong2 va = *reinterpret_cast<const ulonglong2 *>(a + src);
        const PrimeConst P = pc[limb];
        if (pt) {
            ulonglong2 vb = *reinterpret_cast<const ulonglong2 *>(pt + (long long)limb * n + off);
            va.x = mul_mod(va.x, vb.x, P);
            va.y = mul_mod(va.y, vb.y, P);
        } else {
            va.x = mul_shoup(va.x, k.w[limb], k.ws[limb], P.q);
            va.y = mul_shoup(va.y, k.w[limb], k.ws[limb], P.q);
        }
        *reinterpret_cast<ulonglong2 *>(out + x) = va;
    }
}

// d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 for `batch` pairs (a, b at ct stride
// ab_ct, poly stride nl N; d: [3][nl][N] at stride d_ct) -- one launch per batch
__global__ void k_tensor(const uint64_t *__restrict__ a0p, const uint64_t *__restrict__ b0p, long long ab_ct,
                         uint64_t *__restrict__ d0p, long long d_ct, const PrimeConst *__restrict__ pc,
                         int log_n, int nl, int batch) {
    const long long n = 1ll << log_n;
    const long long ps = (long long)nl * n;
    const Div32 dv = mk_div32(nl);
    for (long long xx = blockIdx.x * (long long)blockDim.x + threadIdx.x; xx < ps * batch;
         xx += (long long)gridDim.x * blockDim.x) {
        const uint32_t row = (uint32_t)(xx >> log_n);
        const long long bi = div32(row, dv);
        const long long x = xx - bi * ps;
        const uint64_t *a = a0p + bi * ab_ct, *b = b0p + bi * ab_ct;
        uint64_t *d = d0p + bi * d_ct;
        const PrimeConst P = pc[x >> log_n];
        uint64_t a0 = __ldg(a + x), a1 = __ldg(a + ps + x), b0 = __ldg(b + x), b1 = __ldg(b + ps + x);
        if (P.q < SRK_F64_Q) {  // FP64 pipe: exact FMA-split products (ntt.cuh modmul_f64)
            const double q = __longlong_as_double((long long)P.qd_bits);
            const double qi = __longlong_as_double((long long)P.qinv_bits);
            const double fa0 = f64_of_u64(a0), fa1 = f64_of_u64(a1);
            const double fb0 = f64_of_u64(b0), fb1 = f64_of_u64(b1);
            d[x] = canon_u64_of_small_f64(modmul_f64(fa0, fb0, q, qi), P.q);
            d[ps + x] = canon_u64_of_f64(modmul_f64(fa0, fb1, q, qi) + modmul_f64(fa1, fb0, q, qi), q, qi);
            d[2 * ps + x] = canon_u64_of_small_f64(modmul_f64(fa1, fb1, q, qi), P.q);
            continue;
        }
        d[x] = mul_mod(a0, b0, P);
        U128 m = mul_wide(a0, b1);
        mac(m, a1, b0);
        d[ps + x] = reduce_u128(m, P);
        d[2 * ps + x] = mul_mod(a1, b1, P);
    }
}

// the same over a pointer table: pair i = (a[i], b[i]) (poly stride nl N each),
// d[i] at d + i d_ct -- operands shared between pairs are read where they lie
#define SRK_PAIRS_MAX 32
struct TensorPairs {
    const uint64_t *a[SRK_PAIRS_MAX];
    const uint64_t *b[SRK_PAIRS_MAX];
};
__global__ void k_tensor_pairs(const __grid_constant__ TensorPairs tp, uint64_t *__restrict__ d0p, long long d_ct,
                               const PrimeConst *__restrict__ pc, int log_n, int nl, int batch) {
    const long long n = 1ll << log_n;
    const long long ps = (long long)nl * n;
    const Div32 dv = mk_div32(nl);
    for (long long xx = blockIdx.x * (long long)blockDim.x + threadIdx.x; xx < ps * batch;
         xx += (long long)gridDim.x * blockDim.x) {
        const uint32_t row = (uint32_t)(xx >> log_n);
        const int bi = (int)div32(row, dv);
        const long long x = xx - (long long)bi * ps;
        const uint64_t *a = tp.a[bi], *b = tp.b[bi];
        uint64_t *d = d0p + bi * d_ct;
        const PrimeConst P = pc[x >> log_n];
        uint64_t a0 = __ldg(a + x), a1 = __ldg(a + ps + x), b0 = __ldg(b + x), b1 = __ldg(b + ps + x);
        if (P.q < SRK_F64_Q) {
            const double q = __longlong_as_double((long long)P.qd_bits);
            const double qi = __longlong_as_double((long long)P.qinv_bits);
            const double fa0 = f64_of_u64(a0), fa1 = f64_of_u64(a1);
            const double fb0 = f64_of_u64(b0), fb1 = f64_of_u64(b1);
            d[x] = canon_u64_of_small_f64(modmul_f64(fa0, fb0, q, qi), P.q);
            d[ps + x] = canon_u64_of_f64(modmul_f64(fa0, fb1, q, qi) + modmul_f64(fa1, fb0, q, qi), q, qi);
            d[2 * ps + x] = canon_u64_of_small_f64(modmul_f64(fa1, fb1, q, qi), P.q);
            continue;
        }
        d[x] = mul_mod(a0, b0, P);
        U128 m = mul_wide(a0, b1);
        mac(m, a1, b0);
        d[ps + x] = reduce_u128(m, P);
        d[2 * ps + x] = mul_mod(a1, b1, P);
    }
}

// ---------------------------------------------------------------------
// rescale helpers
// ---------------------------------------------------------------------

// top[b][p] = a[b][p][level] * pt[level]   (rescale of a ct x pt product:
// the dropped limb of the product, before its INTT)
__global__ void k_rescale_top(const uint64_t *__restrict__ a, long long a_ct, long long a_ps,
                              const uint64_t *__restrict__ pt, long long pt_ct, uint64_t *__restrict__ top,
                              const PrimeConst *__restrict__ pc, int log_n, int level, int batch) {
    const long long n = 1ll << log_n;
    const PrimeConst P = pc[level];
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < 2ll * batch * n;
         x += (long long)gridDim.x * blockDim.x) {
        const long long bp = x >> log_n;
        const int b = (int)(bp >> 1), p = (int)(bp & 1);
        const long long off = x & (n - 1);
        top[x] = mul_mod(a[b * a_ct + p * a_ps + (long long)level * n + off],
                         pt[b * pt_ct + (long long)level * n + off], P);
    }
}

// ---------------------------------------------------------------------
// Galois automorphism in the NTT domain (gather, one permutation per limb)
// ---------------------------------------------------------------------
__global__ void k_automorph(const uint64_t *__restrict__ a, uint64_t *__restrict__ out,
                            long long n_limbs_total, uint64_t galois, int log_n) {
    const long long n = 1ll << log_n;
    const long long total = n_limbs_total * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long base = x & ~(n - 1);
        const uint32_t k = (uint32_t)(x & (n - 1));
        out[x] = __ldg(a + base + auto_index(k, galois, log_n));
    }
}

// ---------------------------------------------------------------------
// hybrid key switching, batched over B ciphertexts
// ---------------------------------------------------------------------
// ModUp base conversion for every digit of every ciphertext (ModUpArgs, bconv.cuh):
//   ext[b][j][slot_t] = sum_{i in G_j} y_i * mat_j[i][t]  mod p_t
// y = dc[b][G_j] already multiplied by (Q_j/q_i)^-1 (folded into the INTT).
// grid: x = coefficient blocks, y = b * beta + j, z = chunks of 8 targets.
#define SRK_MODUP_TCH 8

// GS = exact digit size (compile-time: no predicated MACs); digits smaller
// than GS (the last one at some levels) fall back to the runtime loop
template <int GS>
__global__ void __launch_bounds__(256) k_modup(const __grid_constant__ ModUpArgs a,
                                               const PrimeConst *__restrict__ pc, int log_n) {
    const long long n = 1ll << log_n;
    const int b = blockIdx.y / a.beta, j = blockIdx.y - b * a.beta;
    const int g0 = j * a.alpha, gs = min(a.alpha, a.nl - g0);
    const int t0 = blockIdx.z * SRK_MODUP_TCH;
    const int nd = a.n_dst[j];
    if (t0 >= nd) return;
    const int t1 = min(nd, t0 + SRK_MODUP_TCH);
    const uint64_t *src = a.dc + b * a.dc_ct + (long long)g0 * n;
    uint64_t *dst = a.ext + b * a.ext_ct + j * a.ext_dig;
    const uint64_t *mat = a.mat[j];
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        if (gs == GS) {
            uint64_t y[GS];
#pragma unroll
            for (int i = 0; i < GS; i++) y[i] = src[(long long)i * n + x];
            for (int t = t0; t < t1; t++) {
                U128 acc = {0, 0};
#pragma unroll
                for (int i = 0; i < GS; i++) mac(acc, y[i], __ldg(mat + i * nd + t));
                dst[(long long)__ldg(a.slot[j] + t) * n + x] = reduce_u128(acc, pc[__ldg(a.pid[j] + t)]);
            }
        } else {
            for (int t = t0; t < t1; t++) {
                U128 acc = {0, 0};
                for (int i = 0; i < gs; i++) mac(acc, src[(long long)i * n + x], __ldg(mat + i * nd + t));
                dst[(long long)__ldg(a.slot[j] + t) * n + x] = reduce_u128(acc, pc[__ldg(a.pid[j] + t)]);
            }
        }
    }
}

// key-switch inner product:
//   acc[b][r][t][n] = sum_j E_j[t][n] * key[j][r][pid(t)][n]
// E_j[t] = d[b][t] for t in digit j's own limbs G_j (NTT form input), else
// ext[b][j][t].  For a rotation by X -> X^g the key is stored permuted by
// sigma_g^-1 (srk_keygen_galois), so acc here is sigma_g^-1 of the rotated
// accumulator and the ModDown reads it back through sigma_g: the streams in
// this kernel stay coalesced.  Each thread owns one (t, n) for every
// ciphertext of the batch, so each key word is read once per batch (the
// key is the dominant HBM stream of a key switch).
struct KsInnerArgs {
    const uint64_t *d;
    long long d_ct;
    const uint64_t *ext;
    long long ext_ct, ext_dig;
    const uint64_t *key;
    uint64_t *acc;
    long long acc_ct;
    uint64_t galois;
    int n_primes, nl, ne, level, L, alpha, beta, batch;
    int t0;  // first extended-basis limb to produce (nl: special limbs only)
};

// Thread = one coefficient of one limb t, for every ciphertext of the batch:
// its beta x 2 key words are loaded once and kept in registers; ciphertexts
// are processed two at a time so 2 x beta independent ext loads are in flight
// before the MACs need them (the kernel is HBM-latency bound otherwise).
template <int MAXD>
__global__ void __launch_bounds__(256) k_ks_inner(const __grid_constant__ KsInnerArgs a,
                                                  const PrimeConst *__restrict__ pc, int log_n) {
    const long long n = 1ll << log_n;
    const long long total = (long long)a.ne * n;  // acc poly stride
    const long long work = (long long)(a.ne - a.t0) * n;
    const Div32 dalpha = mk_div32(a.alpha);
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < work;
         x += (long long)gridDim.x * blockDim.x) {
        const int t = a.t0 + (int)(x >> log_n);
        const long long off = x & (n - 1);
        const int pid = t <= a.level ? t : t + (a.L - a.level);
        const int jt = t < a.nl ? (int)div32((uint32_t)t, dalpha) : -1;
        uint64_t k0[MAXD], k1[MAXD];
#pragma unroll
        for (int j = 0; j < MAXD; j++) {
            if (j < a.beta) {
                const uint64_t *kj = a.key + ((long long)j * 2 * a.n_primes + pid) * n + off;
                k0[j] = __ldg(kj);
                k1[j] = __ldg(kj + (long long)a.n_primes * n);
            }
        }
        const PrimeConst P = pc[pid];
        const uint64_t *ext = a.ext + (long long)t * n + off;
        const uint64_t *dd = a.d + (long long)t * n + off;
        for (int b = 0; b < a.batch; b += 2) {
            const bool two = b + 1 < a.batch;
            uint64_t e0[MAXD], e1[MAXD];
#pragma unroll
            for (int j = 0; j < MAXD; j++) {
                if (j < a.beta) {
                    const uint64_t *p = j == jt ? dd + b * a.d_ct : ext + b * a.ext_ct + j * a.ext_dig;
                    const long long st = j == jt ? a.d_ct : a.ext_ct;
                    e0[j] = __ldg(p);  // read-only: may overlap the previous pair's stores
                    e1[j] = (two ? __ldg(p + (two ? st : 0)) : 0);
                }
            }
            U128 a0 = {0, 0}, a1 = {0, 0}, c0 = {0, 0}, c1 = {0, 0};
#pragma unroll
            for (int j = 0; j < MAXD; j++) {
                if (j < a.beta) {
                    mac(a0, e0[j], k0[j]);
                    mac(a1, e0[j], k1[j]);
                    mac(c0, e1[j], k0[j]);
                    mac(c1, e1[j], k1[j]);
                }
            }
            uint64_t *o = a.acc + b * a.acc_ct + (long long)t * n + off;
            o[0] = reduce_u128(a0, P);
            o[total] = reduce_u128(a1, P);
            if (two) {
                o[a.acc_ct] = reduce_u128(c0, P);
                o[a.acc_ct + total] = reduce_u128(c1, P);
            }
        }
    }
}

// exact ModDown rounding term per coefficient: v = round(sum_k z_k / p_k)
// (64.64 fixed point, f_k = z_k R1 + hi(z_k R0), R = floor(2^128 / p_k));
// z: B*2 polys (ct stride z_ct, poly stride z_ps) of K limbs; v: [B*2][N]
// (limb k < K under prime pid0 + k; limb K, if present, under prime pid_last)
__global__ void k_moddown_v(const uint64_t *__restrict__ z, long long z_ct, long long z_ps, int K,
                            int pid0, int n_src, int pid_last, uint8_t *__restrict__ v,
                            const PrimeConst *__restrict__ pc, int log_n, int batch) {
    const long long n = 1ll << log_n;
    const long long total = 2ll * batch * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long p = x >> log_n;
        const long long off = x & (n - 1);
        const uint64_t *zp = z + (p >> 1) * z_ct + (p & 1) * z_ps + off;
        U128 frac = {0, 1ull << 63};
        for (int k = 0; k < n_src; k++) {
            const uint64_t zk = zp[k * n];
            const PrimeConst Q = pc[k < K ? pid0 + k : pid_last];
            U128 fr = {0, zk * Q.ratio_hi + mulhi64(zk, Q.ratio_lo)};
            add_to(frac, fr);
        }
        v[x] = (uint8_t)frac.hi;
    }
}

// ---------------------------------------------------------------------
// sampling (counter-based, restated bit for bit in oracle/ckks_oracle.c)
// ---------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// a[k][j] = uniform mod prime(k), stream = stream_base + prime(k)
__global__ void k_uniform(LimbBatch b, const PrimeConst *__restrict__ pc, int log_n,
                          uint64_t seed, uint64_t stream_base) {
    const long long n = 1ll << log_n;
    const long long total = (long long)b.n_limbs * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(x >> log_n);
        const uint64_t j = (uint64_t)(x & (n - 1));
        const int pid = batch_pid(b, k);
        const uint64_t key = mix64(seed ^ mix64(stream_base + (uint64_t)pid));
        U128 v;
        v.hi = mix64(key + 2 * j);
        v.lo = mix64(key + 2 * j + 1);
        b.ptr[x] = reduce_u128(v, pc[pid]);
    }
}

// out[k][j] = v[j] mod prime(k)   (v: small signed integers)
__global__ void k_small_to_res(const int64_t *__restrict__ v, LimbBatch b,
                               const PrimeConst *__restrict__ pc, int log_n) {
    const long long n = 1ll << log_n;
    const long long total = (long long)b.n_limbs * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(x >> log_n);
        const PrimeConst P = pc[batch_pid(b, k)];
        const int64_t s = v[x & (n - 1)];
        uint64_t r = reduce64(s >= 0 ? (uint64_t)s : (uint64_t)(-s), P);
        b.ptr[x] = s >= 0 ? r : neg_mod(r, P.q);
    }
}

// key[j] = (-a s + e + [limb in digit j] * Pmod * sfrom ,  a)   for one digit
// e_ntt, a, s, sfrom: [n_primes][N]; b written over all primes
__global__ void k_keygen_combine(const uint64_t *__restrict__ a, const uint64_t *__restrict__ s,
                                 const uint64_t *__restrict__ sfrom,
                                 const uint64_t *__restrict__ e, uint64_t *__restrict__ b,
                                 LimbConsts pmod, const PrimeConst *__restrict__ pc, int log_n,
                                 int n_primes, int d0, int d1) {
    const long long n = 1ll << log_n;
    const long long total = (long long)n_primes * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x >> log_n);
        const PrimeConst P = pc[i];
        uint64_t v = sub_mod(e[x], mul_mod(a[x], s[x], P), P.q);
        if (i >= d0 && i < d1) v = add_mod(v, mul_shoup(sfrom[x], pmod.w[i], pmod.ws[i], P.q), P.q);
        b[x] = v;
    }
}

// c0 = -c1 s + e + m  over nl limbs
__global__ void k_encrypt_combine(const uint64_t *__restrict__ c1, const uint64_t *__restrict__ s,
                                  const uint64_t *__restrict__ e, const uint64_t *__restrict__ m,
                                  uint64_t *__restrict__ c0, const PrimeConst *__restrict__ pc,
                                  int log_n, int nl) {
    const long long n = 1ll << log_n;
    const long long total = (long long)nl * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const PrimeConst P = pc[x >> log_n];
        uint64_t v = sub_mod(e[x], mul_mod(c1[x], s[x], P), P.q);
        c0[x] = add_mod(v, m[x], P.q);
    }
}

// t = c0 + c1 s on limb 0
__global__ void k_decrypt_limb0(const uint64_t *__restrict__ ct, long long pstride,
                                const uint64_t *__restrict__ s, uint64_t *__restrict__ t,
                                const PrimeConst *__restrict__ pc, int log_n) {
    const long long n = 1ll << log_n;
    const PrimeConst P = pc[0];
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x)
        t[x] = add_mod(ct[x], mul_mod(ct[pstride + x], s[x], P), P.q);
}

__global__ void k_center_limb0(const uint64_t *__restrict__ t, int64_t *__restrict__ m,
                               const PrimeConst *__restrict__ pc, int log_n) {
    const long long n = 1ll << log_n;
    const uint64_t q = pc[0].q;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x)
        m[x] = t[x] > (q >> 1) ? -(int64_t)(q - t[x]) : (int64_t)t[x];
}

// cross-rank modular sum fix-up: limbs hold plain int64 sums (< 2^63)
__global__ void k_reduce_mod(uint64_t *__restrict__ a, const PrimeConst *__restrict__ pc,
                             int log_n, int nl, long long total) {
    const Div32 dv = mk_div32(nl);
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const uint32_t row = (uint32_t)(x >> log_n);
        a[x] = reduce64(a[x], pc[row - div32(row, dv) * nl]);
    }
}

// special limbs of X = acc + P d for the fused HMult rescale:
// zb[b][r][k] = acc[b][r][nl + k] (k < K), zb[b][r][K] = acc[b][r][l] + P d_r[l]  (mod q_l)
__global__ void k_prep_special(const uint64_t *__restrict__ acc, long long acc_ct, long long acc_ps,
                               const uint64_t *__restrict__ d, long long d_ct, long long d_ps,
                               uint64_t *__restrict__ zb, uint64_t pmod_l, uint64_t pmod_l_shoup,
                               const PrimeConst *__restrict__ pc, int log_n, int level, int K,
                               int batch) {
    const long long n = 1ll << log_n;
    const int nl = level + 1;
    const long long per = (long long)(K + 1) * n;
    const long long total = 2ll * batch * per;
    const uint64_t ql = pc[level].q;
    const Div32 dv = mk_div32(K + 1);
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long p = div32((uint32_t)(x >> log_n), dv), xi = x - p * per;
        const int k = (int)(xi >> log_n);
        const long long off = xi & (n - 1);
        const long long b = p >> 1, r = p & 1;
        const uint64_t *a = acc + b * acc_ct + r * acc_ps;
        uint64_t v;
        if (k < K) {
            v = a[(long long)(nl + k) * n + off];
        } else {
            const uint64_t dv = d[b * d_ct + r * d_ps + (long long)level * n + off];
            v = add_mod(a[(long long)level * n + off], mul_shoup(dv, pmod_l, pmod_l_shoup, ql), ql);
        }
        zb[x] = v;
    }
}

// linear combination of ciphertexts (the BSGS leaf sum), before its rescale:
//   out[b][r][j] = sum_i k[i][j] * T_i[b][r][j]   mod q_j,  j < nl
// T_i read as its first nl limbs (terms may sit at higher levels); k: device
// [n_terms][nl] residues; U128 accumulation, one reduction per output word
#define SRK_LC_MAX 64
struct LinCombArgs {
    const uint64_t *term[SRK_LC_MAX];
    long long term_ps[SRK_LC_MAX];  // poly stride (words) of each term
    long long term_ct[SRK_LC_MAX];  // ciphertext stride for batches
    int n_terms, nl, batch;
    const uint64_t *k;
    uint64_t *out;
};

__global__ void k_lincomb(const __grid_constant__ LinCombArgs a, const PrimeConst *__restrict__ pc,
                          int log_n) {
    const long long n = 1ll << log_n;
    const long long per = 2ll * a.nl * n;
    const long long total = per * a.batch;
    const Div32 d2 = mk_div32(2 * a.nl), d1 = mk_div32(a.nl);
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long b = div32((uint32_t)(x >> log_n), d2), xi = x - b * per;
        const long long lr = xi >> log_n;
        const int r = (int)div32((uint32_t)lr, d1), j = (int)(lr - (long long)r * a.nl);
        const long long off = xi & (n - 1);
        U128 acc = {0, 0};
        for (int i = 0; i < a.n_terms; i++) {
            const uint64_t v = __ldg(a.term[i] + b * a.term_ct[i] + r * a.term_ps[i] + (long long)j * n + off);
            mac(acc, v, __ldg(a.k + (long long)i * a.nl + j));
            if ((i & 7) == 7) {  // keep the 128-bit sum bounded: reduce every 8 products
                U128 red = {0, reduce_u128(acc, pc[j])};
                acc = red;
            }
        }
        a.out[x] = reduce_u128(acc, pc[j]);
    }
}

// Several linear combinations of the SAME terms (all BSGS leaf sums of a polynomial share
// the baby-step ciphertexts): out_l = sum_i k[l][i][j] T_i for l < L, every term word
// read once for all L outputs (one launch per 8 outputs instead of one pass over the
// terms per output).  k: device [n_out][n_terms][nl]; outs: n_out destinations.
#define SRK_LC_OUTS 8
struct LinCombOuts {
    uint64_t *out[SRK_LC_OUTS];
    const double *kf;         // k / q per table entry (same layout as k), or null
    int n_out, k_out_stride;  // residue words between consecutive outputs' tables
};
template <int L>
__global__ void __launch_bounds__(256) k_lincomb_multi(const __grid_constant__ LinCombArgs a,
                                                       const __grid_constant__ LinCombOuts o,
                                                       const PrimeConst *__restrict__ pc, int log_n) {
    // this limb's table entries {k, bits of k / q} per (term, output), staged once per
    // 256-element block (the block shares its limb: 256 divides N)
    __shared__ ulonglong2 s_k[SRK_LC_MAX * L];
    const long long n = 1ll << log_n;
    const long long per = 2ll * a.nl * n;
    const long long total = per * a.batch;
    const Div32 d2 = mk_div32(2 * a.nl), d1 = mk_div32(a.nl);
    const int tid = threadIdx.x;
    for (long long x0 = blockIdx.x * (long long)blockDim.x; x0 < total; x0 += (long long)gridDim.x * blockDim.x) {
        const long long x = x0 + tid;
        const long long b = div32((uint32_t)(x0 >> log_n), d2), xi = x0 - b * per;
        const long long lr = xi >> log_n;
        const int r = (int)div32((uint32_t)lr, d1), j = (int)(lr - (long long)r * a.nl);
        const long long off = (xi & (n - 1)) + tid;
        const PrimeConst P = pc[j];
        // under a prime < 2^41 (every scaling prime) with the k / q table: wrapped 64-bit
        // sum S and FP64 quotient T = sum v (k / q), result S - round(T) q (the base
        // conversions' recipe, bconv.cuh: exact while |T error| < 1/2 -- up to 32 terms
        // below 2^41 keep T < 2^46, so 32 FMA roundings of <= 2^-8 plus the table's 2^-53
        // relative error stay below 0.14); else 128-bit sums, reduced after every 8 products
        const bool f64 = o.kf != nullptr && P.q < SRK_F64_Q && a.n_terms <= 32;
        __syncthreads();  // the previous block's reads of s_k are done
        for (int e = tid; e < a.n_terms * L; e += blockDim.x) {
            const int i = e / L, l = e - i * L;  // rows past n_out repeat the last one (never stored)
            const long long kl = (long long)i * a.nl + j + (long long)min(l, o.n_out - 1) * o.k_out_stride;
            s_k[e] = make_ulonglong2(__ldg(a.k + kl),
                                     f64 ? (uint64_t)__double_as_longlong(__ldg(o.kf + kl)) : 0ull);
        }
        __syncthreads();
        U128 acc[L];  // f64 path: lo = S, hi = bits of T
#pragma unroll
        for (int l = 0; l < L; l++) acc[l] = {0, 0};
        for (int i0 = 0; i0 < a.n_terms; i0 += 8) {
            const int ni = min(8, a.n_terms - i0);
            uint64_t v[8];
#pragma unroll
            for (int i = 0; i < 8; i++)  // the group's loads first: all in flight together
                v[i] = (i < ni && x < total)
                           ? __ldg(a.term[i0 + i] + b * a.term_ct[i0 + i] + r * a.term_ps[i0 + i] +
                                   (long long)j * n + off)
                           : 0;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (i < ni) {
                    const ulonglong2 *kp = s_k + (i0 + i) * L;
                    if (f64) {
                        const uint32_t vl = (uint32_t)v[i], vh = (uint32_t)(v[i] >> 32);
                        const double dv = f64_of_u64(v[i]);
#pragma unroll
                        for (int l = 0; l < L; l++) {
                            const ulonglong2 kk = kp[l];
                            uint32_t sl = (uint32_t)acc[l].lo, sh = (uint32_t)(acc[l].lo >> 32);
                            mac_wide(sl, sh, vl, (uint32_t)kk.x);
                            mac_hi(sh, vl, (uint32_t)(kk.x >> 32));
                            mac_hi(sh, vh, (uint32_t)kk.x);
                            acc[l].lo = ((uint64_t)sh << 32) | sl;
                            acc[l].hi = (uint64_t)__double_as_longlong(
                                fma(dv, __longlong_as_double((long long)kk.y),
                                    __longlong_as_double((long long)acc[l].hi)));
                        }
                    } else {
#pragma unroll
                        for (int l = 0; l < L; l++) mac(acc[l], v[i], kp[l].x);
                    }
                }
            }
            if (!f64) {
#pragma unroll
                for (int l = 0; l < L; l++) acc[l] = {0, reduce_u128(acc[l], P)};
            }
        }
        if (x < total) {
#pragma unroll
            for (int l = 0; l < L; l++) {
                if (l < o.n_out)
                    o.out[l][x] = f64 ? bconv_finish((uint32_t)acc[l].lo, (uint32_t)(acc[l].lo >> 32),
                                                     __longlong_as_double((long long)acc[l].hi), P.q)
                                      : acc[l].lo;
            }
        }
    }
}

// square (NTT domain) of s over all primes: relinearisation source key
__global__ void k_square(const uint64_t *__restrict__ s, uint64_t *__restrict__ out,
                         const PrimeConst *__restrict__ pc, int log_n, int n_limbs) {
    const long long n = 1ll << log_n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < (long long)n_limbs * n;
         x += (long long)gridDim.x * blockDim.x)
        out[x] = mul_mod(s[x], s[x], pc[x >> log_n]);
}
