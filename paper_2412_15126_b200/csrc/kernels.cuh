// kernels.cuh -- elementwise / base-conversion / key-switching / sampling
// kernels for the RNS-CKKS engine.  Every kernel is a grid-stride loop over
// (limb, coefficient) with 16-byte (2 x uint64) vectorised accesses where
// the layout allows; all of them are HBM-streaming kernels whose roofline is
// the copy bandwidth ("kernels and their roofs").
#pragma once
#include <cstdint>

#include "modarith.cuh"
#include "ntt.cuh"

#define SRK_MAXP 128

// per-limb constant with Shoup companion, passed by value (<= 2 KiB)
struct LimbConsts {
    uint64_t w[SRK_MAXP];
    uint64_t ws[SRK_MAXP];
};

__device__ __forceinline__ uint32_t auto_index(uint32_t k, uint64_t g, int log_n) {
    const uint64_t mask = (2ull << log_n) - 1;
    uint32_t r = __brev(k) >> (32 - log_n);
    uint64_t e = ((uint64_t)r * 2 + 1) * g & mask;
    return __brev((uint32_t)((e - 1) >> 1)) >> (32 - log_n);
}

// ---------------------------------------------------------------------
// elementwise on ciphertexts [2][nl][N] (poly stride may differ per operand)
// ---------------------------------------------------------------------

// op 0: a+b, 1: a-b, 2: -a
__global__ void k_addsub(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                         uint64_t *__restrict__ out, const PrimeConst *__restrict__ pc, int log_n,
                         int nl, int op) {
    const long long n = 1ll << log_n;
    const long long total = 2ll * nl * n;
    for (long long x = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; x < total;
         x += (long long)gridDim.x * blockDim.x * 2) {
        const int limb = (int)((x >> log_n) % nl);
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

// out = a + (poly0: pt or const k[limb]); poly1 copied.  pt == nullptr -> const
__global__ void k_add_plain(const uint64_t *__restrict__ a, const uint64_t *__restrict__ pt,
                            LimbConsts k, uint64_t *__restrict__ out,
                            const PrimeConst *__restrict__ pc, int log_n, int nl) {
    const long long n = 1ll << log_n;
    const long long total = 2ll * nl * n;
    for (long long x = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; x < total;
         x += (long long)gridDim.x * blockDim.x * 2) {
        const long long limb_all = x >> log_n;
        ulonglong2 va = *reinterpret_cast<const ulonglong2 *>(a + x);
        if (limb_all < nl) {
            const int limb = (int)limb_all;
            const uint64_t q = pc[limb].q;
            ulonglong2 vb;
            if (pt) {
                vb = *reinterpret_cast<const ulonglong2 *>(pt + x);
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
    for (long long x = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; x < total;
         x += (long long)gridDim.x * blockDim.x * 2) {
        const long long la = x >> log_n;
        const int p = (int)(la / nl), limb = (int)(la - (long long)p * nl);
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

// d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1   (d: [3][nl][N])
__global__ void k_tensor(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                         uint64_t *__restrict__ d, const PrimeConst *__restrict__ pc, int log_n,
                         int nl) {
    const long long n = 1ll << log_n;
    const long long ps = (long long)nl * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ps;
         x += (long long)gridDim.x * blockDim.x) {
        const PrimeConst P = pc[x >> log_n];
        uint64_t a0 = a[x], a1 = a[ps + x], b0 = b[x], b1 = b[ps + x];
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

// top[p] = a[p][level] * pre  (pre: const k[level] or pt[level] or none)
__global__ void k_rescale_top(const uint64_t *__restrict__ a, long long a_pstride,
                              const uint64_t *__restrict__ pt, LimbConsts k, int mode,
                              uint64_t *__restrict__ top, const PrimeConst *__restrict__ pc,
                              int log_n, int level) {
    const long long n = 1ll << log_n;
    const PrimeConst P = pc[level];
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < 2 * n;
         x += (long long)gridDim.x * blockDim.x) {
        const int p = (int)(x >> log_n);
        const long long off = x & (n - 1);
        uint64_t v = a[p * a_pstride + (long long)level * n + off];
        if (mode == 1) v = mul_shoup(v, k.w[level], k.ws[level], P.q);
        if (mode == 2) v = mul_mod(v, pt[(long long)level * n + off], P);
        top[x] = v;
    }
}

// t[p][i] = centred(top[p]) mod q_i for i < level
__global__ void k_rescale_spread(const uint64_t *__restrict__ top, uint64_t *__restrict__ t,
                                 const PrimeConst *__restrict__ pc, int log_n, int level) {
    const long long n = 1ll << log_n;
    const long long total = 2ll * level * n;
    const uint64_t ql = pc[level].q;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long la = x >> log_n;
        const int p = (int)(la / level), i = (int)(la - (long long)p * level);
        const long long off = x & (n - 1);
        const PrimeConst P = pc[i];
        uint64_t v = top[(long long)p * n + off];
        uint64_t r;
        if (v > (ql >> 1)) {
            // v - q_l < 0: (v - q_l) mod q_i
            r = sub_mod(reduce64(v, P), reduce64(ql, P), P.q);
        } else {
            r = reduce64(v, P);
        }
        t[x] = r;
    }
}

// out[p][i] = (a[p][i]*pre_i - t[p][i]) * qlinv_i   over i < level
__global__ void k_rescale_combine(const uint64_t *__restrict__ a, long long a_pstride,
                                  const uint64_t *__restrict__ pt, LimbConsts k, int mode,
                                  const uint64_t *__restrict__ t, LimbConsts qlinv,
                                  uint64_t *__restrict__ out, const PrimeConst *__restrict__ pc,
                                  int log_n, int level) {
    const long long n = 1ll << log_n;
    const long long total = 2ll * level * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long la = x >> log_n;
        const int p = (int)(la / level), i = (int)(la - (long long)p * level);
        const long long off = x & (n - 1);
        const PrimeConst P = pc[i];
        uint64_t v = a[p * a_pstride + (long long)i * n + off];
        if (mode == 1) v = mul_shoup(v, k.w[i], k.ws[i], P.q);
        if (mode == 2) v = mul_mod(v, pt[(long long)i * n + off], P);
        v = sub_mod(v, t[x], P.q);
        out[x] = mul_shoup(v, qlinv.w[i], qlinv.ws[i], P.q);
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
// fast base conversion (ModUp / ModDown)
//   y_i = [x_i * hinv_i]_{src prime i}       (Shoup)
//   out_t = sum_i y_i * mat[i][t]  mod dst prime t
// src: n_src limbs (contiguous, coefficient form) ; out limb t written at
// out + dst_off(t) * N for t in [0, n_dst) ; mat row-major [n_src][n_dst]
// ---------------------------------------------------------------------
struct BconvArgs {
    const uint64_t *src;
    long long src_pstride;  // between polys
    int n_src;
    int src_pid0;           // prime of src limb 0 (src limbs are consecutive primes)
    uint64_t *out;
    long long out_pstride;
    int n_dst;
    const uint64_t *mat;    // device [n_src][n_dst]
    const uint64_t *hinv;   // device [n_src] (+ [n_src] Shoup)
    const int *dst_slot;    // device [n_dst]: output limb index for target t
    const int *dst_pid;     // device [n_dst]: prime id of target t
    const uint64_t *dst_corr;  // optional [n_dst]: [prod src primes]_{dst}; rounds exactly
};

template <int MAXS>
__global__ void k_bconv(BconvArgs ba, const PrimeConst *__restrict__ pc, int log_n) {
    __shared__ uint64_t s_mat[MAXS * 72];
    const long long n = 1ll << log_n;
    const int p = blockIdx.y;
    const int tot = ba.n_src * ba.n_dst;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) s_mat[i] = ba.mat[i];
    __syncthreads();
    const uint64_t *src = ba.src + p * ba.src_pstride;
    uint64_t *out = ba.out + p * ba.out_pstride;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        uint64_t y[MAXS];
#pragma unroll
        for (int i = 0; i < MAXS; i++) {
            if (i < ba.n_src) {
                const uint64_t q = pc[ba.src_pid0 + i].q;
                y[i] = mul_shoup(src[(long long)i * n + x], ba.hinv[i], ba.hinv[ba.n_src + i], q);
            }
        }
        // exact conversion: v = round(sum_i y_i / q_i) in 64.64 fixed point
        // (f_i = y_i R1 + hi(y_i R0), R = floor(2^128/q_i)); output - v * Q
        uint64_t v = 0;
        if (ba.dst_corr) {
            U128 frac = {0, 0};
#pragma unroll
            for (int i = 0; i < MAXS; i++) {
                if (i < ba.n_src) {
                    const PrimeConst P = pc[ba.src_pid0 + i];
                    U128 f = {0, y[i] * P.ratio_hi + mulhi64(y[i], P.ratio_lo)};
                    add_to(frac, f);
                }
            }
            U128 half = {0, 1ull << 63};
            add_to(frac, half);
            v = frac.hi;
        }
        for (int t = 0; t < ba.n_dst; t++) {
            U128 acc = {0, 0};
#pragma unroll
            for (int i = 0; i < MAXS; i++)
                if (i < ba.n_src) mac(acc, y[i], s_mat[i * ba.n_dst + t]);
            const PrimeConst P = pc[ba.dst_pid[t]];
            uint64_t r = reduce_u128(acc, P);
            if (ba.dst_corr) r = sub_mod(r, mul_mod(v, ba.dst_corr[t], P), P.q);
            out[(long long)ba.dst_slot[t] * n + x] = r;
        }
    }
}

// ---------------------------------------------------------------------
// key-switch inner product: acc_r[t] = sum_j ext_j[t] * key[j][r][pid(t)]
// ext: [beta][ne][N] ; key: [dnum][2][n_primes][N] ; acc: [2][ne][N]
// ---------------------------------------------------------------------
__global__ void k_ks_inner(const uint64_t *__restrict__ ext, const uint64_t *__restrict__ key,
                           uint64_t *__restrict__ acc, const PrimeConst *__restrict__ pc,
                           int log_n, int ne, int level, int L, int n_primes, int beta) {
    const long long n = 1ll << log_n;
    const long long total = (long long)ne * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(x >> log_n);
        const long long off = x & (n - 1);
        const int pid = t <= level ? t : t + (L - level);
        U128 a0 = {0, 0}, a1 = {0, 0};
        for (int j = 0; j < beta; j++) {
            const uint64_t e = ext[(long long)j * total + x];
            const uint64_t *kj = key + ((long long)j * 2 * n_primes + pid) * n + off;
            mac(a0, e, kj[0]);
            mac(a1, e, kj[(long long)n_primes * n]);
        }
        const PrimeConst P = pc[pid];
        acc[x] = reduce_u128(a0, P);
        acc[total + x] = reduce_u128(a1, P);
    }
}

// ModDown combine: out[r][i] = add_r[i] + (acc[r][i] - conv[r][i]) * P^-1 mod q_i
// add_r may be null (then just the quotient); r in {0,1}
__global__ void k_moddown_combine(const uint64_t *__restrict__ acc, long long acc_pstride,
                                  const uint64_t *__restrict__ conv,
                                  const uint64_t *__restrict__ add0,
                                  const uint64_t *__restrict__ add1, LimbConsts pinv,
                                  uint64_t *__restrict__ out0, uint64_t *__restrict__ out1,
                                  const PrimeConst *__restrict__ pc, int log_n, int nl) {
    const long long n = 1ll << log_n;
    const long long ps = (long long)nl * n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < 2 * ps;
         x += (long long)gridDim.x * blockDim.x) {
        const int r = x >= ps;
        const long long xi = x - r * ps;
        const int i = (int)(xi >> log_n);
        const uint64_t q = pc[i].q;
        uint64_t v = sub_mod(acc[r * acc_pstride + xi], conv[x], q);
        v = mul_shoup(v, pinv.w[i], pinv.ws[i], q);
        const uint64_t *ad = r ? add1 : add0;
        if (ad) v = add_mod(v, ad[xi], q);
        (r ? out1 : out0)[xi] = v;
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

// square (NTT domain) of s over all primes: relinearisation source key
__global__ void k_square(const uint64_t *__restrict__ s, uint64_t *__restrict__ out,
                         const PrimeConst *__restrict__ pc, int log_n, int n_limbs) {
    const long long n = 1ll << log_n;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < (long long)n_limbs * n;
         x += (long long)gridDim.x * blockDim.x)
        out[x] = mul_mod(s[x], s[x], pc[x >> log_n]);
}
