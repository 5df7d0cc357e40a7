/*
 * ckks_oracle.c -- CPU restatement of the RNS-CKKS primitives on the
 * ranking / order-statistics / sorting hot path.  TEST INFRASTRUCTURE ONLY:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the CPU baseline.
 *
 * Parity status: the reference (/root/reference, arXiv 2412.15126 "slotrank")
 * is a cleartext simulator with NO ciphertext arithmetic (reference
 * pkg/src/slotrank/engine.py:1-10); the paper's CKKS ran on an
 * unvendored, unpinned OpenFHE.  There is therefore no
 * reference ciphertext to pin these limbs against: at the ciphertext level
 * this oracle is "parity unpinned" and restates textbook RNS-CKKS (Cheon-Han-
 * Kim-Kim-Song SAC'18 RNS variant; Han-Ki hybrid key switching).  It is pinned
 * at the slot level instead: decrypting its outputs must reproduce the
 * reference simulator's slots (engine.py:190-251) for the same circuit, which
 * tests/test_oracle_*.py check against golden fixtures made from the reference.
 *
 * Everything here is written for obviousness: radix-2 loops and one exact
 * 128-by-64-bit division per general product.  Two standard CPU techniques keep
 * it an honest baseline for bench.py's cpu_baseline / reference arm (a CPU CKKS
 * library does both): the transforms multiply by their precomputed twiddles
 * with Shoup's method (w' = floor(w 2^64 / q), two multiplications and one
 * conditional subtraction, the same canonical result), and on x86-64 the
 * general product's remainder is the hardware divq instead of the __umodti3
 * library call.  OpenMP only splits independent limbs.
 *
 * Conventions shared with the CUDA library (include/slotrank_b200.h):
 *   - prime table: ids 0..L are Q primes (q_0 60-bit base, q_1..q_L scaling),
 *     ids L+1..L+K are the special primes P;
 *   - a ciphertext at level l is uint64[2][l+1][N], limb i under prime i,
 *     every limb in NTT form, values canonical in [0, q);
 *   - an extended polynomial at level l is uint64[l+1+K][N]: limb j < l+1 is
 *     prime j, limb l+1+k is special prime L+1+k;
 *   - forward NTT: natural-order coefficients -> evaluations at
 *     psi^(2*brv(k)+1) in slot k (bit-reversed), psi from params.root_of_unity;
 *   - evaluation keys: uint64[dnum][2][L+1+K][N] indexed by prime id.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define ORC_MAX_PRIMES 128

typedef struct {
    int log_n, n;
    int n_q, n_p, dnum, alpha;
    int n_primes;
    uint64_t prime[ORC_MAX_PRIMES];
    uint64_t *psi_brv[ORC_MAX_PRIMES];  /* psi^brv(k) */
    uint64_t *ipsi_brv[ORC_MAX_PRIMES]; /* psi^-brv(k) */
    uint64_t *psi_sh[ORC_MAX_PRIMES];   /* floor(psi^brv(k) 2^64 / q) */
    uint64_t *ipsi_sh[ORC_MAX_PRIMES];  /* floor(psi^-brv(k) 2^64 / q) */
    uint64_t n_inv[ORC_MAX_PRIMES], n_inv_sh[ORC_MAX_PRIMES];
} orc_ctx;

/* ------------------------------------------------------------------ */
/* scalar modular arithmetic                                           */
/* ------------------------------------------------------------------ */

/* a b mod q for a, b < q: the quotient is below q < 2^64, so the 128-by-64-bit
 * hardware division cannot overflow */
static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
#if defined(__x86_64__) && !defined(ORC_NO_ASM)
    if (a < q && b < q) {
        uint64_t lo, hi, quo, rem;
        __asm__("mulq %3" : "=a"(lo), "=d"(hi) : "a"(a), "rm"(b) : "cc");
        __asm__("divq %4" : "=a"(quo), "=d"(rem) : "a"(lo), "d"(hi), "rm"(q) : "cc");
        (void)quo;
        return rem;
    }
#endif
    return (uint64_t)(((u128)a * b) % q);
}
/* x mod q for any 128-bit x (two hardware divisions: the high word first) */
static inline uint64_t mod128(u128 x, uint64_t q) {
#if defined(__x86_64__) && !defined(ORC_NO_ASM)
    uint64_t hi = (uint64_t)(x >> 64) % q, lo = (uint64_t)x, quo, rem;
    __asm__("divq %4" : "=a"(quo), "=d"(rem) : "a"(lo), "d"(hi), "rm"(q) : "cc");
    (void)quo;
    return rem;
#else
    return (uint64_t)(x % q);
#endif
}
/* Shoup: a w mod q for a < q with ws = floor(w 2^64 / q); exact, canonical */
static inline uint64_t shoup_const(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static inline uint64_t mulmod_shoup(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t hi = (uint64_t)(((u128)a * ws) >> 64);
    uint64_t r = a * w - hi * q; /* in [0, 2q) */
    return r >= q ? r - q : r;
}
static inline uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
static inline uint64_t submod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static inline uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); }

static inline uint32_t brv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) {
        r = (r << 1) | (x & 1);
        x >>= 1;
    }
    return r;
}

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    for (int i = 0; i < c->n_primes; i++) {
        free(c->psi_brv[i]);
        free(c->ipsi_brv[i]);
        free(c->psi_sh[i]);
        free(c->ipsi_sh[i]);
    }
    free(c);
}

orc_ctx *orc_create(int log_n, const uint64_t *primes, const uint64_t *roots, int n_q, int n_p,
                    int dnum) {
    if (n_q + n_p > ORC_MAX_PRIMES || n_q < 1 || dnum < 1) return NULL;
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->log_n = log_n;
    c->n = 1 << log_n;
    c->n_q = n_q;
    c->n_p = n_p;
    c->dnum = dnum;
    c->alpha = (n_q + dnum - 1) / dnum;
    c->n_primes = n_q + n_p;
    for (int i = 0; i < c->n_primes; i++) {
        uint64_t q = primes[i], psi = roots[i], ipsi = invmod(psi, q);
        c->prime[i] = q;
        c->psi_brv[i] = (uint64_t *)malloc(sizeof(uint64_t) * c->n);
        c->ipsi_brv[i] = (uint64_t *)malloc(sizeof(uint64_t) * c->n);
        uint64_t p = 1, ip = 1;
        for (int k = 0; k < c->n; k++) {
            uint32_t r = brv((uint32_t)k, log_n);
            c->psi_brv[i][r] = p;
            c->ipsi_brv[i][r] = ip;
            p = mulmod(p, psi, q);
            ip = mulmod(ip, ipsi, q);
        }
        c->psi_sh[i] = (uint64_t *)malloc(sizeof(uint64_t) * c->n);
        c->ipsi_sh[i] = (uint64_t *)malloc(sizeof(uint64_t) * c->n);
        for (int k = 0; k < c->n; k++) {
            c->psi_sh[i][k] = shoup_const(c->psi_brv[i][k], q);
            c->ipsi_sh[i][k] = shoup_const(c->ipsi_brv[i][k], q);
        }
        c->n_inv[i] = invmod((uint64_t)c->n, q);
        c->n_inv_sh[i] = shoup_const(c->n_inv[i], q);
    }
    return c;
}

/* prime id of limb j of an extended polynomial at level l */
static inline int ext_prime(const orc_ctx *c, int level, int j) {
    return j <= level ? j : c->n_q + (j - level - 1);
}

/* ------------------------------------------------------------------ */
/* NTT (one limb)                                                      */
/* ------------------------------------------------------------------ */

static void ntt_limb(const orc_ctx *c, uint64_t *a, int pid) {
    const uint64_t q = c->prime[pid];
    const uint64_t *w = c->psi_brv[pid], *wsh = c->psi_sh[pid];
    const int n = c->n;
    for (int m = 1, t = n >> 1; m < n; m <<= 1, t >>= 1) {
        for (int i = 0; i < m; i++) {
            uint64_t wi = w[m + i], ws = wsh[m + i];
            int j1 = 2 * i * t;
            for (int j = j1; j < j1 + t; j++) {
                uint64_t u = a[j], v = mulmod_shoup(a[j + t], wi, ws, q);
                a[j] = addmod(u, v, q);
                a[j + t] = submod(u, v, q);
            }
        }
    }
}

static void intt_limb(const orc_ctx *c, uint64_t *a, int pid) {
    const uint64_t q = c->prime[pid];
    const uint64_t *w = c->ipsi_brv[pid], *wsh = c->ipsi_sh[pid];
    const int n = c->n;
    for (int m = n >> 1, t = 1; m >= 1; m >>= 1, t <<= 1) {
        for (int i = 0; i < m; i++) {
            uint64_t wi = w[m + i], ws = wsh[m + i];
            int j1 = 2 * i * t;
            for (int j = j1; j < j1 + t; j++) {
                uint64_t u = a[j], v = a[j + t];
                a[j] = addmod(u, v, q);
                a[j + t] = mulmod_shoup(submod(u, v, q), wi, ws, q);
            }
        }
    }
    for (int j = 0; j < n; j++) a[j] = mulmod_shoup(a[j], c->n_inv[pid], c->n_inv_sh[pid], q);
}

/* a: uint64[nl][N], limb k under prime prime_ids[k] */
void orc_ntt(const orc_ctx *c, uint64_t *a, int nl, const int *prime_ids, int inverse) {
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < nl; k++) {
        uint64_t *limb = a + (size_t)k * c->n;
        if (inverse)
            intt_limb(c, limb, prime_ids[k]);
        else
            ntt_limb(c, limb, prime_ids[k]);
    }
}

/* ------------------------------------------------------------------ */
/* elementwise ciphertext ops (both polys, limbs 0..level)             */
/* ------------------------------------------------------------------ */

/* op: 0 add, 1 sub, 2 negate (b ignored) */
void orc_addsub(const orc_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out, int level,
                int op) {
    const int n = c->n, nl = level + 1;
#pragma omp parallel for
    for (int pl = 0; pl < 2 * nl; pl++) {
        const uint64_t q = c->prime[pl % nl];
        const size_t off = (size_t)pl * n;
        for (int j = 0; j < n; j++) {
            uint64_t x = a[off + j];
            if (op == 0)
                out[off + j] = addmod(x, b[off + j], q);
            else if (op == 1)
                out[off + j] = submod(x, b[off + j], q);
            else
                out[off + j] = x ? q - x : 0;
        }
    }
}

/* add the constant polynomial with residues k[i] to poly 0 (NTT form:
 * every evaluation of a constant polynomial is the constant) */
void orc_add_const(const orc_ctx *c, const uint64_t *a, const uint64_t *k, uint64_t *out,
                   int level) {
    const int n = c->n, nl = level + 1;
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->prime[i];
        for (int j = 0; j < n; j++) {
            out[(size_t)i * n + j] = addmod(a[(size_t)i * n + j], k[i], q);
            out[(size_t)(nl + i) * n + j] = a[(size_t)(nl + i) * n + j];
        }
    }
}

/* out = a * k (residue k[i] per limb), both polys; a may have a larger poly
 * stride (src_limbs >= level+1) so a higher-level ciphertext can be read
 * as its level-`level` modulus-dropped view. */
void orc_mul_const(const orc_ctx *c, const uint64_t *a, int src_limbs, const uint64_t *k,
                   uint64_t *out, int level) {
    const int n = c->n, nl = level + 1;
#pragma omp parallel for
    for (int pl = 0; pl < 2 * nl; pl++) {
        int p = pl / nl, i = pl % nl;
        const uint64_t q = c->prime[i];
        const uint64_t *src = a + ((size_t)p * src_limbs + i) * n;
        uint64_t *dst = out + ((size_t)p * nl + i) * n;
        for (int j = 0; j < n; j++) dst[j] = mulmod(src[j], k[i], q);
    }
}

/* out = a * pt, pt: uint64[level+1][N] NTT form */
void orc_mul_plain(const orc_ctx *c, const uint64_t *a, const uint64_t *pt, uint64_t *out,
                   int level) {
    const int n = c->n, nl = level + 1;
#pragma omp parallel for
    for (int pl = 0; pl < 2 * nl; pl++) {
        int i = pl % nl;
        const uint64_t q = c->prime[i];
        const size_t off = (size_t)pl * n;
        for (int j = 0; j < n; j++) out[off + j] = mulmod(a[off + j], pt[(size_t)i * n + j], q);
    }
}

/* d: uint64[3][level+1][N]; d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 */
void orc_tensor(const orc_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *d, int level) {
    const int n = c->n, nl = level + 1;
    const size_t ps = (size_t)nl * n;
#pragma omp parallel for
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->prime[i];
        for (int j = 0; j < n; j++) {
            size_t x = (size_t)i * n + j;
            uint64_t a0 = a[x], a1 = a[ps + x], b0 = b[x], b1 = b[ps + x];
            d[x] = mulmod(a0, b0, q);
            d[ps + x] = addmod(mulmod(a0, b1, q), mulmod(a1, b0, q), q);
            d[2 * ps + x] = mulmod(a1, b1, q);
        }
    }
}

/* ------------------------------------------------------------------ */
/* rescale: level l -> l-1, rounding division by q_l                   */
/* ------------------------------------------------------------------ */

void orc_rescale(const orc_ctx *c, const uint64_t *a, uint64_t *out, int level) {
    const int n = c->n, nl = level + 1;
    const uint64_t ql = c->prime[level];
    uint64_t *top = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (int p = 0; p < 2; p++) {
        memcpy(top, a + ((size_t)p * nl + level) * n, sizeof(uint64_t) * n);
        intt_limb(c, top, level);
#pragma omp parallel for
        for (int i = 0; i < level; i++) {
            const uint64_t q = c->prime[i];
            const uint64_t qinv = invmod(ql % q, q);
            const uint64_t ql_mod = ql % q;
            uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * n);
            for (int j = 0; j < n; j++) {
                uint64_t v = top[j];
                /* centred representative: v > q_l/2 means v - q_l < 0 */
                t[j] = v > (ql >> 1) ? submod(v % q, ql_mod, q) : v % q;
            }
            ntt_limb(c, t, i);
            const uint64_t *src = a + ((size_t)p * nl + i) * n;
            uint64_t *dst = out + ((size_t)p * level + i) * n;
            for (int j = 0; j < n; j++) dst[j] = mulmod(submod(src[j], t[j], q), qinv, q);
            free(t);
        }
    }
    free(top);
}

/* ------------------------------------------------------------------ */
/* Galois automorphism X -> X^g in the NTT domain                      */
/* ------------------------------------------------------------------ */

static inline uint32_t auto_index(uint32_t k, uint64_t g, int log_n) {
    const uint64_t two_n_mask = (2ull << log_n) - 1;
    uint64_t e = (((uint64_t)brv(k, log_n) * 2 + 1) * g) & two_n_mask;
    return brv((uint32_t)((e - 1) >> 1), log_n);
}

/* a: n_polys x nl limbs; out[k] = a[pi(k)] in every limb */
void orc_automorph(const orc_ctx *c, const uint64_t *a, uint64_t *out, int n_limbs_total,
                   uint64_t galois) {
    const int n = c->n;
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * n);
    for (int k = 0; k < n; k++) perm[k] = auto_index((uint32_t)k, galois, c->log_n);
#pragma omp parallel for
    for (int l = 0; l < n_limbs_total; l++)
        for (int k = 0; k < n; k++) out[(size_t)l * n + k] = a[(size_t)l * n + perm[k]];
    free(perm);
}

/* ------------------------------------------------------------------ */
/* hybrid key switching                                                */
/* ------------------------------------------------------------------ */

static inline uint32_t auto_index(uint32_t k, uint64_t g, int log_n);

/* ModUp of every digit of d (uint64[level+1][N], NTT form): ext is
 * uint64[beta][level+1+K][N], digit jd's limbs over the extended basis
 * Q_level u P in NTT form (its own alpha limbs are copied). */
static void modup_digits(const orc_ctx *c, const uint64_t *d, int level, uint64_t *ext_all) {
    const int n = c->n, nl = level + 1, K = c->n_p, ne = nl + K;
    const int alpha = c->alpha, beta = (nl + alpha - 1) / alpha;
    uint64_t *dc = (uint64_t *)malloc(sizeof(uint64_t) * nl * n);
    memcpy(dc, d, sizeof(uint64_t) * nl * n);
#pragma omp parallel for schedule(dynamic)
    for (int i = 0; i < nl; i++) intt_limb(c, dc + (size_t)i * n, i);
    for (int jd = 0; jd < beta; jd++) {
        uint64_t *ext = ext_all + (size_t)jd * ne * n;
        const int g0 = jd * alpha, g1 = (jd + 1) * alpha < nl ? (jd + 1) * alpha : nl;
        /* y_i = [d_i * (Qhat_i)^-1]_{q_i},  Qhat_i = prod_{G\i} q */
        uint64_t *y = (uint64_t *)malloc(sizeof(uint64_t) * (g1 - g0) * n);
#pragma omp parallel for
        for (int i = g0; i < g1; i++) {
            const uint64_t q = c->prime[i];
            uint64_t qhat = 1;
            for (int m = g0; m < g1; m++)
                if (m != i) qhat = mulmod(qhat, c->prime[m] % q, q);
            const uint64_t qhinv = invmod(qhat, q);
            for (int j = 0; j < n; j++) y[(size_t)(i - g0) * n + j] = mulmod(dc[(size_t)i * n + j], qhinv, q);
        }
#pragma omp parallel for schedule(dynamic)
        for (int t = 0; t < ne; t++) {
            const int pid = ext_prime(c, level, t);
            uint64_t *dst = ext + (size_t)t * n;
            if (t >= g0 && t < g1) {
                memcpy(dst, d + (size_t)t * n, sizeof(uint64_t) * n);
                continue;
            }
            const uint64_t p = c->prime[pid];
            uint64_t coef[ORC_MAX_PRIMES];
            for (int i = g0; i < g1; i++) {
                uint64_t v = 1;
                for (int m = g0; m < g1; m++)
                    if (m != i) v = mulmod(v, c->prime[m] % p, p);
                coef[i - g0] = v;
            }
            for (int j = 0; j < n; j++) {
                u128 s = 0;
                for (int i = g0; i < g1; i++) s += (u128)y[(size_t)(i - g0) * n + j] * coef[i - g0];
                dst[j] = mod128(s, p);
            }
            ntt_limb(c, dst, pid);
        }
        free(y);
    }
    free(dc);
}

/* acc[r] = sum_jd sigma_g(ext_jd) * key[jd][r] over the extended basis
 * (uint64[2][level+1+K][N]); galois != 1 applies X -> X^galois to the extended
 * digits as a gather of NTT slots (after the base extension, so rotations of
 * one ciphertext share it). */
static void ks_inner_from_ext(const orc_ctx *c, const uint64_t *ext_all, const uint64_t *key,
                              int level, uint64_t galois, uint64_t *acc) {
    const int n = c->n, nl = level + 1, K = c->n_p, ne = nl + K, np_all = c->n_primes;
    const int alpha = c->alpha, beta = (nl + alpha - 1) / alpha;
    uint32_t *perm = NULL;
    if (galois != 1) {
        perm = (uint32_t *)malloc(sizeof(uint32_t) * n);
        for (int j = 0; j < n; j++) perm[j] = auto_index((uint32_t)j, galois, c->log_n);
    }
    memset(acc, 0, sizeof(uint64_t) * 2 * ne * n);
#pragma omp parallel for schedule(dynamic)
    for (int t = 0; t < ne; t++) {
        const int pid = ext_prime(c, level, t);
        const uint64_t p = c->prime[pid];
        for (int jd = 0; jd < beta; jd++) {
            const uint64_t *e = ext_all + ((size_t)jd * ne + t) * n;
            for (int r = 0; r < 2; r++) {
                const uint64_t *kk = key + (((size_t)jd * 2 + r) * np_all + pid) * n;
                uint64_t *ac = acc + ((size_t)r * ne + t) * n;
                if (perm)
                    for (int j = 0; j < n; j++) ac[j] = addmod(ac[j], mulmod(e[perm[j]], kk[j], p), p);
                else
                    for (int j = 0; j < n; j++) ac[j] = addmod(ac[j], mulmod(e[j], kk[j], p), p);
            }
        }
    }
    free(perm);
}

/* Base-extend d digit by digit and take the inner product with the switching
 * key: acc[r] over the extended basis Q_level u P (uint64[2][level+1+K][N]). */
static void ks_inner_acc(const orc_ctx *c, const uint64_t *d, const uint64_t *key, int level,
                         uint64_t galois, uint64_t *acc) {
    const int n = c->n, nl = level + 1, ne = nl + c->n_p;
    const int beta = (nl + c->alpha - 1) / c->alpha;
    uint64_t *ext = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)beta * ne * n);
    modup_digits(c, d, level, ext);
    ks_inner_from_ext(c, ext, key, level, galois, acc);
    free(ext);
}

/* Exact ModDown over a special basis S (ns limbs, prime ids sid[]):
 * xs[k] (NTT form, under prime sid[k]); xq[i] (NTT form, i < no, prime i);
 * out[i] = (xq_i - conv_S->q_i(xs)) * (prod S)^-1 mod q_i, with the centred
 * conversion conv = sum_k z_k [S/s_k]_{q_i} - v [prod S]_{q_i},
 * z_k = [x_k (S/s_k)^-1]_{s_k}, v = round(sum_k z_k / s_k) evaluated in 64.64
 * fixed point (f_k = z_k R1 + hi(z_k R0), R = floor(2^128/s_k)) -- the same
 * integer recipe as the GPU, so the rounding decision is bit-identical. */
static void moddown_exact(const orc_ctx *c, const uint64_t *xq, int no, const uint64_t *xs, int ns,
                          const int *sid, uint64_t *out) {
    const int n = c->n;
    uint64_t *z = (uint64_t *)malloc(sizeof(uint64_t) * ns * n);
#pragma omp parallel for
    for (int k = 0; k < ns; k++) {
        const uint64_t p = c->prime[sid[k]];
        memcpy(z + (size_t)k * n, xs + (size_t)k * n, sizeof(uint64_t) * n);
        intt_limb(c, z + (size_t)k * n, sid[k]);
        uint64_t shat = 1;
        for (int m = 0; m < ns; m++)
            if (m != k) shat = mulmod(shat, c->prime[sid[m]] % p, p);
        const uint64_t shinv = invmod(shat, p);
        for (int j = 0; j < n; j++) z[(size_t)k * n + j] = mulmod(z[(size_t)k * n + j], shinv, p);
    }
    uint64_t *vr = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint64_t r1[ORC_MAX_PRIMES], r0[ORC_MAX_PRIMES];
    for (int k = 0; k < ns; k++) {
        const u128 R = (~(u128)0) / c->prime[sid[k]];
        r1[k] = (uint64_t)(R >> 64);
        r0[k] = (uint64_t)R;
    }
#pragma omp parallel for
    for (int j = 0; j < n; j++) {
        u128 frac = 0;
        for (int k = 0; k < ns; k++) {
            const uint64_t zk = z[(size_t)k * n + j];
            frac += (u128)(uint64_t)(zk * r1[k] + (uint64_t)(((u128)zk * r0[k]) >> 64));
        }
        vr[j] = (uint64_t)((frac + ((u128)1 << 63)) >> 64);
    }
#pragma omp parallel for
    for (int i = 0; i < no; i++) {
        const uint64_t q = c->prime[i];
        uint64_t coef[ORC_MAX_PRIMES];
        uint64_t smod = 1;
        for (int k = 0; k < ns; k++) {
            uint64_t v = 1;
            for (int m = 0; m < ns; m++)
                if (m != k) v = mulmod(v, c->prime[sid[m]] % q, q);
            coef[k] = v;
            smod = mulmod(smod, c->prime[sid[k]] % q, q);
        }
        const uint64_t sinv = invmod(smod, q);
        uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * n);
        for (int j = 0; j < n; j++) {
            u128 s = 0;
            for (int k = 0; k < ns; k++) s += (u128)z[(size_t)k * n + j] * coef[k];
            t[j] = submod(mod128(s, q), mulmod(vr[j] % q, smod, q), q);
        }
        ntt_limb(c, t, i);
        for (int j = 0; j < n; j++)
            out[(size_t)i * n + j] = mulmod(submod(xq[(size_t)i * n + j], t[j], q), sinv, q);
        free(t);
    }
    free(vr);
    free(z);
}

/* out0/out1: uint64[level+1][N] NTT form, <(out0,out1),(1,s)> ~ sigma_g(d) * s_from
 * (galois = 1: plain key switch).  Exact ModDown by P. */
void orc_keyswitch_g(const orc_ctx *c, const uint64_t *d, const uint64_t *key, uint64_t *out0,
                     uint64_t *out1, int level, uint64_t galois) {
    const int n = c->n, nl = level + 1, K = c->n_p, ne = nl + K;
    uint64_t *acc = (uint64_t *)malloc(sizeof(uint64_t) * 2 * ne * n);
    ks_inner_acc(c, d, key, level, galois, acc);
    int sid[ORC_MAX_PRIMES];
    for (int k = 0; k < K; k++) sid[k] = c->n_q + k;
    for (int r = 0; r < 2; r++) {
        const uint64_t *a = acc + (size_t)r * ne * n;
        moddown_exact(c, a, nl, a + (size_t)nl * n, K, sid, r ? out1 : out0);
    }
    free(acc);
}

/* HMult with the rescale fused into the key switch:
 * X_r = acc_r + P d_r (d = tensor(a, b), acc = key switch accumulator of d2),
 * out_r = round(X_r / (P q_level)) over Q_{level-1}: one exact ModDown over the
 * special basis P u {q_level}.  Output at level-1. */
void orc_mul_relin_rescale(const orc_ctx *c, const uint64_t *a, const uint64_t *b,
                           const uint64_t *rlk, uint64_t *out, int level) {
    const int n = c->n, nl = level + 1, K = c->n_p, ne = nl + K;
    const size_t ps = (size_t)nl * n;
    uint64_t *d = (uint64_t *)malloc(sizeof(uint64_t) * 3 * ps);
    orc_tensor(c, a, b, d, level);
    uint64_t *acc = (uint64_t *)malloc(sizeof(uint64_t) * 2 * ne * n);
    ks_inner_acc(c, d + 2 * ps, rlk, level, 1, acc);
    int sid[ORC_MAX_PRIMES];
    for (int k = 0; k < K; k++) sid[k] = c->n_q + k;
    sid[K] = level;
    uint64_t *xs = (uint64_t *)malloc(sizeof(uint64_t) * (K + 1) * n);
    uint64_t *xq = (uint64_t *)malloc(sizeof(uint64_t) * nl * n);
    for (int r = 0; r < 2; r++) {
        const uint64_t *ar = acc + (size_t)r * ne * n;
        const uint64_t *dr = d + (size_t)r * ps;
        /* X over Q_level: acc + P d ; over P: acc */
#pragma omp parallel for
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->prime[i];
            uint64_t pm = 1;
            for (int k = 0; k < K; k++) pm = mulmod(pm, c->prime[c->n_q + k] % q, q);
            for (int j = 0; j < n; j++)
                xq[(size_t)i * n + j] = addmod(ar[(size_t)i * n + j], mulmod(dr[(size_t)i * n + j], pm, q), q);
        }
        memcpy(xs, ar + (size_t)nl * n, sizeof(uint64_t) * K * n);
        memcpy(xs + (size_t)K * n, xq + (size_t)level * n, sizeof(uint64_t) * n);
        moddown_exact(c, xq, level, xs, K + 1, sid, out + (size_t)r * level * n);
    }
    free(xq);
    free(xs);
    free(acc);
    free(d);
}

void orc_keyswitch(const orc_ctx *c, const uint64_t *d, const uint64_t *key, uint64_t *out0,
                   uint64_t *out1, int level) {
    orc_keyswitch_g(c, d, key, out0, out1, level, 1);
}

/* out = tensor(a, b) relinearised (no rescale), level unchanged */
void orc_mul_relin(const orc_ctx *c, const uint64_t *a, const uint64_t *b, const uint64_t *rlk,
                   uint64_t *out, int level) {
    const int n = c->n, nl = level + 1;
    const size_t ps = (size_t)nl * n;
    uint64_t *d = (uint64_t *)malloc(sizeof(uint64_t) * 3 * ps);
    orc_tensor(c, a, b, d, level);
    uint64_t *u = (uint64_t *)malloc(sizeof(uint64_t) * 2 * ps);
    orc_keyswitch(c, d + 2 * ps, rlk, u, u + ps, level);
#pragma omp parallel for
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->prime[i];
        for (int j = 0; j < n; j++) {
            size_t x = (size_t)i * n + j;
            out[x] = addmod(d[x], u[x], q);
            out[ps + x] = addmod(d[ps + x], u[ps + x], q);
        }
    }
    free(u);
    free(d);
}

/* out = rotate(a) by Galois element g with key for sigma_g(s) -> s:
 * (sigma_g(c0) + u0, u1) with (u0, u1) = keyswitch_g(c1) */
void orc_rotate(const orc_ctx *c, const uint64_t *a, const uint64_t *gkey, uint64_t *out,
                int level, uint64_t galois) {
    const int n = c->n, nl = level + 1;
    const size_t ps = (size_t)nl * n;
    uint64_t *r0 = (uint64_t *)malloc(sizeof(uint64_t) * ps);
    orc_automorph(c, a, r0, nl, galois);
    uint64_t *u = (uint64_t *)malloc(sizeof(uint64_t) * 2 * ps);
    orc_keyswitch_g(c, a + ps, gkey, u, u + ps, level, galois);
#pragma omp parallel for
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->prime[i];
        for (int j = 0; j < n; j++) {
            size_t x = (size_t)i * n + j;
            out[x] = addmod(r0[x], u[x], q);
            out[ps + x] = u[ps + x];
        }
    }
    free(u);
    free(r0);
}

/* n_rot rotations of one ciphertext sharing one base extension (hoisting):
 * outs[r] = orc_rotate(a, gkeys[r], galois[r]) bit for bit. */
void orc_rotate_hoisted(const orc_ctx *c, const uint64_t *a, const uint64_t *const *gkeys,
                        const uint64_t *galois, int n_rot, uint64_t *const *outs, int level) {
    const int n = c->n, nl = level + 1, K = c->n_p, ne = nl + K;
    const int beta = (nl + c->alpha - 1) / c->alpha;
    const size_t ps = (size_t)nl * n;
    uint64_t *ext = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)beta * ne * n);
    modup_digits(c, a + ps, level, ext);
    uint64_t *acc = (uint64_t *)malloc(sizeof(uint64_t) * 2 * ne * n);
    uint64_t *r0 = (uint64_t *)malloc(sizeof(uint64_t) * ps);
    uint64_t *u0 = (uint64_t *)malloc(sizeof(uint64_t) * ps);
    int sid[ORC_MAX_PRIMES];
    for (int k = 0; k < K; k++) sid[k] = c->n_q + k;
    for (int r = 0; r < n_rot; r++) {
        uint64_t *out = outs[r];
        ks_inner_from_ext(c, ext, gkeys[r], level, galois[r], acc);
        moddown_exact(c, acc, nl, acc + (size_t)nl * n, K, sid, u0);
        moddown_exact(c, acc + (size_t)ne * n, nl, acc + (size_t)ne * n + (size_t)nl * n, K, sid, out + ps);
        orc_automorph(c, a, r0, nl, galois[r]);
#pragma omp parallel for
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->prime[i];
            for (int j = 0; j < n; j++) {
                size_t x = (size_t)i * n + j;
                out[x] = addmod(r0[x], u0[x], q);
            }
        }
    }
    free(u0);
    free(r0);
    free(acc);
    free(ext);
}

/* ------------------------------------------------------------------ */
/* randomness, keys, encryption                                        */
/* ------------------------------------------------------------------ */

/* counter-based generator: word(seed, stream, ctr) -- restated bit for bit
 * by k_uniform in csrc/kernels.cuh so uniform polynomials agree between CPU and GPU */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static inline uint64_t rand_word(uint64_t seed, uint64_t stream, uint64_t ctr) {
    return mix64(mix64(seed ^ mix64(stream)) + ctr);
}
uint64_t orc_uniform(uint64_t seed, uint64_t stream, uint64_t idx, uint64_t q) {
    u128 x = ((u128)rand_word(seed, stream, 2 * idx) << 64) | rand_word(seed, stream, 2 * idx + 1);
    return (uint64_t)(x % q);
}

/* fill uint64[nl][N] (limb k under prime prime_ids[k]) with uniform values;
 * the stream for limb k is stream_base + prime_ids[k] */
void orc_uniform_poly(const orc_ctx *c, uint64_t *a, int nl, const int *prime_ids, uint64_t seed,
                      uint64_t stream_base) {
    for (int k = 0; k < nl; k++) {
        const int pid = prime_ids[k];
        for (int j = 0; j < c->n; j++)
            a[(size_t)k * c->n + j] = orc_uniform(seed, stream_base + (uint64_t)pid, (uint64_t)j, c->prime[pid]);
    }
}

/* small signed coefficients -> NTT-form residues for the given primes */
void orc_small_to_ntt(const orc_ctx *c, const int64_t *v, uint64_t *out, int nl,
                      const int *prime_ids) {
#pragma omp parallel for
    for (int k = 0; k < nl; k++) {
        const int pid = prime_ids[k];
        const uint64_t q = c->prime[pid];
        uint64_t *dst = out + (size_t)k * c->n;
        for (int j = 0; j < c->n; j++) {
            int64_t x = v[j];
            dst[j] = x >= 0 ? (uint64_t)x % q : q - ((uint64_t)(-x) % q);
            if (dst[j] == q) dst[j] = 0;
        }
        ntt_limb(c, dst, pid);
    }
}

/* Switching key from s_from to s (both NTT form over all n_q+n_p primes):
 *   key[j][1] = a_j (uniform, stream (key_id, j)),
 *   key[j][0] = -a_j s + e_j + [prime in digit j] * P * s_from.
 * e: int64[dnum][N] small coefficients. */
void orc_keygen(const orc_ctx *c, const uint64_t *s_ntt, const uint64_t *sfrom_ntt,
                const int64_t *e, uint64_t seed, uint64_t key_id, uint64_t *key) {
    const int n = c->n, np_all = c->n_primes;
    int *ids = (int *)malloc(sizeof(int) * np_all);
    for (int i = 0; i < np_all; i++) ids[i] = i;
    uint64_t *en = (uint64_t *)malloc(sizeof(uint64_t) * np_all * n);
    for (int jd = 0; jd < c->dnum; jd++) {
        uint64_t *b = key + ((size_t)jd * 2 + 0) * np_all * n;
        uint64_t *a = key + ((size_t)jd * 2 + 1) * np_all * n;
        orc_uniform_poly(c, a, np_all, ids, seed, ((key_id << 8) | (uint64_t)jd) << 8);
        orc_small_to_ntt(c, e + (size_t)jd * n, en, np_all, ids);
        for (int i = 0; i < np_all; i++) {
            const uint64_t q = c->prime[i];
            uint64_t pm = 1;
            for (int k = 0; k < c->n_p; k++) pm = mulmod(pm, c->prime[c->n_q + k] % q, q);
            const int in_digit = i < c->n_q && i / c->alpha == jd;
            for (int j = 0; j < n; j++) {
                size_t x = (size_t)i * n + j;
                uint64_t v = submod(en[x], mulmod(a[x], s_ntt[x], q), q);
                if (in_digit) v = addmod(v, mulmod(pm, sfrom_ntt[x], q), q);
                b[x] = v;
            }
        }
    }
    free(en);
    free(ids);
}

/* symmetric encryption at level l: c1 = a (stream 0xE0000000+seq), c0 = -a s + e + m.
 * m_ntt / s_ntt / out over limbs 0..level; e: int64[N]. */
void orc_encrypt(const orc_ctx *c, const uint64_t *m_ntt, const uint64_t *s_ntt, const int64_t *e,
                 uint64_t seed, uint64_t seq, uint64_t *out, int level) {
    const int n = c->n, nl = level + 1;
    if (nl < 1) return;
    int *ids = (int *)malloc(sizeof(int) * nl);
    for (int i = 0; i < nl; i++) ids[i] = i;
    uint64_t *c1 = out + (size_t)nl * n;
    orc_uniform_poly(c, c1, nl, ids, seed, (0xE0000000ull + seq) << 8);
    uint64_t *en = (uint64_t *)malloc(sizeof(uint64_t) * nl * n);
    orc_small_to_ntt(c, e, en, nl, ids);
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->prime[i];
        for (int j = 0; j < n; j++) {
            size_t x = (size_t)i * n + j;
            out[x] = addmod(submod(en[x], mulmod(c1[x], s_ntt[x], q), q), m_ntt[x], q);
        }
    }
    free(en);
    free(ids);
}

/* m = c0 + c1 s on limb 0 only, returned in coefficient form, centred */
void orc_decrypt_limb0(const orc_ctx *c, const uint64_t *ct, const uint64_t *s_ntt, int64_t *m,
                       int level) {
    const int n = c->n, nl = level + 1;
    const uint64_t q = c->prime[0];
    uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (int j = 0; j < n; j++) t[j] = addmod(ct[j], mulmod(ct[(size_t)nl * n + j], s_ntt[j], q), q);
    intt_limb(c, t, 0);
    for (int j = 0; j < n; j++) m[j] = t[j] > (q >> 1) ? -(int64_t)(q - t[j]) : (int64_t)t[j];
    free(t);
}
