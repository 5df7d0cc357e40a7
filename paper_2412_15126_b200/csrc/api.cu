// api.cu -- context, tables and the C-ABI of libslotrank_b200.so.
// See include/slotrank_b200.h for the contract and the reference methods
// each entry point realises.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/slotrank_b200.h"
#include "kernels.cuh"
#include "modarith.cuh"
#include "ntt.cuh"

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------
// error handling
// ---------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            return fail(SRK_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,            \
                        cudaGetErrorString(e_));                                      \
    } while (0)

static std::atomic<unsigned long long> g_launches{0};

#define LAUNCHED()                                                                    \
    do {                                                                              \
        g_launches.fetch_add(1, std::memory_order_relaxed);                           \
        cudaError_t e_ = cudaGetLastError();                                          \
        if (e_ != cudaSuccess)                                                        \
            return fail(SRK_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__,            \
                        cudaGetErrorString(e_));                                      \
    } while (0)

#define TRY(x)                 \
    do {                       \
        int r_ = (x);          \
        if (r_ != SRK_OK) return r_; \
    } while (0)

extern "C" const char *srk_last_error(void) { return g_err.c_str(); }
extern "C" int srk_version(void) { return 1; }
// number of kernels this library has launched in this process
extern "C" unsigned long long srk_kernel_launches(void) { return g_launches.load(); }

// ---------------------------------------------------------------------
// host modular helpers
// ---------------------------------------------------------------------
static inline uint64_t hmul(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t hpow(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = hmul(r, b, q);
        b = hmul(b, b, q);
        e >>= 1;
    }
    return r;
}
static inline uint64_t hinv(uint64_t a, uint64_t q) { return hpow(a % q, q - 2, q); }
static inline uint64_t shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static inline uint32_t hbrv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) {
        r = (r << 1) | (x & 1);
        x >>= 1;
    }
    return r;
}

// ---------------------------------------------------------------------
// context
// ---------------------------------------------------------------------
struct BconvPlan {
    uint64_t *mat = nullptr;   // [n_src][n_dst]
    uint64_t *hinv = nullptr;  // [2][n_src]
    int *dst_slot = nullptr;
    int *dst_pid = nullptr;
    uint64_t *dst_corr = nullptr;  // ModDown: [P]_{q_t} for exact rounding
    int n_src = 0, n_dst = 0, src_pid0 = 0;
};

struct srk_ctx {
    int device;
    int log_n, n, n_q, n_p, L, dnum, alpha, n_primes;
    std::vector<uint64_t> primes;
    PrimeConst *d_pc = nullptr;
    uint64_t *d_tw = nullptr, *d_tws = nullptr, *d_itw = nullptr, *d_itws = nullptr;
    std::vector<void *> allocs;
    // modup[level][digit], moddown[level]
    std::vector<std::vector<BconvPlan>> modup;
    std::vector<BconvPlan> moddown;
    LimbConsts lc_pinv;               // P^-1 mod q_i
    LimbConsts lc_pmod;               // P mod prime_i (all primes)
    std::vector<LimbConsts> lc_qlinv; // [level]: q_level^-1 mod q_i
    int ntt_chunk = 128;              // limbs per L2-resident NTT chunk
};

template <typename T>
static int dalloc(srk_ctx *c, T **p, size_t count) {
    void *ptr = nullptr;
    CU(cudaMalloc(&ptr, sizeof(T) * (count ? count : 1)));
    c->allocs.push_back(ptr);
    *p = (T *)ptr;
    return SRK_OK;
}
template <typename T>
static int dupload(srk_ctx *c, T **p, const std::vector<T> &h) {
    TRY(dalloc(c, p, h.size()));
    CU(cudaMemcpy(*p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return SRK_OK;
}

static inline int ext_pid(const srk_ctx *c, int level, int t) {
    return t <= level ? t : t + (c->L - level);
}

static int build_plan(srk_ctx *c, BconvPlan &pl, const std::vector<int> &src_pids,
                      const std::vector<int> &dst_slots, const std::vector<int> &dst_pids,
                      bool exact = false) {
    const int ns = (int)src_pids.size(), nd = (int)dst_pids.size();
    std::vector<uint64_t> mat((size_t)ns * nd), hv(2 * ns);
    for (int i = 0; i < ns; i++) {
        const uint64_t q = c->primes[src_pids[i]];
        uint64_t h = 1;
        for (int m = 0; m < ns; m++)
            if (m != i) h = hmul(h, c->primes[src_pids[m]] % q, q);
        hv[i] = hinv(h, q);
        hv[ns + i] = shoup(hv[i], q);
        for (int t = 0; t < nd; t++) {
            const uint64_t p = c->primes[dst_pids[t]];
            uint64_t v = 1;
            for (int m = 0; m < ns; m++)
                if (m != i) v = hmul(v, c->primes[src_pids[m]] % p, p);
            mat[(size_t)i * nd + t] = v;
        }
    }
    pl.n_src = ns;
    pl.n_dst = nd;
    pl.src_pid0 = src_pids[0];
    TRY(dupload(c, &pl.mat, mat));
    TRY(dupload(c, &pl.hinv, hv));
    TRY(dupload(c, &pl.dst_slot, dst_slots));
    TRY(dupload(c, &pl.dst_pid, dst_pids));
    if (exact) {
        std::vector<uint64_t> corr(nd);
        for (int t = 0; t < nd; t++) {
            const uint64_t p = c->primes[dst_pids[t]];
            uint64_t v = 1;
            for (int m = 0; m < ns; m++) v = hmul(v, c->primes[src_pids[m]] % p, p);
            corr[t] = v;
        }
        TRY(dupload(c, &pl.dst_corr, corr));
    }
    return SRK_OK;
}

static void fill_consts(LimbConsts &lc, const std::vector<uint64_t> &w,
                        const std::vector<uint64_t> &q) {
    memset(&lc, 0, sizeof lc);
    for (size_t i = 0; i < w.size(); i++) {
        lc.w[i] = w[i];
        lc.ws[i] = shoup(w[i], q[i]);
    }
}

extern "C" int srk_ctx_destroy(srk_ctx *c) {
    if (!c) return SRK_OK;
    cudaSetDevice(c->device);
    for (void *p : c->allocs) cudaFree(p);
    delete c;
    return SRK_OK;
}

extern "C" int srk_ctx_create(int device, int log_n, const uint64_t *primes,
                              const uint64_t *roots, int n_q, int n_p, int dnum, srk_ctx **out) {
    if (!out || !primes || !roots) return fail(SRK_EINVAL, "null argument");
    if (log_n < 10 || log_n > 16) return fail(SRK_EINVAL, "log_n must lie in [10, 16]");
    if (n_q < 1 || n_p < 1 || n_q + n_p > SRK_MAXP)
        return fail(SRK_EINVAL, "prime counts out of range");
    if (dnum < 1 || dnum > n_q) return fail(SRK_EINVAL, "dnum out of range");
    CU(cudaSetDevice(device));
    srk_ctx *c = new srk_ctx();
    c->device = device;
    c->log_n = log_n;
    c->n = 1 << log_n;
    c->n_q = n_q;
    c->n_p = n_p;
    c->L = n_q - 1;
    c->dnum = dnum;
    c->alpha = (n_q + dnum - 1) / dnum;
    c->n_primes = n_q + n_p;
    c->primes.assign(primes, primes + c->n_primes);
    if (c->alpha > 16 || n_p > 16) {
        srk_ctx_destroy(c);
        return fail(SRK_EINVAL, "digit size and special prime count must be <= 16");
    }
    const int n = c->n, np = c->n_primes;
    int rc;
    // prime constants
    std::vector<PrimeConst> pc(np);
    for (int i = 0; i < np; i++) {
        const uint64_t q = primes[i];
        if (q >= (1ull << 62) || (q - 1) % (2ull * n)) {
            srk_ctx_destroy(c);
            return fail(SRK_EINVAL, "prime %d is not an NTT prime below 2^62", i);
        }
        u128 ratio = (~(u128)0) / q;  // floor((2^128-1)/q) == floor(2^128/q) for odd q
        pc[i].q = q;
        pc[i].two_q = 2 * q;
        pc[i].ratio_hi = (uint64_t)(ratio >> 64);
        pc[i].ratio_lo = (uint64_t)ratio;
        pc[i].ninv = hinv((uint64_t)n, q);
        pc[i].ninv_shoup = shoup(pc[i].ninv, q);
    }
    if ((rc = dupload(c, &c->d_pc, pc))) { srk_ctx_destroy(c); return rc; }
    // twiddles
    std::vector<uint64_t> tw((size_t)np * n), tws((size_t)np * n), itw((size_t)np * n),
        itws((size_t)np * n);
    for (int i = 0; i < np; i++) {
        const uint64_t q = primes[i], psi = roots[i] % q, ipsi = hinv(psi, q);
        if (hpow(psi, (uint64_t)n, q) != q - 1) {
            srk_ctx_destroy(c);
            return fail(SRK_EINVAL, "root %d is not a primitive 2N-th root", i);
        }
        uint64_t p = 1, ip = 1;
        for (int k = 0; k < n; k++) {
            const size_t r = (size_t)i * n + hbrv((uint32_t)k, log_n);
            tw[r] = p;
            tws[r] = shoup(p, q);
            itw[r] = ip;
            itws[r] = shoup(ip, q);
            p = hmul(p, psi, q);
            ip = hmul(ip, ipsi, q);
        }
    }
    if ((rc = dupload(c, &c->d_tw, tw)) || (rc = dupload(c, &c->d_tws, tws)) ||
        (rc = dupload(c, &c->d_itw, itw)) || (rc = dupload(c, &c->d_itws, itws))) {
        srk_ctx_destroy(c);
        return rc;
    }
    // base-conversion plans
    c->modup.resize(n_q);
    c->moddown.resize(n_q);
    std::vector<uint64_t> qv(c->primes);
    for (int l = 0; l < n_q; l++) {
        const int nl = l + 1, ne = nl + n_p;
        const int beta = (nl + c->alpha - 1) / c->alpha;
        c->modup[l].resize(beta);
        for (int j = 0; j < beta; j++) {
            const int g0 = j * c->alpha, g1 = std::min(nl, (j + 1) * c->alpha);
            std::vector<int> src, slot, pid;
            for (int i = g0; i < g1; i++) src.push_back(i);
            for (int t = 0; t < ne; t++) {
                if (t >= g0 && t < g1) continue;
                slot.push_back(t);
                pid.push_back(ext_pid(c, l, t));
            }
            if ((rc = build_plan(c, c->modup[l][j], src, slot, pid))) { srk_ctx_destroy(c); return rc; }
        }
        std::vector<int> src, slot, pid;
        for (int k = 0; k < n_p; k++) src.push_back(n_q + k);
        for (int i = 0; i < nl; i++) {
            slot.push_back(i);
            pid.push_back(i);
        }
        if ((rc = build_plan(c, c->moddown[l], src, slot, pid, true))) { srk_ctx_destroy(c); return rc; }
    }
    // P^-1 mod q_i, P mod prime_i, q_l^-1 mod q_i
    std::vector<uint64_t> pinv(n_q), pmod(np);
    for (int i = 0; i < np; i++) {
        uint64_t pm = 1;
        for (int k = 0; k < n_p; k++) pm = hmul(pm, primes[n_q + k] % primes[i], primes[i]);
        pmod[i] = pm;
        if (i < n_q) pinv[i] = hinv(pm, primes[i]);
    }
    fill_consts(c->lc_pinv, pinv, std::vector<uint64_t>(qv.begin(), qv.begin() + n_q));
    fill_consts(c->lc_pmod, pmod, qv);
    c->lc_qlinv.resize(n_q);
    for (int l = 1; l < n_q; l++) {
        std::vector<uint64_t> w(l), qq(l);
        for (int i = 0; i < l; i++) {
            w[i] = hinv(primes[l] % primes[i], primes[i]);
            qq[i] = primes[i];
        }
        fill_consts(c->lc_qlinv[l], w, qq);
    }
    *out = c;
    return SRK_OK;
}

extern "C" size_t srk_workspace_bytes(const srk_ctx *c) {
    const size_t n = c->n, nl = c->n_q, ne = nl + c->n_p;
    const size_t beta = (nl + c->alpha - 1) / c->alpha;
    size_t ks = nl + beta * ne + 2 * ne + 2 * nl;      // keyswitch
    size_t relin = 3 * nl + 2 * nl + ks;               // tensor + ks outputs
    size_t relin_rs = relin + 2 * nl + (2 + 2 * nl);   // + product + rescale
    size_t rot = 2 * nl + 2 * nl + ks;
    size_t keygen = 2 * (size_t)c->n_primes;
    size_t enc = 2 * nl;
    size_t words = std::max({ks, relin_rs, rot, keygen, enc, (size_t)2 + 2 * nl});
    return words * n * sizeof(uint64_t) + 256;
}

// ---------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------
static inline cudaStream_t S(void *s) { return (cudaStream_t)s; }
static inline int grid_for(long long total, int per_thread = 1) {
    long long blocks = (total / per_thread + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 16) blocks = 148 * 16;
    return (int)blocks;
}

static NttTables tables(const srk_ctx *c) {
    NttTables t;
    t.pc = c->d_pc;
    t.tw = c->d_tw;
    t.tws = c->d_tws;
    t.itw = c->d_itw;
    t.itws = c->d_itws;
    return t;
}

template <int LOG_T, bool INV, bool COL>
static int launch_pass(const srk_ctx *c, LimbBatch b, int y0, int ny, cudaStream_t s) {
    using SH = NttShape<LOG_T>;
    const int subs = c->n >> LOG_T;  // sub-transforms per limb
    int cb = 256 / SH::TPS;
    if (cb > subs) cb = subs;
    const int threads = cb * SH::TPS;
    const size_t smem = COL ? (size_t)cb * SH::T * 8 : (size_t)cb * (SH::T + SH::T / SH::E) * 8;
    // shift the batch so blockIdx.y starts at y0
    LimbBatch bb = b;
    const int limb0 = y0 / b.n_polys;
    if (y0 % b.n_polys) return fail(SRK_EINVAL, "ntt chunk must start at a limb boundary");
    bb.ptr = b.ptr + (long long)limb0 * c->n;
    bb.split = b.split - limb0;
    bb.off_a = b.off_a + limb0;
    bb.off_b = b.off_b + limb0;
    bb.n_limbs = ny / b.n_polys;
    dim3 grid(subs / cb, ny);
    ntt_pass_kernel<LOG_T, INV, COL><<<grid, threads, smem, s>>>(bb, tables(c), c->log_n);
    LAUNCHED();
    return SRK_OK;
}

template <bool INV, bool COL>
static int pass_dispatch(const srk_ctx *c, int log_t, LimbBatch b, int y0, int ny, cudaStream_t s) {
    switch (log_t) {
        case 5: return launch_pass<5, INV, COL>(c, b, y0, ny, s);
        case 6: return launch_pass<6, INV, COL>(c, b, y0, ny, s);
        case 7: return launch_pass<7, INV, COL>(c, b, y0, ny, s);
        case 8: return launch_pass<8, INV, COL>(c, b, y0, ny, s);
        default: return fail(SRK_EINVAL, "unsupported NTT pass size 2^%d", log_t);
    }
}

// NTT over a LimbBatch, chunked so one chunk's intermediate stays in L2
static int ntt_batch(const srk_ctx *c, LimbBatch b, bool inverse, cudaStream_t s) {
    if (b.n_limbs <= 0 || b.n_polys <= 0) return SRK_OK;
    const int log_r = (c->log_n + 1) / 2, log_c = c->log_n - log_r;
    // chunk = whole limbs (all polys of a limb index) so pid stays per y-row
    int limbs_per_chunk = c->ntt_chunk / b.n_polys;
    if (limbs_per_chunk < 1) limbs_per_chunk = 1;
    if (limbs_per_chunk > 65535 / b.n_polys) limbs_per_chunk = 65535 / b.n_polys;
    for (int l0 = 0; l0 < b.n_limbs; l0 += limbs_per_chunk) {
        const int nlc = std::min(limbs_per_chunk, b.n_limbs - l0);
        const int y0 = l0 * b.n_polys, ny = nlc * b.n_polys;
        if (!inverse) {
            TRY((pass_dispatch<false, true>(c, log_r, b, y0, ny, s)));
            TRY((pass_dispatch<false, false>(c, log_c, b, y0, ny, s)));
        } else {
            TRY((pass_dispatch<true, false>(c, log_c, b, y0, ny, s)));
            TRY((pass_dispatch<true, true>(c, log_r, b, y0, ny, s)));
        }
    }
    return SRK_OK;
}

static LimbBatch qbatch(uint64_t *p, int n_polys, long long pstride, int n_limbs, int first) {
    LimbBatch b;
    b.ptr = p;
    b.poly_stride = pstride;
    b.n_polys = n_polys;
    b.n_limbs = n_limbs;
    b.split = 1 << 30;
    b.off_a = first;
    b.off_b = first;
    return b;
}
// limbs [t0, t1) of an extended poly at `level`
static LimbBatch ebatch(const srk_ctx *c, uint64_t *p, int n_polys, long long pstride, int level,
                        int t0, int t1) {
    LimbBatch b;
    b.ptr = p + (long long)t0 * c->n;
    b.poly_stride = pstride;
    b.n_polys = n_polys;
    b.n_limbs = t1 - t0;
    b.split = level + 1 - t0;
    b.off_a = t0;
    b.off_b = t0 + c->L - level;
    return b;
}

static int check_level(const srk_ctx *c, int level) {
    if (level < 0 || level > c->L) return fail(SRK_EINVAL, "level %d out of range [0, %d]", level, c->L);
    return SRK_OK;
}

// ---------------------------------------------------------------------
// C-ABI: NTT and elementwise
// ---------------------------------------------------------------------
extern "C" int srk_ntt(srk_ctx *c, uint64_t *data, int n_polys, long long poly_stride,
                       int n_limbs, int first_prime, int inverse, void *stream) {
    if (!c || !data) return fail(SRK_EINVAL, "null argument");
    if (first_prime < 0 || first_prime + n_limbs > c->n_primes)
        return fail(SRK_EINVAL, "prime range out of bounds");
    CU(cudaSetDevice(c->device));
    return ntt_batch(c, qbatch(data, n_polys, poly_stride, n_limbs, first_prime), inverse != 0,
                     S(stream));
}

extern "C" int srk_ntt_ext(srk_ctx *c, uint64_t *data, int n_polys, long long poly_stride,
                           int level, int inverse, void *stream) {
    if (!c || !data) return fail(SRK_EINVAL, "null argument");
    TRY(check_level(c, level));
    return ntt_batch(c, ebatch(c, data, n_polys, poly_stride, level, 0, level + 1 + c->n_p),
                     inverse != 0, S(stream));
}

extern "C" int srk_addsub(srk_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out,
                          int level, int op, void *stream) {
    TRY(check_level(c, level));
    if (op < 0 || op > 2) return fail(SRK_EINVAL, "bad op");
    const long long total = 2ll * (level + 1) * c->n;
    k_addsub<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, b, out, c->d_pc, c->log_n, level + 1, op);
    LAUNCHED();
    return SRK_OK;
}

static LimbConsts host_consts(const srk_ctx *c, const uint64_t *k_res, int nl) {
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    for (int i = 0; i < nl; i++) {
        lc.w[i] = k_res[i] % c->primes[i];
        lc.ws[i] = shoup(lc.w[i], c->primes[i]);
    }
    return lc;
}

extern "C" int srk_add_const(srk_ctx *c, const uint64_t *a, const uint64_t *k_res, uint64_t *out,
                             int level, void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc = host_consts(c, k_res, level + 1);
    const long long total = 2ll * (level + 1) * c->n;
    k_add_plain<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, nullptr, lc, out, c->d_pc, c->log_n,
                                                           level + 1);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_add_plain(srk_ctx *c, const uint64_t *a, const uint64_t *pt, uint64_t *out,
                             int level, void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    const long long total = 2ll * (level + 1) * c->n;
    k_add_plain<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, pt, lc, out, c->d_pc, c->log_n,
                                                           level + 1);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_mul_const(srk_ctx *c, const uint64_t *a, int src_limbs, const uint64_t *k_res,
                             uint64_t *out, int level, void *stream) {
    TRY(check_level(c, level));
    if (src_limbs < level + 1) return fail(SRK_EINVAL, "source has fewer limbs than level+1");
    LimbConsts lc = host_consts(c, k_res, level + 1);
    const long long total = 2ll * (level + 1) * c->n;
    k_mul_pt<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, src_limbs, nullptr, lc, out, c->d_pc,
                                                        c->log_n, level + 1);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_mul_plain(srk_ctx *c, const uint64_t *a, const uint64_t *pt, uint64_t *out,
                             int level, void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    const long long total = 2ll * (level + 1) * c->n;
    k_mul_pt<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, level + 1, pt, lc, out, c->d_pc,
                                                        c->log_n, level + 1);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_tensor(srk_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *d,
                          int level, void *stream) {
    TRY(check_level(c, level));
    const long long total = (long long)(level + 1) * c->n;
    k_tensor<<<grid_for(total), 256, 0, S(stream)>>>(a, b, d, c->d_pc, c->log_n, level + 1);
    LAUNCHED();
    return SRK_OK;
}

// ---------------------------------------------------------------------
// rescale (with optional pre-multiplier: 0 none, 1 per-limb constant, 2 plaintext)
// ---------------------------------------------------------------------
static int rescale_impl(srk_ctx *c, const uint64_t *a, long long a_pstride, const uint64_t *pt,
                        const LimbConsts &k, int mode, uint64_t *out, int level, uint64_t *ws,
                        cudaStream_t s) {
    if (level < 1) return fail(SRK_EINVAL, "cannot rescale a level-0 ciphertext");
    const int n = c->n;
    uint64_t *top = ws;                  // [2][N]
    uint64_t *t = ws + 2ll * n;          // [2][level][N]
    k_rescale_top<<<grid_for(2ll * n), 256, 0, s>>>(a, a_pstride, pt, k, mode, top, c->d_pc,
                                                    c->log_n, level);
    LAUNCHED();
    TRY(ntt_batch(c, qbatch(top, 2, n, 1, level), true, s));
    k_rescale_spread<<<grid_for(2ll * level * n), 256, 0, s>>>(top, t, c->d_pc, c->log_n, level);
    LAUNCHED();
    TRY(ntt_batch(c, qbatch(t, 2, (long long)level * n, level, 0), false, s));
    k_rescale_combine<<<grid_for(2ll * level * n), 256, 0, s>>>(
        a, a_pstride, pt, k, mode, t, c->lc_qlinv[level], out, c->d_pc, c->log_n, level);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_rescale(srk_ctx *c, const uint64_t *a, uint64_t *out, int level, void *ws,
                           void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    return rescale_impl(c, a, (long long)(level + 1) * c->n, nullptr, lc, 0, out, level,
                        (uint64_t *)ws, S(stream));
}

extern "C" int srk_mul_const_rescale(srk_ctx *c, const uint64_t *a, int src_limbs,
                                     const uint64_t *k_res, uint64_t *out, int level, void *ws,
                                     void *stream) {
    TRY(check_level(c, level));
    if (src_limbs < level + 1) return fail(SRK_EINVAL, "source has fewer limbs than level+1");
    LimbConsts lc = host_consts(c, k_res, level + 1);
    return rescale_impl(c, a, (long long)src_limbs * c->n, nullptr, lc, 1, out, level,
                        (uint64_t *)ws, S(stream));
}

extern "C" int srk_mul_plain_rescale(srk_ctx *c, const uint64_t *a, const uint64_t *pt,
                                     uint64_t *out, int level, void *ws, void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    return rescale_impl(c, a, (long long)(level + 1) * c->n, pt, lc, 2, out, level,
                        (uint64_t *)ws, S(stream));
}

// ---------------------------------------------------------------------
// key switching
// ---------------------------------------------------------------------
static int bconv(const srk_ctx *c, const BconvPlan &pl, const uint64_t *src, long long src_ps,
                 uint64_t *out, long long out_ps, int n_polys, cudaStream_t s) {
    if (pl.n_src * pl.n_dst > 16 * 72) return fail(SRK_EINVAL, "base conversion too wide");
    BconvArgs ba;
    ba.src = src;
    ba.src_pstride = src_ps;
    ba.n_src = pl.n_src;
    ba.src_pid0 = pl.src_pid0;
    ba.out = out;
    ba.out_pstride = out_ps;
    ba.n_dst = pl.n_dst;
    ba.mat = pl.mat;
    ba.hinv = pl.hinv;
    ba.dst_slot = pl.dst_slot;
    ba.dst_pid = pl.dst_pid;
    ba.dst_corr = pl.dst_corr;
    dim3 grid((c->n + 255) / 256, n_polys);
    if (pl.n_src <= 4)
        k_bconv<4><<<grid, 256, 0, s>>>(ba, c->d_pc, c->log_n);
    else if (pl.n_src <= 8)
        k_bconv<8><<<grid, 256, 0, s>>>(ba, c->d_pc, c->log_n);
    else
        k_bconv<16><<<grid, 256, 0, s>>>(ba, c->d_pc, c->log_n);
    LAUNCHED();
    return SRK_OK;
}

// adds: optional (add0, add1) fused into the ModDown combine
static int keyswitch_impl(srk_ctx *c, const uint64_t *d, const uint64_t *key, uint64_t *out0,
                          uint64_t *out1, const uint64_t *add0, const uint64_t *add1, int level,
                          uint64_t *ws, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->n_p, ne = nl + K;
    const int beta = (nl + c->alpha - 1) / c->alpha;
    uint64_t *dc = ws;                                  // [nl][N]
    uint64_t *ext = dc + (long long)nl * n;             // [beta][ne][N]
    uint64_t *acc = ext + (long long)beta * ne * n;     // [2][ne][N]
    uint64_t *conv = acc + 2ll * ne * n;                // [2][nl][N]
    CU(cudaMemcpyAsync(dc, d, sizeof(uint64_t) * nl * n, cudaMemcpyDeviceToDevice, s));
    TRY(ntt_batch(c, qbatch(dc, 1, 0, nl, 0), true, s));
    for (int j = 0; j < beta; j++) {
        const int g0 = j * c->alpha, g1 = std::min(nl, (j + 1) * c->alpha);
        uint64_t *ej = ext + (long long)j * ne * n;
        const BconvPlan &pl = c->modup[level][j];
        TRY(bconv(c, pl, dc + (long long)g0 * n, 0, ej, 0, 1, s));
        CU(cudaMemcpyAsync(ej + (long long)g0 * n, d + (long long)g0 * n,
                           sizeof(uint64_t) * (g1 - g0) * n, cudaMemcpyDeviceToDevice, s));
        if (g0 > 0) TRY(ntt_batch(c, ebatch(c, ej, 1, 0, level, 0, g0), false, s));
        TRY(ntt_batch(c, ebatch(c, ej, 1, 0, level, g1, ne), false, s));
    }
    const long long tot = (long long)ne * n;
    k_ks_inner<<<grid_for(tot), 256, 0, s>>>(ext, key, acc, c->d_pc, c->log_n, ne, level, c->L,
                                             c->n_primes, beta);
    LAUNCHED();
    // ModDown: INTT the special limbs of both accumulators, convert to Q_l
    LimbBatch pb;
    pb.ptr = acc + (long long)nl * n;
    pb.poly_stride = (long long)ne * n;
    pb.n_polys = 2;
    pb.n_limbs = K;
    pb.split = 0;
    pb.off_a = c->n_q;
    pb.off_b = c->n_q;
    TRY(ntt_batch(c, pb, true, s));
    TRY(bconv(c, c->moddown[level], acc + (long long)nl * n, (long long)ne * n, conv,
              (long long)nl * n, 2, s));
    TRY(ntt_batch(c, qbatch(conv, 2, (long long)nl * n, nl, 0), false, s));
    k_moddown_combine<<<grid_for(2ll * nl * n), 256, 0, s>>>(acc, (long long)ne * n, conv, add0,
                                                             add1, c->lc_pinv, out0, out1,
                                                             c->d_pc, c->log_n, nl);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_keyswitch(srk_ctx *c, const uint64_t *d, const uint64_t *key, uint64_t *out0,
                             uint64_t *out1, int level, void *ws, void *stream) {
    TRY(check_level(c, level));
    return keyswitch_impl(c, d, key, out0, out1, nullptr, nullptr, level, (uint64_t *)ws,
                          S(stream));
}

static int mul_relin_impl(srk_ctx *c, const uint64_t *a, const uint64_t *b, const uint64_t *rlk,
                          uint64_t *out, int level, uint64_t *ws, cudaStream_t s) {
    const long long ps = (long long)(level + 1) * c->n;
    uint64_t *d = ws;  // [3][nl][N]
    k_tensor<<<grid_for(ps), 256, 0, s>>>(a, b, d, c->d_pc, c->log_n, level + 1);
    LAUNCHED();
    return keyswitch_impl(c, d + 2 * ps, rlk, out, out + ps, d, d + ps, level, ws + 3 * ps, s);
}

extern "C" int srk_mul_relin(srk_ctx *c, const uint64_t *a, const uint64_t *b,
                             const uint64_t *rlk, uint64_t *out, int level, void *ws,
                             void *stream) {
    TRY(check_level(c, level));
    return mul_relin_impl(c, a, b, rlk, out, level, (uint64_t *)ws, S(stream));
}

extern "C" int srk_mul_relin_rescale(srk_ctx *c, const uint64_t *a, const uint64_t *b,
                                     const uint64_t *rlk, uint64_t *out, int level, void *ws,
                                     void *stream) {
    TRY(check_level(c, level));
    if (level < 1) return fail(SRK_EINVAL, "depth exhausted");
    const long long ps = (long long)(level + 1) * c->n;
    uint64_t *w = (uint64_t *)ws;
    uint64_t *prod = w;  // [2][nl][N]
    TRY(mul_relin_impl(c, a, b, rlk, prod, level, w + 2 * ps, S(stream)));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    return rescale_impl(c, prod, ps, nullptr, lc, 0, out, level, w + 2 * ps, S(stream));
}

extern "C" int srk_automorph(srk_ctx *c, const uint64_t *a, uint64_t *out,
                             long long n_limbs_total, uint64_t galois, void *stream) {
    if (!(galois & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
    const long long total = n_limbs_total * c->n;
    k_automorph<<<grid_for(total), 256, 0, S(stream)>>>(a, out, n_limbs_total, galois, c->log_n);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_rotate(srk_ctx *c, const uint64_t *a, const uint64_t *gkey, uint64_t *out,
                          int level, uint64_t galois, void *ws, void *stream) {
    TRY(check_level(c, level));
    if (!(galois & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
    const long long ps = (long long)(level + 1) * c->n;
    uint64_t *r = (uint64_t *)ws;  // [2][nl][N] automorphed input
    k_automorph<<<grid_for(2 * ps), 256, 0, S(stream)>>>(a, r, 2ll * (level + 1), galois, c->log_n);
    LAUNCHED();
    return keyswitch_impl(c, r + ps, gkey, out, out + ps, r, nullptr, level, r + 2 * ps,
                          S(stream));
}

// ---------------------------------------------------------------------
// sampling, keys, encryption
// ---------------------------------------------------------------------
extern "C" int srk_uniform(srk_ctx *c, uint64_t *a, int n_limbs, int first_prime, uint64_t seed,
                           uint64_t stream_base, void *stream) {
    if (first_prime < 0 || first_prime + n_limbs > c->n_primes)
        return fail(SRK_EINVAL, "prime range out of bounds");
    LimbBatch b = qbatch(a, 1, 0, n_limbs, first_prime);
    k_uniform<<<grid_for((long long)n_limbs * c->n), 256, 0, S(stream)>>>(b, c->d_pc, c->log_n,
                                                                          seed, stream_base);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_small_to_ntt(srk_ctx *c, const int64_t *v, uint64_t *out, int n_limbs,
                                int first_prime, void *stream) {
    if (first_prime < 0 || first_prime + n_limbs > c->n_primes)
        return fail(SRK_EINVAL, "prime range out of bounds");
    LimbBatch b = qbatch(out, 1, 0, n_limbs, first_prime);
    k_small_to_res<<<grid_for((long long)n_limbs * c->n), 256, 0, S(stream)>>>(v, b, c->d_pc,
                                                                               c->log_n);
    LAUNCHED();
    return ntt_batch(c, b, false, S(stream));
}

extern "C" int srk_square(srk_ctx *c, const uint64_t *s, uint64_t *out, int n_limbs,
                          void *stream) {
    k_square<<<grid_for((long long)n_limbs * c->n), 256, 0, S(stream)>>>(s, out, c->d_pc,
                                                                         c->log_n, n_limbs);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_keygen(srk_ctx *c, const uint64_t *s_ntt, const uint64_t *sfrom_ntt,
                          const int64_t *e, uint64_t seed, uint64_t key_id, uint64_t *key,
                          void *ws, void *stream) {
    const int n = c->n, np = c->n_primes;
    uint64_t *en = (uint64_t *)ws;
    for (int j = 0; j < c->dnum; j++) {
        uint64_t *b = key + ((long long)j * 2 + 0) * np * n;
        uint64_t *a = key + ((long long)j * 2 + 1) * np * n;
        TRY(srk_uniform(c, a, np, 0, seed, ((key_id << 8) | (uint64_t)j) << 8, stream));
        TRY(srk_small_to_ntt(c, e + (long long)j * n, en, np, 0, stream));
        const int d0 = j * c->alpha, d1 = std::min(c->n_q, (j + 1) * c->alpha);
        k_keygen_combine<<<grid_for((long long)np * n), 256, 0, S(stream)>>>(
            a, s_ntt, sfrom_ntt, en, b, c->lc_pmod, c->d_pc, c->log_n, np, d0, d1);
        LAUNCHED();
    }
    return SRK_OK;
}

extern "C" int srk_encrypt(srk_ctx *c, const int64_t *m, const uint64_t *s_ntt, const int64_t *e,
                           uint64_t seed, uint64_t seq, uint64_t *out, int level, void *ws,
                           void *stream) {
    TRY(check_level(c, level));
    const int n = c->n, nl = level + 1;
    uint64_t *en = (uint64_t *)ws, *mn = en + (long long)nl * n;
    uint64_t *c1 = out + (long long)nl * n;
    TRY(srk_uniform(c, c1, nl, 0, seed, (0xE0000000ull + seq) << 8, stream));
    TRY(srk_small_to_ntt(c, e, en, nl, 0, stream));
    TRY(srk_small_to_ntt(c, m, mn, nl, 0, stream));
    k_encrypt_combine<<<grid_for((long long)nl * n), 256, 0, S(stream)>>>(c1, s_ntt, en, mn, out,
                                                                          c->d_pc, c->log_n, nl);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_decrypt_limb0(srk_ctx *c, const uint64_t *ct, const uint64_t *s_ntt,
                                 int64_t *m_out, int level, void *ws, void *stream) {
    TRY(check_level(c, level));
    uint64_t *t = (uint64_t *)ws;
    k_decrypt_limb0<<<grid_for(c->n), 256, 0, S(stream)>>>(ct, (long long)(level + 1) * c->n, s_ntt,
                                                           t, c->d_pc, c->log_n);
    LAUNCHED();
    TRY(ntt_batch(c, qbatch(t, 1, 0, 1, 0), true, S(stream)));
    k_center_limb0<<<grid_for(c->n), 256, 0, S(stream)>>>(t, m_out, c->d_pc, c->log_n);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_encode_plain(srk_ctx *c, const int64_t *coeffs, uint64_t *pt_out, int level,
                                void *stream) {
    TRY(check_level(c, level));
    return srk_small_to_ntt(c, coeffs, pt_out, level + 1, 0, stream);
}
