// api.cu -- context, tables and the C-ABI of libslotrank_b200.so.
// See include/slotrank_b200.h for the contract and the reference methods
// each entry point realises.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/slotrank_b200.h"
#include "kernels.cuh"
#include "modarith.cuh"
#include "ntt.cuh"

#ifndef SRK_WS_BATCH
#define SRK_WS_BATCH 32  // ciphertexts per internal chunk of a batched call (keys read once per chunk)
#endif

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

// FP64 pipe probe: 8 independent FMA chains per thread (the NTT passes' binding pipe;
// bench.py divides the transforms' FP64 instruction count by this rate)
__global__ void __launch_bounds__(256) k_fp64_probe(int iters, double *sink) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
    const double m = 1.0000000001, c = 1e-12;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fma(a[i], m, c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += a[i];
    if (s == 12345.678) sink[0] = s;  // never true: keeps the chains alive
}
extern "C" int srk_fp64_probe(int ctas, int iters, double *sink, void *stream) {
    if (ctas < 1 || iters < 1 || !sink) return fail(SRK_EINVAL, "bad FP64 probe arguments");
    k_fp64_probe<<<ctas, 256, 0, (cudaStream_t)stream>>>(iters, sink);
    LAUNCHED();
    return SRK_OK;
}

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
    ulonglong2 *mat2 = nullptr;  // [n_src][n_dst] {m, floor(m 2^64 / q_t)} (Shoup)
    ulonglong2 *mhl = nullptr;   // [n_src][n_dst] {m, m 2^32 mod q_t}       (k_moddown_conv_f64,
    double2 *fhl = nullptr;      // [n_src][n_dst] {m / q_t, (m 2^32 mod q_t) / q_t}  q_t < 2^41)
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
    ulonglong2 *d_tw = nullptr, *d_itw = nullptr;  // {w, Shoup(w)} interleaved
    double *d_twd = nullptr, *d_itwd = nullptr;     // w as double (FP64-mode limbs)
    std::vector<void *> allocs;
    // modup[level][digit], moddown[level]
    std::vector<std::vector<BconvPlan>> modup;
    std::vector<BconvPlan> moddown;
    std::vector<BconvPlan> moddown_rs;        // [level]: P u {q_level} -> q_0..q_{level-1}
    std::vector<LimbConsts> lc_rs_scale;      // [level]: N^-1 (S/s_k)^-1 mod s_k, S = P q_level
    std::vector<LimbConsts> lc_rs_mulc;       // [level]: (P q_level)^-1 mod q_i
    std::vector<LimbConsts> lc_modup_scale;  // [level]: N^-1 (Q_j/q_i)^-1 mod q_i (INTT fold)
    LimbConsts lc_moddown_scale;      // N^-1 (P/p_k)^-1 mod p_k (INTT fold)
    LimbConsts lc_pinv;               // P^-1 mod q_i
    LimbConsts lc_pmod;               // P mod prime_i (all primes)
    std::vector<LimbConsts> lc_qlinv; // [level]: q_level^-1 mod q_i
    int ntt_chunk = 128;              // limb-polys per L2-resident NTT chunk (SRK_NTT_CHUNK: tests force chunking)
    int ks_streams = 2;               // hoisted outputs alternate over two streams
    cudaStream_t side = nullptr;      // the second lane
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // NTT chunk lanes: independent limb chunks of one NTT alternate between the
    // caller's stream and nside[lane], so one chunk's pass tail overlaps the
    // next chunk's passes (lane = 1 when called from the key-switch side lane)
    int ntt_streams = 2;
    int ws_batch = SRK_WS_BATCH;  // ciphertexts per internal chunk (SRK_WS_BATCH env: smaller workspace)
    int ntt_cta_threads = 128;  // threads per NTT pass CTA (128: 8 CTAs/SM, cheaper barriers)
    unsigned conv_cpt = 4;  // coefficients per thread of the conversions (amortises their staging)
    cudaStream_t nside[2] = {nullptr, nullptr};
    cudaStream_t branch = nullptr;  // the caller's second stream (srk_ctx_set_branch_stream): NTT lane 1
    cudaEvent_t ev_nfork[2] = {nullptr, nullptr}, ev_njoin[2] = {nullptr, nullptr};
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
    std::vector<ulonglong2> mat2((size_t)ns * nd);
    for (int i = 0; i < ns; i++)
        for (int t = 0; t < nd; t++) {
            const uint64_t m = mat[(size_t)i * nd + t];
            mat2[(size_t)i * nd + t] = make_ulonglong2(m, shoup(m, c->primes[dst_pids[t]]));
        }
    TRY(dupload(c, &pl.mat2, mat2));
    {
        std::vector<ulonglong2> mhl((size_t)ns * nd);
        std::vector<double2> fhl((size_t)ns * nd);
        for (int i = 0; i < ns; i++)
            for (int t = 0; t < nd; t++) {
                const uint64_t p = c->primes[dst_pids[t]], m = mat[(size_t)i * nd + t];
                const uint64_t mh = (uint64_t)(((u128)m << 32) % p);
                mhl[(size_t)i * nd + t] = make_ulonglong2(m, mh);
                fhl[(size_t)i * nd + t] = make_double2((double)m / (double)p, (double)mh / (double)p);
            }
        TRY(dupload(c, &pl.mhl, mhl));
        TRY(dupload(c, &pl.fhl, fhl));
    }
    TRY(dupload(c, &pl.hinv, hv));
    TRY(dupload(c, &pl.dst_slot, dst_slots));
    TRY(dupload(c, &pl.dst_pid, dst_pids));
    if (exact) {  // table [v][t] = v * [prod src]_{q_t}, v = 0..n_src
        std::vector<uint64_t> corr((size_t)(ns + 1) * nd);
        for (int t = 0; t < nd; t++) {
            const uint64_t p = c->primes[dst_pids[t]];
            uint64_t v = 1;
            for (int m = 0; m < ns; m++) v = hmul(v, c->primes[src_pids[m]] % p, p);
            for (int k = 0; k <= ns; k++) corr[(size_t)k * nd + t] = hmul((uint64_t)k, v, p);
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
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (int i = 0; i < 2; i++) {
        if (c->nside[i]) cudaStreamDestroy(c->nside[i]);
        if (c->ev_nfork[i]) cudaEventDestroy(c->ev_nfork[i]);
        if (c->ev_njoin[i]) cudaEventDestroy(c->ev_njoin[i]);
    }
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
    // two run-time settings: the NTT chunk (tests force multi-chunk launches) and the
    // key-switch workspace batch (several ranks sharing one GPU need a smaller one)
    if (const char *e = getenv("SRK_NTT_CHUNK")) c->ntt_chunk = std::max(1, atoi(e));
    if (const char *e = getenv("SRK_WS_BATCH")) c->ws_batch = std::max(1, atoi(e));
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        srk_ctx_destroy(c);
        return fail(SRK_ECUDA, "stream / event creation failed");
    }
    for (int i = 0; i < 2; i++) {
        if (cudaStreamCreateWithFlags(&c->nside[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_nfork[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_njoin[i], cudaEventDisableTiming) != cudaSuccess) {
            srk_ctx_destroy(c);
            return fail(SRK_ECUDA, "stream / event creation failed");
        }
    }
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
        const double qd = (double)q, qi = 1.0 / qd;
        memcpy(&pc[i].qd_bits, &qd, 8);
        memcpy(&pc[i].qinv_bits, &qi, 8);
    }
    if ((rc = dupload(c, &c->d_pc, pc))) { srk_ctx_destroy(c); return rc; }
    // twiddles
    std::vector<ulonglong2> tw((size_t)np * n), itw((size_t)np * n);
    std::vector<double> twd((size_t)np * n), itwd((size_t)np * n);
    for (int i = 0; i < np; i++) {
        const uint64_t q = primes[i], psi = roots[i] % q, ipsi = hinv(psi, q);
        if (hpow(psi, (uint64_t)n, q) != q - 1) {
            srk_ctx_destroy(c);
            return fail(SRK_EINVAL, "root %d is not a primitive 2N-th root", i);
        }
        uint64_t p = 1, ip = 1;
        for (int k = 0; k < n; k++) {
            const size_t r = (size_t)i * n + hbrv((uint32_t)k, log_n);
            tw[r] = make_ulonglong2(p, shoup(p, q));
            itw[r] = make_ulonglong2(ip, shoup(ip, q));
            twd[r] = (double)p;   // exact for the q < 2^41 limbs that use it
            itwd[r] = (double)ip;
            p = hmul(p, psi, q);
            ip = hmul(ip, ipsi, q);
        }
    }
    if ((rc = dupload(c, &c->d_tw, tw)) || (rc = dupload(c, &c->d_itw, itw)) ||
        (rc = dupload(c, &c->d_twd, twd)) || (rc = dupload(c, &c->d_itwd, itwd))) {
        srk_ctx_destroy(c);
        return rc;
    }
    // base-conversion plans
    c->modup.resize(n_q);
    c->moddown.resize(n_q);
    c->moddown_rs.resize(n_q);
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
        if (l >= 1) {  // fused HMult rescale: special basis P u {q_l}, targets q_0..q_{l-1}
            std::vector<int> src2(src), slot2, pid2;
            src2.push_back(l);
            for (int i = 0; i < l; i++) {
                slot2.push_back(i);
                pid2.push_back(i);
            }
            if ((rc = build_plan(c, c->moddown_rs[l], src2, slot2, pid2, true))) { srk_ctx_destroy(c); return rc; }
        }
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
    {
        std::vector<uint64_t> w(n_p), qq(n_p);
        for (int k = 0; k < n_p; k++) {
            const uint64_t p = primes[n_q + k];
            uint64_t h = 1;
            for (int m = 0; m < n_p; m++)
                if (m != k) h = hmul(h, primes[n_q + m] % p, p);
            w[k] = hmul(hinv((uint64_t)n, p), hinv(h, p), p);
            qq[k] = p;
        }
        fill_consts(c->lc_moddown_scale, w, qq);
    }
    c->lc_rs_scale.resize(n_q);
    c->lc_rs_mulc.resize(n_q);
    for (int l = 1; l < n_q; l++) {
        std::vector<int> sid;
        for (int k = 0; k < n_p; k++) sid.push_back(n_q + k);
        sid.push_back(l);
        std::vector<uint64_t> w(sid.size()), qq(sid.size());
        for (size_t k = 0; k < sid.size(); k++) {
            const uint64_t p = primes[sid[k]];
            uint64_t h = 1;
            for (size_t m = 0; m < sid.size(); m++)
                if (m != k) h = hmul(h, primes[sid[m]] % p, p);
            w[k] = hmul(hinv((uint64_t)n, p), hinv(h, p), p);
            qq[k] = p;
        }
        fill_consts(c->lc_rs_scale[l], w, qq);
        std::vector<uint64_t> mc(l), q2(l);
        for (int i = 0; i < l; i++) {
            uint64_t s = pmod[i];
            s = hmul(s, primes[l] % primes[i], primes[i]);
            mc[i] = hinv(s, primes[i]);
            q2[i] = primes[i];
        }
        fill_consts(c->lc_rs_mulc[l], mc, q2);
    }
    c->lc_modup_scale.resize(n_q);
    for (int l = 0; l < n_q; l++) {
        std::vector<uint64_t> w(l + 1), qq(l + 1);
        for (int i = 0; i <= l; i++) {
            const uint64_t q = primes[i];
            const int g0 = (i / c->alpha) * c->alpha, g1 = std::min(l + 1, g0 + c->alpha);
            uint64_t h = 1;
            for (int m = g0; m < g1; m++)
                if (m != i) h = hmul(h, primes[m] % q, q);
            w[i] = hmul(hinv((uint64_t)n, q), hinv(h, q), q);
            qq[i] = q;
        }
        fill_consts(c->lc_modup_scale[l], w, qq);
    }
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


// words of scratch (x N) each op needs for a chunk of B ciphertexts at level l
static size_t ks_limbs(const srk_ctx *c, int level, int B) {
    const size_t nl = level + 1, ne = nl + c->n_p, beta = (nl + c->alpha - 1) / c->alpha;
    // + two stream lanes of {acc, conversion, special limbs z, rounding bytes}
    return (size_t)B * (nl + beta * ne + 2 * (2 * ne + 2 * nl + 2 * (c->n_p + 1) + 1));
}
static size_t rescale_limbs(int level, int B) { return (size_t)B * (2 + 2 * (size_t)level); }
static size_t relin_limbs(const srk_ctx *c, int level, int B) {
    const size_t nl = level + 1;
    return (size_t)B * (3 * nl + 2 * nl) + std::max(ks_limbs(c, level, B), rescale_limbs(level, B));
}

// Two op sequences issued alternately on the caller's main stream and on this
// branch stream run side by side: ops on the branch stream use the context's second
// set of internal NTT streams and events instead of queueing behind the main stream's.
extern "C" int srk_ctx_set_branch_stream(srk_ctx *c, void *stream) {
    if (!c) return fail(SRK_EINVAL, "null context");
    c->branch = (cudaStream_t)stream;
    return SRK_OK;
}

extern "C" size_t srk_workspace_bytes(const srk_ctx *c) {
    const int L = c->L;
    const int WB = c->ws_batch;
    size_t limbs = std::max({relin_limbs(c, L, WB), ks_limbs(c, L, WB) + 4 * (L + 1),
                             rescale_limbs(L, WB) + 2 * (size_t)(L + 1) * WB,
                             (size_t)4 * c->n_primes, (size_t)2 * (L + 1)});
    return limbs * c->n * sizeof(uint64_t) + 256;
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
    t.itw = c->d_itw;
    t.twd = c->d_twd;
    t.itwd = c->d_itwd;
    return t;
}

static FuseArgs no_fuse() {
    FuseArgs f;
    memset(&f, 0, sizeof f);
    f.galois = 1;
    f.out_galois = 1;
    f.out_galois_inv = 1;
    return f;
}

// cudaLaunchKernelEx wrapper (explicit config; arguments converted to the kernel's types)
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args &&...args) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <int LOG_T, bool INV, bool COL, int IO, int KM, int LOGN>
static void launch_kernel_n(dim3 grid, int threads, size_t smem, cudaStream_t s, const LimbBatch &bb,
                            const NttTables &tb, int log_n, const FuseArgs &ff) {
    // the attribute is per device: one bit per device ordinal
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_relaxed) & bit)) {
        cudaFuncSetAttribute(ntt_pass_kernel<LOG_T, INV, COL, IO, KM, LOGN>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr_done.fetch_or(bit, std::memory_order_relaxed);
    }
    launch_ex(ntt_pass_kernel<LOG_T, INV, COL, IO, KM, LOGN>, grid, dim3(threads), smem, s, bb, tb, log_n, ff);
}
// ring 2^16 (every BASELINE config past config 1): compile-time shape
template <int LOG_T, bool INV, bool COL, int IO, int KM>
static void launch_kernel(dim3 grid, int threads, size_t smem, cudaStream_t s, const LimbBatch &bb,
                          const NttTables &tb, int log_n, const FuseArgs &ff) {
    if constexpr (LOG_T == 8) {
        if (log_n == 16) {
            launch_kernel_n<LOG_T, INV, COL, IO, KM, 16>(grid, threads, smem, s, bb, tb, log_n, ff);
            return;
        }
    }
    launch_kernel_n<LOG_T, INV, COL, IO, KM, 0>(grid, threads, smem, s, bb, tb, log_n, ff);
}

template <int LOG_T, bool INV, bool COL, int IO>
static int launch_pass(const srk_ctx *c, LimbBatch b, int l0, int nlc, const FuseArgs &f,
                       cudaStream_t s, bool f64) {
    using SH = NttShape<LOG_T>;
    const int subs = c->n >> LOG_T;  // sub-transforms per limb
    int cb = c->ntt_cta_threads / SH::TPS;
    if (cb > subs) cb = subs;
    // small batches (single-ciphertext ops): narrower tiles so the grid covers
    // several waves of the 148 SMs instead of ~1 wave plus a long tail
    while (cb > 4 && (long long)(subs / cb) * nlc * b.n_polys < 148 * 3 * 4) cb >>= 1;
    const int threads = cb * SH::TPS;
    const size_t smem = COL ? (size_t)cb * SH::T * 8 : (size_t)cb * (SH::T + SH::T / SH::E) * 8;
    // shift the batch to start at limb l0 (mode 0: pointer + prime offsets; mode 1 keeps the
    // slot map, which is absolute, so only chunk by whole batches there)
    LimbBatch bb = b;
    FuseArgs ff = f;
    if (l0) {
        bb.ptr = b.ptr + (long long)l0 * c->n;
        bb.split = b.split - l0;
        bb.off_a = b.off_a + l0;
        bb.off_b = b.off_b + l0;
        if (ff.src && (IO == LD_PLAIN || IO == LD_AUTO) && COL != INV) ff.src += (long long)l0 * c->n;
        if (ff.out) ff.out += (long long)l0 * c->n;
        if (ff.acc) ff.acc += (long long)l0 * c->n;
        if (ff.add0) ff.add0 += (long long)l0 * c->n;
        if (ff.add1) ff.add1 += (long long)l0 * c->n;
        if (ff.pt) ff.pt += (long long)l0 * c->n;
        if (ff.ks_d) ff.ks_d += (long long)l0 * c->n;
        if (ff.ks_ext) ff.ks_ext += (long long)l0 * c->n;
        if (ff.ks_key) ff.ks_key += (long long)l0 * c->n;
        for (int k = 0; k + l0 < SRK_MAXP; k++) {
            ff.mulc.w[k] = f.mulc.w[k + l0];
            ff.mulc.ws[k] = f.mulc.ws[k + l0];
            ff.pre.w[k] = f.pre.w[k + l0];
            ff.pre.ws[k] = f.pre.ws[k + l0];
            ff.addc.w[k] = f.addc.w[k + l0];
            ff.addc.ws[k] = f.addc.ws[k + l0];
        }
    }
    bb.n_limbs = nlc;
    dim3 grid(subs / cb, b.n_polys, nlc);
    // FP64-only kernel for q < 2^41 chunks, Harvey-only integer kernel otherwise; both
    // passes of a transform use the same one (the intermediate format differs).  The
    // rescale's FP64 spread needs the dropped prime < 2^41 too (IO 2 on either pass:
    // LD_SPREAD first, ST_RESCALE last)
    if (f64 && (IO != 2 || f.top_q < SRK_F64_Q))
        launch_kernel<LOG_T, INV, COL, IO, 1>(grid, threads, smem, s, bb, tables(c), c->log_n, ff);
    else
        launch_kernel<LOG_T, INV, COL, IO, 2>(grid, threads, smem, s, bb, tables(c), c->log_n, ff);
    LAUNCHED();
    return SRK_OK;
}

template <bool INV, bool COL, int IO>
static int pass_t(const srk_ctx *c, int log_t, LimbBatch b, int l0, int nlc, const FuseArgs &f,
                  cudaStream_t s, bool f64) {
    switch (log_t) {
        case 5: return launch_pass<5, INV, COL, IO>(c, b, l0, nlc, f, s, f64);
        case 6: return launch_pass<6, INV, COL, IO>(c, b, l0, nlc, f, s, f64);
        case 7: return launch_pass<7, INV, COL, IO>(c, b, l0, nlc, f, s, f64);
        case 8: return launch_pass<8, INV, COL, IO>(c, b, l0, nlc, f, s, f64);
        default: return fail(SRK_EINVAL, "unsupported NTT pass size 2^%d", log_t);
    }
}

// forward: first pass fused load `ld` (LD_PLAIN/LD_SPREAD), last pass store `st`
// (ST_PLAIN/ST_KSC/ST_RESCALE); inverse: ld in {LD_PLAIN, LD_AUTO}, st in {ST_PLAIN, ST_SCALE}
static int ntt_run(const srk_ctx *c, LimbBatch b, bool inverse, const FuseArgs &f, int ld, int st,
                   cudaStream_t s) {
    if (b.n_limbs <= 0 || b.n_polys <= 0) return SRK_OK;
    const int log_r = (c->log_n + 1) / 2, log_c = c->log_n - log_r;
    // chunk whole limb indices (all polys of a limb) so the intermediate stays in L2
    int per = c->ntt_chunk / b.n_polys;
    if (per < 1) per = 1;
    if (per > 65535 / b.n_polys) per = 65535 / b.n_polys;
    if (b.mode == 1 && per < b.n_limbs) per = b.n_limbs;  // slot map is absolute
    if ((long long)per * b.n_polys > 65535) return fail(SRK_EINVAL, "NTT batch too large");
    // mode-0 batches: split chunks where the prime class changes, so runs of
    // limbs under primes < 2^41 use the FP64-only pass kernels
    auto f64_limb = [&](int i) {
        const int pid = i + (i < b.split ? b.off_a : b.off_b);
        return c->primes[pid] < SRK_F64_Q;
    };
    struct Chunk {
        int l0, nlc;
        bool f64;
        int cls;
    };
    std::vector<Chunk> chunks;
    if (b.mode == 1) {
        // ModUp targets mix 40-bit and 60-bit primes per digit: one FP64 launch that
        // skips the >= 2^41 limbs and one integer launch that skips the rest
        // (independent, so they run on the two streams side by side)
        chunks.push_back({0, b.n_limbs, true, 1});
        chunks.push_back({0, b.n_limbs, false, 2});
    }
    for (int l0 = 0, nlc = 0; b.mode == 0 && l0 < b.n_limbs; l0 += nlc) {
        nlc = std::min(per, b.n_limbs - l0);
        const bool f64 = f64_limb(l0);
        int k = 1;
        while (k < nlc && f64_limb(l0 + k) == f64) k++;
        nlc = k;
        chunks.push_back({l0, nlc, f64, 0});
    }
    // independent chunks alternate between s and this lane's NTT side stream
    const int lane = (s == c->side || (c->branch && s == c->branch)) ? 1 : 0;
    const bool two = c->ntt_streams >= 2 && chunks.size() >= 2 && c->nside[lane];
    if (two) {
        CU(cudaEventRecord(c->ev_nfork[lane], s));
        CU(cudaStreamWaitEvent(c->nside[lane], c->ev_nfork[lane], 0));
    }
    for (size_t ci = 0; ci < chunks.size(); ci++) {
        const int l0 = chunks[ci].l0, nlc = chunks[ci].nlc;
        const bool f64 = chunks[ci].f64;
        b.cls = chunks[ci].cls;
        cudaStream_t cs = (two && (ci & 1)) ? c->nside[lane] : s;
        if (!inverse) {
            switch (ld) {
                case LD_PLAIN: TRY((pass_t<false, true, LD_PLAIN>(c, log_r, b, l0, nlc, f, cs, f64))); break;
                case LD_SPREAD: TRY((pass_t<false, true, LD_SPREAD>(c, log_r, b, l0, nlc, f, cs, f64))); break;
                default: return fail(SRK_EINVAL, "bad forward load mode");
            }
            switch (st) {
                case ST_PLAIN: TRY((pass_t<false, false, ST_PLAIN>(c, log_c, b, l0, nlc, f, cs, f64))); break;
                case ST_KSC: TRY((pass_t<false, false, ST_KSC>(c, log_c, b, l0, nlc, f, cs, f64))); break;
                case ST_RESCALE: TRY((pass_t<false, false, ST_RESCALE>(c, log_c, b, l0, nlc, f, cs, f64))); break;
                default: return fail(SRK_EINVAL, "bad forward store mode");
            }
        } else {
            switch (ld) {
                case LD_PLAIN: TRY((pass_t<true, false, LD_PLAIN>(c, log_c, b, l0, nlc, f, cs, f64))); break;
                case LD_AUTO: TRY((pass_t<true, false, LD_AUTO>(c, log_c, b, l0, nlc, f, cs, f64))); break;
                default: return fail(SRK_EINVAL, "bad inverse load mode");
            }
            switch (st) {
                case ST_PLAIN: TRY((pass_t<true, true, ST_PLAIN>(c, log_r, b, l0, nlc, f, cs, f64))); break;
                case ST_SCALE: TRY((pass_t<true, true, ST_SCALE>(c, log_r, b, l0, nlc, f, cs, f64))); break;
                default: return fail(SRK_EINVAL, "bad inverse store mode");
            }
        }
    }
    if (two) {
        CU(cudaEventRecord(c->ev_njoin[lane], c->nside[lane]));
        CU(cudaStreamWaitEvent(s, c->ev_njoin[lane], 0));
    }
    return SRK_OK;
}

static int ntt_batch(const srk_ctx *c, LimbBatch b, bool inverse, cudaStream_t s) {
    return ntt_run(c, b, inverse, no_fuse(), LD_PLAIN, ST_PLAIN, s);
}

// n_polys polys of n_limbs limbs (limb i under prime first + i), uniform poly stride
static LimbBatch qbatch(uint64_t *p, int n_polys, long long pstride, int n_limbs, int first) {
    LimbBatch b;
    memset(&b, 0, sizeof b);
    b.ptr = p;
    b.poly_stride = pstride;
    b.ct_stride = 0;
    b.ppc = n_polys > 0 ? n_polys : 1;
    b.n_polys = n_polys;
    b.n_limbs = n_limbs;
    b.mode = 0;
    b.split = 1 << 30;
    b.off_a = first;
    b.off_b = first;
    return b;
}
// B ciphertexts of ppc polys each: poly (b, r) at p + b*ct + r*ps
static LimbBatch cbatch(uint64_t *p, int B, int ppc, long long ct, long long ps, int n_limbs,
                        int first) {
    LimbBatch b = qbatch(p, B * ppc, ps, n_limbs, first);
    b.ppc = ppc;
    b.ct_stride = ct;
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
    LimbBatch b = qbatch(data, n_polys, poly_stride, level + 1 + c->n_p, 0);
    b.split = level + 1;
    b.off_b = c->L - level;
    return ntt_batch(c, b, inverse != 0, S(stream));
}

extern "C" int srk_addsub(srk_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out,
                          int level, int op, void *stream) {
    TRY(check_level(c, level));
    if (op < 0 || op > 2) return fail(SRK_EINVAL, "bad op");
    const long long total = 2ll * (level + 1) * c->n;
    k_addsub<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, b, out, c->d_pc, c->log_n, level + 1, op,
                                                        total);
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

extern "C" int srk_addsub_batch(srk_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out,
                                int batch, int level, int op, void *stream) {
    TRY(check_level(c, level));
    if (op < 0 || op > 2 || batch < 1) return fail(SRK_EINVAL, "bad op or batch");
    const long long total = 2ll * batch * (level + 1) * c->n;
    k_addsub<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, b, out, c->d_pc, c->log_n, level + 1, op,
                                                        total);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_add_const(srk_ctx *c, const uint64_t *a, const uint64_t *k_res, uint64_t *out,
                             int level, void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc = host_consts(c, k_res, level + 1);
    const long long total = 2ll * (level + 1) * c->n;
    k_add_plain<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, nullptr, 0, lc, out, c->d_pc, c->log_n,
                                                           level + 1, 1);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_add_plain(srk_ctx *c, const uint64_t *a, const uint64_t *pt, uint64_t *out,
                             int level, void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    const long long total = 2ll * (level + 1) * c->n;
    k_add_plain<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, pt, 0, lc, out, c->d_pc, c->log_n,
                                                           level + 1, 1);
    LAUNCHED();
    return SRK_OK;
}

// batched add of a constant (pt == NULL, residues k_res) or plaintexts pt
// (stride pt_ct words, 0 = one plaintext for all) to poly 0 of every ciphertext
extern "C" int srk_add_plain_batch(srk_ctx *c, const uint64_t *a, const uint64_t *pt, long long pt_ct,
                                   const uint64_t *k_res, uint64_t *out, int batch, int level,
                                   void *stream) {
    TRY(check_level(c, level));
    LimbConsts lc;
    memset(&lc, 0, sizeof lc);
    if (!pt) {
        if (!k_res) return fail(SRK_EINVAL, "need a plaintext or constant residues");
        lc = host_consts(c, k_res, level + 1);
    }
    const long long total = 2ll * batch * (level + 1) * c->n;
    k_add_plain<<<grid_for(total, 2), 256, 0, S(stream)>>>(a, pt, pt_ct, lc, out, c->d_pc, c->log_n,
                                                           level + 1, batch);
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
    k_tensor<<<grid_for(total), 256, 0, S(stream)>>>(a, b, 0, d, 0, c->d_pc, c->log_n, level + 1, 1);
    LAUNCHED();
    return SRK_OK;
}

// ---------------------------------------------------------------------
// rescale: B ciphertexts (a: ct stride a_ct, poly stride a_ps) at `level`
// -> out (ct stride out_ct, poly stride level*N), dividing by q_level with
// rounding.  Optional pre-multiplier: mode 1 per-limb constant k, mode 2
// plaintext pt [level+1][N].  Two fused transforms:
//   INTT(top limb) [x k folded into the N^-1 scale]  ->  top
//   NTT(centred(top) mod q_i) with the combine (a*pre - .) q_l^-1 in its store
// ---------------------------------------------------------------------
static int rescale_impl(srk_ctx *c, const uint64_t *a, long long a_ct, long long a_ps,
                        const uint64_t *pt, const LimbConsts *k, uint64_t *out, long long out_ct,
                        int level, int B, uint64_t *ws, cudaStream_t s, long long pt_ct = 0) {
    if (level < 1) return fail(SRK_EINVAL, "cannot rescale a level-0 ciphertext");
    const long long n = c->n;
    uint64_t *top = ws;              // [B][2][N]
    uint64_t *tb = ws + 2ll * B * n; // [B][2][level][N]
    const int mode = pt ? 2 : (k ? 1 : 0);
    FuseArgs f = no_fuse();
    LimbBatch bt = cbatch(top, B, 2, 2 * n, n, 1, level);
    if (mode == 2) {
        k_rescale_top<<<grid_for(2ll * B * n), 256, 0, s>>>(a, a_ct, a_ps, pt, pt_ct, top, c->d_pc,
                                                             c->log_n, level, B);
        LAUNCHED();
        TRY(ntt_run(c, bt, true, f, LD_PLAIN, ST_PLAIN, s));
    } else {
        f.src = a + (long long)level * n;
        f.src_ct = a_ct;
        f.src_ps = a_ps;
        if (mode == 1) {
            const uint64_t q = c->primes[level];
            const uint64_t w = hmul(hinv((uint64_t)c->n, q), k->w[level], q);
            f.mulc.w[0] = w;
            f.mulc.ws[0] = shoup(w, q);
        }
        TRY(ntt_run(c, bt, true, f, LD_PLAIN, mode == 1 ? ST_SCALE : ST_PLAIN, s));
    }
    FuseArgs g = no_fuse();
    g.src = top;
    g.src_ct = 2 * n;
    g.src_ps = n;
    g.top_q = c->primes[level];
    g.out = out;
    g.out_ct = out_ct;
    g.out_ps = (long long)level * n;
    g.acc = a;
    g.acc_ct = a_ct;
    g.acc_ps = a_ps;
    g.pre_mode = mode;
    g.pt = pt ? pt : a;  // never null: the store's loads may be speculated
    g.pt_ct = pt ? pt_ct : 0;
    if (k) g.pre = *k;
    g.mulc = c->lc_qlinv[level];
    LimbBatch bq = cbatch(tb, B, 2, 2ll * level * n, (long long)level * n, level, 0);
    return ntt_run(c, bq, false, g, LD_SPREAD, ST_RESCALE, s);
}

// chunk a batch of B into balanced pieces of at most c->ws_batch (36 -> 18 + 18,
// not 32 + 4: a small remainder chunk runs its kernels at a fraction of the GPU)
static inline int chunk_size(int B, int ws) {
    const int pieces = (B + ws - 1) / ws;
    return pieces > 0 ? (B + pieces - 1) / pieces : 1;
}
#define FOR_CHUNKS(B, b0, nb)                                                                        \
    for (int b0 = 0, cs_ = chunk_size((B), c->ws_batch), nb = std::min(cs_, (B)); b0 < (B);         \
         b0 += nb, nb = std::min(cs_, (B) - b0))

extern "C" int srk_rescale(srk_ctx *c, const uint64_t *a, uint64_t *out, int level, void *ws,
                           void *stream) {
    TRY(check_level(c, level));
    const long long ps = (long long)(level + 1) * c->n;
    return rescale_impl(c, a, 2 * ps, ps, nullptr, nullptr, out, 2ll * level * c->n, level, 1,
                        (uint64_t *)ws, S(stream));
}

extern "C" int srk_rescale_batch(srk_ctx *c, const uint64_t *a, long long a_ct, uint64_t *out,
                                 long long out_ct, int batch, int level, void *ws, void *stream) {
    TRY(check_level(c, level));
    const long long ps = (long long)(level + 1) * c->n;
    FOR_CHUNKS(batch, b0, nb) {
        TRY(rescale_impl(c, a + b0 * a_ct, a_ct, ps, nullptr, nullptr, out + b0 * out_ct, out_ct,
                         level, nb, (uint64_t *)ws, S(stream)));
    }
    return SRK_OK;
}

extern "C" int srk_mul_const_rescale(srk_ctx *c, const uint64_t *a, int src_limbs,
                                     const uint64_t *k_res, uint64_t *out, int level, void *ws,
                                     void *stream) {
    TRY(check_level(c, level));
    if (src_limbs < level + 1) return fail(SRK_EINVAL, "source has fewer limbs than level+1");
    LimbConsts lc = host_consts(c, k_res, level + 1);
    const long long ps = (long long)src_limbs * c->n;
    return rescale_impl(c, a, 2 * ps, ps, nullptr, &lc, out, 2ll * level * c->n, level, 1,
                        (uint64_t *)ws, S(stream));
}

// batch versions: a at ct stride a_ct read as a level-`level` view (src_limbs
// limbs per poly); outputs packed [batch][2][level][N]
extern "C" int srk_mul_const_rescale_batch(srk_ctx *c, const uint64_t *a, long long a_ct, int src_limbs,
                                           const uint64_t *k_res, uint64_t *out, int batch, int level,
                                           void *ws, void *stream) {
    TRY(check_level(c, level));
    if (src_limbs < level + 1) return fail(SRK_EINVAL, "source has fewer limbs than level+1");
    LimbConsts lc = host_consts(c, k_res, level + 1);
    const long long ps = (long long)src_limbs * c->n, oct = 2ll * level * c->n;
    FOR_CHUNKS(batch, b0, nb) {
        TRY(rescale_impl(c, a + b0 * a_ct, a_ct, ps, nullptr, &lc, out + b0 * oct, oct, level, nb,
                         (uint64_t *)ws, S(stream)));
    }
    return SRK_OK;
}

extern "C" int srk_mul_plain_rescale_batch(srk_ctx *c, const uint64_t *a, const uint64_t *pt,
                                           long long pt_ct, uint64_t *out, int batch, int level,
                                           void *ws, void *stream) {
    TRY(check_level(c, level));
    const long long ps = (long long)(level + 1) * c->n, oct = 2ll * level * c->n;
    FOR_CHUNKS(batch, b0, nb) {
        TRY(rescale_impl(c, a + b0 * 2 * ps, 2 * ps, ps, pt + b0 * pt_ct, nullptr, out + b0 * oct, oct,
                         level, nb, (uint64_t *)ws, S(stream), pt_ct));
    }
    return SRK_OK;
}

extern "C" int srk_mul_plain_rescale(srk_ctx *c, const uint64_t *a, const uint64_t *pt,
                                     uint64_t *out, int level, void *ws, void *stream) {
    TRY(check_level(c, level));
    const long long ps = (long long)(level + 1) * c->n;
    return rescale_impl(c, a, 2 * ps, ps, pt, nullptr, out, 2ll * level * c->n, level, 1,
                        (uint64_t *)ws, S(stream));
}

// ---------------------------------------------------------------------
// hybrid key switching (keyswitch_impl below)
// ---------------------------------------------------------------------
// conversion grids (x = target groups, y = polys, z = coefficient tiles): z shrunk by up
// to conv_cpt tiles per CTA (to amortise the CTA's constant staging) only while >= ~3
// waves of CTAs remain, so the one-ciphertext ops of the pipelines keep enough CTAs in flight
static inline dim3 conv_grid(const srk_ctx *c, dim3 g) {
    const unsigned long long ctas = (unsigned long long)g.x * g.y * g.z;
    unsigned cpt = c->conv_cpt;
    while (cpt > 1 && ctas / cpt < 148ull * 8 * 3) cpt >>= 1;
    return dim3(g.x, g.y, std::max(1u, g.z / cpt));
}

// source-tile buffers of a conversion launch: two (the next tile streams in while
// this one is converted) when a CTA walks several tiles and two CTAs of that size
// still fit an SM, else one
static inline int bconv_nbuf(const srk_ctx *c, int n_src, bool multi_tile) {
    (void)c;
    return multi_tile && bconv_smem_bytes(n_src, 2) <= 100 * 1024 ? 2 : 1;
}
// opt in to > 48 KiB of dynamic shared memory (once per kernel and device)
template <typename K>
static int bconv_attr(K kern, size_t smem) {
    if (smem <= 32 * 1024) return SRK_OK;  // static tables (< 8 KiB) + this stay under the 48 KiB default
    static std::mutex mu;
    static std::vector<std::pair<const void *, unsigned long long>> done;  // kernel -> device bits
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : done)
        if (e.first == (const void *)kern) {
            if (e.second & bit) return SRK_OK;
            CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            e.second |= bit;
            return SRK_OK;
        }
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    done.emplace_back((const void *)kern, bit);
    return SRK_OK;
}

// ModDown base conversion P (or P u {q_l}) -> q_0..q_{nout-1} with exact rounding,
// coefficient domain, into conv [B][2][nout] (ct stride cv_ct, poly stride cv_ps):
//   conv[t] = sum_k z_k m_kt - v [prod src]_{q_t},  v = round(sum_k z_k / p_k)
static int moddown_conv(srk_ctx *c, const BconvPlan &pl, const uint64_t *z, long long z_ct, long long z_ps,
                        const uint8_t *vround, uint64_t *conv, long long cv_ct, long long cv_ps, int B,
                        int nout, cudaStream_t s) {
    const long long n = c->n;
    const int ns = pl.n_src;
    if (ns > SRK_BCONV_MAXSRC) return fail(SRK_EINVAL, "ModDown with more than 17 source primes");
    if (ns <= 4) {
        // few sources: one coefficient per thread, sources in registers (bconv.cuh)
        dim3 grid((nout + SRK_BCONV_TG - 1) / SRK_BCONV_TG, 2 * B, (unsigned)((n + 255) / 256));
        const dim3 g2 = conv_grid(c, grid);
#define SRK_CONV_SMALL(K)                                                                                  \
    case K:                                                                                                \
        launch_ex(k_moddown_conv_small<K>, g2, dim3(256), 0, s, z, z_ct, z_ps, vround, pl.mhl, pl.fhl,     \
                  pl.n_dst, pl.dst_corr, conv, cv_ct, cv_ps, c->d_pc, c->log_n);                           \
        break;
        switch (ns) { SRK_CONV_SMALL(1) SRK_CONV_SMALL(2) SRK_CONV_SMALL(3) SRK_CONV_SMALL(4) }
#undef SRK_CONV_SMALL
        LAUNCHED();
        return SRK_OK;
    }
    const int tg = SRK_BCONV_TG;
    dim3 grid((nout + tg - 1) / tg, 2 * B, (unsigned)((n + SRK_BCONV_TILE - 1) / SRK_BCONV_TILE));
    const dim3 g2 = conv_grid(c, grid);
    const int nbuf = bconv_nbuf(c, ns, g2.z < grid.z);
    const size_t smem = bconv_smem_bytes(ns, nbuf);
#define SRK_MODDOWN_CONV(NB, TG)                                                                            \
    do {                                                                                                    \
        TRY(bconv_attr(k_moddown_conv<NB, TG>, smem));                                                      \
        launch_ex(k_moddown_conv<NB, TG>, g2, dim3(256), smem, s, z, z_ct, z_ps, ns, vround, pl.mhl, pl.fhl, \
                  pl.n_dst, pl.dst_corr, conv, cv_ct, cv_ps, c->d_pc, c->log_n);                            \
    } while (0)
    if (nbuf == 2) SRK_MODDOWN_CONV(2, 8); else SRK_MODDOWN_CONV(1, 8);
#undef SRK_MODDOWN_CONV
    LAUNCHED();
    return SRK_OK;
}

struct KsOut {
    uint64_t *out;
    long long out_ct, out_ps;
    const uint64_t *key;
    uint64_t galois;
    const uint64_t *add0, *add1;  // optional addends (nullptr: none)
    long long add_ct;
};

// Hybrid key switching of B polys d (ct stride d_ct, NTT form, level `level`):
//   1. INTT(d) with (Q_j/q_i)^-1 folded into the N^-1 scale  -> dc
//   2. ModUp base conversion of every digit                   -> ext (coef)
//   3. NTT of every ModUp target limb (one batched call)
// then, for each output o (Galois element g; 1 = relinearisation):
//   4. inner product with key g over the special limbs only    -> acc_P
//   5. INTT of acc_P with (P/p_k)^-1 folded in, rounding term v
//   6. ModDown conversion P -> Q (coefficient domain)          -> conv
//   7. NTT(conv) whose row pass computes, per output limb t,
//        out = sigma_g(add + (sum_j e_j key_j - NTT(conv)) P^-1)
//      -- the ciphertext-modulus limbs' inner product is never written to HBM
//      (ST_KSC, ntt.cuh ksc_epilogue).
// Rotations run in sigma_g^-1 space (rotation-layout keys): exact ModDown commutes
// with sigma_g, so only the last store permutes.
// rescale_d: fused HMult rescale -- outs[0].add0/add1 are d0/d1 (ct stride add_ct,
// poly stride = level+1 limbs) and the output is round((acc + P d) / (P q_level)) at
// level-1: special basis S = P u {q_level}, bit-identical to ModDown then rescale
// (consecutive roundings by odd moduli compose exactly).
static uint64_t galois_inverse(const srk_ctx *c, uint64_t g) {
    // (Z/2N)^* has order N, so g^-1 = g^(N-1) mod 2N
    const uint64_t two_n = 2ull * c->n;
    uint64_t r = 1, b = g % two_n, e = (uint64_t)c->n - 1;
    while (e) {
        if (e & 1) r = r * b % two_n;
        b = b * b % two_n;
        e >>= 1;
    }
    return r;
}

static int keyswitch_impl(srk_ctx *c, const uint64_t *d, long long d_ct, const KsOut *outs,
                          int n_out, int level, int B, uint64_t *ws, cudaStream_t s,
                          bool rescale_d = false) {
    const long long n = c->n;
    const int nl = level + 1, K = c->n_p, ne = nl + K;
    const int alpha = c->alpha, beta = (nl + alpha - 1) / alpha;
    if (beta > SRK_MAX_DIGITS) return fail(SRK_EINVAL, "too many digits");
    if (rescale_d && level < 1) return fail(SRK_EINVAL, "cannot rescale a level-0 ciphertext");
    // the base conversions move coefficient pairs with 16-byte copies and stores
    if (((uintptr_t)ws & 15) || (n & 1)) return fail(SRK_EINVAL, "key-switch workspace must be 16-byte aligned");
    uint64_t *dc = ws;                                 // [B][nl]
    uint64_t *ext = dc + (long long)B * nl * n;        // [B][beta][ne]
    // per-output scratch, one set per stream lane (outputs alternate between the
    // caller's stream and the context's side stream so their small latency-bound
    // kernels overlap the large ones)
    uint64_t *lane_acc[2], *lane_conv[2], *lane_zb[2];
    uint8_t *lane_vround[2];
    {
        uint64_t *q = ext + (long long)B * beta * ne * n;
        for (int l = 0; l < 2; l++) {
            lane_acc[l] = q;                                          // [B][2][ne]
            lane_conv[l] = q + (long long)B * 2 * ne * n;             // [B][2][nl]
            lane_zb[l] = lane_conv[l] + (long long)B * 2 * nl * n;    // [B][2][K(+1)] special limbs, coef
            lane_vround[l] = (uint8_t *)(lane_zb[l] + (long long)B * 2 * (K + 1) * n);  // [B][2][N] bytes
            q = (uint64_t *)lane_vround[l] + (long long)B * n;
        }
    }
    const bool dual = n_out >= 2 && !rescale_d && c->ks_streams >= 2 && c->side;
    cudaStream_t lane_s[2] = {s, dual ? c->side : s};

    // 1. INTT with the ModUp scale folded in
    {
        FuseArgs f = no_fuse();
        f.src = d;
        f.src_ct = d_ct;
        f.src_ps = 0;
        f.mulc = c->lc_modup_scale[level];
        TRY(ntt_run(c, cbatch(dc, B, 1, (long long)nl * n, 0, nl, 0), true, f, LD_PLAIN, ST_SCALE, s));
    }
    // 2. ModUp conversion, all digits
    {
        ModUpArgs m;
        memset(&m, 0, sizeof m);
        m.dc = dc;
        m.dc_ct = (long long)nl * n;
        m.ext = ext;
        m.ext_ct = (long long)beta * ne * n;
        m.ext_dig = (long long)ne * n;
        m.nl = nl;
        m.beta = beta;
        m.alpha = alpha;
        int maxd = 0;
        for (int j = 0; j < beta; j++) {
            const BconvPlan &pl = c->modup[level][j];
            m.mat[j] = pl.mat;
            m.slot[j] = pl.dst_slot;
            m.pid[j] = pl.dst_pid;
            m.n_dst[j] = pl.n_dst;
            m.mhl[j] = pl.mhl;
            m.fhl[j] = pl.fhl;
            maxd = std::max(maxd, pl.n_dst);
        }
        // FP64-pipe conversion when every source but a digit's first is < 2^41
        bool f64ok = true, wide0 = false;
        for (int j = 0; j < beta; j++)
            for (int i = 0; i < alpha && j * alpha + i < nl; i++)
                if (c->primes[j * alpha + i] >= SRK_F64_Q) {
                    if (i == 0 && j == 0)
                        wide0 = true;
                    else
                        f64ok = false;
                }
        dim3 grid((unsigned)((n + 255) / 256), B * beta, (maxd + SRK_MODUP_TCH - 1) / SRK_MODUP_TCH);
        if (f64ok && alpha <= 16) {
            dim3 gb((maxd + SRK_BCONV_TG - 1) / SRK_BCONV_TG, B * beta, (unsigned)((n + SRK_BCONV_TILE - 1) / SRK_BCONV_TILE));
            const dim3 g2 = conv_grid(c, gb);
            const int nbuf = bconv_nbuf(c, alpha, g2.z < gb.z);
            const size_t smem = bconv_smem_bytes(alpha, nbuf);
#define SRK_MODUP_CONV(W, NB)                                                     \
    do {                                                                          \
        TRY(bconv_attr(k_modup_conv<W, NB>, smem));                               \
        launch_ex(k_modup_conv<W, NB>, g2, dim3(256), smem, s, m, c->d_pc, c->log_n); \
    } while (0)
            if (nbuf == 2) {
                if (wide0) SRK_MODUP_CONV(true, 2); else SRK_MODUP_CONV(false, 2);
            } else {
                if (wide0) SRK_MODUP_CONV(true, 1); else SRK_MODUP_CONV(false, 1);
            }
#undef SRK_MODUP_CONV
        } else {
            // general parameter sets (wide scaling primes): 128-bit MAC + Barrett
            switch (alpha) {
                case 1: launch_ex(k_modup<1>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 2: launch_ex(k_modup<2>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 3: launch_ex(k_modup<3>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 4: launch_ex(k_modup<4>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 5: launch_ex(k_modup<5>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 6: launch_ex(k_modup<6>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 7: launch_ex(k_modup<7>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 8: launch_ex(k_modup<8>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 9: launch_ex(k_modup<9>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 10: launch_ex(k_modup<10>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 11: launch_ex(k_modup<11>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 12: launch_ex(k_modup<12>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 13: launch_ex(k_modup<13>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 14: launch_ex(k_modup<14>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 15: launch_ex(k_modup<15>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
                default: launch_ex(k_modup<16>, grid, dim3(256), 0, s, m, (const PrimeConst *)c->d_pc, c->log_n); break;
            }
        }
        LAUNCHED();
    }
    // 3. NTT of all ModUp targets
    {
        LimbBatch b = cbatch(ext, B, beta, (long long)beta * ne * n, (long long)ne * n, 0, 0);
        const int glast = nl - (beta - 1) * alpha;
        b.mode = 1;
        b.n_limbs = ne - glast;
        b.alpha = alpha;
        b.nl = nl;
        b.level = level;
        b.L = c->L;
        b.ne = ne;
        TRY(ntt_run(c, b, false, no_fuse(), LD_PLAIN, ST_PLAIN, s));
    }
    if (dual) {
        CU(cudaEventRecord(c->ev_fork, s));
        CU(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    }
    for (int o = 0; o < n_out; o++) {
        const KsOut &ko = outs[o];
        const int lane = dual ? (o & 1) : 0;
        cudaStream_t so = lane_s[lane];
        uint64_t *acc = lane_acc[lane], *conv = lane_conv[lane], *zb = lane_zb[lane];
        uint8_t *vround = lane_vround[lane];
        // 4. inner product over the special limbs (+ limb `level` for the fused rescale)
        KsInnerArgs ka;
        ka.d = d;
        ka.d_ct = d_ct;
        ka.ext = ext;
        ka.ext_ct = (long long)beta * ne * n;
        ka.ext_dig = (long long)ne * n;
        ka.key = ko.key;
        ka.acc = acc;
        ka.acc_ct = 2ll * ne * n;
        ka.galois = ko.galois;
        ka.n_primes = c->n_primes;
        ka.nl = nl;
        ka.ne = ne;
        ka.level = level;
        ka.L = c->L;
        ka.alpha = alpha;
        ka.beta = beta;
        ka.batch = B;
        ka.t0 = rescale_d ? level : nl;
        {
            const int blocks = grid_for((long long)(ne - ka.t0) * n);
            switch (beta) {
                case 1: launch_ex(k_ks_inner<1>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 2: launch_ex(k_ks_inner<2>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 3: launch_ex(k_ks_inner<3>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n); break;
                case 4: launch_ex(k_ks_inner<4>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n); break;
                default:
                    if (beta <= 8)
                        launch_ex(k_ks_inner<8>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n);
                    else if (beta <= 16)
                        launch_ex(k_ks_inner<16>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n);
                    else
                        launch_ex(k_ks_inner<64>, dim3(blocks), dim3(256), 0, so, ka, (const PrimeConst *)c->d_pc, c->log_n);
            }
            LAUNCHED();
        }
        // the store's arguments: out = sigma_g(add + (sum_j e_j key_j - NTT(conv)) mulc)
        FuseArgs g = no_fuse();
        g.out = ko.out;
        g.out_ct = ko.out_ct;
        g.out_ps = ko.out_ps;
        g.has_add0 = ko.add0 != nullptr;
        g.has_add1 = ko.add1 != nullptr;
        g.add0 = ko.add0 ? ko.add0 : d;  // valid dummies: loads are never speculated from null
        g.add1 = ko.add1 ? ko.add1 : d;
        g.add_ct = ko.add_ct;
        g.ks_d = d;
        g.ks_d_ct = d_ct;
        g.ks_ext = ext;
        g.ks_ext_ct = (long long)beta * ne * n;
        g.ks_ext_dig = (long long)ne * n;
        g.ks_key = ko.key;
        g.ks_key_j = 2ll * c->n_primes * n;
        g.ks_key_r = (long long)c->n_primes * n;
        g.ks_alpha = alpha;
        g.ks_beta = beta;
        int nout;
        const BconvPlan *plan;
        const uint64_t *zsrc;
        long long z_ct, z_ps;
        if (rescale_d) {
            // 5'. special basis S = P u {q_l}: X_S = (acc_P, acc_l + P d_l), INTT with
            //     N^-1 (S/s_k)^-1 folded in; rounding term over K+1 limbs
            const int ns = K + 1;
            const uint64_t pm = c->lc_pmod.w[level], pms = c->lc_pmod.ws[level];
            launch_ex(k_prep_special, dim3(grid_for(2ll * B * ns * n)), dim3(256), 0, so,
                      (const uint64_t *)acc, 2ll * ne * n, (long long)ne * n, ko.add0, ko.add_ct,
                      (long long)nl * n, zb, pm, pms, (const PrimeConst *)c->d_pc, c->log_n, level, K, B);
            LAUNCHED();
            FuseArgs f = no_fuse();
            f.mulc = c->lc_rs_scale[level];
            LimbBatch b = cbatch(zb, B, 2, 2ll * ns * n, (long long)ns * n, ns, 0);
            b.split = K;
            b.off_a = c->n_q;
            b.off_b = level - K;
            TRY(ntt_run(c, b, true, f, LD_PLAIN, ST_SCALE, so));
            launch_ex(k_moddown_v, dim3(grid_for(2ll * B * n)), dim3(256), 0, so, (const uint64_t *)zb,
                      2ll * ns * n, (long long)ns * n, K, c->n_q, ns, level, vround, (const PrimeConst *)c->d_pc,
                      c->log_n, B);
            LAUNCHED();
            // out = (acc - conv) (P q_l)^-1 + d q_l^-1 over q_0..q_{l-1}
            nout = level;
            plan = &c->moddown_rs[level];
            zsrc = zb;
            z_ct = 2ll * ns * n;
            z_ps = (long long)ns * n;
            g.mulc = c->lc_rs_mulc[level];
            g.add_scaled = 1;
            g.addc = c->lc_qlinv[level];
        } else {
            // 5. INTT of the special limbs, (P/p_k)^-1 folded in -> zb; rounding term
            FuseArgs f = no_fuse();
            f.mulc = c->lc_moddown_scale;
            f.src = acc + (long long)nl * n;
            f.src_ct = 2ll * ne * n;
            f.src_ps = (long long)ne * n;
            LimbBatch b = cbatch(zb, B, 2, 2ll * K * n, (long long)K * n, K, 0);
            b.split = 0;
            b.off_b = c->n_q;
            TRY(ntt_run(c, b, true, f, LD_PLAIN, ST_SCALE, so));
            launch_ex(k_moddown_v, dim3(grid_for(2ll * B * n)), dim3(256), 0, so, (const uint64_t *)zb,
                      2ll * K * n, (long long)K * n, K, c->n_q, K, 0, vround, (const PrimeConst *)c->d_pc,
                      c->log_n, B);
            LAUNCHED();
            nout = nl;
            plan = &c->moddown[level];
            zsrc = zb;
            z_ct = 2ll * K * n;
            z_ps = (long long)K * n;
            g.mulc = c->lc_pinv;
            g.out_galois = ko.galois;
            g.out_galois_inv = galois_inverse(c, ko.galois);
        }
        // 6. conversion, 7. NTT with the key-switch combine in its store
        TRY(moddown_conv(c, *plan, zsrc, z_ct, z_ps, vround, conv, 2ll * nout * n, (long long)nout * n, B,
                         nout, so));
        TRY(ntt_run(c, cbatch(conv, B, 2, 2ll * nout * n, (long long)nout * n, nout, 0), false, g, LD_PLAIN,
                    ST_KSC, so));
    }
    if (dual) {
        CU(cudaEventRecord(c->ev_join, c->side));
        CU(cudaStreamWaitEvent(s, c->ev_join, 0));
    }
    return SRK_OK;
}

extern "C" int srk_keyswitch(srk_ctx *c, const uint64_t *d, const uint64_t *key, uint64_t *out0,
                             uint64_t *out1, int level, void *ws, void *stream) {
    TRY(check_level(c, level));
    if (out1 - out0 <= 0) return fail(SRK_EINVAL, "out1 must follow out0");
    KsOut o = {out0, 0, (long long)(out1 - out0), key, 1, nullptr, nullptr, 0};
    return keyswitch_impl(c, d, 0, &o, 1, level, 1, (uint64_t *)ws, S(stream));
}

// B products a[b] x b[b] (both ct stride ab_ct) -> out (ct stride out_ct)
static int mul_relin_chunk(srk_ctx *c, const uint64_t *a, const uint64_t *b, long long ab_ct,
                           const uint64_t *rlk, uint64_t *out, long long out_ct, int level, int B,
                           bool rescale, uint64_t *ws, cudaStream_t s) {
    const long long n = c->n, nl = level + 1, ps = nl * n;
    uint64_t *d = ws;                       // [B][3][nl]
    uint64_t *prod = d + (long long)B * 3 * ps;  // [B][2][nl]
    uint64_t *rest = prod + (long long)B * 2 * ps;
    k_tensor<<<grid_for(B * ps), 256, 0, s>>>(a, b, ab_ct, d, 3 * ps, c->d_pc, c->log_n, level + 1, B);
    LAUNCHED();
    (void)prod;
    if (rescale) {  // HMult rescale fused into the key switch's ModDown
        KsOut o = {out, out_ct, (long long)level * n, rlk, 1, d, d + ps, 3 * ps};
        return keyswitch_impl(c, d + 2 * ps, 3 * ps, &o, 1, level, B, rest, s, true);
    }
    KsOut o = {out, out_ct, ps, rlk, 1, d, d + ps, 3 * ps};
    return keyswitch_impl(c, d + 2 * ps, 3 * ps, &o, 1, level, B, rest, s);
}

extern "C" int srk_mul_relin(srk_ctx *c, const uint64_t *a, const uint64_t *b,
                             const uint64_t *rlk, uint64_t *out, int level, void *ws,
                             void *stream) {
    TRY(check_level(c, level));
    const long long ps = (long long)(level + 1) * c->n;
    return mul_relin_chunk(c, a, b, 2 * ps, rlk, out, 2 * ps, level, 1, false, (uint64_t *)ws, S(stream));
}

extern "C" int srk_mul_relin_rescale(srk_ctx *c, const uint64_t *a, const uint64_t *b,
                                     const uint64_t *rlk, uint64_t *out, int level, void *ws,
                                     void *stream) {
    TRY(check_level(c, level));
    if (level < 1) return fail(SRK_EINVAL, "depth exhausted");
    const long long ps = (long long)(level + 1) * c->n;
    return mul_relin_chunk(c, a, b, 2 * ps, rlk, out, 2ll * level * c->n, level, 1, true,
                           (uint64_t *)ws, S(stream));
}

extern "C" int srk_mul_relin_batch(srk_ctx *c, const uint64_t *a, const uint64_t *b, long long ab_ct,
                                   const uint64_t *rlk, uint64_t *out, long long out_ct, int batch,
                                   int level, int rescale, void *ws, void *stream) {
    TRY(check_level(c, level));
    if (rescale && level < 1) return fail(SRK_EINVAL, "depth exhausted");
    FOR_CHUNKS(batch, b0, nb) {
        TRY(mul_relin_chunk(c, a + b0 * ab_ct, b + b0 * ab_ct, ab_ct, rlk, out + b0 * out_ct,
                            out_ct, level, nb, rescale != 0, (uint64_t *)ws, S(stream)));
    }
    return SRK_OK;
}

// pairs a[i] x b[i] (host table of device pointers), chunked like the batch form
extern "C" int srk_mul_relin_ptrs(srk_ctx *c, const uint64_t *const *a, const uint64_t *const *b, int batch,
                                  const uint64_t *rlk, uint64_t *out, long long out_ct, int level, int rescale,
                                  void *ws, void *stream) {
    TRY(check_level(c, level));
    if (!a || !b || batch < 1) return fail(SRK_EINVAL, "need a non-empty pair table");
    if (rescale && level < 1) return fail(SRK_EINVAL, "depth exhausted");
    const long long n = c->n, nl = level + 1, ps = nl * n;
    const int ws_b = std::min(c->ws_batch, SRK_PAIRS_MAX);
    const int pieces = (batch + ws_b - 1) / ws_b;
    const int per = (batch + pieces - 1) / pieces;
    for (int b0 = 0; b0 < batch; b0 += per) {
        const int nb = std::min(per, batch - b0);
        uint64_t *d = (uint64_t *)ws;  // [nb][3][nl]
        uint64_t *rest = d + (long long)nb * 5 * ps;
        TensorPairs tp;
        memset(&tp, 0, sizeof tp);
        for (int i = 0; i < nb; i++) {
            if (!a[b0 + i] || !b[b0 + i]) return fail(SRK_EINVAL, "null operand in the pair table");
            tp.a[i] = a[b0 + i];
            tp.b[i] = b[b0 + i];
        }
        k_tensor_pairs<<<grid_for((long long)nb * ps), 256, 0, S(stream)>>>(tp, d, 3 * ps, c->d_pc, c->log_n,
                                                                          (int)nl, nb);
        LAUNCHED();
        uint64_t *o = out + (long long)b0 * out_ct;
        if (rescale) {
            KsOut ko = {o, out_ct, (long long)level * n, rlk, 1, d, d + ps, 3 * ps};
            TRY(keyswitch_impl(c, d + 2 * ps, 3 * ps, &ko, 1, level, nb, rest, S(stream), true));
        } else {
            KsOut ko = {o, out_ct, ps, rlk, 1, d, d + ps, 3 * ps};
            TRY(keyswitch_impl(c, d + 2 * ps, 3 * ps, &ko, 1, level, nb, rest, S(stream)));
        }
    }
    return SRK_OK;
}

extern "C" int srk_automorph(srk_ctx *c, const uint64_t *a, uint64_t *out,
                             long long n_limbs_total, uint64_t galois, void *stream) {
    if (!(galois & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
    const long long total = n_limbs_total * c->n;
    k_automorph<<<grid_for(total), 256, 0, S(stream)>>>(a, out, n_limbs_total, galois, c->log_n);
    LAUNCHED();
    return SRK_OK;
}

// rotation = key switch of c1 composed with X -> X^g, + sigma_g(c0)
extern "C" int srk_rotate_batch(srk_ctx *c, const uint64_t *a, long long a_ct, const uint64_t *gkey,
                                uint64_t *out, long long out_ct, int batch, int level,
                                uint64_t galois, void *ws, void *stream) {
    TRY(check_level(c, level));
    if (!(galois & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
    const long long ps = (long long)(level + 1) * c->n;
    FOR_CHUNKS(batch, b0, nb) {
        const uint64_t *ab = a + b0 * a_ct;
        KsOut o = {out + b0 * out_ct, out_ct, ps, gkey, galois, ab, nullptr, a_ct};
        TRY(keyswitch_impl(c, ab + ps, a_ct, &o, 1, level, nb, (uint64_t *)ws, S(stream)));
    }
    return SRK_OK;
}

extern "C" int srk_rotate(srk_ctx *c, const uint64_t *a, const uint64_t *gkey, uint64_t *out,
                          int level, uint64_t galois, void *ws, void *stream) {
    const long long ct = 2ll * (level + 1) * c->n;
    return srk_rotate_batch(c, a, ct, gkey, out, ct, 1, level, galois, ws, stream);
}

// several rotations of each ciphertext sharing one ModUp (hoisting)
extern "C" int srk_rotate_hoisted(srk_ctx *c, const uint64_t *a, long long a_ct, int batch,
                                  int n_rot, const uint64_t *const *gkeys, const uint64_t *galois,
                                  uint64_t *const *outs, long long out_ct, int level, void *ws,
                                  void *stream) {
    TRY(check_level(c, level));
    if (n_rot < 1 || n_rot > 64) return fail(SRK_EINVAL, "n_rot must lie in [1, 64]");
    const long long ps = (long long)(level + 1) * c->n;
    std::vector<KsOut> o(n_rot);
    FOR_CHUNKS(batch, b0, nb) {
        const uint64_t *ab = a + b0 * a_ct;
        for (int r = 0; r < n_rot; r++) {
            if (!(galois[r] & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
            o[r] = {outs[r] + b0 * out_ct, out_ct, ps, gkeys[r], galois[r], ab, nullptr, a_ct};
        }
        TRY(keyswitch_impl(c, ab + ps, a_ct, o.data(), n_rot, level, nb, (uint64_t *)ws, S(stream)));
    }
    return SRK_OK;
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


// key (dnum x 2 x n_primes limbs) <- sigma_g^-1(key), limb by limb, via tmp (2 x n_primes limbs)
extern "C" int srk_permute_key(srk_ctx *c, uint64_t *key, uint64_t galois, void *tmp_ws,
                               void *stream) {
    if (!(galois & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
    const long long np = c->n_primes, n = c->n;
    const uint64_t two_n = 2ull * c->n;
    // inverse of g in (Z/2N)^*: g^(N/2 - 1) has order dividing N/2 ... use g^(phi-1), phi = N
    uint64_t ginv = 1, b = galois % two_n, e = (uint64_t)c->n - 1;
    while (e) {
        if (e & 1) ginv = ginv * b % two_n;
        b = b * b % two_n;
        e >>= 1;
    }
    uint64_t *tmp = (uint64_t *)tmp_ws;
    for (int j = 0; j < c->dnum; j++) {
        uint64_t *kj = key + (long long)j * 2 * np * n;
        k_automorph<<<grid_for(2 * np * n), 256, 0, S(stream)>>>(kj, tmp, 2 * np, ginv, c->log_n);
        LAUNCHED();
        CU(cudaMemcpyAsync(kj, tmp, sizeof(uint64_t) * 2 * np * n, cudaMemcpyDeviceToDevice, S(stream)));
    }
    return SRK_OK;
}

// Galois key for X -> X^g in the rotation layout: every limb of the
// switching key sigma_g(s) -> s permuted by sigma_g^-1 (see k_ks_inner)
extern "C" int srk_keygen_galois(srk_ctx *c, const uint64_t *s_ntt, const int64_t *e, uint64_t seed,
                                 uint64_t key_id, uint64_t galois, uint64_t *key, void *ws,
                                 void *stream) {
    if (!(galois & 1)) return fail(SRK_EINVAL, "Galois element must be odd");
    const long long np = c->n_primes, n = c->n;
    uint64_t *sg = (uint64_t *)ws;           // sigma_g(s)
    uint64_t *tmp = sg + np * n;             // one key digit
    k_automorph<<<grid_for(np * n), 256, 0, S(stream)>>>(s_ntt, sg, np, galois, c->log_n);
    LAUNCHED();
    // ws after sg: keygen needs np limbs of scratch -> place it after tmp region
    TRY(srk_keygen(c, s_ntt, sg, e, seed, key_id, key, tmp + 2 * np * n, stream));
    return srk_permute_key(c, key, galois, tmp, stream);
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

// out = sum_i k[i] * terms[i] over the first level+1 limbs (no rescale);
// terms: host array of device pointers, term_limbs: limbs per poly of each
// term (>= level+1), k: DEVICE [n_terms][level+1] residues, batch packed
// ciphertexts per term (ct stride 2 * term_limbs * N), out [batch][2][level+1][N]
extern "C" int srk_lincomb(srk_ctx *c, const uint64_t *const *terms, const int *term_limbs,
                           int n_terms, const uint64_t *k, uint64_t *out, int batch, int level,
                           void *stream) {
    TRY(check_level(c, level));
    if (n_terms < 1 || n_terms > SRK_LC_MAX) return fail(SRK_EINVAL, "1..64 terms");
    LinCombArgs la;
    memset(&la, 0, sizeof la);
    for (int i = 0; i < n_terms; i++) {
        if (term_limbs[i] < level + 1) return fail(SRK_EINVAL, "term below the output level");
        la.term[i] = terms[i];
        la.term_ps[i] = (long long)term_limbs[i] * c->n;
        la.term_ct[i] = 2ll * term_limbs[i] * c->n;
    }
    la.n_terms = n_terms;
    la.nl = level + 1;
    la.batch = batch;
    la.k = k;
    la.out = out;
    const long long total = 2ll * batch * (level + 1) * c->n;
    k_lincomb<<<grid_for(total), 256, 0, S(stream)>>>(la, c->d_pc, c->log_n);
    LAUNCHED();
    return SRK_OK;
}

// n_out linear combinations of the same terms: outs[l] = sum_i k[l][i] * terms[i]
// (k: DEVICE residues [n_out][n_terms][level+1]; kf: k / q as doubles in the same layout,
// or null); eight outputs per pass over the terms
extern "C" int srk_lincomb_multi(srk_ctx *c, const uint64_t *const *terms, const int *term_limbs,
                                 int n_terms, const uint64_t *k, const double *kf,
                                 uint64_t *const *outs, int n_out, int batch, int level, void *stream) {
    TRY(check_level(c, level));
    if (n_terms < 1 || n_terms > SRK_LC_MAX) return fail(SRK_EINVAL, "1..64 terms");
    if (n_out < 1) return fail(SRK_EINVAL, "no outputs");
    if (c->n % 256) return fail(SRK_EINVAL, "srk_lincomb_multi needs a ring degree divisible by 256");
    LinCombArgs la;
    memset(&la, 0, sizeof la);
    for (int i = 0; i < n_terms; i++) {
        if (term_limbs[i] < level + 1) return fail(SRK_EINVAL, "term below the output level");
        la.term[i] = terms[i];
        la.term_ps[i] = (long long)term_limbs[i] * c->n;
        la.term_ct[i] = 2ll * term_limbs[i] * c->n;
    }
    la.n_terms = n_terms;
    la.nl = level + 1;
    la.batch = batch;
    const long long total = 2ll * batch * (level + 1) * c->n;
    const int stride = n_terms * (level + 1);
    for (int l0 = 0; l0 < n_out; l0 += SRK_LC_OUTS) {
        LinCombOuts lo;
        memset(&lo, 0, sizeof lo);
        lo.n_out = std::min(SRK_LC_OUTS, n_out - l0);
        lo.k_out_stride = stride;
        for (int l = 0; l < SRK_LC_OUTS; l++) lo.out[l] = outs[l0 + std::min(l, lo.n_out - 1)];
        la.k = k + (long long)l0 * stride;
        lo.kf = kf ? kf + (long long)l0 * stride : nullptr;
        if (lo.n_out <= 1)
            k_lincomb_multi<1><<<grid_for(total), 256, 0, S(stream)>>>(la, lo, c->d_pc, c->log_n);
        else if (lo.n_out <= 2)
            k_lincomb_multi<2><<<grid_for(total), 256, 0, S(stream)>>>(la, lo, c->d_pc, c->log_n);
        else if (lo.n_out <= 4)
            k_lincomb_multi<4><<<grid_for(total), 256, 0, S(stream)>>>(la, lo, c->d_pc, c->log_n);
        else
            k_lincomb_multi<8><<<grid_for(total), 256, 0, S(stream)>>>(la, lo, c->d_pc, c->log_n);
        LAUNCHED();
    }
    return SRK_OK;
}

extern "C" int srk_reduce_mod(srk_ctx *c, uint64_t *data, int n_polys, int level, void *stream) {
    TRY(check_level(c, level));
    const long long total = (long long)n_polys * (level + 1) * c->n;
    k_reduce_mod<<<grid_for(total), 256, 0, S(stream)>>>(data, c->d_pc, c->log_n, level + 1, total);
    LAUNCHED();
    return SRK_OK;
}

extern "C" int srk_encode_plain(srk_ctx *c, const int64_t *coeffs, uint64_t *pt_out, int level,
                                void *stream) {
    TRY(check_level(c, level));
    return srk_small_to_ntt(c, coeffs, pt_out, level + 1, 0, stream);
}
