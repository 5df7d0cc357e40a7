// bconv.cuh -- RNS base conversions (ModUp digit extension, ModDown P -> Q) with
// the quotient on the FP64 pipe and the remainder in wrapping 64-bit integers.
//
//   out_t = sum_i y_i m_it  (mod q_t),   m_it the CRT constant of source i under q_t
//
// is computed as  S = sum_i y_i m_it (mod 2^64),  T = sum_i y_i (m_it / q_t) in
// FP64,  r = S - round(T) q_t:  |r| < q_t < 2^63 whenever T is within 1/2 of the
// true quotient, so the wrapped 64-bit difference is the exact signed remainder
// and one conditional +q_t makes it canonical.  The result is S mod q_t whatever
// the summation order and whichever neighbouring integer round(T) lands on.
//
// Loop order: sources outer, the CTA's 8 targets inner.  Per (source, target)
// the work is one or two 16-byte broadcast loads of the constants from shared
// memory, the FMAs of the quotient, and 32-bit multiply-adds written so that every
// one of them accumulates in place:
//     (SH:SL) += lo32(y) * lo32(m)     one IMAD.WIDE.U32 (64-bit accumulate)
//     SH      += lo32(y) * hi32(m)     one IMAD        (the 2^32 column, wrapping)
// A thread owns two adjacent coefficients (one constant load serves both, 16-byte
// loads and stores).  The source limbs of a 512-coefficient tile are staged in
// shared memory with cp.async -- every source's load is in flight at once and none
// of them occupies a register; each thread reads back only what it copied itself,
// so a cp.async.wait_group is the only synchronisation.  With NBUF = 2 the next
// tile's sources stream in while the current tile is converted.
#pragma once
#include <cstdint>

#include "modarith.cuh"
#include "ntt.cuh"

#define SRK_BCONV_TG 8      // targets per CTA (blockIdx.x groups)
#define SRK_BCONV_MAXSRC 17  // ModDown sources: K special primes (+ q_l for the fused rescale)
#define SRK_BCONV_TILE 512   // coefficients per CTA tile (256 threads x 2)

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// bytes of dynamic shared memory a conversion launch needs
static inline size_t bconv_smem_bytes(int n_src, int nbuf) { return (size_t)nbuf * n_src * 256 * 16; }

// (hi:lo) += a * b, wrapping mod 2^64: the carry-chain pair below is what ptxas
// fuses into ONE IMAD.WIDE.U32 with a 64-bit addend (a mad.wide.u32 on a u64
// variable is split into a multiply and a separate IADD3 pair)
__device__ __forceinline__ void mac_wide(uint32_t &lo, uint32_t &hi, uint32_t a, uint32_t b) {
    asm("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// the 2^32 column: hi += lo32(a * b), one IMAD
__device__ __forceinline__ void mac_hi(uint32_t &hi, uint32_t a, uint32_t b) {
    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(hi) : "r"(a), "r"(b));
}
// value < 2^32 as a double (one LOP-free register pair + one DADD)
__device__ __forceinline__ double f64_of_u32(uint32_t v) {
    return __hiloint2double(0x43300000, (int)v) - SRK_F64_TWO52;
}
// canonical remainder from the wrapped sum and the FP64 quotient
__device__ __forceinline__ uint64_t bconv_finish(uint32_t sl, uint32_t sh, double T, uint64_t q) {
    const uint64_t S = ((uint64_t)sh << 32) | sl;
    const long long tq = __double_as_longlong(T + SRK_F64_MAGIC) - 0x4338000000000000ll;
    const long long rr = (long long)(S - (uint64_t)tq * q);
    return (uint64_t)(rr < 0 ? rr + (long long)q : rr);
}

// ---------------------------------------------------------------------
// ModDown conversion P (or P u {q_l}) -> q_0..q_{n_dst-1}, coefficient domain:
//   conv[t] = sum_k z_k m_kt - v [prod src]_{q_t},  v = round(sum_k z_k / p_k)
// z_k < 2^62 enters as halves z = zh 2^32 + zl with m' = m 2^32 mod q_t:
//   S = sum zl m + zh m',  T = sum zl (m/q) + zh (m'/q)   (terms < 2^32, error < 2^-16).
// The rounding correction is folded into the start values: S0 = (q - v P) mod q,
// T0 = S0 / q, so the finished remainder is already conv[t].
// z: B*2 polys (ct stride z_ct, poly stride z_ps) of n_src limbs; mhl / fhl:
// [n_src][n_dst] {m, m'} / {m/q, m'/q}; corr: [n_src+1][n_dst] = v P mod q_t.
// Grid: x = target groups, y = (b, r), z = tiles of 512 coefficients (grid-stride):
// the CTAs that share a tile's source words are dispatched together, so the words
// come from HBM once and from L2 for the other groups.
// ---------------------------------------------------------------------
template <int NBUF, int TG>
__global__ void __launch_bounds__(256, 2) k_moddown_conv(
    const uint64_t *__restrict__ z, long long z_ct, long long z_ps, int n_src,
    const uint8_t *__restrict__ vround, const ulonglong2 *__restrict__ mhl,
    const double2 *__restrict__ fhl, int n_dst, const uint64_t *__restrict__ corr,
    uint64_t *__restrict__ conv, long long c_ct, long long c_ps, const PrimeConst *__restrict__ pc,
    int log_n) {
    extern __shared__ __align__(16) unsigned char bconv_dyn[];
    ulonglong2 *sy = reinterpret_cast<ulonglong2 *>(bconv_dyn);  // [NBUF][n_src][256]
    __shared__ double2 s_f[SRK_BCONV_MAXSRC][TG];
    __shared__ uint4 s_m[SRK_BCONV_MAXSRC][TG];           // {lo(m), hi(m), lo(m'), hi(m')}
    __shared__ ulonglong2 s_c[SRK_BCONV_MAXSRC + 1][TG];  // per v: {(q - v P) mod q, bits of it / q}
    __shared__ uint64_t s_q[TG];
    const long long n = 1ll << log_n;
    const int p = blockIdx.y;  // (b, r)
    const int b = p >> 1, r = p & 1;
    const int t0 = blockIdx.x * TG, nt = min(n_dst - t0, TG);
    const int tid = threadIdx.x;
    for (int i = tid; i < n_src * TG; i += blockDim.x) {
        const int k = i / TG, tt = i - k * TG;
        const ulonglong2 m = tt < nt ? __ldg(mhl + k * n_dst + t0 + tt) : make_ulonglong2(0, 0);
        s_f[k][tt] = tt < nt ? __ldg(fhl + k * n_dst + t0 + tt) : make_double2(0.0, 0.0);
        s_m[k][tt] = make_uint4((uint32_t)m.x, (uint32_t)(m.x >> 32), (uint32_t)m.y, (uint32_t)(m.y >> 32));
    }
    for (int i = tid; i < (n_src + 1) * TG; i += blockDim.x) {
        const int v = i / TG, tt = i - v * TG;
        uint64_t nc = 0;
        double fc = 0.0;
        if (tt < nt) {
            const uint64_t q = pc[t0 + tt].q, cv = __ldg(corr + v * n_dst + t0 + tt);
            nc = cv ? q - cv : 0;
            fc = (double)nc / (double)q;
        }
        s_c[v][tt] = make_ulonglong2(nc, (uint64_t)__double_as_longlong(fc));
    }
    if (tid < TG) s_q[tid] = tid < nt ? pc[t0 + tid].q : 1;
    __syncthreads();
    const uint64_t *zp = z + b * z_ct + r * z_ps;
    const long long tiles = (n + SRK_BCONV_TILE - 1) / SRK_BCONV_TILE;
    // stage tile `tile`'s sources (this thread's two coefficients of every limb)
    auto stage = [&](long long tile, int buf) {
        const long long x = min(tile * SRK_BCONV_TILE + 2 * tid, n - 2);
        for (int k = 0; k < n_src; k++) cp_async16(sy + ((long long)buf * n_src + k) * 256 + tid, zp + k * n + x);
        cp_async_commit();
    };
    long long tile = blockIdx.z;
    if (tile < tiles) stage(tile, 0);
    for (int it = 0; tile < tiles; tile += gridDim.z, it++) {
        const int buf = NBUF == 2 ? (it & 1) : 0;
        const long long x = tile * SRK_BCONV_TILE + 2 * tid;
        const long long xl = min(x, n - 2);
        const uint32_t v2 = *reinterpret_cast<const uint16_t *>(vround + (long long)p * n + xl);
        if (NBUF == 2) {
            if (tile + gridDim.z < tiles) {
                stage(tile + gridDim.z, buf ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
        } else {
            cp_async_wait<0>();
        }
        double T[2][TG];
        uint32_t SL[2][TG], SH[2][TG];
#pragma unroll
        for (int c = 0; c < 2; c++) {
            const int v = (v2 >> (8 * c)) & 0xff;
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                const ulonglong2 cv = s_c[v][tt];
                SL[c][tt] = (uint32_t)cv.x;
                SH[c][tt] = (uint32_t)(cv.x >> 32);
                T[c][tt] = __longlong_as_double((long long)cv.y);
            }
        }
        const ulonglong2 *yb = sy + (long long)buf * n_src * 256 + tid;
        for (int k = 0; k < n_src; k++) {
            const ulonglong2 zz = yb[k * 256];
            const uint32_t zl[2] = {(uint32_t)zz.x, (uint32_t)zz.y};
            const uint32_t zh[2] = {(uint32_t)(zz.x >> 32), (uint32_t)(zz.y >> 32)};
            const double dl[2] = {f64_of_u32(zl[0]), f64_of_u32(zl[1])};
            const double dh[2] = {f64_of_u32(zh[0]), f64_of_u32(zh[1])};
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                const double2 f = s_f[k][tt];
                const uint4 m = s_m[k][tt];
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    T[c][tt] = fma(dh[c], f.y, fma(dl[c], f.x, T[c][tt]));
                    mac_wide(SL[c][tt], SH[c][tt], zl[c], m.x);
                    mac_hi(SH[c][tt], zl[c], m.y);
                    mac_wide(SL[c][tt], SH[c][tt], zh[c], m.z);
                    mac_hi(SH[c][tt], zh[c], m.w);
                }
            }
        }
        if (NBUF == 1 && tile + gridDim.z < tiles) stage(tile + gridDim.z, 0);  // own slots: already consumed
        if (x < n) {
            uint64_t *out = conv + b * c_ct + r * c_ps + (long long)t0 * n + x;
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                if (tt >= nt) break;
                const uint64_t q = s_q[tt];
                *reinterpret_cast<ulonglong2 *>(out + (long long)tt * n) = make_ulonglong2(
                    bconv_finish(SL[0][tt], SH[0][tt], T[0][tt], q), bconv_finish(SL[1][tt], SH[1][tt], T[1][tt], q));
            }
        }
    }
}

// ---------------------------------------------------------------------
// The same conversion for K <= 4 sources (config 2's three special primes): the few
// source words of a coefficient stay in registers, targets are the outer loop, and
// the light per-thread state (one coefficient, 64 registers) lets four CTAs per SM
// keep enough stores in flight -- the tile-staged kernel above is built for many
// sources and runs this shape ~12% slower (473 vs 422 us per 32-ciphertext launch;
// a variant with the constants in registers and the coefficients streaming: 720 us).
// The next coefficient's sources are loaded before this one's stores (which loads
// cannot pass).
// ---------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(256, 4) k_moddown_conv_small(
    const uint64_t *__restrict__ z, long long z_ct, long long z_ps, const uint8_t *__restrict__ vround,
    const ulonglong2 *__restrict__ mhl, const double2 *__restrict__ fhl, int n_dst,
    const uint64_t *__restrict__ corr, uint64_t *__restrict__ conv, long long c_ct, long long c_ps,
    const PrimeConst *__restrict__ pc, int log_n) {
    constexpr int TG = SRK_BCONV_TG;
    __shared__ double2 s_f[TG][K];
    __shared__ uint4 s_m[TG][K];           // {lo(m), hi(m), lo(m'), hi(m')}
    __shared__ ulonglong2 s_c[K + 1][TG];  // per v: {(q - v P) mod q, bits of it / q}
    __shared__ uint64_t s_q[TG];
    const long long n = 1ll << log_n;
    const int p = blockIdx.y;  // (b, r)
    const int b = p >> 1, r = p & 1;
    const int t0 = blockIdx.x * TG, nt = min(n_dst - t0, TG);
    for (int i = threadIdx.x; i < nt * K; i += blockDim.x) {
        const int tt = i / K, k = i - tt * K;
        const ulonglong2 m = __ldg(mhl + k * n_dst + t0 + tt);
        s_f[tt][k] = __ldg(fhl + k * n_dst + t0 + tt);
        s_m[tt][k] = make_uint4((uint32_t)m.x, (uint32_t)(m.x >> 32), (uint32_t)m.y, (uint32_t)(m.y >> 32));
    }
    for (int i = threadIdx.x; i < (K + 1) * nt; i += blockDim.x) {
        const int v = i / nt, tt = i - v * nt;
        const uint64_t q = pc[t0 + tt].q, cv = __ldg(corr + v * n_dst + t0 + tt);
        const uint64_t nc = cv ? q - cv : 0;
        s_c[v][tt] = make_ulonglong2(nc, (uint64_t)__double_as_longlong((double)nc / (double)q));
    }
    if (threadIdx.x < nt) s_q[threadIdx.x] = pc[t0 + threadIdx.x].q;
    __syncthreads();
    const uint64_t *zp = z + b * z_ct + r * z_ps;
    const long long stride = (long long)gridDim.z * blockDim.x;
    long long x = blockIdx.z * (long long)blockDim.x + threadIdx.x;
    uint64_t zn[K];
    int vn = 0;
    if (x < n) {
#pragma unroll
        for (int k = 0; k < K; k++) zn[k] = __ldg(zp + k * n + x);
        vn = __ldg(vround + (long long)p * n + x);
    }
    for (; x < n; x += stride) {
        uint32_t zl[K], zh[K];
        double dl[K], dh[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            zl[k] = (uint32_t)zn[k];
            zh[k] = (uint32_t)(zn[k] >> 32);
            dl[k] = f64_of_u32(zl[k]);
            dh[k] = f64_of_u32(zh[k]);
        }
        const int v = vn;
        if (x + stride < n) {
#pragma unroll
            for (int k = 0; k < K; k++) zn[k] = __ldg(zp + k * n + x + stride);
            vn = __ldg(vround + (long long)p * n + x + stride);
        }
        uint64_t *out = conv + b * c_ct + r * c_ps + (long long)t0 * n + x;
#pragma unroll 4
        for (int tt = 0; tt < TG; tt++) {
            if (tt >= nt) break;
            const ulonglong2 cv = s_c[v][tt];
            uint32_t sl = (uint32_t)cv.x, sh = (uint32_t)(cv.x >> 32);
            double T0 = __longlong_as_double((long long)cv.y), T1 = 0.0;
#pragma unroll
            for (int k = 0; k < K; k++) {
                const double2 f = s_f[tt][k];
                const uint4 m = s_m[tt][k];
                T0 = fma(dl[k], f.x, T0);
                T1 = fma(dh[k], f.y, T1);
                mac_wide(sl, sh, zl[k], m.x);
                mac_hi(sh, zl[k], m.y);
                mac_wide(sl, sh, zh[k], m.z);
                mac_hi(sh, zh[k], m.w);
            }
            *out = bconv_finish(sl, sh, T0 + T1, s_q[tt]);
            out += n;
        }
    }
}

// ---------------------------------------------------------------------
// ModUp conversion of every digit (hybrid key switching): digit j's alpha source
// limbs y_i (already scaled by (Q_j/q_i)^-1 in the INTT) -> every extended-basis
// limb outside the digit, for targets q_t < 2^62.
// Sources under primes < 2^41 enter whole (|term| < 2^41, T error < 2^-4 over 16
// terms); a wider source (q_0 in digit 0: WIDE0) enters as halves with
// m' = m 2^32 mod q_t like the ModDown sources.
// Grid: x = target groups, y = b * beta + j, z = tiles of 512 coefficients (grid-stride).
// ---------------------------------------------------------------------
#ifndef SRK_MAX_DIGITS
#define SRK_MAX_DIGITS 64
#endif
struct ModUpArgs {
    const uint64_t *dc;   // [B][nl] coefficient-domain limbs (ct stride dc_ct)
    long long dc_ct;
    uint64_t *ext;        // [B][beta][ne]
    long long ext_ct, ext_dig;
    int nl, beta, alpha;
    const uint64_t *mat[SRK_MAX_DIGITS];
    const int *slot[SRK_MAX_DIGITS];
    const int *pid[SRK_MAX_DIGITS];
    int n_dst[SRK_MAX_DIGITS];
    // {m, m 2^32 mod q_t}, {m/q_t, (m 2^32 mod q_t)/q_t} per (source, target)
    const ulonglong2 *mhl[SRK_MAX_DIGITS];
    const double2 *fhl[SRK_MAX_DIGITS];
};

template <bool WIDE0, int NBUF>
__global__ void __launch_bounds__(256, 2) k_modup_conv(const __grid_constant__ ModUpArgs a,
                                                      const PrimeConst *__restrict__ pc, int log_n) {
    constexpr int TG = SRK_BCONV_TG;
    extern __shared__ __align__(16) unsigned char bconv_dyn[];
    ulonglong2 *sy = reinterpret_cast<ulonglong2 *>(bconv_dyn);  // [NBUF][alpha][256]
    __shared__ uint4 s_mf[16][TG];  // {lo(m), hi(m), bits(m / q)} per (source, target)
    __shared__ uint4 s_w0[TG];      // the wide source's {lo(m'), hi(m'), bits(m' / q)}
    __shared__ uint64_t s_q[TG];
    __shared__ int s_slot[TG];
    const long long n = 1ll << log_n;
    const int b = blockIdx.y / a.beta, j = blockIdx.y - b * a.beta;
    const int g0 = j * a.alpha, gs = min(a.alpha, a.nl - g0);
    const int t0 = blockIdx.x * TG;
    const int nd = a.n_dst[j];
    if (t0 >= nd) return;
    const int nt = min(nd - t0, TG);
    const int tid = threadIdx.x;
    for (int i = tid; i < gs * TG; i += blockDim.x) {
        const int k = i / TG, tt = i - k * TG;
        ulonglong2 m = make_ulonglong2(0, 0);
        double2 f = make_double2(0.0, 0.0);
        if (tt < nt) {
            m = __ldg(a.mhl[j] + k * nd + t0 + tt);
            f = __ldg(a.fhl[j] + k * nd + t0 + tt);
        }
        const uint64_t fb = (uint64_t)__double_as_longlong(f.x);
        s_mf[k][tt] = make_uint4((uint32_t)m.x, (uint32_t)(m.x >> 32), (uint32_t)fb, (uint32_t)(fb >> 32));
        if (k == 0) {
            const uint64_t gb = (uint64_t)__double_as_longlong(f.y);
            s_w0[tt] = make_uint4((uint32_t)m.y, (uint32_t)(m.y >> 32), (uint32_t)gb, (uint32_t)(gb >> 32));
        }
    }
    if (tid < TG) {
        const bool ok = tid < nt;
        s_q[tid] = ok ? pc[__ldg(a.pid[j] + t0 + tid)].q : 1;
        s_slot[tid] = ok ? __ldg(a.slot[j] + t0 + tid) : 0;
    }
    __syncthreads();
    const uint64_t *src = a.dc + b * a.dc_ct + (long long)g0 * n;
    uint64_t *dst = a.ext + b * a.ext_ct + j * a.ext_dig;
    const bool wide = WIDE0 && j == 0;
    const long long tiles = (n + SRK_BCONV_TILE - 1) / SRK_BCONV_TILE;
    auto stage = [&](long long tile, int buf) {
        const long long x = min(tile * SRK_BCONV_TILE + 2 * tid, n - 2);
        for (int k = 0; k < gs; k++) cp_async16(sy + ((long long)buf * a.alpha + k) * 256 + tid, src + k * n + x);
        cp_async_commit();
    };
    long long tile = blockIdx.z;
    if (tile < tiles) stage(tile, 0);
    for (int it = 0; tile < tiles; tile += gridDim.z, it++) {
        const int buf = NBUF == 2 ? (it & 1) : 0;
        const long long x = tile * SRK_BCONV_TILE + 2 * tid;
        if (NBUF == 2) {
            if (tile + gridDim.z < tiles) {
                stage(tile + gridDim.z, buf ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
        } else {
            cp_async_wait<0>();
        }
        double T[2][TG];
        uint32_t SL[2][TG], SH[2][TG];
#pragma unroll
        for (int c = 0; c < 2; c++) {
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                T[c][tt] = 0.0;
                SL[c][tt] = 0;
                SH[c][tt] = 0;
            }
        }
        const ulonglong2 *yb = sy + (long long)buf * a.alpha * 256 + tid;
        int i0 = 0;
        if (wide) {
            // source 0 under the wide prime: halves against {m, m'}
            const ulonglong2 yy = yb[0];
            const uint32_t yl[2] = {(uint32_t)yy.x, (uint32_t)yy.y};
            const uint32_t yh[2] = {(uint32_t)(yy.x >> 32), (uint32_t)(yy.y >> 32)};
            const double dl[2] = {f64_of_u32(yl[0]), f64_of_u32(yl[1])};
            const double dh[2] = {f64_of_u32(yh[0]), f64_of_u32(yh[1])};
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                const uint4 mf = s_mf[0][tt], w0 = s_w0[tt];
                const double f = __hiloint2double((int)mf.w, (int)mf.z);
                const double g = __hiloint2double((int)w0.w, (int)w0.z);
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    T[c][tt] = fma(dh[c], g, fma(dl[c], f, T[c][tt]));
                    mac_wide(SL[c][tt], SH[c][tt], yl[c], mf.x);
                    mac_hi(SH[c][tt], yl[c], mf.y);
                    mac_wide(SL[c][tt], SH[c][tt], yh[c], w0.x);
                    mac_hi(SH[c][tt], yh[c], w0.y);
                }
            }
            i0 = 1;
        }
        for (int i = i0; i < gs; i++) {
            const ulonglong2 yy = yb[i * 256];  // both < 2^41
            const uint32_t yl[2] = {(uint32_t)yy.x, (uint32_t)yy.y};
            const uint32_t yh[2] = {(uint32_t)(yy.x >> 32), (uint32_t)(yy.y >> 32)};
            const double dy[2] = {f64_of_u64(yy.x), f64_of_u64(yy.y)};
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                const uint4 mf = s_mf[i][tt];
                const double f = __hiloint2double((int)mf.w, (int)mf.z);
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    T[c][tt] = fma(dy[c], f, T[c][tt]);
                    mac_wide(SL[c][tt], SH[c][tt], yl[c], mf.x);
                    mac_hi(SH[c][tt], yl[c], mf.y);
                    mac_hi(SH[c][tt], yh[c], mf.x);
                }
            }
        }
        if (NBUF == 1 && tile + gridDim.z < tiles) stage(tile + gridDim.z, 0);  // own slots: already consumed
        if (x < n) {
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                if (tt >= nt) break;
                const uint64_t q = s_q[tt];
                *reinterpret_cast<ulonglong2 *>(dst + (long long)s_slot[tt] * n + x) = make_ulonglong2(
                    bconv_finish(SL[0][tt], SH[0][tt], T[0][tt], q), bconv_finish(SL[1][tt], SH[1][tt], T[1][tt], q));
            }
        }
    }
}
