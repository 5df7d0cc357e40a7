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

// A batch of limbs: poly p (0..n_polys-1), limb i (0..n_limbs-1) lives at
// ptr + p * poly_stride + i * N and is reduced modulo prime
//   pid(i) = i + (i < split ? off_a : off_b).
struct LimbBatch {
    uint64_t *ptr;
    long long poly_stride;
    int n_polys;
    int n_limbs;
    int split;
    int off_a;
    int off_b;
};

__device__ __forceinline__ int batch_pid(const LimbBatch &b, int i) {
    return i + (i < b.split ? b.off_a : b.off_b);
}

struct NttTables {
    const PrimeConst *pc;
    const uint64_t *tw;    // [n_primes][N] psi^brv(k)
    const uint64_t *tws;   // Shoup constants of tw
    const uint64_t *itw;   // psi^-brv(k)
    const uint64_t *itws;
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

// One pass of the NTT.  COL = column pass (sub-transforms strided by C),
// else row pass (contiguous chunks).  Grid: x = sub-transform groups of
// one limb, y = limb of the batch (poly fastest, so one prime's twiddles
// are reused across consecutive CTAs).
template <int LOG_T, bool INV, bool COL>
__global__ void __launch_bounds__(256) ntt_pass_kernel(LimbBatch b, NttTables tb, int log_n) {
    using S = NttShape<LOG_T>;
    constexpr int T = S::T, E = S::E, TPS = S::TPS, LE1 = S::LE1, LE2 = S::LE2;
    extern __shared__ uint64_t smem[];

    const int n = 1 << log_n;
    const int CB = blockDim.x / TPS;  // sub-transforms per CTA
    const int y = blockIdx.y;
    const int limb = y / b.n_polys, poly = y - limb * b.n_polys;
    const int pid = batch_pid(b, limb);
    uint64_t *data = b.ptr + (long long)poly * b.poly_stride + (long long)limb * n;
    const PrimeConst pc = tb.pc[pid];
    const uint64_t q = pc.q, two_q = pc.two_q;
    const uint64_t *tw = (INV ? tb.itw : tb.tw) + (long long)pid * n;
    const uint64_t *tws = (INV ? tb.itws : tb.tws) + (long long)pid * n;

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
    const int C = n >> LOG_T;               // COL: #columns ; ROW: T == C
    // element c of this sub-transform lives at data[addr(c)]
    auto gaddr = [&](int c) -> long long {
        return COL ? (long long)c * C + sub : (long long)sub * T + c;
    };
    const int R = n >> LOG_T;  // ROW pass: number of rows (chunks)
    const int base = COL ? 1 : (R + sub);
    auto tw_at = [&](int stage, int c, uint64_t &w, uint64_t &ws) {
        int idx = (base << stage) + (c >> (LOG_T - stage));
        w = __ldg(tw + idx);
        ws = __ldg(tws + idx);
    };
    auto sidx = [&](int c) -> int {
        return COL ? c * CB + sb : row_sidx<LOG_T>(sb, c);
    };

    uint64_t x[E];
    if (!INV) {
        // ---- round 1: strided ownership c = u + TPS e, strides T/2 .. TPS
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = data[gaddr(u + TPS * e)];
#pragma unroll
        for (int s = 0; s < LE1; s++) {
            const int half = E >> (s + 1);
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & half) continue;
                uint64_t w, ws;
                tw_at(s, u + TPS * e, w, ws);
                ct_bfly(x[e], x[e + half], w, ws, q, two_q);
            }
        }
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = x[e];
        __syncthreads();
        // ---- round 2: contiguous ownership c = u E + e, strides TPS/2 .. 1
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
#pragma unroll
        for (int s = 0; s < LE2; s++) {
            const int half = TPS >> (s + 1);
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & half) continue;
                uint64_t w, ws;
                tw_at(LE1 + s, u * E + e, w, ws);
                ct_bfly(x[e], x[e + half], w, ws, q, two_q);
            }
        }
        if (COL) {
#pragma unroll
            for (int e = 0; e < E; e++) data[gaddr(u * E + e)] = x[e];  // [0,4q)
        } else {
            // final pass: canonical values, staged through smem for coalescing
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) {
                uint64_t v = x[e];
                v = v >= two_q ? v - two_q : v;
                v = v >= q ? v - q : v;
                smem[sidx(u * E + e)] = v;
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) data[gaddr(u + TPS * e)] = smem[sidx(u + TPS * e)];
        }
    } else {
        // ---- round 1: contiguous ownership, strides 1 .. E/2
        if (COL) {
#pragma unroll
            for (int e = 0; e < E; e++) x[e] = data[gaddr(u * E + e)];
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = data[gaddr(u + TPS * e)];
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
        }
#pragma unroll
        for (int s = 0; s < LE1; s++) {
            const int half = 1 << s;  // stride in elements == in registers
            const int stage = LOG_T - 1 - s;
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & half) continue;
                uint64_t w, ws;
                tw_at(stage, u * E + e, w, ws);
                gs_bfly(x[e], x[e + half], w, ws, q, two_q);
            }
        }
        if (!COL) __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u * E + e)] = x[e];
        __syncthreads();
        // ---- round 2: strided ownership c = u + TPS e, strides E .. T/2
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u + TPS * e)];
#pragma unroll
        for (int s = 0; s < LE2; s++) {
            const int half = (E / TPS) << s;  // register stride
            const int stage = LE2 - 1 - s;
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & half) continue;
                uint64_t w, ws;
                tw_at(stage, u + TPS * e, w, ws);
                gs_bfly(x[e], x[e + half], w, ws, q, two_q);
            }
        }
        if (COL) {
            // last pass of the inverse: * N^-1, canonical
#pragma unroll
            for (int e = 0; e < E; e++)
                data[gaddr(u + TPS * e)] = mul_shoup(x[e], pc.ninv, pc.ninv_shoup, q);
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) data[gaddr(u + TPS * e)] = x[e];  // [0,2q)
        }
    }
}
