// ntt_cluster.cuh -- forward 2^16-point NTT of one limb per 8-CTA thread-block
// cluster, FP64 arithmetic (limbs under primes < 2^41), column -> row exchange
// through distributed shared memory.
//
// The two-pass kernels in ntt.cuh write the 256 x 256 intermediate to global
// memory (L2) between the column and the row pass and pay a second launch.
// Here the limb is split over the cluster instead: CTA c owns columns
// [32c, 32c + 32) for the column pass and keeps its 256 x 32 result in its own
// shared memory (64 KiB); after a cluster barrier it owns rows [32c, 32c + 32)
// for the row pass and reads each row's 256 elements straight out of the eight
// CTAs' shared memory (32 contiguous words from each).  HBM sees exactly one
// read and one write of the limb; there is no intermediate in L2 and one
// launch per chunk.  Same arithmetic, twiddle indices and output order as
// ntt_pass_kernel<8, false, COL, LD_PLAIN/ST_PLAIN, KM=1, 16>, so results are
// bit-identical to the two-pass path.
#pragma once
#include <cooperative_groups.h>

#include "ntt.cuh"

#define SRK_CL_CTAS 8                       // CTAs per limb (cluster size)
#define SRK_CL_COLS (256 / SRK_CL_CTAS)     // columns (and rows) per CTA
#define SRK_CL_THREADS (SRK_CL_COLS * 16)   // 16 threads per 256-point sub-transform
// padded row-pass layout of ntt.cuh (row_sidx<8>): one pad word every 16
#define SRK_CL_SMEM_WORDS (SRK_CL_COLS * (256 + 16))

__global__ void __cluster_dims__(SRK_CL_CTAS, 1, 1) __launch_bounds__(SRK_CL_THREADS, 2)
    ntt_fwd_cluster_f64(LimbBatch b, NttTables tb, const __grid_constant__ FuseArgs f) {
    namespace cg = cooperative_groups;
    using S = NttShape<8>;
    constexpr int T = 256, E = S::E, TPS = S::TPS, LE1 = S::LE1, LE2 = S::LE2;
    constexpr int CB = SRK_CL_COLS;
    constexpr int log_n = 16;
    constexpr long long n = 1ll << log_n;
    extern __shared__ uint64_t smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank();  // == blockIdx.x

    const int limb = blockIdx.z, poly = blockIdx.y;
    const int bi = b.ppc == 2 ? poly >> 1 : (b.ppc == 1 ? poly : poly / b.ppc);
    const int r = poly - bi * b.ppc;
    int t, pid;
    // whole clusters exit together (the limb decides), so no barrier is orphaned
    if (!limb_map(b, r, limb, t, pid)) return;
    const PrimeConst pc = tb.pc[pid];
    if (pc.q >= SRK_F64_Q) return;
    uint64_t *data = b.ptr + (long long)bi * b.ct_stride + (long long)r * b.poly_stride + (long long)t * n;
    const uint64_t *src = f.src ? f.src + (long long)bi * f.src_ct + (long long)r * f.src_ps + (long long)t * n
                                : data;
    const TwPtr tw = {tb.tw + (long long)pid * n, tb.twd + (long long)pid * n};
    const F64Q fq = {__longlong_as_double((long long)pc.qd_bits), __longlong_as_double((long long)pc.qinv_bits)};
    const uint64_t q = pc.q, two_q = pc.two_q;
    const int tid = threadIdx.x;
    uint64_t x[E];

    // ---- column pass: CTA columns [crank*CB, +CB); thread (sb, u) = (tid % CB, tid / CB)
    {
        const int sb = tid % CB, u = tid / CB;
        const int col = crank * CB + sb;
        auto sidx = [&](int c) { return c * CB + sb; };
#pragma unroll
        for (int e = 0; e < E; e++)
            x[e] = (uint64_t)__double_as_longlong(f64_of_u64(src[(long long)(u + TPS * e) * 256 + col]));
        FwdR1<E, LE1, 2>::run(x, tw, 1, q, two_q, fq);
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u + TPS * e)] = x[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = smem[sidx(u * E + e)];
        FwdR2<E, TPS, LE1, LE2, 2>::run(x, tw, 1, u, q, two_q, fq);
        __syncthreads();
        // column pass result of row rho = u E + e, local column sb: A[rho][sb]
#pragma unroll
        for (int e = 0; e < E; e++) smem[sidx(u * E + e)] = x[e];
    }
    cluster.sync();
    // ---- row pass: CTA rows [crank*CB, +CB); thread (sb, u) = (tid / TPS, tid % TPS)
    const int sb = tid / TPS, u = tid % TPS;
    const int row = crank * CB + sb;
    // element c = u + TPS e of the row lives in CTA c / CB at A[row][c % CB]
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int c = u + TPS * e;
        const uint64_t *rs = cluster.map_shared_rank(smem, c / CB);
        x[e] = rs[row * CB + (c % CB)];
    }
    cluster.sync();  // every CTA's A has been read: reuse the buffer
    auto rsidx = [&](int c) { return row_sidx<8>(sb, c); };
    const int base = 256 + row;  // C + sub of the two-pass row kernel
    FwdR1<E, LE1, 2>::run(x, tw, base, q, two_q, fq);
#pragma unroll
    for (int e = 0; e < E; e++) smem[rsidx(u + TPS * e)] = x[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++) x[e] = smem[rsidx(u * E + e)];
    FwdR2<E, TPS, LE1, LE2, 2>::run(x, tw, base, u, q, two_q, fq);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++)
        smem[rsidx(u * E + e)] = canon_u64_of_f64(__longlong_as_double((long long)x[e]), fq.q, fq.qinv);
    __syncthreads();
    uint64_t *o = data + (long long)row * T;
#pragma unroll
    for (int e = 0; e < E; e++) o[u + TPS * e] = smem[rsidx(u + TPS * e)];
}
