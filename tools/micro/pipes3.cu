// Is FRND.F64 (rint) on its own pipe, i.e. does replacing the magic-constant rounding
// (DFMA + DADD) of the FP64 modular product by DMUL + FRND shorten the butterfly? (B200)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/pipes3 tools/micro/pipes3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2048
#define MAGIC 6755399441055744.0
template <int MODE>
__device__ __forceinline__ double modmul(double y, double w, double q, double qinv) {
    const double hi = y * w;
    const double lo = fma(y, w, -hi);
    double t;
    if (MODE == 0) t = fma(hi, qinv, MAGIC) - MAGIC;
    else t = rint(hi * qinv);
    return fma(-t, q, hi) + lo;
}
template <int MODE>
__global__ void k_bfly(double *out, double w, double q, double qinv) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; i++) {
        double t;
        t = modmul<MODE>(x1, w, q, qinv); x1 = x0 - t; x0 = x0 + t;
        t = modmul<MODE>(x3, w, q, qinv); x3 = x2 - t; x2 = x2 + t;
        t = modmul<MODE>(x5, w, q, qinv); x5 = x4 - t; x4 = x4 + t;
        t = modmul<MODE>(x7, w, q, qinv); x7 = x6 - t; x6 = x6 + t;
        t = modmul<MODE>(x2, w, q, qinv); x2 = x0 - t; x0 = x0 + t;
        t = modmul<MODE>(x3, w, q, qinv); x3 = x1 - t; x1 = x1 + t;
        t = modmul<MODE>(x6, w, q, qinv); x6 = x4 - t; x4 = x4 + t;
        t = modmul<MODE>(x7, w, q, qinv); x7 = x5 - t; x5 = x5 + t;
        // keep magnitudes bounded (one centred reduction per 2 stages; same in both modes)
        x0 = fma(-rint(x0 * qinv), q, x0); x4 = fma(-rint(x4 * qinv), q, x4);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    const int blocks = 148 * 6, threads = 128;
    double *dd; cudaMalloc(&dd, blocks * threads * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const double q = 1099511480321.0, qinv = 1.0 / q, w = 734298172113.0;
    for (int rep = 0; rep < 2; rep++)
    for (int mode = 0; mode < 2; mode++) {
        if (mode == 0) k_bfly<0><<<blocks, threads>>>(dd, w, q, qinv); else k_bfly<1><<<blocks, threads>>>(dd, w, q, qinv);
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) { if (mode == 0) k_bfly<0><<<blocks, threads>>>(dd, w, q, qinv); else k_bfly<1><<<blocks, threads>>>(dd, w, q, qinv); }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%s: %.3f ms  (%.2f G butterflies/s)\n", mode ? "DMUL+FRND " : "magic const", ms / 5,
               (double)blocks * threads * ITERS * 8 / (ms / 5) / 1e6);
    }
    return 0;
}
