// Do DFMA and IMAD pipes overlap? Is rint (FRND.F64) full rate? (B200)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/pipes2 tools/micro/pipes2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_mix(double *out, uint32_t *o2, double a, double b, uint32_t ia, int mode) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    uint32_t y0 = threadIdx.x, y1 = y0 + 1, y2 = y0 + 2, y3 = y0 + 3;
    for (int i = 0; i < ITERS; i++) {
        if (mode & 1) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); }
        if (mode & 2) { y0 = y0 * ia + 7; y1 = y1 * ia + 7; y2 = y2 * ia + 7; y3 = y3 * ia + 7; }
        if (mode & 4) { x0 = rint(x0 * a); x1 = rint(x1 * a); x2 = rint(x2 * a); x3 = rint(x3 * a); }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
    o2[blockIdx.x * blockDim.x + threadIdx.x] = y0 ^ y1 ^ y2 ^ y3;
}
int main() {
    const int blocks = 148 * 8, threads = 256;
    double *dd; uint32_t *d32;
    cudaMalloc(&dd, blocks * threads * 8); cudaMalloc(&d32, blocks * threads * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char *names[] = {"", "DFMA only", "IMAD only", "DFMA+IMAD", "rint(DMUL)", "", "", ""};
    for (int mode : {1, 2, 3, 4}) {
        k_mix<<<blocks, threads>>>(dd, d32, 1.0000001, 0.5, 2654435761u, mode);
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) k_mix<<<blocks, threads>>>(dd, d32, 1.0000001, 0.5, 2654435761u, mode);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-12s %.3f ms  (%.2f G iterations x4 per s)\n", names[mode], ms / 5,
               (double)blocks * threads * ITERS / (ms / 5) / 1e6);
    }
    return 0;
}
