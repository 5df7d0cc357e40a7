// Pipe-throughput microbenchmark (B200): DFMA, IMAD.WIDE (64x64 mulhi), I2F/F2I 64-bit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/pipes tools/micro/pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_dfma(double *out, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; i++) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_mulhi(uint64_t *out, uint64_t a) {
    uint64_t x0 = threadIdx.x, x1 = x0 + 11, x2 = x0 + 22, x3 = x0 + 33, x4 = x0 + 44, x5 = x0 + 55, x6 = x0 + 66, x7 = x0 + 77;
    for (int i = 0; i < ITERS; i++) {
        x0 = __umul64hi(x0, a) + a; x1 = __umul64hi(x1, a) + a; x2 = __umul64hi(x2, a) + a; x3 = __umul64hi(x3, a) + a;
        x4 = __umul64hi(x4, a) + a; x5 = __umul64hi(x5, a) + a; x6 = __umul64hi(x6, a) + a; x7 = __umul64hi(x7, a) + a;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
}
__global__ void k_imad(uint32_t *out, uint32_t a) {
    uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; i++) {
        x0 = x0 * a + 7; x1 = x1 * a + 7; x2 = x2 * a + 7; x3 = x3 * a + 7;
        x4 = x4 * a + 7; x5 = x5 * a + 7; x6 = x6 * a + 7; x7 = x7 * a + 7;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
}
__global__ void k_cvt(double *out, uint64_t a) {
    uint64_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double acc = 0;
    for (int i = 0; i < ITERS; i++) {
        double d0 = (double)x0, d1 = (double)x1, d2 = (double)x2, d3 = (double)x3;
        x0 = (uint64_t)(d0 * 0.5) + a; x1 = (uint64_t)(d1 * 0.5) + a; x2 = (uint64_t)(d2 * 0.5) + a; x3 = (uint64_t)(d3 * 0.5) + a;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (double)(x0 ^ x1 ^ x2 ^ x3);
}
template <typename F>
float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; r++) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}
int main() {
    const int blocks = 148 * 8, threads = 256;
    double *dd; uint64_t *du; uint32_t *d32;
    cudaMalloc(&dd, blocks * threads * 8); cudaMalloc(&du, blocks * threads * 8); cudaMalloc(&d32, blocks * threads * 4);
    const double n = (double)blocks * threads * ITERS * 8;
    float t = timeit([&] { k_dfma<<<blocks, threads>>>(dd, 1.0000001, 0.5); });
    printf("DFMA:      %.2f T ops/s  (%.1f per clk per SM @1.965GHz)\n", n / t / 1e9, n / t / 1e9 * 1e12 / 148 / 1.965e9 / 1e12 * 1e0);
    t = timeit([&] { k_mulhi<<<blocks, threads>>>(du, 0x9e3779b97f4a7c15ull); });
    printf("mulhi64:   %.2f T ops/s  (%.1f per clk per SM)\n", n / t / 1e9, n / t / 1e9 / 148 / 1.965);
    t = timeit([&] { k_imad<<<blocks, threads>>>(d32, 2654435761u); });
    printf("IMAD32:    %.2f T ops/s  (%.1f per clk per SM)\n", n / t / 1e9, n / t / 1e9 / 148 / 1.965);
    const double nc = (double)blocks * threads * ITERS * 4;
    t = timeit([&] { k_cvt<<<blocks, threads>>>(dd, 3); });
    printf("I2F+DMUL+F2I (u64): %.2f T round-trips/s  (%.1f per clk per SM)\n", nc / t / 1e9, nc / t / 1e9 / 148 / 1.965);
    return 0;
}
