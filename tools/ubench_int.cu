// Throughput microbenchmark of integer / fp64 multiply primitives on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define ILP 8

__global__ void k_imad(uint32_t *out, uint32_t a, uint32_t b) {
    uint32_t x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = x[i] * a + b;
    uint32_t s = 0;
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imadwide(uint64_t *out, uint32_t a) {
    uint64_t x[ILP];
    uint32_t y[ILP];
    for (int i = 0; i < ILP; ++i) { x[i] = threadIdx.x + i; y[i] = threadIdx.x * 3 + i; }
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[i]) : "r"(y[i]), "r"(a));
        }
    uint64_t s = 0;
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mulhi32(uint32_t *out, uint32_t a) {
    uint32_t x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i + 12345;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __umulhi(x[i], a) + x[i];
    uint32_t s = 0;
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mul64lo(uint64_t *out, uint64_t a) {
    uint64_t x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i + 12345;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = x[i] * a;
    uint64_t s = 0;
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mul64hi(uint64_t *out, uint64_t a) {
    uint64_t x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i + 12345;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __umul64hi(x[i], a) ^ x[i];
    uint64_t s = 0;
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double *out, double a, double b) {
    double x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_iadd3(uint32_t *out, uint32_t a, uint32_t b) {
    uint32_t x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = (x[i] + a + b) ^ a;
    uint32_t s = 0;
    for (int i = 0; i < ILP; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void run(const char *name, F launch, double ops_per_thread_iter) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    launch(blocks, threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch(blocks, threads);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * ITERS * ILP * ops_per_thread_iter;
    const double per_s = ops / (ms * 1e-3);
    printf("%-12s %8.3f ms  %8.2f Gops/s  %6.1f ops/clk/SM (at %d MHz max)\n", name, ms, per_s / 1e9,
           per_s / sms / (clk * 1e3), clk / 1000);
}

int main() {
    void *buf;
    cudaMalloc(&buf, 1 << 26);
    run("IMAD", [&](int b, int t) { k_imad<<<b, t>>>((uint32_t *)buf, 3, 7); }, 1);
    run("IMAD.WIDE", [&](int b, int t) { k_imadwide<<<b, t>>>((uint64_t *)buf, 12345); }, 1);
    run("IMAD.HI32", [&](int b, int t) { k_mulhi32<<<b, t>>>((uint32_t *)buf, 12345); }, 1);
    run("mul.lo.u64", [&](int b, int t) { k_mul64lo<<<b, t>>>((uint64_t *)buf, 1234567891234ull); }, 1);
    run("mul.hi.u64", [&](int b, int t) { k_mul64hi<<<b, t>>>((uint64_t *)buf, 1234567891234ull); }, 1);
    run("DFMA", [&](int b, int t) { k_dfma<<<b, t>>>((double *)buf, 1.0000001, 0.5); }, 1);
    run("IADD3+LOP", [&](int b, int t) { k_iadd3<<<b, t>>>((uint32_t *)buf, 3, 7); }, 1);
    cudaDeviceSynchronize();
    return 0;
}
