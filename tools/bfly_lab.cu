// bfly_lab.cu — register-only butterfly throughput on sm_100a (not product code).
//
// Measures how many radix-2 CT butterflies per clock per SM the exact FP64
// two-product Shoup butterfly reaches when nothing but arithmetic runs:
//   A: ntt16::ct_f with twiddles held in registers
//   B: same, twiddles read from shared memory per butterfly (as the NTT does)
//   C: A with half the butterflies on the integer pipe (quotient from one DFMA,
//      remainder as a 64-bit wrap-around difference y*w - t*q)
//   nvcc -O3 -std=c++17 --fmad=false -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2409_07751_b200/csrc tools/bfly_lab.cu -o tools/bfly_lab
#include <cstdio>
#include <cstdint>

#include "ntt16.cuh"

using namespace ntt16;

constexpr int kIters = 256;

__device__ __forceinline__ void ct_i(double &x, double &y, double2 w, uint64_t wi, uint64_t q, const FpMod &m) {
    // t = round(y * w / q) on the FP64 pipe; r = y*w - t*q mod 2^64 on the integer pipe
    const double t = __dsub_rn(__fma_rn(y, w.y, kMagic), kMagic);
    const long long mb = __double_as_longlong(kMagic);
    const uint64_t yi = (uint64_t)(__double_as_longlong(__dadd_rn(y, kMagic)) - mb);  // signed |y| < 2^51
    const uint64_t ti = (uint64_t)(__double_as_longlong(__dadd_rn(t, kMagic)) - mb);
    const long long r = (long long)(yi * wi - ti * q);
    const double rd = __dsub_rn(__longlong_as_double(r + mb), kMagic);
    const double U = x;
    x = __dadd_rn(U, rd);
    y = __dsub_rn(U, rd);
}

template <int V>
__global__ void __launch_bounds__(256, 4) k_bfly(double *out, const double2 *__restrict__ tw, FpMod m, uint64_t q) {
    __shared__ double2 st[256];
    st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = (double)(threadIdx.x * 16 + u + blockIdx.x);
    double2 w[4];
    uint64_t wi[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        w[s] = tw[s + 1];
        wi[s] = (uint64_t)w[s].x;
    }
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int d = 8 >> s;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) {
                    if (V == 0) ct_f<false>(x[u], x[u + d], w[s], m);
                    if (V == 1) ct_f<false>(x[u], x[u + d], st[(1 << s) + (u >> (4 - s)) + (it & 1)], m);
                    if (V == 2) {
                        if (u & 1) ct_i(x[u], x[u + d], w[s], wi[s], q, m);
                        else ct_f<false>(x[u], x[u + d], w[s], m);
                    }
                }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = f_center(x[u], m);
    }
    double s = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) s += x[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
float run(double *out, const double2 *tw, FpMod m, uint64_t q, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_bfly<V><<<blocks, 256>>>(out, tw, m, q);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_bfly<V><<<blocks, 256>>>(out, tw, m, q);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const uint64_t q = (1ull << 46) + 0x12345 * 2 + 1;
    FpMod m{(double)q, 1.0 / (double)q};
    double2 h[256];
    for (int i = 0; i < 256; ++i) {
        const double w = (double)((0x9E3779B97F4A7C15ull * (i + 1)) % q);
        h[i] = make_double2(w, w / (double)q);
    }
    double2 *tw;
    double *out;
    cudaMalloc(&tw, sizeof h);
    cudaMemcpy(tw, h, sizeof h, cudaMemcpyHostToDevice);
    const int blocks = sms * 4 * 8;
    cudaMalloc(&out, sizeof(double) * blocks * 256);
    const double bf = (double)blocks * 256 * kIters * 32;  // butterflies per launch
    const char *names[] = {"A fp64, twiddles in regs", "B fp64, twiddles from smem", "C half integer-pipe"};
    for (int v = 0; v < 3; ++v) {
        const float ms = v == 0 ? run<0>(out, tw, m, q, blocks) : v == 1 ? run<1>(out, tw, m, q, blocks)
                                                                        : run<2>(out, tw, m, q, blocks);
        const double per_clk_sm = bf / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("%-28s %8.3f ms  %6.2f butterflies/clk/SM (%s)\n", names[v], ms, per_clk_sm,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
