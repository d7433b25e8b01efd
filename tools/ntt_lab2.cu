// ntt_lab2.cu — variants of the production 16-CTA forward NTT (not product code).
//
//   P  production ntt16::fwd_kernel<ProPlain, EpiPlain>
//   L<F, MINB> lab copy of its small-prime path with
//      F & 1  split cluster barrier: arrive.release after the column stores, L2
//             prefetch of the row's twist factors, then wait.acquire
//      F & 2  column phase in two 128-thread groups (8 columns each) joined by
//             named barriers instead of one 256-thread __syncthreads
//      MINB   __launch_bounds__ min blocks (4 = 64 registers, 3 = 80)
// Tables are random; only timings are meaningful.
//   nvcc -O3 -std=c++17 --fmad=false -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2409_07751_b200/csrc tools/ntt_lab2.cu -o tools/ntt_lab2
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ntt16.cuh"

using namespace ntt16;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int F>
__device__ __forceinline__ void lab_cols(const uint64_t *in, long long P, double *inter, int tile, const double2 *T,
                                         const FpMod &m, double *sm) {
    constexpr bool kGroups = F & 2;
    const int t = kGroups ? (threadIdx.x & 127) : threadIdx.x;
    const int g = kGroups ? (threadIdx.x >> 7) : 0;
    constexpr int kW = kGroups ? 8 : 16;  // columns per barrier group
    const int c = t % kW, k = t / kW, col = tile * 16 + g * kW + c;
    double *s = sm + g * (256 * kW);
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = u2d(in[(P << 16) + (k + 16 * u) * 256 + col]);
#pragma unroll
    for (int st = 0; st < 4; ++st) {
        const int d = 8 >> st;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<false>(x[u], x[u + d], T[(1 << st) + (u >> (4 - st))], m);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) s[(k + 16 * u) * kW + c] = x[u];
    if (kGroups) named_bar(1 + g, 128);
    else __syncthreads();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = s[(16 * k + v) * kW + c];
#pragma unroll
    for (int st = 4; st < 8; ++st) {
        const int d = 128 >> st;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) ct_f<false>(x[v], x[v + d], T[(1 << st) + ((16 * k + v) >> (8 - st))], m);
    }
#pragma unroll
    for (int v = 0; v < 16; ++v) inter[(16 * k + v) * 256 + col] = x[v];
}

template <int F, int MINB>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kTh, MINB)
    lab_fwd(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
            const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % kCl;
    const long long P = blockIdx.x / kCl;
    stage_table(st, tw);
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    const int rs = threadIdx.x >> 4, r = c * kTc + rs;
    lab_cols<F>(in, P, inter, c, st, m, smd);
    if (F & 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        const int k = threadIdx.x & 15;
        const char *tr = reinterpret_cast<const char *>(twist + r * 256 + k * 16);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(tr));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(tr + 128));
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        cluster_sync_all();
    }
    fwd_row<false>(EpiPlain{out, kLogN}, 0, P, inter, r, twist, st, m, smd + rs * kRowPad);
}

template <class K>
float time_it(K launch, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

template <int F, int MINB>
void run_lab(const char *name, int polys, const uint64_t *in, uint64_t *inter, uint64_t *out, const double2 *tw,
             const double2 *twist, FpMod m, int reps) {
    CK(cudaFuncSetAttribute(lab_fwd<F, MINB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(lab_fwd<F, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    const float ms = time_it([&] { lab_fwd<F, MINB><<<kCl * polys, kTh, kSmem>>>(in, inter, out, tw, twist, m); }, reps);
    printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", name, ms, 1e3 * ms / polys);
}

int main(int argc, char **argv) {
    const int polys = argc > 1 ? atoi(argv[1]) : 1184;
    const int reps = 10;
    const double q = 70368744177629.0;  // ~2^46
    FpMod m{q, 1.0 / q};
    std::vector<double2> h(kN);
    srand(1);
    for (int i = 0; i < kN; ++i) {
        const double w = (double)(((uint64_t)rand() << 31 ^ rand()) % (uint64_t)q);
        h[i] = make_double2(w, w / q);
    }
    double2 *tw, *twist;
    FpMod *fm;
    uint64_t *in, *inter, *out;
    CK(cudaMalloc(&tw, kN * sizeof(double2)));
    CK(cudaMalloc(&twist, kN * sizeof(double2)));
    CK(cudaMalloc(&fm, sizeof(FpMod)));
    CK(cudaMemcpy(tw, h.data(), kN * sizeof(double2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(twist, h.data(), kN * sizeof(double2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(fm, &m, sizeof m, cudaMemcpyHostToDevice));
    const size_t bytes = (size_t)polys * kN * 8;
    CK(cudaMalloc(&in, bytes));
    CK(cudaMalloc(&inter, bytes));
    CK(cudaMalloc(&out, bytes));
    CK(cudaMemset(in, 0, bytes));
    {
        auto kf = fwd_kernel<ProPlain, EpiPlain>;
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        // one prime: limb0 = 0, B = polys (all polynomials share table 0)
        const float ms = time_it(
            [&] {
                kf<<<kCl * polys, kTh, kSmem>>>(inter, 0, polys, tw, twist, fm, ProPlain{in, kLogN},
                                                EpiPlain{out, kLogN});
            },
            reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "P production", ms, 1e3 * ms / polys);
    }
    {
        auto ki = inv_kernel<ProPlain, EpiPlain>;
        CK(cudaFuncSetAttribute(ki, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(ki, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        double2 *ninv;
        CK(cudaMalloc(&ninv, 2 * sizeof(double2)));
        CK(cudaMemcpy(ninv, h.data(), 2 * sizeof(double2), cudaMemcpyHostToDevice));
        const float ms = time_it(
            [&] {
                ki<<<kCl * polys, kTh, kSmem>>>(inter, 0, polys, tw, twist, ninv, fm, ProPlain{in, kLogN},
                                                EpiPlain{out, kLogN});
            },
            reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "P production inverse", ms, 1e3 * ms / polys);
    }
    run_lab<0, 4>("L0 lab copy", polys, in, inter, out, tw, twist, m, reps);
    run_lab<1, 4>("L1 split barrier + L2 prefetch", polys, in, inter, out, tw, twist, m, reps);
    run_lab<2, 4>("L2 128-thread column groups", polys, in, inter, out, tw, twist, m, reps);
    run_lab<3, 4>("L3 = L1 + L2", polys, in, inter, out, tw, twist, m, reps);
    run_lab<0, 3>("L0 minBlocks 3", polys, in, inter, out, tw, twist, m, reps);
    run_lab<3, 3>("L3 minBlocks 3", polys, in, inter, out, tw, twist, m, reps);
    return 0;
}
