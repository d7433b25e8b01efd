// ntt_lab2.cu — variants of the production 16-CTA forward NTT (not product code).
//
//   P  production ntt16::fwd_kernel<ProPlain, EpiPlain, CPP> at CPP = 16 (the former layout)
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
#include <algorithm>

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

// persistent: each cluster loops over polynomials P = cluster, cluster + n_cl, ...;
// STAGGER > 0 delays cluster c by (c % 4) * STAGGER ns once at start so the four
// CTAs resident on an SM run their latency phases at different times.
template <int STAGGER>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kTh, 4)
    lab_persist(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
                const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m, int polys) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % kCl;
    const int cl = blockIdx.x / kCl, ncl = gridDim.x / kCl;
    if (STAGGER > 0) __nanosleep((unsigned)((cl & 3) * STAGGER));
    stage_table(st, tw);
    __syncthreads();
    const int rs = threadIdx.x >> 4, r = c * kTc + rs;
    for (long long P = cl; P < polys; P += ncl) {
        double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
        lab_cols<0>(in, P, inter, c, st, m, smd);
        cluster_sync_all();
        fwd_row<false>(EpiPlain{out, kLogN}, 0, P, inter, r, twist, st, m, smd + rs * kRowPad);
        __syncthreads();  // row buffers are reused by the next column phase
    }
}

template <int STAGGER>
void run_persist(const char *name, int polys, int ncl, const uint64_t *in, uint64_t *inter, uint64_t *out,
                 const double2 *tw, const double2 *twist, FpMod m, int reps) {
    CK(cudaFuncSetAttribute(lab_persist<STAGGER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(lab_persist<STAGGER>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    const float ms = time_it(
        [&] { lab_persist<STAGGER><<<kCl * ncl, kTh, kSmem>>>(in, inter, out, tw, twist, m, polys); }, reps);
    printf("%-26s ncl=%-4d %8.3f ms  %6.3f us/limb-poly\n", name, ncl, ms, 1e3 * ms / polys);
}

// production-shaped kernel that records each CTA's start / end (globaltimer, ns)
// and SM id, to measure how many CTAs are co-resident
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kTh, 4)
    lab_timed(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
              const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m, ulonglong2 *rec, int *smid) {
    extern __shared__ double smd[];
    const unsigned long long t0 = gtime();
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % kCl;
    const long long P = blockIdx.x / kCl;
    stage_table(st, tw);
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    const int rs = threadIdx.x >> 4, r = c * kTc + rs;
    lab_cols<0>(in, P, inter, c, st, m, smd);
    cluster_sync_all();
    fwd_row<false>(EpiPlain{out, kLogN}, 0, P, inter, r, twist, st, m, smd + rs * kRowPad);
    __syncthreads();
    if (threadIdx.x == 0) {
        rec[blockIdx.x] = make_ulonglong2(t0, gtime());
        int id;
        asm("mov.u32 %0, %%smid;" : "=r"(id));
        smid[blockIdx.x] = id;
    }
}

// cooperative persistent kernel without clusters: groups of 16 CTAs (one
// polynomial at a time) joined by a self-resetting software barrier in global
// memory; the grid fills every SM (4 CTAs each), unlike 16-CTA clusters which
// leave whole SMs idle when a GPC's SM count is not a multiple of 4.
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void group_bar(unsigned *cnt, unsigned *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(gen);
        __threadfence();
        if (atomicAdd(cnt, 1u) == kCl - 1) {
            atomicExch(cnt, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (ld_acquire(gen) == g) {
            }
        }
    }
    __syncthreads();
}
template <int SLEEP>
__global__ void __launch_bounds__(kTh, 4)
    lab_coop(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
             const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m, int polys, unsigned *bars) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % kCl;
    const int grp = blockIdx.x / kCl, ngrp = gridDim.x / kCl;
    unsigned *cnt = bars + 64 * grp, *gen = cnt + 32;
    if (SLEEP > 0) __nanosleep((unsigned)((blockIdx.x / (gridDim.x / 4)) * SLEEP));
    stage_table(st, tw);
    __syncthreads();
    const int rs = threadIdx.x >> 4, r = c * kTc + rs;
    for (long long P = grp; P < polys; P += ngrp) {
        double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
        lab_cols<0>(in, P, inter, c, st, m, smd);
        group_bar(cnt, gen);
        fwd_row<false>(EpiPlain{out, kLogN}, 0, P, inter, r, twist, st, m, smd + rs * kRowPad);
        __syncthreads();
    }
}

// one CTA per polynomial, no cluster: 16 column passes, a CTA barrier, 16 row
// passes (inter through L2 / HBM). CTAs are independent, so nothing couples the
// phases of the four CTAs on an SM and every SM can be used.
__global__ void __launch_bounds__(kTh, 4)
    lab_single(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
               const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const long long P = blockIdx.x;
    stage_table(st, tw);
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    for (int t = 0; t < 16; ++t) {
        lab_cols<0>(in, P, inter, t, st, m, smd);
        __syncthreads();
    }
    const int rs = threadIdx.x >> 4;
    for (int t = 0; t < 16; ++t) {
        fwd_row<false>(EpiPlain{out, kLogN}, 0, P, inter, t * kTc + rs, twist, st, m, smd + rs * kRowPad);
        __syncwarp();
    }
}

// CPP CTAs per polynomial (cluster of CPP, or a lone CTA for CPP = 1): each CTA
// runs 16 / CPP column tiles, the cluster barrier, then 16 / CPP row blocks.
template <int CPP, int MINB = 4>
__global__ void __launch_bounds__(kTh, MINB)
    lab_multi(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
              const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % CPP;
    const long long P = blockIdx.x / CPP;
    stage_table(st, tw);
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    constexpr int kT = 16 / CPP;
    for (int t = 0; t < kT; ++t) {
        lab_cols<0>(in, P, inter, c * kT + t, st, m, smd);
        __syncthreads();
    }
    if (CPP > 1) cluster_sync_all();
    const int rs = threadIdx.x >> 4;
    for (int t = 0; t < kT; ++t) {
        fwd_row<false>(EpiPlain{out, kLogN}, 0, P, inter, (c * kT + t) * kTc + rs, twist, st, m, smd + rs * kRowPad);
        __syncwarp();
    }
}

template <int CPP, int MINB = 4>
void run_multi(int polys, const uint64_t *in, uint64_t *inter, uint64_t *out, const double2 *tw, const double2 *twist,
               FpMod m, int reps) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CPP * polys);
    cfg.blockDim = dim3(kTh);
    cfg.dynamicSmemBytes = kSmem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = CPP;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    CK(cudaFuncSetAttribute(lab_multi<CPP, MINB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(lab_multi<CPP, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    const float ms =
        time_it([&] { CK(cudaLaunchKernelEx(&cfg, lab_multi<CPP, MINB>, in, inter, out, tw, twist, m)); }, reps);
    printf("M%-2d minB %d %5d polys %8.3f ms  %6.3f us/limb-poly\n", CPP, MINB, polys, ms, 1e3 * ms / polys);
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
    if (argc > 2) {  // sweep: CTAs-per-polynomial variants over launch sizes
        auto kf = fwd_kernel<ProPlain, EpiPlain, 16>;
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        for (int n : {64, 416, 600, 800, 1184, 2368, 4736}) {
            if (n > polys) break;
            const float ms = time_it(
                [&] {
                    CK(launch_clustered(kf, 16, n, 0, (uint64_t *)inter, 0, n, (const double2 *)tw, (const double2 *)twist, (const FpMod *)fm, ProPlain{in, kLogN}, EpiPlain{out, kLogN}, 0));
                },
                reps);
            printf("P   %5d polys %8.3f ms  %6.3f us/limb-poly\n", n, ms, 1e3 * ms / n);
            run_multi<1>(n, in, inter, out, tw, twist, m, reps);
            run_multi<2>(n, in, inter, out, tw, twist, m, reps);
            run_multi<4>(n, in, inter, out, tw, twist, m, reps);
            run_multi<8>(n, in, inter, out, tw, twist, m, reps);
            run_multi<16>(n, in, inter, out, tw, twist, m, reps);
            run_multi<4, 5>(n, in, inter, out, tw, twist, m, reps);
            run_multi<4, 6>(n, in, inter, out, tw, twist, m, reps);
        }
        return 0;
    }
    {
        auto kf = fwd_kernel<ProPlain, EpiPlain, 16>;
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        // one prime: limb0 = 0, B = polys (all polynomials share table 0)
        const float ms = time_it(
            [&] {
                CK(launch_clustered(kf, 16, polys, 0, (uint64_t *)inter, 0, polys, (const double2 *)tw, (const double2 *)twist,
                                    (const FpMod *)fm, ProPlain{in, kLogN}, EpiPlain{out, kLogN}, 0));
            },
            reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "P production", ms, 1e3 * ms / polys);
    }
    {
        auto ki = inv_kernel<ProPlain, EpiPlain, 16>;
        CK(cudaFuncSetAttribute(ki, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(ki, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        double2 *ninv;
        CK(cudaMalloc(&ninv, 2 * sizeof(double2)));
        CK(cudaMemcpy(ninv, h.data(), 2 * sizeof(double2), cudaMemcpyHostToDevice));
        const float ms = time_it(
            [&] {
                CK(launch_clustered(ki, 16, polys, 0, (uint64_t *)inter, 0, polys, (const double2 *)tw, (const double2 *)twist,
                                    (const double2 *)ninv, (const FpMod *)fm, ProPlain{in, kLogN}, EpiPlain{out, kLogN}));
            },
            reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "P production inverse", ms, 1e3 * ms / polys);
    }
    {
        int ncl = 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kCl * 1024);
        cfg.blockDim = dim3(kTh);
        cfg.dynamicSmemBytes = kSmem;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = kCl;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        CK(cudaFuncSetAttribute(lab_persist<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(lab_persist<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        CK(cudaOccupancyMaxActiveClusters(&ncl, (void *)lab_persist<0>, &cfg));
        printf("max active 16-CTA clusters: %d\n", ncl);
        for (int f : {1, 2}) {
            run_persist<0>("T1 persistent", polys, ncl * f, in, inter, out, tw, twist, m, reps);
            run_persist<2000>("T2 persistent stagger 2us", polys, ncl * f, in, inter, out, tw, twist, m, reps);
            run_persist<5000>("T3 persistent stagger 5us", polys, ncl * f, in, inter, out, tw, twist, m, reps);
        }
    }
    {
        ulonglong2 *rec;
        int *smid;
        CK(cudaMalloc(&rec, sizeof(ulonglong2) * kCl * polys));
        CK(cudaMalloc(&smid, sizeof(int) * kCl * polys));
        CK(cudaFuncSetAttribute(lab_timed, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(lab_timed, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        for (int i = 0; i < 2; ++i) lab_timed<<<kCl * polys, kTh, kSmem>>>(in, inter, out, tw, twist, m, rec, smid);
        CK(cudaDeviceSynchronize());
        std::vector<ulonglong2> h(kCl * polys);
        std::vector<int> sm(kCl * polys);
        CK(cudaMemcpy(h.data(), rec, sizeof(ulonglong2) * h.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sm.data(), smid, sizeof(int) * sm.size(), cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull, t1 = 0;
        double life = 0;
        for (auto &x : h) {
            t0 = std::min(t0, (unsigned long long)x.x);
            t1 = std::max(t1, (unsigned long long)x.y);
            life += (double)(x.y - x.x);
        }
        // sample concurrency every 1 us
        int maxc = 0;
        double sumc = 0;
        int ns = 0;
        for (unsigned long long t = t0; t < t1; t += 1000, ++ns) {
            int cnt = 0;
            for (auto &x : h) cnt += (x.x <= t && t < x.y);
            maxc = std::max(maxc, cnt);
            sumc += cnt;
        }
        std::vector<int> per(256, 0);
        for (int v : sm) per[v & 255]++;
        int nsm = 0;
        for (int v : per) nsm += v > 0;
        printf("timed: span %.1f us, mean CTA life %.2f us, co-resident CTAs max %d mean %.1f, SMs used %d\n",
               (t1 - t0) / 1e3, life / h.size() / 1e3, maxc, sumc / ns, nsm);
    }
    {
        unsigned *bars;
        CK(cudaMalloc(&bars, 4096 * 64 * 4));
        CK(cudaMemset(bars, 0, 4096 * 64 * 4));
        CK(cudaFuncSetAttribute(lab_coop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        int per_sm = 0, sms = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lab_coop<0>, kTh, kSmem));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
        const int grid = (per_sm * sms / kCl) * kCl;
        printf("coop: %d CTAs/SM, grid %d CTAs (%d groups)\n", per_sm, grid, grid / kCl);
        int np = polys;
        void *args[] = {(void *)&in, (void *)&inter, (void *)&out, (void *)&tw, (void *)&twist, (void *)&m, (void *)&np,
                        (void *)&bars};
        float ms = time_it(
            [&] { CK(cudaLaunchCooperativeKernel((void *)lab_coop<0>, dim3(grid), dim3(kTh), args, kSmem, 0)); }, reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "T4 cooperative, software barrier", ms, 1e3 * ms / polys);
        CK(cudaFuncSetAttribute(lab_coop<2000>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        CK(cudaFuncSetAttribute(lab_coop<4000>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        ms = time_it(
            [&] { CK(cudaLaunchCooperativeKernel((void *)lab_coop<2000>, dim3(grid), dim3(kTh), args, kSmem, 0)); }, reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "T5 coop, stagger 2us per quarter", ms, 1e3 * ms / polys);
        ms = time_it(
            [&] { CK(cudaLaunchCooperativeKernel((void *)lab_coop<4000>, dim3(grid), dim3(kTh), args, kSmem, 0)); }, reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "T6 coop, stagger 4us per quarter", ms, 1e3 * ms / polys);
    }
    {
        CK(cudaFuncSetAttribute(lab_single, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        const float ms = time_it([&] { lab_single<<<polys, kTh, kSmem>>>(in, inter, out, tw, twist, m); }, reps);
        printf("%-34s %8.3f ms  %6.3f us/limb-poly\n", "T7 one CTA per polynomial", ms, 1e3 * ms / polys);
    }
    run_lab<0, 4>("L0 lab copy", polys, in, inter, out, tw, twist, m, reps);
    run_lab<1, 4>("L1 split barrier + L2 prefetch", polys, in, inter, out, tw, twist, m, reps);
    run_lab<2, 4>("L2 128-thread column groups", polys, in, inter, out, tw, twist, m, reps);
    run_lab<3, 4>("L3 = L1 + L2", polys, in, inter, out, tw, twist, m, reps);
    run_lab<0, 3>("L0 minBlocks 3", polys, in, inter, out, tw, twist, m, reps);
    run_lab<3, 3>("L3 minBlocks 3", polys, in, inter, out, tw, twist, m, reps);
    return 0;
}
