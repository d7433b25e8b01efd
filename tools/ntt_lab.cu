// ntt_lab.cu — timing lab for the fused N = 2^16 forward NTT (not product code).
//
// Times copies of ntt16::fwd_kernel with pieces removed, to attribute the
// kernel's time: V0 production data flow, V1 synthetic column input (no
// global loads), V2 twist factors from shared memory (no table loads), V3 row
// phase from own shared memory (no between-phase exchange, no cluster
// barrier), V4 = V1+V2+V3 with stores suppressed (arithmetic floor).
// Values are meaningless (random tables); only the timings are reported.
//   nvcc -O3 -std=c++17 --fmad=false -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2409_07751_b200/csrc tools/ntt_lab.cu -o tools/ntt_lab
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ntt16.cuh"

using namespace ntt16;

constexpr int kSmem32 = 32 * kRowPad * 8 + 256 * 16;  // 8-CTA variants (512 threads, 32 columns)

template <int V>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 2)
    lab_fwd(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
            const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m) {
    constexpr bool kVec = V == 7;
    constexpr bool kSynth = V == 1 || V == 4, kNoTau = V == 2 || V == 4, kNoX = V == 3 || V == 4, kNoSt = V == 4;
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + 32 * kRowPad);
    const int cb = blockIdx.x & 7;
    const long long P = blockIdx.x >> 3;
    if (threadIdx.x < 256) st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    // ---- column phase
    {
        const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = cb * 32 + c;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
            x[u] = kSynth ? (double)((k + 16 * u) * 256 + col + (int)P) : u2d(in[P * kN + (k + 16 * u) * 256 + col]);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int d = 8 >> s;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << s) + (u >> (4 - s))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) smd[(k + 16 * u) * 32 + c] = x[u];
        __syncthreads();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = smd[(16 * k + v) * 32 + c];
#pragma unroll
        for (int s = 4; s < 8; ++s) {
            const int d = 128 >> s;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << s) + ((16 * k + v) >> (8 - s))], m);
        }
        if (kNoX) {
            __syncthreads();
#pragma unroll
            for (int v = 0; v < 16; ++v) smd[(16 * k + v) * 32 + c] = f_center(x[v], m);
            __syncthreads();
        } else {
#pragma unroll
            for (int v = 0; v < 16; ++v) inter[(16 * k + v) * 256 + col] = f_center(x[v], m);
        }
    }
    if (!kNoX) cluster_sync_all();
    // ---- row phase
    {
        const int rs = threadIdx.x >> 4, r = cb * 32 + rs;
        const int k = threadIdx.x & 15;
        double *srow = smd + rs * kRowPad;
        double x[16];
        if (kNoX) {
#pragma unroll
            for (int u = 0; u < 16; ++u) x[u] = smd[(rs * 8 + (u & 7)) * 32 + ((k + 16 * u) & 31)];
            __syncthreads();
        } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) x[u] = __ldcg(inter + r * 256 + k + 16 * u);
        }
        const double2 *tr = twist + r * 256;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double2 t = kNoTau ? st[(k + 16 * u) & 255] : __ldg(tr + k + 16 * u);
            x[u] = f_mulmod(x[u], t.x, t.y, m.q);
        }
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
            const int d = 8 >> sp;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
        for (int sp = 4; sp < 8; ++sp) {
            const int d = 128 >> sp;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << sp) + ((16 * k + v) >> (8 - sp))], m);
        }
        if (kVec) {
            ulonglong2 *o2 = reinterpret_cast<ulonglong2 *>(out + P * kN + r * 256 + 16 * k);
#pragma unroll
            for (int v = 0; v < 16; v += 2) o2[v >> 1] = make_ulonglong2(d2canon(x[v], m), d2canon(x[v + 1], m));
        } else {
            __syncwarp();
            uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
            for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint64_t v = su[pad16(k + 16 * u)];
                if (!kNoSt || v == 0x123456789ull) out[P * kN + r * 256 + k + 16 * u] = v;
            }
        }
    }
}


// V5: between-phase exchange through distributed shared memory: each CTA's
// column tile stays in its own shared memory; the row phase reads the 8 tiles
// of the cluster remotely; a split arrive/wait barrier protects reuse.
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ double ld_dsmem(const double *local, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 2)
    lab_fwd5(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, const double2 *__restrict__ tw,
             const double2 *__restrict__ twist, FpMod m) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + 32 * kRowPad);
    const int cb = blockIdx.x & 7;
    const long long P = blockIdx.x >> 3;
    if (threadIdx.x < 256) st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    {
        const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = cb * 32 + c;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = u2d(in[P * kN + (k + 16 * u) * 256 + col]);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int d = 8 >> s;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << s) + (u >> (4 - s))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) smd[(k + 16 * u) * 32 + c] = x[u];
        __syncthreads();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = smd[(16 * k + v) * 32 + c];
#pragma unroll
        for (int s = 4; s < 8; ++s) {
            const int d = 128 >> s;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << s) + ((16 * k + v) >> (8 - s))], m);
        }
#pragma unroll
        for (int v = 0; v < 16; ++v) smd[(16 * k + v) * 32 + c] = f_center(x[v], m);  // own tile [row][32]
    }
    cl_arrive();
    cl_wait();
    {
        const int rs = threadIdx.x >> 4, r = cb * 32 + rs;
        const int k = threadIdx.x & 15;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = ld_dsmem(smd + r * 32 + k + 16 * (u & 1), (unsigned)(u >> 1));
        cl_arrive();  // this CTA's remote reads are done
        const double2 *tr = twist + r * 256;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double2 t = __ldg(tr + k + 16 * u);
            x[u] = f_mulmod(x[u], t.x, t.y, m.q);
        }
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
            const int d = 8 >> sp;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m);
        }
        cl_wait();  // every CTA has read this CTA's tile: reuse it
        double *srow = smd + rs * kRowPad;
#pragma unroll
        for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
        for (int sp = 4; sp < 8; ++sp) {
            const int d = 128 >> sp;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << sp) + ((16 * k + v) >> (8 - sp))], m);
        }
        __syncwarp();
        uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
        for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 16; ++u) out[P * kN + r * 256 + k + 16 * u] = su[pad16(k + 16 * u)];
    }
}


__device__ __forceinline__ void st_dsmem(double *local, unsigned rank, double v) {
    unsigned a = (unsigned)__cvta_generic_to_shared(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// V6: push exchange: after the column transpose every CTA's buffer is free
// (barrier 1, arrive early / wait late); the column results are stored into
// the owning row CTA's buffer (row layout, padded); barrier 2; the row phase
// reads local shared memory.
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 2)
    lab_fwd6(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, const double2 *__restrict__ tw,
             const double2 *__restrict__ twist, FpMod m) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + 32 * kRowPad);
    const int cb = blockIdx.x & 7;
    const long long P = blockIdx.x >> 3;
    if (threadIdx.x < 256) st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    {
        const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = cb * 32 + c;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = u2d(in[P * kN + (k + 16 * u) * 256 + col]);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int d = 8 >> s;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << s) + (u >> (4 - s))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) smd[(k + 16 * u) * 32 + c] = x[u];
        __syncthreads();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = smd[(16 * k + v) * 32 + c];
        cl_arrive();  // this CTA's transpose buffer is free
#pragma unroll
        for (int s = 4; s < 8; ++s) {
            const int d = 128 >> s;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << s) + ((16 * k + v) >> (8 - s))], m);
        }
        cl_wait();
        // rows 16k + v go to CTA (16k+v) >> 5 = k >> 1, local row (16k+v) & 31
#pragma unroll
        for (int v = 0; v < 16; ++v)
            st_dsmem(smd + ((16 * k + v) & 31) * kRowPad + pad16(col), (unsigned)(k >> 1), f_center(x[v], m));
    }
    cl_arrive();
    cl_wait();
    {
        const int rs = threadIdx.x >> 4, r = cb * 32 + rs;
        const int k = threadIdx.x & 15;
        double *srow = smd + rs * kRowPad;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = srow[pad16(k + 16 * u)];
        const double2 *tr = twist + r * 256;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double2 t = __ldg(tr + k + 16 * u);
            x[u] = f_mulmod(x[u], t.x, t.y, m.q);
        }
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
            const int d = 8 >> sp;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
        for (int sp = 4; sp < 8; ++sp) {
            const int d = 128 >> sp;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << sp) + ((16 * k + v) >> (8 - sp))], m);
        }
        __syncwarp();
        uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
        for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 16; ++u) out[P * kN + r * 256 + k + 16 * u] = su[pad16(k + 16 * u)];
    }
}


// V8: 16-CTA cluster of 256 threads: CTA owns 16 columns / 16 rows.
constexpr int kSmem8 = 16 * kRowPad * 8 + 256 * 16;
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, 4)
    lab_fwd8(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
             const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + 16 * kRowPad);
    const int cb = blockIdx.x & 15;
    const long long P = blockIdx.x >> 4;
    st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    {
        const int c = threadIdx.x & 15, k = threadIdx.x >> 4, col = cb * 16 + c;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = u2d(in[P * kN + (k + 16 * u) * 256 + col]);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int d = 8 >> s;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << s) + (u >> (4 - s))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) smd[(k + 16 * u) * 17 + c] = x[u];
        __syncthreads();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = smd[(16 * k + v) * 17 + c];
#pragma unroll
        for (int s = 4; s < 8; ++s) {
            const int d = 128 >> s;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << s) + ((16 * k + v) >> (8 - s))], m);
        }
#pragma unroll
        for (int v = 0; v < 16; ++v) inter[(16 * k + v) * 256 + col] = f_center(x[v], m);
    }
    cluster_sync_all();
    {
        const int rs = threadIdx.x >> 4, r = cb * 16 + rs;
        const int k = threadIdx.x & 15;
        double *srow = smd + rs * kRowPad;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = __ldcg(inter + r * 256 + k + 16 * u);
        const double2 *tr = twist + r * 256;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double2 t = __ldg(tr + k + 16 * u);
            x[u] = f_mulmod(x[u], t.x, t.y, m.q);
        }
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
            const int d = 8 >> sp;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
        for (int sp = 4; sp < 8; ++sp) {
            const int d = 128 >> sp;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << sp) + ((16 * k + v) >> (8 - sp))], m);
        }
        __syncwarp();
        uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
        for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 16; ++u) out[P * kN + r * 256 + k + 16 * u] = su[pad16(k + 16 * u)];
    }
}


// V9: V8 (16-CTA clusters) with the CTA-uniform twiddles T[1..15] of stages 0-3 of
// both phases read from constant memory (DFMA operands, no LDS)
__constant__ double2 cT[64][16];
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, 4)
    lab_fwd9(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
             const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m, int mi) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + 16 * kRowPad);
    const int cb = blockIdx.x & 15;
    const long long P = blockIdx.x >> 4;
    st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    {
        const int c = threadIdx.x & 15, k = threadIdx.x >> 4, col = cb * 16 + c;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = u2d(in[P * kN + (k + 16 * u) * 256 + col]);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int d = 8 >> s;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], cT[mi][(1 << s) + (u >> (4 - s))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) smd[(k + 16 * u) * 16 + c] = x[u];
        __syncthreads();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = smd[(16 * k + v) * 16 + c];
#pragma unroll
        for (int s = 4; s < 8; ++s) {
            const int d = 128 >> s;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << s) + ((16 * k + v) >> (8 - s))], m);
        }
#pragma unroll
        for (int v = 0; v < 16; ++v) inter[(16 * k + v) * 256 + col] = f_center(x[v], m);
    }
    cluster_sync_all();
    {
        const int rs = threadIdx.x >> 4, r = cb * 16 + rs;
        const int k = threadIdx.x & 15;
        double *srow = smd + rs * kRowPad;
        double x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = __ldcg(inter + r * 256 + k + 16 * u);
        const double2 *tr = twist + r * 256;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double2 t = __ldg(tr + k + 16 * u);
            x[u] = f_mulmod(x[u], t.x, t.y, m.q);
        }
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
            const int d = 8 >> sp;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (!(u & d)) ct_f<false>(x[u], x[u + d], cT[mi][(1 << sp) + (u >> (4 - sp))], m);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
        for (int sp = 4; sp < 8; ++sp) {
            const int d = 128 >> sp;
#pragma unroll
            for (int v = 0; v < 16; ++v)
                if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << sp) + ((16 * k + v) >> (8 - sp))], m);
        }
        __syncwarp();
        uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
        for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 16; ++u) out[P * kN + r * 256 + k + 16 * u] = su[pad16(k + 16 * u)];
    }
}


// V10: persistent, software-pipelined 16-CTA clusters: the next polynomial's
// column phase runs between the cluster barrier's arrive and wait of the current
// one, hiding the barrier; the twiddle table is staged once per CTA.
__device__ __forceinline__ void v10_col(const uint64_t *__restrict__ in, double *inter, long long P, int cb,
                                        const double2 *st, const FpMod &m, double *smd) {
    const int c = threadIdx.x & 15, k = threadIdx.x >> 4, col = cb * 16 + c;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = u2d(in[P * kN + (k + 16 * u) * 256 + col]);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int d = 8 >> s;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << s) + (u >> (4 - s))], m);
    }
    __syncthreads();  // previous row phase done with smd
#pragma unroll
    for (int u = 0; u < 16; ++u) smd[(k + 16 * u) * 16 + c] = x[u];
    __syncthreads();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = smd[(16 * k + v) * 16 + c];
#pragma unroll
    for (int s = 4; s < 8; ++s) {
        const int d = 128 >> s;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << s) + ((16 * k + v) >> (8 - s))], m);
    }
#pragma unroll
    for (int v = 0; v < 16; ++v) inter[P * kN + (16 * k + v) * 256 + col] = x[v];
}
__device__ __forceinline__ void v10_row(const double *inter, uint64_t *__restrict__ out, long long P, int cb,
                                        const double2 *__restrict__ twist, const double2 *st, const FpMod &m,
                                        double *smd) {
    const int rs = threadIdx.x >> 4, r = cb * 16 + rs;
    const int k = threadIdx.x & 15;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = __ldcg(inter + P * kN + r * 256 + k + 16 * u);
    const double2 *tr = twist + r * 256;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const double2 t = __ldg(tr + k + 16 * u);
        x[u] = f_mulmod(x[u], t.x, t.y, m.q);
    }
#pragma unroll
    for (int sp = 0; sp < 4; ++sp) {
        const int d = 8 >> sp;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<false>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m);
    }
    __syncthreads();  // column phase done with smd (it is reused as row buffers)
    double *srow = smd + rs * kRowPad;
#pragma unroll
    for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
    for (int sp = 4; sp < 8; ++sp) {
        const int d = 128 >> sp;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) ct_f<false>(x[v], x[v + d], st[(1 << sp) + ((16 * k + v) >> (8 - sp))], m);
    }
    __syncwarp();
    uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
    for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 16; ++u) out[P * kN + r * 256 + k + 16 * u] = su[pad16(k + 16 * u)];
}
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, 4)
    lab_fwd10(const uint64_t *__restrict__ in, uint64_t *__restrict__ inter_base, uint64_t *__restrict__ out,
              const double2 *__restrict__ tw, const double2 *__restrict__ twist, FpMod m, int polys) {
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + 16 * kRowPad);
    const int cb = blockIdx.x & 15;
    const int cl = blockIdx.x >> 4, ncl = gridDim.x >> 4;
    double *inter = reinterpret_cast<double *>(inter_base);
    st[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    long long p = cl;
    if (p >= polys) return;
    v10_col(in, inter, p, cb, st, m, smd);
    cl_arrive();
    for (;;) {
        const long long pn = p + ncl;
        const bool more = pn < polys;
        if (more) v10_col(in, inter, pn, cb, st, m, smd);
        cl_wait();
        v10_row(inter, out, p, cb, twist, st, m, smd);
        if (!more) break;
        cl_arrive();
        p = pn;
    }
}

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                             \
        }                                                                        \
    } while (0)

template <int V>
float run(int polys, const uint64_t *in, uint64_t *inter, uint64_t *out, const double2 *tw, const double2 *twist,
          FpMod m, int reps) {
    CK(cudaFuncSetAttribute(lab_fwd<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem32));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    lab_fwd<V><<<8 * polys, 512, kSmem32>>>(in, inter, out, tw, twist, m);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) lab_fwd<V><<<8 * polys, 512, kSmem32>>>(in, inter, out, tw, twist, m);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
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
    uint64_t *in, *inter, *out;
    CK(cudaMalloc(&tw, kN * sizeof(double2)));
    CK(cudaMalloc(&twist, kN * sizeof(double2)));
    CK(cudaMemcpy(tw, h.data(), kN * sizeof(double2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(twist, h.data(), kN * sizeof(double2), cudaMemcpyHostToDevice));
    const size_t bytes = (size_t)polys * kN * 8;
    CK(cudaMalloc(&in, bytes));
    CK(cudaMalloc(&inter, bytes));
    CK(cudaMalloc(&out, bytes));
    CK(cudaMemset(in, 0, bytes));
    const char *names[] = {"V0 production", "V1 synthetic input", "V2 twist from smem", "V3 no exchange",
                           "V4 arithmetic floor"};
    float t[5];
    t[0] = run<0>(polys, in, inter, out, tw, twist, m, reps);
    t[1] = run<1>(polys, in, inter, out, tw, twist, m, reps);
    t[2] = run<2>(polys, in, inter, out, tw, twist, m, reps);
    t[3] = run<3>(polys, in, inter, out, tw, twist, m, reps);
    t[4] = run<4>(polys, in, inter, out, tw, twist, m, reps);
    {
        CK(cudaFuncSetAttribute(lab_fwd5, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem32));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        lab_fwd5<<<8 * polys, 512, kSmem32>>>(in, out, tw, twist, m);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) lab_fwd5<<<8 * polys, 512, kSmem32>>>(in, out, tw, twist, m);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-22s %8.3f ms  %6.3f us/limb-poly\n", "V5 DSMEM exchange", ms / reps, 1e3 * ms / reps / polys);
    }
    {
        CK(cudaFuncSetAttribute(lab_fwd6, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem32));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        lab_fwd6<<<8 * polys, 512, kSmem32>>>(in, out, tw, twist, m);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) lab_fwd6<<<8 * polys, 512, kSmem32>>>(in, out, tw, twist, m);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-22s %8.3f ms  %6.3f us/limb-poly\n", "V6 DSMEM push", ms / reps, 1e3 * ms / reps / polys);
    }
    printf("%-22s %8.3f ms\n", "V7 direct vec stores", run<7>(polys, in, inter, out, tw, twist, m, reps));
    {
        CK(cudaFuncSetAttribute(lab_fwd8, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(lab_fwd8, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem8));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        lab_fwd8<<<16 * polys, 256, kSmem8>>>(in, inter, out, tw, twist, m);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) lab_fwd8<<<16 * polys, 256, kSmem8>>>(in, inter, out, tw, twist, m);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-22s %8.3f ms  %6.3f us/limb-poly\n", "V8 cluster16 x 256", ms / reps, 1e3 * ms / reps / polys);
    }
    {
        std::vector<double2> ct(64 * 16);
        for (int j = 0; j < 64; ++j)
            for (int i = 0; i < 16; ++i) ct[j * 16 + i] = h[i];
        CK(cudaMemcpyToSymbol(cT, ct.data(), sizeof(double2) * 64 * 16));
        CK(cudaFuncSetAttribute(lab_fwd9, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(lab_fwd9, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem8));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        lab_fwd9<<<16 * polys, 256, kSmem8>>>(in, inter, out, tw, twist, m, 3);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) lab_fwd9<<<16 * polys, 256, kSmem8>>>(in, inter, out, tw, twist, m, 3);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-22s %8.3f ms  %6.3f us/limb-poly\n", "V9 const twiddles", ms / reps, 1e3 * ms / reps / polys);
    }
    for (int cpm : {4, 8, 16}) {  // clusters per 148 SMs x 4 CTAs: 37 resident clusters
        CK(cudaFuncSetAttribute(lab_fwd10, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(lab_fwd10, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem8));
        const int ncl = 37 * cpm / 4;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        lab_fwd10<<<16 * ncl, 256, kSmem8>>>(in, inter, out, tw, twist, m, polys);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) lab_fwd10<<<16 * ncl, 256, kSmem8>>>(in, inter, out, tw, twist, m, polys);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("V10 pipelined ncl=%-4d %8.3f ms  %6.3f us/limb-poly\n", ncl, ms / reps, 1e3 * ms / reps / polys);
    }
    for (int i = 0; i < 5; ++i)
        printf("%-22s %8.3f ms  %6.3f us/limb-poly\n", names[i], t[i], 1e3 * t[i] / polys);
    return 0;
}
