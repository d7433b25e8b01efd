// ntt.cu — negacyclic NTT / inverse NTT over limb-major RNS buffers (sm_100a).
//
// Convention (identical to oracle/ckks_oracle.c ntt_fwd_1/ntt_inv_1): forward =
// Cooley-Tukey, natural-order coefficients -> bit-reversed evaluations, stage s
// (0..logN-1) pairs (j, j + N/2^(s+1)) with twiddle psi^brv(2^s + (j >> (logN-s)));
// inverse = Gentleman-Sande in reverse stage order with psi^-brv, then * N^-1.
//
// N = 2^16 fast path: one 8-CTA thread-block cluster per polynomial.
//   stages 0..7 act along rows r of the 256x256 view j = 256 r + c -> column
//     phase: CTA c owns columns [32c, 32c+32): 4 radix-2 stages in registers,
//     one shared-memory transpose, 4 more stages; 256 B coalesced row segments;
//   a cluster barrier (release/acquire) publishes the in-place intermediate,
//     which stays in L2 (512 KiB live per cluster);
//   stages 8..15 act within a row -> row phase: CTA c owns rows [32c, 32c+32),
//     a half-warp per row, both exchanges inside a warp (__syncwarp) through a
//     bank-conflict-free padded tile.
// DRAM therefore sees one read and one write per coefficient.
// Arithmetic: lazy Harvey butterflies with an approximate-quotient Shoup
// multiply (3 IMAD.WIDE for the quotient instead of a 64-bit mulhi).
// Other N (parity tests at small sizes): one canonical launch per stage.
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kLogN16 = 16;
constexpr int kN16 = 1 << kLogN16;
constexpr int kRowPad = 272;  // 256 + 16: pad one element every 16

__device__ __forceinline__ int pad16(int c) { return c + (c >> 4); }

// Canonical butterflies (generic per-stage path).
__device__ __forceinline__ void ct_bfly(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q) {
    const uint64_t U = x, V = mul_shoup(y, w.x, w.y, q);
    x = add_mod(U, V, q);
    y = sub_mod(U, V, q);
}
__device__ __forceinline__ void gs_bfly(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q) {
    const uint64_t U = x, V = y;
    x = add_mod(U, V, q);
    y = mul_shoup(sub_mod(U, V, q), w.x, w.y, q);
}

// ---------------------------------------------------------------- FP64 arithmetic
// Inside the fused kernels residues live in float64 registers as exact
// integers (|x| < 2^51). The DFMA/DMUL pipe (64/clk/SM on B200, otherwise idle
// here) carries the modular arithmetic:
//   y*w = h + l exactly (two-product), t = round(y*w/q) via y*(w/q) + M - M,
//   r = (h - t q) + l exactly, |r| <= 1.5 q                      (6 FP64 ops).
// Small primes (q < 2^47): a phase of 8 stages from |x| < q stays below 13 q <
// 2^51, so no reductions are needed inside a phase; the column->row boundary
// recentres (|x| <= q/2). Large primes (q_0 ~ 2^50): recentre after every stage.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;  // 2^52
constexpr uint64_t kSmallPrime = 1ull << 47;

struct FpMod {
    double q, qinv;
};

__device__ __forceinline__ double f_round(double x) { return __dsub_rn(__fma_rn(x, 1.0, kMagic), kMagic); }
__device__ __forceinline__ double f_mulmod(double y, double w, double wq, double q) {
    const double h = __dmul_rn(y, w);
    const double l = __fma_rn(y, w, -h);
    const double t = __dsub_rn(__fma_rn(y, wq, kMagic), kMagic);
    return __dadd_rn(__fma_rn(-t, q, h), l);
}
// centred reduction: |result| <= q/2 (+1)
__device__ __forceinline__ double f_center(double x, const FpMod &m) {
    const double t = __dsub_rn(__fma_rn(x, m.qinv, kMagic), kMagic);
    return __fma_rn(-t, m.q, x);
}
__device__ __forceinline__ double u2d(uint64_t x) {  // exact for x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), kTwo52);
}
// centred value -> canonical residue as u64
__device__ __forceinline__ uint64_t d2canon(double x, const FpMod &m) {
    double c = f_center(x, m);
    c = c < 0.0 ? __dadd_rn(c, m.q) : c;
    c = c >= m.q ? __dsub_rn(c, m.q) : c;
    return (uint64_t)__double_as_longlong(__dadd_rn(c, kTwo52)) & 0xFFFFFFFFFFFFFull;
}

template <bool kBig>
__device__ __forceinline__ void ct_f(double &x, double &y, double2 w, const FpMod &m) {
    const double r = f_mulmod(y, w.x, w.y, m.q);
    const double U = x;
    x = __dadd_rn(U, r);
    y = __dsub_rn(U, r);
    if (kBig) {
        x = f_center(x, m);
        y = f_center(y, m);
    }
}
template <bool kBig>
__device__ __forceinline__ void gs_f(double &x, double &y, double2 w, const FpMod &m) {
    const double U = x, V = y;
    x = f_center(__dadd_rn(U, V), m);
    y = f_mulmod(__dsub_rn(U, V), w.x, w.y, m.q);
    if (kBig) y = f_center(y, m);
}

// ---------------------------------------------------------------- phases
// column phase, forward: stages 0..7 on columns [32 tile, 32 tile + 32);
// canonical u64 in, recentred doubles out (in place)
template <bool kBig>
__device__ __forceinline__ void fwd_cols(uint64_t *poly, int tile, const double2 *__restrict__ T, const FpMod &m,
                                         double *sm) {
    const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = tile * 32 + c;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = u2d(poly[(k + 16 * u) * 256 + col]);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int d = 8 >> s;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<kBig>(x[u], x[u + d], T[(1 << s) + (u >> (4 - s))], m);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[(k + 16 * u) * 32 + c] = x[u];
    __syncthreads();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = sm[(16 * k + v) * 32 + c];
#pragma unroll
    for (int s = 4; s < 8; ++s) {
        const int d = 128 >> s;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) ct_f<kBig>(x[v], x[v + d], T[(1 << s) + ((16 * k + v) >> (8 - s))], m);
    }
    double *pd = reinterpret_cast<double *>(poly);
#pragma unroll
    for (int v = 0; v < 16; ++v) pd[(16 * k + v) * 256 + col] = kBig ? x[v] : f_center(x[v], m);
}

// row phase, forward: stages 8..15 of row r (16 threads per row), canonical out
template <bool kBig>
__device__ __forceinline__ void fwd_row(uint64_t *row, int r, const double2 *__restrict__ T, const FpMod &m,
                                        double *srow) {
    const int k = threadIdx.x & 15;
    const double *rd = reinterpret_cast<const double *>(row);
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = __ldcg(rd + k + 16 * u);
#pragma unroll
    for (int sp = 0; sp < 4; ++sp) {
        const int d = 8 >> sp;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<kBig>(x[u], x[u + d], T[(256 << sp) + (r << sp) + (u >> (4 - sp))], m);
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
            if (!(v & d))
                ct_f<kBig>(x[v], x[v + d], T[(256 << sp) + (r << sp) + ((16 * k + v) >> (8 - sp))], m);
    }
    __syncwarp();
    uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
    for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 16; ++u) row[k + 16 * u] = su[pad16(k + 16 * u)];
}

// row phase, inverse: stages 15..8 of row r; canonical u64 in, centred doubles out
template <bool kBig>
__device__ __forceinline__ void inv_row(uint64_t *row, int r, const double2 *__restrict__ T, const FpMod &m,
                                        double *srow) {
    const int k = threadIdx.x & 15;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = u2d(row[k + 16 * u]);
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
    for (int sp = 7; sp >= 4; --sp) {
        const int d = 128 >> sp;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d))
                gs_f<kBig>(x[v], x[v + d], T[(256 << sp) + (r << sp) + ((16 * k + v) >> (8 - sp))], m);
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) srow[pad16(16 * k + v)] = x[v];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = srow[pad16(k + 16 * u)];
#pragma unroll
    for (int sp = 3; sp >= 0; --sp) {
        const int d = 8 >> sp;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) gs_f<kBig>(x[u], x[u + d], T[(256 << sp) + (r << sp) + (u >> (4 - sp))], m);
    }
    double *rd = reinterpret_cast<double *>(row);
#pragma unroll
    for (int u = 0; u < 16; ++u) rd[k + 16 * u] = kBig ? x[u] : f_center(x[u], m);
}

// column phase, inverse: stages 7..0, times N^-1, canonical out
template <bool kBig>
__device__ __forceinline__ void inv_cols(uint64_t *poly, int tile, const double2 *__restrict__ T, double2 ni,
                                         const FpMod &m, double *sm) {
    const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = tile * 32 + c;
    const double *pd = reinterpret_cast<const double *>(poly);
    double x[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = __ldcg(pd + (16 * k + v) * 256 + col);
#pragma unroll
    for (int s = 7; s >= 4; --s) {
        const int d = 128 >> s;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) gs_f<kBig>(x[v], x[v + d], T[(1 << s) + ((16 * k + v) >> (8 - s))], m);
    }
#pragma unroll
    for (int v = 0; v < 16; ++v) sm[(16 * k + v) * 32 + c] = x[v];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[(k + 16 * u) * 32 + c];
#pragma unroll
    for (int s = 3; s >= 0; --s) {
        const int d = 8 >> s;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) gs_f<kBig>(x[u], x[u + d], T[(1 << s) + (u >> (4 - s))], m);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u)
        poly[(k + 16 * u) * 256 + col] = d2canon(f_mulmod(x[u], ni.x, ni.y, m.q), m);
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- fused kernels
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 2)
    ntt16_fwd_fused(uint64_t *__restrict__ buf, int limb0, int B, const double2 *__restrict__ tw,
                    const FpMod *__restrict__ fm) {
    extern __shared__ double smd[];
    const int c = blockIdx.x & 7;
    const long long P = blockIdx.x >> 3;  // polynomial index = l * B + b
    const int mi = limb0 + (int)(P / B);
    const FpMod m = fm[mi];
    const double2 *T = tw + (size_t)mi * kN16;
    uint64_t *poly = buf + P * kN16;
    const int rs = threadIdx.x >> 4, r = c * 32 + rs;
    if (m.q < (double)kSmallPrime) {
        fwd_cols<false>(poly, c, T, m, smd);
        cluster_sync_all();
        fwd_row<false>(poly + r * 256, r, T, m, smd + rs * kRowPad);
    } else {
        fwd_cols<true>(poly, c, T, m, smd);
        cluster_sync_all();
        fwd_row<true>(poly + r * 256, r, T, m, smd + rs * kRowPad);
    }
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 2)
    ntt16_inv_fused(uint64_t *__restrict__ buf, int limb0, int B, const double2 *__restrict__ itw,
                    const double2 *__restrict__ ninv, const FpMod *__restrict__ fm) {
    extern __shared__ double smd[];
    const int c = blockIdx.x & 7;
    const long long P = blockIdx.x >> 3;
    const int mi = limb0 + (int)(P / B);
    const FpMod m = fm[mi];
    const double2 *T = itw + (size_t)mi * kN16;
    uint64_t *poly = buf + P * kN16;
    const int rs = threadIdx.x >> 4, r = c * 32 + rs;
    if (m.q < (double)kSmallPrime) {
        inv_row<false>(poly + r * 256, r, T, m, smd + rs * kRowPad);
        cluster_sync_all();
        inv_cols<false>(poly, c, T, ninv[mi], m, smd);
    } else {
        inv_row<true>(poly + r * 256, r, T, m, smd + rs * kRowPad);
        cluster_sync_all();
        inv_cols<true>(poly, c, T, ninv[mi], m, smd);
    }
}

// ---------------------------------------------------------------- generic N
__global__ void ntt_stage_fwd(uint64_t *__restrict__ buf, int limb0, int B, int log_n, int s,
                              const ulonglong2 *__restrict__ tw, const ModQ *__restrict__ mq, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int N = 1 << log_n, half = N >> 1;
    const long long poly_idx = gid / half;
    const int bi = (int)(gid - poly_idx * half);
    const int l = (int)(poly_idx / B), m = limb0 + l;
    const int t = N >> (s + 1);
    const int i = bi / t, j = 2 * i * t + (bi - i * t);
    uint64_t *a = buf + poly_idx * N;
    ct_bfly(a[j], a[j + t], tw[(size_t)m * N + (1 << s) + i], mq[m].q);
}

__global__ void ntt_stage_inv(uint64_t *__restrict__ buf, int limb0, int B, int log_n, int s,
                              const ulonglong2 *__restrict__ itw, const ModQ *__restrict__ mq, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int N = 1 << log_n, half = N >> 1;
    const long long poly_idx = gid / half;
    const int bi = (int)(gid - poly_idx * half);
    const int l = (int)(poly_idx / B), m = limb0 + l;
    const int t = N >> (s + 1);
    const int i = bi / t, j = 2 * i * t + (bi - i * t);
    uint64_t *a = buf + poly_idx * N;
    gs_bfly(a[j], a[j + t], itw[(size_t)m * N + (1 << s) + i], mq[m].q);
}

__global__ void scale_ninv(uint64_t *__restrict__ buf, int limb0, int B, int log_n, const ulonglong2 *__restrict__ ninv,
                           const ModQ *__restrict__ mq, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int m = limb0 + (int)(gid >> log_n) / B;
    const ulonglong2 ni = ninv[m];
    buf[gid] = mul_shoup(buf[gid], ni.x, ni.y, mq[m].q);
}

constexpr int kFusedSmem = 32 * kRowPad * 8;  // >= 256 * 32 * 8 for the column phase

void ntt16_set_attrs() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(ntt16_fwd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem);
    cudaFuncSetAttribute(ntt16_inv_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem);
    done = true;
}

}  // namespace

int ntt_fwd_launch(hk_ctx *c, uint64_t *buf, int limb0, int n_limbs, int B, int) {
    if (n_limbs <= 0 || B <= 0) return HK_OK;
    if (c->log_n == kLogN16) {
        ntt16_set_attrs();
        const unsigned blocks = 8u * (unsigned)n_limbs * (unsigned)B;
        ntt16_fwd_fused<<<blocks, 512, kFusedSmem, c->stream>>>(buf, limb0, B, (const double2 *)c->d_twf,
                                                                 (const FpMod *)c->d_fmod);
        ++c->launches;
    } else {
        const long long total = (long long)n_limbs * B * (c->n / 2);
        for (int s = 0; s < c->log_n; ++s) {
            ntt_stage_fwd<<<hk_grid(total, 256), 256, 0, c->stream>>>(buf, limb0, B, c->log_n, s, c->d_tw,
                                                                     c->d_modq, total);
            ++c->launches;
        }
    }
    HK_LAUNCH_CHECK(c, "ntt_fwd");
    return HK_OK;
}

int ntt_inv_launch(hk_ctx *c, uint64_t *buf, int limb0, int n_limbs, int B, int) {
    if (n_limbs <= 0 || B <= 0) return HK_OK;
    if (c->log_n == kLogN16) {
        ntt16_set_attrs();
        const unsigned blocks = 8u * (unsigned)n_limbs * (unsigned)B;
        ntt16_inv_fused<<<blocks, 512, kFusedSmem, c->stream>>>(buf, limb0, B, (const double2 *)c->d_itwf,
                                                                 (const double2 *)c->d_ninvf, (const FpMod *)c->d_fmod);
        ++c->launches;
    } else {
        const long long total = (long long)n_limbs * B * (c->n / 2);
        for (int s = c->log_n - 1; s >= 0; --s) {
            ntt_stage_inv<<<hk_grid(total, 256), 256, 0, c->stream>>>(buf, limb0, B, c->log_n, s, c->d_itw,
                                                                     c->d_modq, total);
            ++c->launches;
        }
        const long long all = (long long)n_limbs * B * c->n;
        scale_ninv<<<hk_grid(all, 256), 256, 0, c->stream>>>(buf, limb0, B, c->log_n, c->d_ninv, c->d_modq, all);
        ++c->launches;
    }
    HK_LAUNCH_CHECK(c, "ntt_inv");
    return HK_OK;
}

extern "C" int hk_ntt_fwd(hk_ctx *c, uint64_t *buf, int32_t limb0, int32_t nl, int32_t B) {
    if (limb0 < 0 || nl < 0 || limb0 + nl > c->n_mod || B < 0) return hk_fail(c, HK_E_ARG, "ntt: bad limb range");
    return ntt_fwd_launch(c, buf, limb0, nl, B, 0);
}

extern "C" int hk_ntt_inv(hk_ctx *c, uint64_t *buf, int32_t limb0, int32_t nl, int32_t B) {
    if (limb0 < 0 || nl < 0 || limb0 + nl > c->n_mod || B < 0) return hk_fail(c, HK_E_ARG, "intt: bad limb range");
    return ntt_inv_launch(c, buf, limb0, nl, B, 0);
}
