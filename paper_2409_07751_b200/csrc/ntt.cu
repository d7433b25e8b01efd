// ntt.cu — negacyclic NTT / inverse NTT over limb-major RNS buffers (sm_100a).
//
// Convention (identical to oracle/ckks_oracle.c ntt_fwd_1/ntt_inv_1): forward =
// Cooley-Tukey, natural-order coefficients -> bit-reversed evaluations, stage s
// (0..logN-1) pairs (j, j + N/2^(s+1)) with twiddle psi^brv(2^s + (j >> (logN-s)));
// inverse = Gentleman-Sande in reverse stage order with psi^-brv, then * N^-1.
//
// N = 2^16 fast path: the 16 stages split as 256 x 256.
//   stages 0..7  act along rows r of the 256x256 view j = 256 r + c  -> "column"
//                kernel: one CTA = 32 columns x 256 rows of one polynomial,
//                4 radix-2 stages in registers, one shared-memory transpose,
//                4 more stages in registers; all global accesses are 256 B
//                coalesced row segments.
//   stages 8..15 act within a row -> "row" kernel: one CTA = 32 rows, a
//                half-warp per row; the two exchanges stay inside a warp
//                (__syncwarp) through a bank-conflict-free padded tile.
// Other N (parity tests at small sizes): one launch per stage.
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
// Lazy (Harvey) butterflies for the 2^16 path; all primes are < 2^52.
// Forward: inputs < c q, outputs < (c + 2) q, no reductions at all; after the
// 16 stages values are < 33 q < 2^58 and get one Barrett reduction at the end.
__device__ __forceinline__ void ct_lazy(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q2) {
    const uint64_t T = y * w.x - __umul64hi(y, w.y) * (q2 >> 1);  // [0, 2q)
    const uint64_t U = x;
    x = U + T;
    y = U + q2 - T;
}
// Inverse: invariant [0, 2q): X' = U + V folded once, Y' = (U - V + 2q) w.
__device__ __forceinline__ void gs_lazy(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q2) {
    const uint64_t U = x, V = y;
    uint64_t s = U + V;
    x = s >= q2 ? s - q2 : s;
    const uint64_t d = U + q2 - V;
    y = d * w.x - __umul64hi(d, w.y) * (q2 >> 1);
}

// ---------------------------------------------------------------- forward
__global__ void __launch_bounds__(512, 2) ntt16_fwd_cols(uint64_t *__restrict__ buf, int limb0, int B,
                                                      const ulonglong2 *__restrict__ tw,
                                                      const ModQ *__restrict__ mq) {
    extern __shared__ uint64_t sm[];  // 256 x 32
    const int tile = blockIdx.x & 7, b = blockIdx.x >> 3, l = blockIdx.y, m = limb0 + l;
    const uint64_t q2 = 2 * mq[m].q;
    const ulonglong2 *T = tw + (size_t)m * kN16;
    uint64_t *poly = buf + ((size_t)l * B + b) * kN16;
    const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = tile * 32 + c;
    uint64_t x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = poly[(k + 16 * u) * 256 + col];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int d = 8 >> s;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_lazy(x[u], x[u + d], T[(1 << s) + (u >> (4 - s))], q2);
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
            if (!(v & d)) ct_lazy(x[v], x[v + d], T[(1 << s) + ((16 * k + v) >> (8 - s))], q2);
    }
#pragma unroll
    for (int v = 0; v < 16; ++v) poly[(16 * k + v) * 256 + col] = x[v];
}

__global__ void __launch_bounds__(512, 2) ntt16_fwd_rows(uint64_t *__restrict__ buf, int limb0, int B,
                                                      const ulonglong2 *__restrict__ tw,
                                                      const ModQ *__restrict__ mq) {
    extern __shared__ uint64_t sm[];  // 32 x kRowPad
    const int l = blockIdx.y, m = limb0 + l;
    const uint64_t q2 = 2 * mq[m].q;
    const ulonglong2 *T = tw + (size_t)m * kN16;
    const int k = threadIdx.x & 15, rs = threadIdx.x >> 4;
    const int job = blockIdx.x * 32 + rs;
    const int r = job / B, b = job - r * B;
    uint64_t *row = buf + ((size_t)l * B + b) * kN16 + r * 256;
    uint64_t *srow = sm + rs * kRowPad;
    uint64_t x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = row[k + 16 * u];
#pragma unroll
    for (int sp = 0; sp < 4; ++sp) {
        const int d = 8 >> sp;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_lazy(x[u], x[u + d], T[(256 << sp) + (r << sp) + (u >> (4 - sp))], q2);
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
                ct_lazy(x[v], x[v + d], T[(256 << sp) + (r << sp) + ((16 * k + v) >> (8 - sp))], q2);
    }
    const ModQ mm = mq[m];
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) srow[pad16(16 * k + v)] = reduce128(0, x[v], mm);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 16; ++u) row[k + 16 * u] = srow[pad16(k + 16 * u)];
}

// ---------------------------------------------------------------- inverse
__global__ void __launch_bounds__(512, 2) ntt16_inv_rows(uint64_t *__restrict__ buf, int limb0, int B,
                                                      const ulonglong2 *__restrict__ itw,
                                                      const ModQ *__restrict__ mq) {
    extern __shared__ uint64_t sm[];  // 32 x kRowPad
    const int l = blockIdx.y, m = limb0 + l;
    const uint64_t q2 = 2 * mq[m].q;
    const ulonglong2 *T = itw + (size_t)m * kN16;
    const int k = threadIdx.x & 15, rs = threadIdx.x >> 4;
    const int job = blockIdx.x * 32 + rs;
    const int r = job / B, b = job - r * B;
    uint64_t *row = buf + ((size_t)l * B + b) * kN16 + r * 256;
    uint64_t *srow = sm + rs * kRowPad;
    uint64_t x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = row[k + 16 * u];
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
    for (int sp = 7; sp >= 4; --sp) {
        const int d = 128 >> sp;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d))
                gs_lazy(x[v], x[v + d], T[(256 << sp) + (r << sp) + ((16 * k + v) >> (8 - sp))], q2);
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
            if (!(u & d)) gs_lazy(x[u], x[u + d], T[(256 << sp) + (r << sp) + (u >> (4 - sp))], q2);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) row[k + 16 * u] = x[u];
}

__global__ void __launch_bounds__(512, 2) ntt16_inv_cols(uint64_t *__restrict__ buf, int limb0, int B,
                                                      const ulonglong2 *__restrict__ itw,
                                                      const ulonglong2 *__restrict__ ninv,
                                                      const ModQ *__restrict__ mq) {
    extern __shared__ uint64_t sm[];  // 256 x 32
    const int tile = blockIdx.x & 7, b = blockIdx.x >> 3, l = blockIdx.y, m = limb0 + l;
    const uint64_t q2 = 2 * mq[m].q;
    const ulonglong2 *T = itw + (size_t)m * kN16;
    uint64_t *poly = buf + ((size_t)l * B + b) * kN16;
    const int c = threadIdx.x & 31, k = threadIdx.x >> 5, col = tile * 32 + c;
    uint64_t x[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = poly[(16 * k + v) * 256 + col];
#pragma unroll
    for (int s = 7; s >= 4; --s) {
        const int d = 128 >> s;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) gs_lazy(x[v], x[v + d], T[(1 << s) + ((16 * k + v) >> (8 - s))], q2);
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
            if (!(u & d)) gs_lazy(x[u], x[u + d], T[(1 << s) + (u >> (4 - s))], q2);
    }
    const ulonglong2 ni = ninv[m];
    const uint64_t q = q2 >> 1;
#pragma unroll
    for (int u = 0; u < 16; ++u) poly[(k + 16 * u) * 256 + col] = mul_shoup(x[u], ni.x, ni.y, q);
}

// ---------------------------------------------------------------- generic N
__global__ void ntt_stage_fwd(uint64_t *__restrict__ buf, int limb0, int B, int log_n, int s,
                              const ulonglong2 *__restrict__ tw, const ModQ *__restrict__ mq,
                              long long total) {
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
                              const ulonglong2 *__restrict__ itw, const ModQ *__restrict__ mq,
                              long long total) {
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

__global__ void scale_ninv(uint64_t *__restrict__ buf, int limb0, int B, int log_n,
                           const ulonglong2 *__restrict__ ninv, const ModQ *__restrict__ mq,
                           long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int m = limb0 + (int)(gid >> log_n) / B;
    const ulonglong2 ni = ninv[m];
    buf[gid] = mul_shoup(buf[gid], ni.x, ni.y, mq[m].q);
}

constexpr int kColSmem = 256 * 32 * 8;
constexpr int kRowSmem = 32 * kRowPad * 8;

void ntt16_set_attrs() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(ntt16_fwd_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmem);
    cudaFuncSetAttribute(ntt16_inv_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmem);
    cudaFuncSetAttribute(ntt16_fwd_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmem);
    cudaFuncSetAttribute(ntt16_inv_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmem);
    done = true;
}

}  // namespace

int ntt_fwd_launch(hk_ctx *c, uint64_t *buf, int limb0, int n_limbs, int B, int) {
    if (n_limbs <= 0 || B <= 0) return HK_OK;
    if (c->log_n == kLogN16) {
        ntt16_set_attrs();
        dim3 gc(8 * B, n_limbs), gr(8 * B, n_limbs);
        ntt16_fwd_cols<<<gc, 512, kColSmem, c->stream>>>(buf, limb0, B, c->d_tw, c->d_modq); ++c->launches;
        ntt16_fwd_rows<<<gr, 512, kRowSmem, c->stream>>>(buf, limb0, B, c->d_tw, c->d_modq); ++c->launches;
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
        dim3 gc(8 * B, n_limbs), gr(8 * B, n_limbs);
        ntt16_inv_rows<<<gr, 512, kRowSmem, c->stream>>>(buf, limb0, B, c->d_itw, c->d_modq); ++c->launches;
        ntt16_inv_cols<<<gc, 512, kColSmem, c->stream>>>(buf, limb0, B, c->d_itw, c->d_ninv, c->d_modq); ++c->launches;
    } else {
        const long long total = (long long)n_limbs * B * (c->n / 2);
        for (int s = c->log_n - 1; s >= 0; --s) {
            ntt_stage_inv<<<hk_grid(total, 256), 256, 0, c->stream>>>(buf, limb0, B, c->log_n, s, c->d_itw,
                                                                     c->d_modq, total);
            ++c->launches;
        }
        const long long all = (long long)n_limbs * B * c->n;
        scale_ninv<<<hk_grid(all, 256), 256, 0, c->stream>>>(buf, limb0, B, c->log_n, c->d_ninv, c->d_modq,
                                                              all); ++c->launches;
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
