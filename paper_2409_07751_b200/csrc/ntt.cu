// ntt.cu — negacyclic NTT / inverse NTT over limb-major RNS buffers (sm_100a).
//
// Convention (identical to oracle/ckks_oracle.c ntt_fwd_1/ntt_inv_1): forward =
// Cooley-Tukey, natural-order coefficients -> bit-reversed evaluations, stage s
// (0..logN-1) pairs (j, j + N/2^(s+1)) with twiddle psi^brv(2^s + (j >> (logN-s)));
// inverse = Gentleman-Sande in reverse stage order with psi^-brv, then * N^-1.
//
// N = 2^16: the fused cluster kernels of ntt16.cuh (one 4-CTA cluster per
// polynomial, 256 x 256 split, intermediate in L2, FP64-pipe butterflies),
// here with plain in-place prologue/epilogue. N = 2^17: one radix-2 stage +
// twist pass, then the 2^16 kernels on both halves (below). Other N (parity
// tests at small sizes): one canonical integer launch per stage.
#include "ntt16.cuh"

namespace {

constexpr int kLogN16 = 16;

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

}  // namespace

int ntt_fwd_launch(hk_ctx *c, uint64_t *buf, int limb0, int n_limbs, int B, int) {
    if (n_limbs <= 0 || B <= 0) return HK_OK;
    if (ntt16::fused(c)) {
        return ntt16::launch_fwd(c, buf, limb0, n_limbs, B, ntt16::ProPlain{buf, c->log_n},
                                 ntt16::EpiPlain{buf, c->log_n});
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
    if (ntt16::fused(c)) {
        return ntt16::launch_inv(c, buf, limb0, n_limbs, B, ntt16::ProPlain{buf, c->log_n},
                                 ntt16::EpiPlain{buf, c->log_n});
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
