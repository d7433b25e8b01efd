// ops.cu — slot-wise arithmetic, rescale, relinearised product, rotation.
//
// Each extern "C" entry replaces one branch of HeBackend.slotwise/rotate
// (hekan/backend.py:192-245); see include/hekan.h for the argument contract.
// Data layout: ct u64 [2][l+1][B][N] limb-major, NTT domain, canonical residues.
//
// Key switching is hybrid (Han-Ki): ModUp per digit of alpha primes (fast
// basis conversion + NTT), key inner product (128-bit lazy accumulation over
// digits, one Barrett reduction), ModDown by the special primes P.
#include <algorithm>
#include <cstring>

#include "ntt16.cuh"

int automorph_launch(hk_ctx *c, const uint64_t *in, uint64_t *out, uint32_t g, long long n_polys);

namespace {

constexpr int kMacMax = 192;    // operands per mac_plain launch (BSGS block: c4 80, c5 157)

struct Residues { uint64_t v[HK_MAX_MOD]; };
struct PtrList { const uint64_t *p[kMacMax]; };

__device__ __forceinline__ uint32_t auto_src(uint32_t j, uint32_t g, int log_n) {
    const uint32_t M = 2u << log_n;
    const uint32_t e = 2u * brev_bits(j, log_n) + 1u;
    const uint32_t eg = (uint32_t)(((uint64_t)e * g) & (M - 1));
    return brev_bits((eg - 1u) >> 1, log_n);
}

// All element kernels use grid (ceil(B*N / 256), limbs, polys): blockIdx.y is
// the limb, blockIdx.z the polynomial, x runs over the B*N coefficients of one
// limb (no 64-bit divisions in index math).
#define ELEM_INDEX                                                               \
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;       \
    if (e >= BN) return;                                                         \
    const int l = blockIdx.y, p = blockIdx.z;

// ------------------------------------------------------------ add / sub
__global__ void k_addsub(const uint64_t *__restrict__ a, int la, const uint64_t *__restrict__ b, int lb,
                         uint64_t *__restrict__ out, int lo, long long BN, int neg, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const uint64_t q = mq[l].q;
    const uint64_t x = a[((long long)p * (la + 1) + l) * BN + e];
    const uint64_t y = b[((long long)p * (lb + 1) + l) * BN + e];
    out[((long long)p * (lo + 1) + l) * BN + e] = neg ? sub_mod(x, y, q) : add_mod(x, y, q);
}

// same, four elements per thread as two 16-byte accesses (BN % 1024 == 0): the scalar
// kernel reaches 4.4 TB/s of DRAM traffic on 37 x 128 limbs, this one see profiles/r2_notes.md §9
__global__ void __launch_bounds__(256) k_addsub4(const ulonglong2 *__restrict__ a, int la,
                                                 const ulonglong2 *__restrict__ b, int lb,
                                                 ulonglong2 *__restrict__ out, int lo, long long BN2, int neg,
                                                 const ModQ *__restrict__ mq) {
    const long long e = (long long)blockIdx.x * 512 + threadIdx.x;  // in 16-byte units
    const int l = blockIdx.y, p = blockIdx.z;
    const uint64_t q = mq[l].q;
    const ulonglong2 *pa = a + ((long long)p * (la + 1) + l) * BN2 + e;
    const ulonglong2 *pb = b + ((long long)p * (lb + 1) + l) * BN2 + e;
    ulonglong2 *po = out + ((long long)p * (lo + 1) + l) * BN2 + e;
    const ulonglong2 x0 = pa[0], x1 = pa[256], y0 = pb[0], y1 = pb[256];
    ulonglong2 r0, r1;
    r0.x = neg ? sub_mod(x0.x, y0.x, q) : add_mod(x0.x, y0.x, q);
    r0.y = neg ? sub_mod(x0.y, y0.y, q) : add_mod(x0.y, y0.y, q);
    r1.x = neg ? sub_mod(x1.x, y1.x, q) : add_mod(x1.x, y1.x, q);
    r1.y = neg ? sub_mod(x1.y, y1.y, q) : add_mod(x1.y, y1.y, q);
    po[0] = r0;
    po[256] = r1;
}

// c0 +/- pt (pt_batch 1 or B), c1 copied
__global__ void k_add_plain(const uint64_t *__restrict__ a, int la, const uint64_t *__restrict__ pt, int pb,
                            int neg, uint64_t *__restrict__ out, long long BN, int log_n,
                            const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const long long o = ((long long)p * (la + 1) + l) * BN + e;
    if (p == 1) { out[o] = a[o]; return; }
    const int N = 1 << log_n;
    const long long b = e >> log_n;
    const uint64_t y = pt[((long long)l * pb + (pb == 1 ? 0 : b)) * N + (e & (N - 1))];
    const uint64_t q = mq[l].q;
    out[o] = neg ? sub_mod(a[o], y, q) : add_mod(a[o], y, q);
}

__global__ void k_add_const(const uint64_t *__restrict__ a, int la, Residues r, uint64_t *__restrict__ out,
                            long long BN, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const long long o = ((long long)p * (la + 1) + l) * BN + e;
    out[o] = p == 1 ? a[o] : add_mod(a[o], r.v[l], mq[l].q);
}

// add_plain / add_const with 16-byte accesses, four elements per thread (BN % 1024 == 0;
// grid (BN / 1024, limbs, 2)), as k_addsub4
__global__ void __launch_bounds__(256) k_add_plain4(const ulonglong2 *__restrict__ a, int la,
                                                    const ulonglong2 *__restrict__ pt, int pb, int neg,
                                                    ulonglong2 *__restrict__ out, long long BN2, int log_n,
                                                    const ModQ *__restrict__ mq) {
    const long long e = (long long)blockIdx.x * 512 + threadIdx.x;  // in 16-byte units
    const int l = blockIdx.y, p = blockIdx.z;
    const long long o = ((long long)p * (la + 1) + l) * BN2 + e;
    const ulonglong2 x0 = a[o], x1 = a[o + 256];
    if (p == 1) {
        out[o] = x0;
        out[o + 256] = x1;
        return;
    }
    const int N2 = 1 << (log_n - 1);
    const long long e1 = e + 256;
    const ulonglong2 y0 = pt[((long long)l * pb + (pb == 1 ? 0 : e >> (log_n - 1))) * N2 + (e & (N2 - 1))];
    const ulonglong2 y1 = pt[((long long)l * pb + (pb == 1 ? 0 : e1 >> (log_n - 1))) * N2 + (e1 & (N2 - 1))];
    const uint64_t q = mq[l].q;
    ulonglong2 r0, r1;
    r0.x = neg ? sub_mod(x0.x, y0.x, q) : add_mod(x0.x, y0.x, q);
    r0.y = neg ? sub_mod(x0.y, y0.y, q) : add_mod(x0.y, y0.y, q);
    r1.x = neg ? sub_mod(x1.x, y1.x, q) : add_mod(x1.x, y1.x, q);
    r1.y = neg ? sub_mod(x1.y, y1.y, q) : add_mod(x1.y, y1.y, q);
    out[o] = r0;
    out[o + 256] = r1;
}
__global__ void __launch_bounds__(256) k_add_const4(const ulonglong2 *__restrict__ a, int la, Residues r,
                                                    ulonglong2 *__restrict__ out, long long BN2,
                                                    const ModQ *__restrict__ mq) {
    const long long e = (long long)blockIdx.x * 512 + threadIdx.x;
    const int l = blockIdx.y, p = blockIdx.z;
    const long long o = ((long long)p * (la + 1) + l) * BN2 + e;
    ulonglong2 x0 = a[o], x1 = a[o + 256];
    if (p == 0) {
        const uint64_t c = r.v[l], q = mq[l].q;
        x0.x = add_mod(x0.x, c, q);
        x0.y = add_mod(x0.y, c, q);
        x1.x = add_mod(x1.x, c, q);
        x1.y = add_mod(x1.y, c, q);
    }
    out[o] = x0;
    out[o + 256] = x1;
}

// tmp = a (.) pt for both polys (limbs 0..la)
__global__ void k_mul_plain(const uint64_t *__restrict__ a, int la, const uint64_t *__restrict__ pt, int pb,
                            uint64_t *__restrict__ out, long long BN, int log_n, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const int N = 1 << log_n;
    const long long b = e >> log_n;
    const long long o = ((long long)p * (la + 1) + l) * BN + e;
    const uint64_t y = pt[((long long)l * pb + (pb == 1 ? 0 : b)) * N + (e & (N - 1))];
    out[o] = mul_mod(a[o], y, mq[l]);
}

__global__ void k_mul_const(const uint64_t *__restrict__ a, int la, Residues r, uint64_t *__restrict__ out,
                            long long BN, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const long long o = ((long long)p * (la + 1) + l) * BN + e;
    out[o] = mul_mod(a[o], r.v[l], mq[l]);
}

// out = sum_i babies[i] (.) pts[i], both polys; `init` adds the previous out
__global__ void k_mac(PtrList babies, PtrList pts, int n, int la, int ps, uint64_t *__restrict__ out, long long BN,
                      int log_n, int init, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const int N = 1 << log_n;
    const long long o = ((long long)p * (la + 1) + l) * BN + e;
    const long long pe = (long long)l * ps * N + (e & (N - 1));
    Acc3 acc;
    acc3_zero(acc);
    if (init) acc.s0 = out[o];
    for (int i = 0; i < n; ++i) acc3_mac(acc, babies.p[i][o], pts.p[i][pe]);
    out[o] = acc3_reduce(acc, mq[l]);
}

// G consecutive BSGS giant-step blocks at once (hk_mac_plain_blocks): every baby
// value is read ONCE for the group instead of once per block.
//   acc_g[p][l][b][k] = sum_{i < cnt_g} babies[i][p][l][b][k] * pt[l][g*nb + i][k]   (mod q_l)
// CTA = 16 coefficients x 16 (poly, sample) lanes of one limb; the group's plaintext
// tile [G][n][16] is staged in shared memory as 25-bit halves; Karatsuba split MACs
// into 3-word accumulators, one Barrett reduction per output.
constexpr int kBlkK = 16;
template <int G>
__global__ void __launch_bounds__(256) k_mac_blocks(PtrList babies, int n, int nb, int4 cnt_lo, int4 cnt_hi,
                                                   const uint64_t *__restrict__ pt, int pt_count, int la,
                                                   uint64_t *__restrict__ acc, long long BN, int B, int log_n,
                                                   const ModQ *__restrict__ mq) {
    extern __shared__ uint2 shp[];  // [G][n][kBlkK] (y0, y1)
    const int N = 1 << log_n, l = blockIdx.y;
    const int k0 = blockIdx.x * kBlkK;
    const int cnt[8] = {cnt_lo.x, cnt_lo.y, cnt_lo.z, cnt_lo.w, cnt_hi.x, cnt_hi.y, cnt_hi.z, cnt_hi.w};
    // stage the tile with 8 independent loads in flight per thread
    const int tile = G * n * kBlkK;
    for (int t0 = threadIdx.x; t0 < tile; t0 += 8 * blockDim.x) {
        uint64_t y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int t = t0 + u * blockDim.x;
            y[u] = 0;
            if (t < tile) {
                const int kk = t % kBlkK, gi = t / kBlkK, g = gi / n, i = gi - g * n;
                if (i < cnt[g]) y[u] = __ldg(pt + ((long long)l * pt_count + g * nb + i) * N + k0 + kk);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int t = t0 + u * blockDim.x;
            if (t < tile) shp[t] = make_uint2((uint32_t)y[u] & HK_M25, (uint32_t)(y[u] >> 25));
        }
    }
    __syncthreads();
    const int kk = threadIdx.x % kBlkK, lane = threadIdx.x / kBlkK;
    const ModQ m = mq[l];
    const size_t gstride = (size_t)2 * (la + 1) * BN;
    for (int pb = lane; pb < 2 * B; pb += 256 / kBlkK) {
        const int p = pb >= B ? 1 : 0, b = pb - p * B;
        const long long o = ((long long)p * (la + 1) + l) * BN + (long long)b * N + k0 + kk;
        uint64_t a0[G], a2[G], am[G];
#pragma unroll
        for (int g = 0; g < G; ++g) a0[g] = a2[g] = am[g] = 0;
        constexpr int U = G <= 4 ? 16 : 8;  // babies' loads in flight (registers permitting)
        int i = 0;
        for (; i + U <= n; i += U) {
            uint64_t xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = babies.p[i + u][o];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                uint32_t x0, x1;
                split25(xv[u], x0, x1);
                const uint32_t xs = x0 + x1;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint2 y = shp[(g * n + i + u) * kBlkK + kk];
                    a0[g] = mad_wide(x0, y.x, a0[g]);
                    a2[g] = mad_wide(x1, y.y, a2[g]);
                    am[g] = mad_wide(xs, y.x + y.y, am[g]);
                }
            }
        }
        for (; i < n; ++i) {
            uint32_t x0, x1;
            split25(babies.p[i][o], x0, x1);
            const uint32_t xs = x0 + x1;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const uint2 y = shp[(g * n + i) * kBlkK + kk];
                a0[g] = mad_wide(x0, y.x, a0[g]);
                a2[g] = mad_wide(x1, y.y, a2[g]);
                am[g] = mad_wide(xs, y.x + y.y, am[g]);
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const Acc3 A{a0[g], am[g] - a0[g] - a2[g], a2[g]};
            acc[g * gstride + o] = acc3_reduce(A, m);
        }
    }
}

// ------------------------------------------------------------ rescale
// R[i][pb][k] = centered(L[pb][k] mod q_l) mod q_i, i < l ; grid (BN2 / 256, l)
__global__ void k_rs_center(const uint64_t *__restrict__ L, uint64_t *__restrict__ R, int l, long long BN2,
                            const ModQ *__restrict__ mq) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= BN2) return;
    const int i = blockIdx.y;
    const uint64_t ql = mq[l].q, x = L[e];
    const bool neg = x > (ql >> 1);
    const uint64_t mag = neg ? ql - x : x;
    const ModQ m = mq[i];
    const uint64_t r = reduce128(0, mag, m);
    R[(long long)i * BN2 + e] = neg ? (r ? m.q - r : 0) : r;
}

// out[p][i] = (in[p][i] - R[i][p]) * q_l^-1 ; grid (BN / 256, l, 2)
__global__ void k_rs_finish(const uint64_t *__restrict__ in, const uint64_t *__restrict__ R,
                            uint64_t *__restrict__ out, int lvl, long long BN, const ulonglong2 *__restrict__ qinv,
                            const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const uint64_t q = mq[l].q;
    const ulonglong2 w = qinv[l];
    const uint64_t x = in[((long long)p * (lvl + 1) + l) * BN + e];
    const uint64_t y = R[(long long)l * 2 * BN + (long long)p * BN + e];
    out[((long long)p * lvl + l) * BN + e] = mul_shoup(sub_mod(x, y, q), w.x, w.y, q);
}

// ------------------------------------------------------------ tensor product ; grid (BN/256, l+1)
__global__ void k_tensor(const uint64_t *__restrict__ a, int la, const uint64_t *__restrict__ b, int lb, int lt,
                         uint64_t *__restrict__ d, long long BN, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    (void)p;
    const ModQ m = mq[l];
    const long long o = (long long)l * BN + e;
    const uint64_t a0 = a[o], a1 = a[(long long)(la + 1) * BN + o];
    const uint64_t b0 = b[o], b1 = b[(long long)(lb + 1) * BN + o];
    const long long pl = (long long)(lt + 1) * BN;
    d[o] = mul_mod(a0, b0, m);
    uint64_t hi = 0, lo = 0;
    mac128(hi, lo, a0, b1);
    mac128(hi, lo, a1, b0);
    d[pl + o] = reduce128(hi, lo, m);
    d[2 * pl + o] = mul_mod(a1, b1, m);
}

// d += tensor(a, b) (generic-ring path of hk_mul2)
__global__ void k_tensor_add(const uint64_t *__restrict__ a, int la, const uint64_t *__restrict__ b, int lb, int lt,
                             uint64_t *__restrict__ d, long long BN, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    (void)p;
    const ModQ m = mq[l];
    const long long o = (long long)l * BN + e;
    const uint64_t a0 = a[o], a1 = a[(long long)(la + 1) * BN + o];
    const uint64_t b0 = b[o], b1 = b[(long long)(lb + 1) * BN + o];
    const long long pl = (long long)(lt + 1) * BN;
    d[o] = add_mod(d[o], mul_mod(a0, b0, m), m.q);
    uint64_t hi = 0, lo = 0;
    mac128(hi, lo, a0, b1);
    mac128(hi, lo, a1, b0);
    d[pl + o] = add_mod(d[pl + o], reduce128(hi, lo, m), m.q);
    d[2 * pl + o] = add_mod(d[2 * pl + o], mul_mod(a1, b1, m), m.q);
}

// ------------------------------------------------------------ key switching
// Fast basis conversion: dst[t] = sum_i [src_i * inv_i]_{q_i} * hat[t][i] mod q_t.
// The source residues of one coefficient stay in registers (NS >= n_src), the
// hat matrix and target moduli sit in shared memory (broadcast reads).
// mode 0 (ModUp): dst limb of chain prime m = (m <= l ? m : l + 1 + m - n_q)
// mode 1 (ModDown): dst limb = target position d
template <int NS>
__global__ void __launch_bounds__(128) k_conv(const uint64_t *__restrict__ src, int n_src,
                                              const uint64_t *__restrict__ inv, const uint64_t *__restrict__ inv_sh,
                                              const uint64_t *__restrict__ hat, const int32_t *__restrict__ src_mod,
                                              const int32_t *__restrict__ dst_mod, int n_dst,
                                              uint64_t *__restrict__ dst, int mode, int l, int n_q, long long BN,
                                              const ModQ *__restrict__ mq, int prescaled,
                                              const double *__restrict__ src_invd,
                                              const uint64_t *__restrict__ neg_m) {
    // NS == n_src exactly (one instantiation per source count): no guards
    // hat [n_dst][kHs] as 25-bit halves and their sum (h0, h1, h0 + h1) per source, ModQ [n_dst], out index [n_dst]
    constexpr int kHs = (3 * NS + 3) & ~3;  // words per target, 16-byte aligned rows
    extern __shared__ uint4 sh4[];
    uint32_t *sh = reinterpret_cast<uint32_t *>(sh4);
    ModQ *smq = (ModQ *)(sh + n_dst * kHs);
    int *sidx = (int *)(smq + n_dst);
    for (int i = threadIdx.x; i < n_dst * NS; i += blockDim.x) {
        const uint64_t h = hat[i];
        const uint32_t h0 = (uint32_t)h & HK_M25, h1 = (uint32_t)(h >> 25);
        uint32_t *w = sh + (i / NS) * kHs + 3 * (i % NS);
        w[0] = h0;
        w[1] = h1;
        w[2] = h0 + h1;
    }
    for (int d = threadIdx.x; d < n_dst; d += blockDim.x) {
        const int m = dst_mod[d];
        smq[d] = mq[m];
        sidx[d] = mode == 0 ? (m <= l ? m : l + 1 + m - n_q) : d;
    }
    __syncthreads();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= BN) return;
    {
    // Karatsuba split MAC: s0 = sum x0 y0, s2 = sum x1 y1, sm = sum (x0+x1)(y0+y1),
    // s1 = sm - s0 - s2 (once per target): three IMAD.WIDE per multiply-add.
    uint32_t v0[NS], v1[NS], vs[NS];
    double frac = 0.0;  // sum_i v_i / m_i (exact mode), fixed order, no contraction
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const uint64_t x = src[(long long)i * BN + e];
        const uint64_t v = prescaled ? x : mul_shoup(x, inv[i], inv_sh[i], mq[src_mod[i]].q);
        if (neg_m) frac = __dadd_rn(frac, __dmul_rn(ntt16::u2d(v), src_invd[i]));
        split25(v, v0[i], v1[i]);
        vs[i] = v0[i] + v1[i];
    }
    // centred remainder: subtract u * M with u = round(frac) (u <= NS)
    const uint64_t u = neg_m ? (uint64_t)floor(__dadd_rn(frac, 0.5)) : 0;
    int d = 0;
    for (; d + 1 < n_dst; d += 2) {  // two targets in flight
        const uint32_t *h0 = sh + d * kHs;
        const uint32_t *h1 = h0 + kHs;
        uint64_t a0 = 0, a2 = 0, am = 0, b0 = 0, b2 = 0, bm = 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            a0 = mad_wide(v0[i], h0[3 * i], a0);
            a2 = mad_wide(v1[i], h0[3 * i + 1], a2);
            am = mad_wide(vs[i], h0[3 * i + 2], am);
            b0 = mad_wide(v0[i], h1[3 * i], b0);
            b2 = mad_wide(v1[i], h1[3 * i + 1], b2);
            bm = mad_wide(vs[i], h1[3 * i + 2], bm);
        }
        Acc3 A{a0, am - a0 - a2, a2}, Bc{b0, bm - b0 - b2, b2};
        if (neg_m) {
            A.s0 += u * __ldg(neg_m + d);
            Bc.s0 += u * __ldg(neg_m + d + 1);
        }
        dst[(long long)sidx[d] * BN + e] = acc3_reduce(A, smq[d]);
        dst[(long long)sidx[d + 1] * BN + e] = acc3_reduce(Bc, smq[d + 1]);
    }
    if (d < n_dst) {
        const uint32_t *h0 = sh + d * kHs;
        uint64_t a0 = 0, a2 = 0, am = 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            a0 = mad_wide(v0[i], h0[3 * i], a0);
            a2 = mad_wide(v1[i], h0[3 * i + 1], a2);
            am = mad_wide(vs[i], h0[3 * i + 2], am);
        }
        Acc3 A{a0, am - a0 - a2, a2};
        if (neg_m) A.s0 += u * __ldg(neg_m + d);
        dst[(long long)sidx[d] * BN + e] = acc3_reduce(A, smq[d]);
    }
    }
}

// Relinearisation fold: the merged ModDown + rescale divides Y_p = acc_p + P d_p
// by P q_l, so the key inner product writes Y_p directly for the q limbs
// (t <= l): d_p is formed here from the operands (d0 = a0 b0, d1 = a0 b1 +
// a1 b0, plus a second product for hk_mul2 and k x_p for hk_mul_lin) on the
// FP64 pipe, in a streaming kernel whose loads are all in flight together,
// instead of inside the ModDown NTT's epilogue (where they were latency bound
// at 2.3x the time of a plain NTT, profiles/r2_notes.md).
struct FoldD {
    const uint64_t *a, *b, *a2, *b2, *x;  // x: linear term (optional), a2 / b2: second product (optional)
    long long pa, pb, pa2, pb2, px;       // offsets of poly 1
    const ulonglong2 *pmod;               // [n_q] P mod q (Shoup pair; .x used)
    Residues k;                           // linear-term constant per limb
};
__device__ __forceinline__ double fold_prod(const uint64_t *a, const uint64_t *b, long long oa, long long ob,
                                            const ntt16::FpMod &M) {
    using namespace ntt16;
    const double y = u2d(b[ob]);
    return f_mulmod(u2d(a[oa]), y, __dmul_rn(y, M.qinv), M.q);
}

// acc_p[t] = sum_j sigma_g(ext_j[t]) * key_j[p][chain(t)] ; grid (BN/256, ne)
// acc_p[t] = sum_j sigma_g(ext_j[t]) * key_j,p[t]  (p = 0, 1) on the FP64 pipe:
// exact two-product Shoup (ntt16::f_mulmod) with w/q formed once per thread;
// each thread owns one (coefficient k, limb t) and walks `bb` batch entries so
// the key pair, the galois index and the address math are paid once.
// grid (N/min(N,256) * B/bb, ne); every residue is exact, results canonical.
template <int ND, bool FOLD, bool kBig>
__device__ __forceinline__ void key_ip_body(const uint64_t *__restrict__ ext, const uint64_t *__restrict__ d,
                                            const uint64_t *__restrict__ dm, int alpha, int ne, int l, int n_q,
                                            int nm, int ksp0, int log_n, int bb, const uint64_t *__restrict__ key,
                                            uint32_t g, uint64_t *__restrict__ acc0, uint64_t *__restrict__ acc1,
                                            const double2 *__restrict__ fmod, long long BN, int accum,
                                            const FoldD &fd) {
    using namespace ntt16;
    const int N = 1 << log_n;
    const int kblocks = N / (int)blockDim.x;
    const int k = (blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
    const int b0 = (blockIdx.x / kblocks) * bb;
    const int t = blockIdx.y;
    const int m = t <= l ? t : n_q + (t - l - 1);
    const int kr = t <= l ? t : ksp0 + (t - l - 1);  // key row: nm rows, specials from ksp0
    const double2 fm = fmod[m];
    const FpMod M{fm.x, fm.y};
    // Small primes (q < 2^47, every prime but q_0) never recentre: each product is below
    // 0.75 q and at most 8 + 5 of them add up, far inside the 2^51 > 16 q that keeps
    // f_mulmod and d2canon exact; the large prime keeps the centring steps.
    auto cen = [&](double v) { return kBig ? f_center(v, M) : v; };
    const int ks = g == 1u ? k : (int)auto_src((uint32_t)k, g, log_n);
    double w0[ND], v0[ND], w1[ND], v1[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) {
        const uint64_t *kj = key + ((size_t)j * 2 * nm + kr) * N;
        w0[j] = u2d(kj[k]);
        w1[j] = u2d(kj[(size_t)nm * N + k]);
        v0[j] = __dmul_rn(w0[j], M.qinv);
        v1[j] = __dmul_rn(w1[j], M.qinv);
    }
    const int own_j = t <= l ? t / alpha : -1;  // digit whose own limb t is: NTT form of d itself
    const long long row = (long long)b0 * N;
    const uint64_t *xe = ext + (long long)t * BN + row + ks;
    const long long dstride = (long long)ne * BN;
    const uint64_t *xd = d + (long long)t * BN + row + ks;
    const uint64_t *xm = dm ? dm + (long long)t * BN + row + ks : nullptr;
    uint64_t *o0 = acc0 + (long long)t * BN + row + k;
    uint64_t *o1 = acc1 + (long long)t * BN + row + k;
    const bool fold = FOLD && t <= l;
    // two samples per step: every load of both is issued before the arithmetic of the
    // first (the operand pointers of the fold are not restrict-qualified, so the compiler
    // would not hoist them above the previous sample's stores): 6.18 -> see profiles/r2_notes.md §9
    for (int b = 0; b < bb; b += 2) {
        const int nu = min(2, bb - b);
        uint64_t rx[2][ND], ry[2] = {0, 0}, rm[2] = {0, 0}, rs0[2] = {0, 0}, rs1[2] = {0, 0};
        uint64_t fa0[2] = {0, 0}, fa1[2] = {0, 0}, fb0[2] = {0, 0}, fb1[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (u < nu) {
#pragma unroll
                for (int j = 0; j < ND; ++j) rx[u][j] = j == own_j ? 0 : xe[u * N + j * dstride];
                if (own_j >= 0) {
                    ry[u] = xd[u * N];
                    if (xm) rm[u] = xm[u * N];
                }
                if (accum) {
                    rs0[u] = o0[u * N];
                    rs1[u] = o1[u * N];
                }
                if (fold) {  // g = 1: ks = k
                    const long long o = (long long)t * BN + row + (long long)(b + u) * N + k;
                    fa0[u] = fd.a[o];
                    fa1[u] = fd.a[fd.pa + o];
                    fb0[u] = fd.b[o];
                    fb1[u] = fd.b[fd.pb + o];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (u < nu) {
                double x[ND];
#pragma unroll
                for (int j = 0; j < ND; ++j) x[j] = u2d(rx[u][j]);
                if (own_j >= 0) {
                    double y = u2d(ry[u]);
                    if (xm) {  // relinearisation: d = a1 (.) b1 on the fly
                        const double w = u2d(rm[u]);
                        y = cen(f_mulmod(y, w, __dmul_rn(w, M.qinv), M.q));
                    }
#pragma unroll
                    for (int j = 0; j < ND; ++j)
                        if (j == own_j) x[j] = y;
                }
                // accum: add onto the running sum of earlier key switches (hk_rotate_sum)
                double s0 = accum ? u2d(rs0[u]) : 0.0, s1 = accum ? u2d(rs1[u]) : 0.0;
                if (fold) {  // Y_p = acc_p + P d_p
                    const long long o = (long long)t * BN + row + (long long)(b + u) * N + k;
                    const double a0 = u2d(fa0[u]), a1 = u2d(fa1[u]), b0 = u2d(fb0[u]), b1 = u2d(fb1[u]);
                    const double b0q = __dmul_rn(b0, M.qinv), b1q = __dmul_rn(b1, M.qinv);
                    double d0 = f_mulmod(a0, b0, b0q, M.q);
                    double d1 = __dadd_rn(f_mulmod(a0, b1, b1q, M.q), f_mulmod(a1, b0, b0q, M.q));
                    if (fd.a2) {
                        d0 = __dadd_rn(d0, fold_prod(fd.a2, fd.b2, o, o, M));
                        d1 = cen(d1);
                        d1 = __dadd_rn(d1, __dadd_rn(fold_prod(fd.a2, fd.b2, o, fd.pb2 + o, M),
                                                     fold_prod(fd.a2, fd.b2, fd.pa2 + o, o, M)));
                    }
                    if (fd.x) {
                        const double kk = u2d(fd.k.v[t]), kq = __dmul_rn(kk, M.qinv);
                        d0 = __dadd_rn(cen(d0), f_mulmod(u2d(fd.x[o]), kk, kq, M.q));
                        d1 = __dadd_rn(cen(d1), f_mulmod(u2d(fd.x[fd.px + o]), kk, kq, M.q));
                    }
                    const double pm = u2d(fd.pmod[t].x), pq = __dmul_rn(pm, M.qinv);
                    s0 = cen(__dadd_rn(s0, f_mulmod(cen(d0), pm, pq, M.q)));
                    s1 = cen(__dadd_rn(s1, f_mulmod(cen(d1), pm, pq, M.q)));
                }
#pragma unroll
                for (int j = 0; j < ND; ++j) {  // |f_mulmod| < 2.5 q: recentre every second term
                    s0 = __dadd_rn(s0, f_mulmod(x[j], w0[j], v0[j], M.q));
                    s1 = __dadd_rn(s1, f_mulmod(x[j], w1[j], v1[j], M.q));
                    if (j & 1) {
                        s0 = cen(s0);
                        s1 = cen(s1);
                    }
                }
                o0[u * N] = d2canon(s0, M);
                o1[u * N] = d2canon(s1, M);
            }
        }
        xe += 2 * N;
        xd += 2 * N;
        if (xm) xm += 2 * N;
        o0 += 2 * N;
        o1 += 2 * N;
    }
}

template <int ND, bool FOLD>
__global__ void __launch_bounds__(256, 3) k_key_ip(const uint64_t *__restrict__ ext, const uint64_t *__restrict__ d,
                                                const uint64_t *__restrict__ dm, int alpha, int ne, int l, int n_q,
                                                int nm, int ksp0, int log_n, int bb, const uint64_t *__restrict__ key,
                                                uint32_t g, uint64_t *__restrict__ acc0, uint64_t *__restrict__ acc1,
                                                const double2 *__restrict__ fmod, long long BN, int accum, FoldD fd) {
    const int t = blockIdx.y;
    if (fmod[t <= l ? t : n_q + (t - l - 1)].x < (double)ntt16::kSmallPrime)
        key_ip_body<ND, FOLD, false>(ext, d, dm, alpha, ne, l, n_q, nm, ksp0, log_n, bb, key, g, acc0, acc1, fmod, BN,
                                     accum, fd);
    else
        key_ip_body<ND, FOLD, true>(ext, d, dm, alpha, ne, l, n_q, nm, ksp0, log_n, bb, key, g, acc0, acc1, fmod, BN,
                                    accum, fd);
}

// out (+)= sigma_g(in) over [l+1][B][N] ; grid (BN/256, l+1)
__global__ void k_auto_acc(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, uint32_t g, int log_n,
                           long long BN, int init, const ModQ *__restrict__ mq) {
    ELEM_INDEX
    (void)p;
    const long long o = (long long)l * BN + e;
    long long src = o;
    if (g != 1u) {
        const int k = (int)(e & ((1 << log_n) - 1));
        src = o - k + auto_src((uint32_t)k, g, log_n);
    }
    const uint64_t v = in[src];
    out[o] = init ? v : add_mod(out[o], v, mq[l].q);
}

// out_i = (acc_i - conv_i) * P^-1 (+ optional addend, optionally automorphed) ; grid (BN/256, l+1)
__global__ void k_md_finish(const uint64_t *__restrict__ acc, const uint64_t *__restrict__ conv,
                            uint64_t *__restrict__ out, const uint64_t *__restrict__ addend, uint32_t g,
                            int log_n, long long BN, const ulonglong2 *__restrict__ pinv,
                            const ModQ *__restrict__ mq) {
    ELEM_INDEX
    (void)p;
    const uint64_t q = mq[l].q;
    const ulonglong2 w = pinv[l];
    const long long o = (long long)l * BN + e;
    uint64_t r = mul_shoup(sub_mod(acc[o], conv[o], q), w.x, w.y, q);
    if (addend) {
        long long src = o;
        if (g != 1u) {
            const int N = 1 << log_n;
            const int k = (int)(e & (N - 1));
            src = o - k + auto_src((uint32_t)k, g, log_n);
        }
        r = add_mod(r, addend[src], q);
    }
    out[o] = r;
}


// ---------------------------------------------------------------------------
// N = 2^16 fused flows: prologue/epilogue functors for ntt16::launch_fwd/inv
// ---------------------------------------------------------------------------
enum { SRC_PLAIN = 0, SRC_MULPT = 1, SRC_MULCONST = 2, SRC_MAC = 3, SRC_SUM2 = 4 };

// Value X(p, l, b, idx) of the ciphertext about to be rescaled, produced on
// the fly: a, a (.) pt, a * k, sum_i babies_i (.) pts_i, or a + a2.
template <int KIND>
struct RsSrc {
    const uint64_t *a;
    const uint64_t *a2;
    const uint64_t *pt;
    int la, pb, n, log_n;
    int ps;  // plaintext limb stride in units of N (SRC_MAC)
    long long BN;
    const ModQ *mq;
    const double2 *fmod;  // {q, 1/q} per prime
    Residues k, ksh;    // constant residues and Shoup companions (SRC_MULCONST)
    PtrList babies, pts;
    __device__ __forceinline__ uint64_t operator()(int p, int l, int b, int idx) const {
        const long long o = ((long long)p * (la + 1) + l) * BN + ((long long)b << log_n) + idx;
        if (KIND == SRC_PLAIN) return a[o];
        if (KIND == SRC_SUM2) return add_mod(a[o], a2[o], mq[l].q);
        if (KIND == SRC_MULCONST) return mul_shoup_fast(a[o], k.v[l], ksh.v[l], mq[l].q);
        if (KIND == SRC_MULPT) {
            // FP64 two-product Shoup step (pt/q formed in-register)
            const uint64_t y = pt[(((long long)l * pb + (pb == 1 ? 0 : b)) << log_n) + idx];
            const double2 f = fmod[l];
            const ntt16::FpMod fm{f.x, f.y};
            const double yd = ntt16::u2d(y);
            return ntt16::d2canon(ntt16::f_mulmod(ntt16::u2d(a[o]), yd, __dmul_rn(yd, fm.qinv), fm.q), fm);
        }
        Acc3 acc;
        acc3_zero(acc);
        const long long pe = (((long long)l * ps) << log_n) + idx;
        for (int i = 0; i < n; ++i) acc3_mac(acc, babies.p[i][o], pts.p[i][pe]);
        return acc3_reduce(acc, mq[l]);
    }
};

// iNTT prologue for the dropped limb: launch P = p * B + b, prime index la
template <int KIND>
struct ProLast {
    RsSrc<KIND> src;
    int B;
    __device__ __forceinline__ uint64_t operator()(int, long long P, int idx) const {
        const int pb = (int)P, p = pb >= B ? 1 : 0;
        return src(p, src.la, pb - p * B, idx);
    }
};

// NTT prologue: centred remainder of the dropped limb, reduced mod q_l
struct ProRsBcast {
    const uint64_t *L;
    uint64_t ql;
    int B2, log_n;
    const ModQ *mq;
    __device__ __forceinline__ uint64_t operator()(int l, long long P, int idx) const {
        const long long pb = P - (long long)l * B2;
        const uint64_t x = L[(pb << log_n) + idx];
        const bool neg = x > (ql >> 1);
        const uint64_t mag = neg ? ql - x : x;
        // KAN chains: mag <= q_l / 2 < 2^46 and every prime exceeds 2^44, so mag < 4 q
        // and two conditional subtractions reduce it; Barrett otherwise
        const ModQ m = mq[l];
        const uint64_t q = m.q;
        uint64_t r;
        if (mag < 4 * q) {
            r = mag >= 2 * q ? mag - 2 * q : mag;
            r = r >= q ? r - q : r;
        } else {
            r = reduce128(0, mag, m);
        }
        return neg ? (r ? q - r : 0) : r;
    }
    // ntt16::HasDval: the centred remainder itself as a signed double. `fast` (set on the
    // host) says |remainder| <= q_l / 2 <= 4 q_t for every target prime, which the forward
    // NTT's lazy range absorbs (8 stages from 4 q stay below 10 q < 2^51 for q < 2^47; for
    // the large prime q_0 the remainder is already below q_0 / 2).
    int fast = 0;
    __device__ __forceinline__ double dval(int l, long long P, int idx, const ntt16::FpMod &, bool) const {
        if (!fast) return ntt16::u2d((*this)(l, P, idx));
        const long long pb = P - (long long)l * B2;
        const uint64_t x = L[(pb << log_n) + idx];
        const double xd = ntt16::u2d(x);
        return x > (ql >> 1) ? __dsub_rn(xd, ntt16::u2d(ql)) : xd;
    }
};

// NTT epilogue: out[p][l][b] = (X - v) * q_la^-1
template <int KIND>
struct EpiRescale {
    static constexpr bool kDiscardInter = true;  // output != between-phase buffer (ntt16.cuh)
    RsSrc<KIND> src;
    uint64_t *out;
    const ulonglong2 *qinv;
    int B;
    // integer path (generic rings, N = 2^17 halves)
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        const int pb = (int)(P - (long long)l * 2 * B), p = pb >= B ? 1 : 0, b = pb - p * B;
        const uint64_t q = src.mq[l].q;
        const ulonglong2 w = qinv[l];
        __stcs(out + ((long long)p * src.la + l) * src.BN + ((long long)b << src.log_n) + idx,
               mul_shoup(sub_mod(src(p, l, b, idx), v, q), w.x, w.y, q));
    }
    // FP64 finish (ntt16::HasFactor / HasOperandD): the raw operands are loaded in `prep`
    // (all 16 of a thread before its first store) and X is formed as a double
    struct Pre2 {
        uint64_t a, b;
    };
    static constexpr bool kTwo = KIND == SRC_MULPT || KIND == SRC_SUM2;  // two raw operands per output
    using Pre = std::conditional_t<kTwo, Pre2, uint64_t>;
    __device__ __forceinline__ Pre prep(int l, long long P, int idx) const {
        const int pb = (int)(P - (long long)l * 2 * B), p = pb >= B ? 1 : 0, b = pb - p * B;
        const long long o = ((long long)p * (src.la + 1) + l) * src.BN + ((long long)b << src.log_n) + idx;
        if constexpr (kTwo) {
            if (KIND == SRC_SUM2) return Pre2{src.a[o], src.a2[o]};
            return Pre2{src.a[o], src.pt[(((long long)l * src.pb + (src.pb == 1 ? 0 : b)) << src.log_n) + idx]};
        } else {
            if (KIND == SRC_MAC) return src(p, l, b, idx);
            return src.a[o];
        }
    }
    __device__ __forceinline__ double operand_d(const Pre &pr, int l, const ntt16::FpMod &m, bool big) const {
        using namespace ntt16;
        if constexpr (kTwo) {
            const double a = u2d(pr.a), y = u2d(pr.b);
            if (KIND == SRC_SUM2) {
                const double s2 = __dadd_rn(a, y);
                return big ? f_center(s2, m) : s2;
            }
            return f_mulmod(a, y, __dmul_rn(y, m.qinv), m.q);
        } else {
            const double a = u2d(pr);
            if (KIND == SRC_MULCONST) {
                const double y = u2d(src.k.v[l]);
                return f_mulmod(a, y, __dmul_rn(y, m.qinv), m.q);
            }
            return a;
        }
    }
    __device__ __forceinline__ double2 factor(int l) const { return make_double2(ntt16::u2d(qinv[l].x), 0.0); }
    __device__ __forceinline__ void store(int l, long long P, int idx, const Pre &, uint64_t r) const {
        const int pb = (int)(P - (long long)l * 2 * B), p = pb >= B ? 1 : 0, b = pb - p * B;
        __stcs(out + ((long long)p * src.la + l) * src.BN + ((long long)b << src.log_n) + idx, r);
    }
};

// iNTT epilogue: scale by a per-limb constant (basis-conversion inv_i)
struct EpiScale {
    uint64_t *out;
    const uint64_t *inv, *inv_sh;
    const ModQ *mq;
    int mi0, log_n;
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        out[(P << log_n) + idx] = mul_shoup(v, inv[l], inv_sh[l], mq[mi0 + l].q);
    }
    // ntt16::HasScale: the kernel folds inv[l] into its N^-1 stage
    __device__ __forceinline__ uint64_t scale(int l) const { return inv[l]; }
    __device__ __forceinline__ void store(int, long long P, int idx, uint64_t v) const { out[(P << log_n) + idx] = v; }
};
// same, per-digit tables (ModUp sources at one level)
struct EpiScaleDigits {
    uint64_t *out;
    const uint64_t *inv[8], *inv_sh[8];
    int alpha, log_n;
    const ModQ *mq;
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        const int j = l / alpha, i = l - j * alpha;
        out[(P << log_n) + idx] = mul_shoup(v, inv[j][i], inv_sh[j][i], mq[l].q);
    }
    // ntt16::HasScale
    __device__ __forceinline__ uint64_t scale(int l) const {
        const int j = l / alpha;
        return inv[j][l - j * alpha];
    }
    __device__ __forceinline__ void store(int, long long P, int idx, uint64_t v) const { out[(P << log_n) + idx] = v; }
};

// NTT epilogue: ModDown finish (acc - v) * P^-1 (+ sigma_g(addend))
struct EpiModDown {
    static constexpr bool kDiscardInter = true;  // output != between-phase buffer (ntt16.cuh)
    const uint64_t *acc, *addend;
    uint64_t *out;
    const ulonglong2 *pinv;
    const ModQ *mq;
    uint32_t g;
    int B, log_n;
    long long BN;
    struct Pre {
        uint64_t a, add;
    };
    __device__ __forceinline__ Pre prep(int l, long long P, int idx) const {
        const long long o = (long long)l * BN + ((P - (long long)l * B) << log_n) + idx;
        Pre r{acc[o], 0};
        if (addend) r.add = addend[g == 1u ? o : o - idx + auto_src((uint32_t)idx, g, log_n)];
        return r;
    }
    __device__ __forceinline__ void fin(int l, long long P, int idx, Pre pr, uint64_t v) const {
        const long long o = (long long)l * BN + ((P - (long long)l * B) << log_n) + idx;
        const uint64_t q = mq[l].q;
        const ulonglong2 w = pinv[l];
        uint64_t r = mul_shoup(sub_mod(pr.a, v, q), w.x, w.y, q);
        if (addend) r = add_mod(r, pr.add, q);
        out[o] = r;
    }
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        fin(l, P, idx, prep(l, P, idx), v);
    }
};

// merged ModDown + rescale helpers
__global__ void k_mdrs_y(const uint64_t *__restrict__ acc_l, const uint64_t *__restrict__ d_l, uint64_t *__restrict__ y,
                         const ulonglong2 *__restrict__ pmod_l, const ModQ *__restrict__ mq_l, long long BN) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= BN) return;
    const uint64_t q = mq_l->q;
    const ulonglong2 P = *pmod_l;
    y[e] = add_mod(acc_l[e], mul_shoup(d_l[e], P.x, P.y, q), q);
}
__global__ void k_mdrs_finish(const uint64_t *__restrict__ acc, const uint64_t *__restrict__ d,
                              const uint64_t *__restrict__ conv, uint64_t *__restrict__ out,
                              const ulonglong2 *__restrict__ pmod, const ulonglong2 *__restrict__ mqinv,
                              const ModQ *__restrict__ mq, long long BN) {
    ELEM_INDEX
    (void)p;
    const long long o = (long long)l * BN + e;
    const uint64_t q = mq[l].q;
    const ulonglong2 P = pmod[l], w = mqinv[l];
    const uint64_t y = add_mod(acc[o], mul_shoup(d[o], P.x, P.y, q), q);
    out[o] = mul_shoup(sub_mod(y, conv[o], q), w.x, w.y, q);
}
// tensor-product terms of (a, b) at limb l, element o (NTT domain):
// d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1
// With a second pair (a2, b2: hk_mul2) the terms are those of a (x) b + a2 (x) b2,
// relinearised and rescaled once.
struct Tensor {
    const uint64_t *a, *b;
    long long pa, pb;  // offset of poly 1 in a / b
    const ModQ *mq;
    const uint64_t *a2 = nullptr, *b2 = nullptr;
    long long pa2 = 0, pb2 = 0;
    __device__ __forceinline__ uint64_t d(int which, int l, long long o) const {
        const ModQ m = mq[l];
        if (!a2) {
            if (which == 0) return mul_mod(a[o], b[o], m);
            if (which == 2) return mul_mod(a[pa + o], b[pb + o], m);
        }
        Acc3 acc;
        acc3_zero(acc);
        if (which == 0) {
            acc3_mac(acc, a[o], b[o]);
            acc3_mac(acc, a2[o], b2[o]);
        } else if (which == 2) {
            acc3_mac(acc, a[pa + o], b[pb + o]);
            acc3_mac(acc, a2[pa2 + o], b2[pb2 + o]);
        } else {
            acc3_mac(acc, a[o], b[pb + o]);
            acc3_mac(acc, a[pa + o], b[o]);
            if (a2) {
                acc3_mac(acc, a2[o], b2[pb2 + o]);
                acc3_mac(acc, a2[pa2 + o], b2[o]);
            }
        }
        return acc3_reduce(acc, m);
    }
};
// Optional linear term k * x folded into a relinearised product before its
// merged ModDown + rescale (hk_mul_lin): d_p += k_l * x_p at limb l, so the
// product and k x share one division by P q_l. x is a ciphertext at level
// >= l (poly 1 at offset px); k / ksh are the constant's residues and Shoup
// companions per limb.
struct LinTerm {
    const uint64_t *x;
    long long px;
    Residues k, ksh;
    __device__ __forceinline__ uint64_t apply(int which, int l, long long o, uint64_t d, uint64_t q) const {
        if (!x) return d;
        const uint64_t xv = x[which ? px + o : o];
        return add_mod(d, mul_shoup_fast(xv, k.v[l], ksh.v[l], q), q);
    }
};
// Optional affine finish of a relinearised product (hk_mul_affine):
// out = mult * out (+ c on poly 0), bit-identical to hk_add(out, out) and
// hk_add_const on the result (the Chebyshev power step T_2k = 2 T_k^2 - 1).
struct Affine {
    int dbl, has_c;
    Residues c;
    __device__ __forceinline__ uint64_t apply(int which, int l, uint64_t r, uint64_t q) const {
        if (dbl) r = add_mod(r, r, q);
        if (has_c && which == 0) r = add_mod(r, c.v[l], q);
        return r;
    }
};
__global__ void k_d2_sum(Tensor T, uint64_t *__restrict__ d2, long long BN) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= BN) return;
    const int l = blockIdx.y;
    const long long o = (long long)l * BN + e;
    d2[o] = T.d(2, l, o);
}
// iNTT prologue for the relinearisation ModUp: d2 = a1 b1 on the fly
struct ProD2 {
    Tensor T;
    long long BN;
    int B, log_n;
    __device__ __forceinline__ uint64_t operator()(int l, long long P, int idx) const {
        return T.d(2, l, (long long)l * BN + ((P - (long long)l * B) << log_n) + idx);
    }
    // the same product on the FP64 pipe (ntt16::HasDval): exact two-product Shoup step on
    // the operands instead of a 128-bit Barrett product on the integer pipe
    __device__ __forceinline__ double dval(int l, long long P, int idx, const ntt16::FpMod &m, bool big) const {
        using namespace ntt16;
        const long long o = (long long)l * BN + ((P - (long long)l * B) << log_n) + idx;
        const double b = u2d(T.b[T.pb + o]);
        double r = f_mulmod(u2d(T.a[T.pa + o]), b, __dmul_rn(b, m.qinv), m.q);
        if (T.a2) {
            const double b2 = u2d(T.b2[T.pb2 + o]);
            r = __dadd_rn(r, f_mulmod(u2d(T.a2[T.pa2 + o]), b2, __dmul_rn(b2, m.qinv), m.q));
        }
        return big ? f_center(r, m) : r;
    }
};
// Merged ModDown + rescale of both halves of a relinearised product: launches
// run over 2B "samples" pb = 2 b + p, so the two halves of one sample sit in
// adjacent clusters and the tensor operands a0 / b0 both read are shared in L2.
// iNTT prologue of the special limbs: acc_p limb (l + 1 + j), sample b
struct ProAccSp2 {
    const uint64_t *acc;
    long long BN, pne;  // pne: offset of half 1 in acc
    int l, B, log_n;
    __device__ __forceinline__ uint64_t operator()(int j, long long P, int idx) const {
        const long long pb = P - (long long)j * 2 * B;
        return acc[(pb & 1) * pne + (long long)(l + 1 + j) * BN + ((pb >> 1) << log_n) + idx];
    }
};
// Folded relinearisation (FoldD): acc_p already holds Y_p = acc_p + P d_p on
// the q limbs, so the q_l source of the merged ModDown + rescale is acc_p[l]
// and its epilogue reads one operand.
struct ProAccL2 {
    const uint64_t *acc;
    long long BN, pne;
    int l, log_n;
    __device__ __forceinline__ uint64_t operator()(int, long long P, int idx) const {
        return acc[(P & 1) * pne + (long long)l * BN + ((P >> 1) << log_n) + idx];
    }
};
struct EpiMdRsY2 {  // out_p = aff((Y_p - v) (P q_l)^-1)
    static constexpr bool kDiscardInter = true;  // output != between-phase buffer (ntt16.cuh)
    const uint64_t *acc;
    uint64_t *out;
    const ulonglong2 *mqinv;
    const ModQ *mq;
    int B, log_n;
    long long BN, pne, pout;
    Affine aff;
    using Pre = uint64_t;
    __device__ __forceinline__ Pre prep(int l, long long P, int idx) const {
        const long long pb = P - (long long)l * 2 * B;
        return __ldcs(acc + (pb & 1) * pne + (long long)l * BN + ((pb >> 1) << log_n) + idx);
    }
    __device__ __forceinline__ void fin(int l, long long P, int idx, Pre y, uint64_t v) const {
        const long long pb = P - (long long)l * 2 * B;
        const int p = (int)(pb & 1);
        const long long o = (long long)l * BN + ((pb >> 1) << log_n) + idx;
        const uint64_t q = mq[l].q;
        const ulonglong2 w = mqinv[l];
        __stcs(out + p * pout + o, aff.apply(p, l, mul_shoup(sub_mod(y, v, q), w.x, w.y, q), q));
    }
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        fin(l, P, idx, prep(l, P, idx), v);
    }
    // FP64 finish (ntt16::HasFactor): out_p = aff((Y_p - v) (P q_l)^-1)
    __device__ __forceinline__ uint64_t operand(const Pre &y) const { return y; }
    __device__ __forceinline__ double2 factor(int l) const { return make_double2(ntt16::u2d(mqinv[l].x), 0.0); }
    __device__ __forceinline__ void store(int l, long long P, int idx, const Pre &, uint64_t r) const {
        const long long pb = P - (long long)l * 2 * B;
        const int p = (int)(pb & 1);
        const long long o = (long long)l * BN + ((pb >> 1) << log_n) + idx;
        __stcs(out + p * pout + o, aff.apply(p, l, r, mq[l].q));
    }
};
// ModDown of both halves of a key switch (interleaved samples 2 b + p):
// out_p = (acc_p - v) P^-1 (+ sigma_g(add_p))
struct EpiModDown2 {
    static constexpr bool kDiscardInter = true;  // output != between-phase buffer (ntt16.cuh)
    const uint64_t *acc, *add0, *add1;
    uint64_t *out0, *out1;
    const ulonglong2 *pinv;
    const ModQ *mq;
    uint32_t g;
    int B, log_n;
    long long BN, pne;
    struct Pre {
        uint64_t a, add;
    };
    __device__ __forceinline__ Pre prep(int l, long long P, int idx) const {
        const long long pb = P - (long long)l * 2 * B;
        const int p = (int)(pb & 1);
        const long long o = (long long)l * BN + ((pb >> 1) << log_n) + idx;
        Pre r{__ldcs(acc + p * pne + o), 0};
        const uint64_t *addend = p ? add1 : add0;
        if (addend) r.add = addend[g == 1u ? o : o - idx + auto_src((uint32_t)idx, g, log_n)];
        return r;
    }
    __device__ __forceinline__ void fin(int l, long long P, int idx, Pre pr, uint64_t v) const {
        const long long pb = P - (long long)l * 2 * B;
        const int p = (int)(pb & 1);
        const long long o = (long long)l * BN + ((pb >> 1) << log_n) + idx;
        const uint64_t q = mq[l].q;
        const ulonglong2 w = pinv[l];
        uint64_t r = mul_shoup(sub_mod(pr.a, v, q), w.x, w.y, q);
        if (p ? add1 : add0) r = add_mod(r, pr.add, q);
        __stcs((p ? out1 : out0) + o, r);
    }
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        fin(l, P, idx, prep(l, P, idx), v);
    }
    // FP64 finish (ntt16::HasFactor): out_p = (acc_p - v) P^-1 (+ sigma_g(add_p))
    __device__ __forceinline__ uint64_t operand(const Pre &pr) const { return pr.a; }
    __device__ __forceinline__ double2 factor(int l) const { return make_double2(ntt16::u2d(pinv[l].x), 0.0); }
    __device__ __forceinline__ void store(int l, long long P, int idx, const Pre &pr, uint64_t r) const {
        const long long pb = P - (long long)l * 2 * B;
        const int p = (int)(pb & 1);
        const long long o = (long long)l * BN + ((pb >> 1) << log_n) + idx;
        if (p ? add1 : add0) r = add_mod(r, pr.add, mq[l].q);
        __stcs((p ? out1 : out0) + o, r);
    }
};

// generic-ring path of hk_mul_affine: out_p = mult out_p (+ c on poly 0), l limbs
__global__ void k_affine(uint64_t *__restrict__ out, long long pl, Affine aff, long long BN,
                         const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const long long o = p * pl + (long long)l * BN + e;
    out[o] = aff.apply(p, l, out[o], mq[l].q);
}
// generic-ring path of hk_mul_lin: d_p += k x_p over the materialised tensor
__global__ void k_add_lin(uint64_t *__restrict__ d, long long pl, LinTerm lin, long long BN,
                          const ModQ *__restrict__ mq) {
    ELEM_INDEX
    const long long o = (long long)l * BN + e;
    d[p * pl + o] = lin.apply(p, l, o, d[p * pl + o], mq[l].q);
}

// iNTT prologue: y = acc_l + P d_l (prime l)
struct ProMdY {
    const uint64_t *acc_l, *d_l;
    const ulonglong2 *pmod;
    const ModQ *mq;
    int l, log_n;
    __device__ __forceinline__ uint64_t operator()(int, long long P, int idx) const {
        const long long o = (P << log_n) + idx;
        const uint64_t q = mq[l].q;
        const ulonglong2 Pm = pmod[l];
        return add_mod(acc_l[o], mul_shoup(d_l[o], Pm.x, Pm.y, q), q);
    }
};
// NTT epilogue: out_t = (acc_t + P d_t - v) * (P q_l)^-1
struct EpiMdRs {
    static constexpr bool kDiscardInter = true;  // output != between-phase buffer (ntt16.cuh)
    const uint64_t *acc, *d;
    uint64_t *out;
    const ulonglong2 *pmod, *mqinv;
    const ModQ *mq;
    int B, log_n;
    long long BN;
    using Pre = uint64_t;  // y = acc + P d
    __device__ __forceinline__ Pre prep(int l, long long P, int idx) const {
        const long long o = (long long)l * BN + ((P - (long long)l * B) << log_n) + idx;
        const uint64_t q = mq[l].q;
        const ulonglong2 Pm = pmod[l];
        return add_mod(acc[o], mul_shoup(d[o], Pm.x, Pm.y, q), q);
    }
    __device__ __forceinline__ void fin(int l, long long P, int idx, Pre y, uint64_t v) const {
        const long long o = (long long)l * BN + ((P - (long long)l * B) << log_n) + idx;
        const uint64_t q = mq[l].q;
        const ulonglong2 w = mqinv[l];
        out[o] = mul_shoup(sub_mod(y, v, q), w.x, w.y, q);
    }
    __device__ __forceinline__ void operator()(int l, long long P, int idx, uint64_t v) const {
        fin(l, P, idx, prep(l, P, idx), v);
    }
};

}  // namespace

static dim3 egrid(long long BN, int limbs, int polys) {
    return dim3((unsigned)((BN + 255) / 256), (unsigned)limbs, (unsigned)polys);
}

// basis conversion launcher: picks the register-array size, stages hat in smem
static int conv_launch(hk_ctx *c, const ConvTable &T, const uint64_t *src, uint64_t *dst, int mode, int l,
                       long long BN, int n_dst = -1, int prescaled = 0) {
    if (n_dst < 0) n_dst = T.n_dst;
    if (conv_tc_ok(c, T, n_dst, BN, prescaled)) return conv_tc_launch(c, T, src, dst, mode, l, BN, n_dst);
    const size_t smem =
        sizeof(uint32_t) * (size_t)n_dst * ((3 * T.n_src + 3) & ~3) + sizeof(ModQ) * n_dst + sizeof(int) * n_dst;
    const dim3 grid((unsigned)((BN + 127) / 128));
#define CONV_CASE(NSV)                                                                                        \
    case NSV:                                                                                                 \
        if (smem > 48 * 1024)                                                                                 \
            cudaFuncSetAttribute(k_conv<NSV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
        k_conv<NSV><<<grid, 128, smem, c->stream>>>(src, T.n_src, T.d_inv, T.d_inv_sh, T.d_hat, T.d_src_mod, \
                                                     T.d_dst_mod, n_dst, dst, mode, l, c->n_q, BN, c->d_modq, \
                                                     prescaled, T.d_src_invd, T.d_neg_m);                     \
        ++c->launches;                                                                                        \
        HK_LAUNCH_CHECK(c, "basis conversion");                                                              \
        return HK_OK;
    switch (T.n_src) {
        CONV_CASE(1) CONV_CASE(2) CONV_CASE(3) CONV_CASE(4) CONV_CASE(5) CONV_CASE(6) CONV_CASE(7) CONV_CASE(8)
        CONV_CASE(9) CONV_CASE(10) CONV_CASE(11) CONV_CASE(12) CONV_CASE(13) CONV_CASE(14) CONV_CASE(15)
        CONV_CASE(16) CONV_CASE(17) CONV_CASE(18) CONV_CASE(19) CONV_CASE(20)
        default: break;
    }
#undef CONV_CASE
    return hk_fail(c, HK_E_ARG, "basis conversion with %d sources exceeds 20", T.n_src);
}

// words of scratch the key switch at level l needs

static size_t rs_scratch_words(const hk_ctx *c, int l, int B) {
    return (size_t)B * c->n * (2 + 2 * (size_t)l);
}

int rescale_launch(hk_ctx *c, const uint64_t *in, int l, int B, uint64_t *out, uint64_t *scratch) {
    const long long BN = (long long)B * c->n;
    uint64_t *L = scratch, *R = scratch + 2 * BN;
    HK_CUDA(c, cudaMemcpyAsync(L, in + (long long)l * BN, sizeof(uint64_t) * BN, cudaMemcpyDeviceToDevice,
                               c->stream));
    HK_CUDA(c, cudaMemcpyAsync(L + BN, in + (long long)(2 * l + 1) * BN, sizeof(uint64_t) * BN,
                               cudaMemcpyDeviceToDevice, c->stream));
    int rc = ntt_inv_launch(c, L, l, 1, 2 * B, 0);
    if (rc) return rc;
    k_rs_center<<<egrid(2 * BN, l, 1), 256, 0, c->stream>>>(L, R, l, 2 * BN, c->d_modq); ++c->launches;
    rc = ntt_fwd_launch(c, R, 0, l, 2 * B, 0);
    if (rc) return rc;
    k_rs_finish<<<egrid(BN, l, 2), 256, 0, c->stream>>>(in, R, out, l, BN, c->d_rs_qinv + (size_t)l * c->n_q,
                                                        c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "rescale");
    return HK_OK;
}

// ---------------------------------------------------------------------------
// fused rescale / key switch (N = 2^16)
// ---------------------------------------------------------------------------
template <int KIND>
static int rescale_fused(hk_ctx *c, const RsSrc<KIND> &src, int l, int B, uint64_t *out, uint64_t *scratch) {
    const long long BN = (long long)B * c->n;
    uint64_t *L = scratch, *inter = scratch + 2 * BN;
    int rc = ntt16::launch_inv(c, L, l, 1, 2 * B, ProLast<KIND>{src, B}, ntt16::EpiPlain{L, c->log_n});
    if (rc) return rc;
    ProRsBcast pro{L, c->mod_h[l], 2 * B, c->log_n, c->d_modq};
    static const int rs_fast = getenv("HK_RS_FAST") ? atoi(getenv("HK_RS_FAST")) : 1;  // A/B knob
    pro.fast = rs_fast;
    for (int t = 0; t < l; ++t)  // |remainder| <= q_l / 2 must stay within 4 q_t (below q_t for a large prime)
        if ((c->mod_h[t] < ntt16::kSmallPrime && c->mod_h[l] / 2 > 4 * c->mod_h[t]) ||
            (c->mod_h[t] >= ntt16::kSmallPrime && c->mod_h[l] / 2 >= c->mod_h[t]))
            pro.fast = 0;
    EpiRescale<KIND> epi{src, out, c->d_rs_qinv + (size_t)l * c->n_q, B};
    return ntt16::launch_fwd(c, inter, 0, l, 2 * B, pro, epi, true);
}

template <int KIND>
static RsSrc<KIND> make_src(hk_ctx *c, const uint64_t *a, int la, int B) {
    RsSrc<KIND> s;
    memset(&s, 0, sizeof s);
    s.a = a;
    s.la = la;
    s.log_n = c->log_n;
    s.BN = (long long)B * c->n;
    s.mq = c->d_modq;
    s.fmod = c->d_fmod;
    s.ps = 1;
    return s;
}

// ---------------------------------------------------------------------------
// hybrid key switching, staged: ModUp -> key inner product -> ModDown
// (or ModDown merged with the following rescale for relinearisation)
// scratch layout: dc [l+1] | ext [nd][ne] | acc [2][ne] | sp [K+1] | conv [l+1]   (units of B*N words)
// ---------------------------------------------------------------------------
struct KsBufs {
    uint64_t *dc, *ext, *acc, *sp, *conv;
};

static size_t ks_words(const hk_ctx *c, int l, int B) {
    const int ne = l + 1 + c->n_p, nd = l / c->alpha + 1;
    return (size_t)B * c->n * ((size_t)(l + 1) + (size_t)nd * ne + 2 * (size_t)ne + 2 * (c->n_p + 1) + 2 * (l + 1));
}

static KsBufs ks_bufs(const hk_ctx *c, int l, int B, uint64_t *scratch) {
    const int ne = l + 1 + c->n_p, nd = l / c->alpha + 1;
    const size_t BN = (size_t)B * c->n;
    KsBufs k;
    k.dc = scratch;
    k.ext = k.dc + (size_t)(l + 1) * BN;
    k.acc = k.ext + (size_t)nd * ne * BN;
    k.sp = k.acc + 2 * (size_t)ne * BN;
    k.conv = k.sp + 2 * (size_t)(c->n_p + 1) * BN;  // sp / conv hold both halves in the merged ModDown
    return k;
}

// ModUp of d (NTT, [l+1][B][N]) into ext [nd][ne][B][N] (own-digit limbs are
// not copied: the key inner product reads them from d)
static int ks_modup(hk_ctx *c, const uint64_t *d, int l, int B, const KsBufs &kb) {
    const int ne = l + 1 + c->n_p, nd = l / c->alpha + 1, np = c->n_p;
    const long long BN = (long long)B * c->n;
    const bool fused = ntt16::fused(c);
    int rc;
    if (fused) {
        EpiScaleDigits esd;
        memset(&esd, 0, sizeof esd);
        esd.out = kb.dc;
        esd.alpha = c->alpha;
        esd.log_n = c->log_n;
        esd.mq = c->d_modq;
        if (nd > 8) return hk_fail(c, HK_E_ARG, "more than 8 key-switching digits");
        for (int j = 0; j < nd; ++j) {
            esd.inv[j] = c->modup[l][j].d_inv;
            esd.inv_sh[j] = c->modup[l][j].d_inv_sh;
        }
        if ((rc = ntt16::launch_inv(c, kb.dc, 0, l + 1, B, ntt16::ProPlain{d, c->log_n}, esd))) return rc;
    } else {
        HK_CUDA(c, cudaMemcpyAsync(kb.dc, d, sizeof(uint64_t) * (l + 1) * BN, cudaMemcpyDeviceToDevice, c->stream));
        if ((rc = ntt_inv_launch(c, kb.dc, 0, l + 1, B, 0))) return rc;
    }
    for (int j = 0; j < nd; ++j) {
        const ConvTable &T = c->modup[l][j];
        const int d0 = j * c->alpha, d1 = std::min((j + 1) * c->alpha, l + 1);
        uint64_t *ej = kb.ext + (size_t)j * ne * BN;
        if ((rc = conv_launch(c, T, kb.dc + (size_t)d0 * BN, ej, 0, l, BN, -1, fused ? 1 : 0))) return rc;
        if (d0 > 0 && (rc = ntt_fwd_launch(c, ej, 0, d0, B, 0))) return rc;
        if (d1 < l + 1 && (rc = ntt_fwd_launch(c, ej + (size_t)d1 * BN, d1, l + 1 - d1, B, 0))) return rc;
        if ((rc = ntt_fwd_launch(c, ej + (size_t)(l + 1) * BN, c->n_q, np, B, 0))) return rc;
    }
    return HK_OK;
}

// key layout: rows = key level + 1 + K, specials from row (key level + 1)
struct KeyRef {
    const uint64_t *p;
    int level;
};

static int ks_ip(hk_ctx *c, const uint64_t *d, int l, int B, const KsBufs &kb, KeyRef key, uint32_t g,
                 const uint64_t *dm = nullptr, int accum = 0, const FoldD *fold = nullptr) {
    FoldD fd;
    memset(&fd, 0, sizeof fd);
    if (fold) fd = *fold;
    const int ne = l + 1 + c->n_p, nd = l / c->alpha + 1;
    if (key.level < l) return hk_fail(c, HK_E_NOKEY, "key for element %u serves level %d < %d", g, key.level, l);
    const int krows = key.level + 1 + c->n_p;
    const long long BN = (long long)B * c->n;
    // samples per thread: each key pair is read (and converted) once per bb samples (bb = 1 / 2 /
    // 4: 24.3 / 25.1 / 25.5 c1 inf/s at the start of round 2, profiles/r2_notes.md)
    static const int bb_max = getenv("HK_KEYIP_BB") ? atoi(getenv("HK_KEYIP_BB")) : 16;  // A/B knob: 4 / 8 / 16 -> 24.87 / 24.47 (24.80) / 24.57 ms per relinearisation
    const int bb = B % 16 == 0 && bb_max >= 16 ? 16 : B % 8 == 0 && bb_max >= 8 ? 8 : B % 4 == 0 && bb_max >= 4 ? 4 : B % 2 == 0 && bb_max >= 2 ? 2 : 1;
    const int ipt = std::min(256, c->n);
    const dim3 ipg((unsigned)((c->n / ipt) * (B / bb)), (unsigned)ne);
#define HK_KEY_IP(ND)                                                                                          \
    if (fold)                                                                                                  \
        k_key_ip<ND, true><<<ipg, ipt, 0, c->stream>>>(kb.ext, d, dm, c->alpha, ne, l, c->n_q, krows,          \
                                                       key.level + 1, c->log_n, bb, key.p, g, kb.acc,          \
                                                       kb.acc + (size_t)ne * BN, c->d_fmod, BN, accum, fd);    \
    else                                                                                                       \
        k_key_ip<ND, false><<<ipg, ipt, 0, c->stream>>>(kb.ext, d, dm, c->alpha, ne, l, c->n_q, krows,         \
                                                        key.level + 1, c->log_n, bb, key.p, g, kb.acc,         \
                                                        kb.acc + (size_t)ne * BN, c->d_fmod, BN, accum, fd)
    switch (nd) {
        case 1: HK_KEY_IP(1); break;
        case 2: HK_KEY_IP(2); break;
        case 3: HK_KEY_IP(3); break;
        case 4: HK_KEY_IP(4); break;
        case 5: HK_KEY_IP(5); break;
        case 6: HK_KEY_IP(6); break;
        case 7: HK_KEY_IP(7); break;
        case 8: HK_KEY_IP(8); break;
        default: return hk_fail(c, HK_E_ARG, "key switch: more than 8 digits");
    }
#undef HK_KEY_IP
    ++c->launches;
    HK_LAUNCH_CHECK(c, "key inner product");
    return HK_OK;
}

// ModDown of one half acc_p ([ne][B][N]) into out ([l+1][B][N]); adds sigma_g(add0) if given
static int ks_moddown(hk_ctx *c, const uint64_t *a, int l, int B, const KsBufs &kb, uint64_t *out,
                      const uint64_t *add0, uint32_t g) {
    const int np = c->n_p;
    const long long BN = (long long)B * c->n;
    const ConvTable &T = c->moddown;
    int rc;
    if (ntt16::fused(c)) {
        EpiScale es{kb.sp, T.d_inv, T.d_inv_sh, c->d_modq, c->n_q, c->log_n};
        if ((rc = ntt16::launch_inv(c, kb.sp, c->n_q, np, B, ntt16::ProPlain{a + (size_t)(l + 1) * BN, c->log_n}, es))) return rc;
        if ((rc = conv_launch(c, T, kb.sp, kb.conv, 1, l, BN, l + 1, 1))) return rc;
        EpiModDown epi{a, add0, out, c->d_pinv, c->d_modq, g, B, c->log_n, BN};
        return ntt16::launch_fwd(c, kb.conv, 0, l + 1, B, ntt16::ProPlain{kb.conv, c->log_n}, epi);
    }
    HK_CUDA(c, cudaMemcpyAsync(kb.sp, a + (size_t)(l + 1) * BN, sizeof(uint64_t) * np * BN, cudaMemcpyDeviceToDevice,
                               c->stream));
    if ((rc = ntt_inv_launch(c, kb.sp, c->n_q, np, B, 0))) return rc;
    if ((rc = conv_launch(c, T, kb.sp, kb.conv, 1, l, BN, l + 1))) return rc;
    if ((rc = ntt_fwd_launch(c, kb.conv, 0, l + 1, B, 0))) return rc;
    k_md_finish<<<egrid(BN, l + 1, 1), 256, 0, c->stream>>>(a, kb.conv, out, add0, g, c->log_n, BN, c->d_pinv,
                                                           c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "moddown finish");
    return HK_OK;
}

// ModDown of both halves (acc [2][ne][B][N]) into out0 / out1 ([l+1][B][N]), adding
// sigma_g(add0) to half 0 and sigma_g(add1) to half 1 when given. The fused rings
// run both halves as one launch chain over 2B interleaved samples.
static int ks_moddown2(hk_ctx *c, int l, int B, const KsBufs &kb, uint64_t *out0, uint64_t *out1,
                       const uint64_t *add0, const uint64_t *add1, uint32_t g) {
    const int ne = l + 1 + c->n_p, np = c->n_p;
    const long long BN = (long long)B * c->n;
    if (!ntt16::fused(c)) {
        int rc = ks_moddown(c, kb.acc, l, B, kb, out0, add0, g);
        if (!rc) rc = ks_moddown(c, kb.acc + (size_t)ne * BN, l, B, kb, out1, add1, g);
        return rc;
    }
    const ConvTable &T = c->moddown;
    const long long pne = (long long)ne * BN;
    int rc;
    EpiScale es{kb.sp, T.d_inv, T.d_inv_sh, c->d_modq, c->n_q, c->log_n};
    if ((rc = ntt16::launch_inv(c, kb.sp, c->n_q, np, 2 * B, ProAccSp2{kb.acc, BN, pne, l, B, c->log_n}, es)))
        return rc;
    if ((rc = conv_launch(c, T, kb.sp, kb.conv, 1, l, 2 * BN, l + 1, 1))) return rc;
    EpiModDown2 epi{kb.acc, add0, add1, out0, out1, c->d_pinv, c->d_modq, g, B, c->log_n, BN, pne};
    return ntt16::launch_fwd(c, kb.conv, 0, l + 1, 2 * B, ntt16::ProPlain{kb.conv, c->log_n}, epi);
}

// ModDown merged with rescale: out ([l][B][N]) = (acc_p + P d_p) / (P q_l)
static int ks_moddown_rescale(hk_ctx *c, const uint64_t *a, const uint64_t *dp, int l, int B, const KsBufs &kb,
                              uint64_t *out) {
    const int np = c->n_p;
    const long long BN = (long long)B * c->n;
    const ConvTable &T = c->mdrs[l];
    const ulonglong2 *mqinv = c->d_mqinv + (size_t)l * c->n_q;
    int rc;
    if (ntt16::fused(c)) {
        EpiScale es{kb.sp, T.d_inv, T.d_inv_sh, c->d_modq, c->n_q, c->log_n};
        if ((rc = ntt16::launch_inv(c, kb.sp, c->n_q, np, B, ntt16::ProPlain{a + (size_t)(l + 1) * BN, c->log_n}, es))) return rc;
        ProMdY py{a + (size_t)l * BN, dp + (size_t)l * BN, c->d_pmod, c->d_modq, l, c->log_n};
        EpiScale es2{kb.sp + (size_t)np * BN, T.d_inv + np, T.d_inv_sh + np, c->d_modq, l, c->log_n};
        if ((rc = ntt16::launch_inv(c, kb.sp + (size_t)np * BN, l, 1, B, py, es2))) return rc;
        if ((rc = conv_launch(c, T, kb.sp, kb.conv, 1, l, BN, l, 1))) return rc;
        EpiMdRs epi{a, dp, out, c->d_pmod, mqinv, c->d_modq, B, c->log_n, BN};
        return ntt16::launch_fwd(c, kb.conv, 0, l, B, ntt16::ProPlain{kb.conv, c->log_n}, epi);
    }
    HK_CUDA(c, cudaMemcpyAsync(kb.sp, a + (size_t)(l + 1) * BN, sizeof(uint64_t) * np * BN, cudaMemcpyDeviceToDevice,
                               c->stream));
    k_mdrs_y<<<egrid(BN, 1, 1), 256, 0, c->stream>>>(a + (size_t)l * BN, dp + (size_t)l * BN, kb.sp + (size_t)np * BN,
                                                     c->d_pmod + l, c->d_modq + l, BN);
    ++c->launches;
    if ((rc = ntt_inv_launch(c, kb.sp, c->n_q, np, B, 0))) return rc;
    if ((rc = ntt_inv_launch(c, kb.sp + (size_t)np * BN, l, 1, B, 0))) return rc;
    if ((rc = conv_launch(c, T, kb.sp, kb.conv, 1, l, BN, l))) return rc;
    if ((rc = ntt_fwd_launch(c, kb.conv, 0, l, B, 0))) return rc;
    k_mdrs_finish<<<egrid(BN, l, 1), 256, 0, c->stream>>>(a, dp, kb.conv, out, c->d_pmod, mqinv, c->d_modq, BN);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "moddown-rescale finish");
    return HK_OK;
}

// ct x ct at N = 2^16: the tensor product is never materialised — d2 feeds the
// ModUp iNTT prologue, d0 / d1 are recomputed inside the merged ModDown +
// rescale (prologue of the q_l limb, epilogue of every output limb).
struct Pair2 {
    const uint64_t *a, *b;
    int la, lb;
};

static int mul_fused(hk_ctx *c, const uint64_t *a, int la, const uint64_t *b, int lb, int l, int B,
                     const KsBufs &kb, uint64_t *out, const LinTerm &lin, const Affine &aff,
                     const Pair2 *pair2 = nullptr, uint64_t *d2buf = nullptr) {
    const int ne = l + 1 + c->n_p, nd = l / c->alpha + 1, np = c->n_p;
    const long long BN = (long long)B * c->n;
    Tensor T{a, b, (long long)(la + 1) * BN, (long long)(lb + 1) * BN, c->d_modq};
    if (pair2) {
        T.a2 = pair2->a;
        T.b2 = pair2->b;
        T.pa2 = (long long)(pair2->la + 1) * BN;
        T.pb2 = (long long)(pair2->lb + 1) * BN;
    }
    EpiScaleDigits esd;
    memset(&esd, 0, sizeof esd);
    esd.out = kb.dc;
    esd.alpha = c->alpha;
    esd.log_n = c->log_n;
    esd.mq = c->d_modq;
    if (nd > 8) return hk_fail(c, HK_E_ARG, "more than 8 key-switching digits");
    for (int j = 0; j < nd; ++j) {
        esd.inv[j] = c->modup[l][j].d_inv;
        esd.inv_sh[j] = c->modup[l][j].d_inv_sh;
    }
    int rc = ntt16::launch_inv(c, kb.dc, 0, l + 1, B, ProD2{T, BN, B, c->log_n}, esd);
    if (rc) return rc;
    for (int j = 0; j < nd; ++j) {
        const ConvTable &Tc = c->modup[l][j];
        const int d0 = j * c->alpha, d1 = std::min((j + 1) * c->alpha, l + 1);
        uint64_t *ej = kb.ext + (size_t)j * ne * BN;
        if ((rc = conv_launch(c, Tc, kb.dc + (size_t)d0 * BN, ej, 0, l, BN, -1, 1))) return rc;
        if (d0 > 0 && (rc = ntt_fwd_launch(c, ej, 0, d0, B, 0))) return rc;
        if (d1 < l + 1 && (rc = ntt_fwd_launch(c, ej + (size_t)d1 * BN, d1, l + 1 - d1, B, 0))) return rc;
        if ((rc = ntt_fwd_launch(c, ej + (size_t)(l + 1) * BN, c->n_q, np, B, 0))) return rc;
    }
    // the key IP writes Y_p = acc_p + P d_p on the q limbs (d_p from the operands)
    FoldD fold;
    memset(&fold, 0, sizeof fold);
    fold.a = a;
    fold.b = b;
    fold.pa = T.pa;
    fold.pb = T.pb;
    fold.a2 = T.a2;
    fold.b2 = T.b2;
    fold.pa2 = T.pa2;
    fold.pb2 = T.pb2;
    fold.x = lin.x;
    fold.px = lin.px;
    fold.k = lin.k;
    fold.pmod = c->d_pmod;
    if (pair2) {
        // two products: the key IP reads the own-digit limbs of d2 = a1 b1 + a2_1 b2_1
        // from a materialised copy (limbs 0..l, NTT form)
        k_d2_sum<<<egrid(BN, l + 1, 1), 256, 0, c->stream>>>(T, d2buf, BN);
        ++c->launches;
        HK_LAUNCH_CHECK(c, "d2 of two products");
        if ((rc = ks_ip(c, d2buf, l, B, kb, KeyRef{c->d_relin, c->n_q - 1}, 1u, nullptr, 0, &fold))) return rc;
    } else if ((rc = ks_ip(c, a + (size_t)(la + 1) * BN, l, B, kb, KeyRef{c->d_relin, c->n_q - 1}, 1u,
                           b + (size_t)(lb + 1) * BN, 0, &fold))) {
        // own-digit limbs of d2 are formed inside the key IP from a1 (.) b1
        return rc;
    }
    const ConvTable &Tm = c->mdrs[l];
    const ulonglong2 *mqinv = c->d_mqinv + (size_t)l * c->n_q;
    // both halves at once: sp [K+1][2B][N], conv [l][2B][N], sample index 2 b + p
    const long long pne = (long long)ne * BN;
    EpiScale es{kb.sp, Tm.d_inv, Tm.d_inv_sh, c->d_modq, c->n_q, c->log_n};
    if ((rc = ntt16::launch_inv(c, kb.sp, c->n_q, np, 2 * B, ProAccSp2{kb.acc, BN, pne, l, B, c->log_n}, es)))
        return rc;
    ProAccL2 py{kb.acc, BN, pne, l, c->log_n};
    EpiScale es2{kb.sp + (size_t)np * 2 * BN, Tm.d_inv + np, Tm.d_inv_sh + np, c->d_modq, l, c->log_n};
    if ((rc = ntt16::launch_inv(c, kb.sp + (size_t)np * 2 * BN, l, 1, 2 * B, py, es2))) return rc;
    if ((rc = conv_launch(c, Tm, kb.sp, kb.conv, 1, l, 2 * BN, l, 1))) return rc;
    EpiMdRsY2 epi{kb.acc, out, mqinv, c->d_modq, B, c->log_n, BN, pne, (long long)l * BN, aff};
    if ((rc = ntt16::launch_fwd(c, kb.conv, 0, l, 2 * B, ntt16::ProPlain{kb.conv, c->log_n}, epi))) return rc;
    return HK_OK;
}

// Key switch d under n keys (hoisted ModUp); for key r writes
//   out0[r] = ks0 (+ sigma_g(add0) if add0) and out1[r] = ks1, each [l+1][B][N].
static int keyswitch(hk_ctx *c, const uint64_t *d, int l, int B, int n, const KeyRef *keys,
                     const uint32_t *gal, uint64_t *const *out0, uint64_t *const *out1, const uint64_t *add0,
                     uint64_t *scratch) {
    const KsBufs kb = ks_bufs(c, l, B, scratch);
    const int ne = l + 1 + c->n_p;
    const long long BN = (long long)B * c->n;
    int rc = ks_modup(c, d, l, B, kb);
    if (rc) return rc;
    for (int r = 0; r < n; ++r) {
        if ((rc = ks_ip(c, d, l, B, kb, keys[r], gal[r]))) return rc;
        if ((rc = ks_moddown2(c, l, B, kb, out0[r], out1[r], add0, nullptr, gal[r]))) return rc;
    }
    return HK_OK;
}

extern "C" {

int hk_add(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, uint64_t *o, int32_t B) {
    if (la < 0 || lb < 0 || la >= c->n_q || lb >= c->n_q) return hk_fail(c, HK_E_ARG, "add: level out of range");
    const int lo = std::min(la, lb);
    const long long BN = (long long)B * c->n;
    if (BN % 1024 == 0)
        k_addsub4<<<dim3((unsigned)(BN / 1024), (unsigned)(lo + 1), 2), 256, 0, c->stream>>>(
            (const ulonglong2 *)a, la, (const ulonglong2 *)b, lb, (ulonglong2 *)o, lo, BN / 2, 0, c->d_modq);
    else
        k_addsub<<<egrid(BN, lo + 1, 2), 256, 0, c->stream>>>(a, la, b, lb, o, lo, BN, 0, c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "add");
    return HK_OK;
}

int hk_sub(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, uint64_t *o, int32_t B) {
    if (la < 0 || lb < 0 || la >= c->n_q || lb >= c->n_q) return hk_fail(c, HK_E_ARG, "sub: level out of range");
    const int lo = std::min(la, lb);
    const long long BN = (long long)B * c->n;
    if (BN % 1024 == 0)
        k_addsub4<<<dim3((unsigned)(BN / 1024), (unsigned)(lo + 1), 2), 256, 0, c->stream>>>(
            (const ulonglong2 *)a, la, (const ulonglong2 *)b, lb, (ulonglong2 *)o, lo, BN / 2, 1, c->d_modq);
    else
        k_addsub<<<egrid(BN, lo + 1, 2), 256, 0, c->stream>>>(a, la, b, lb, o, lo, BN, 1, c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "sub");
    return HK_OK;
}

int hk_add_plain(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *pt, int32_t lp, int32_t pb,
                 int32_t negate, uint64_t *out, int32_t B) {
    if (la < 0 || la >= c->n_q || lp < la) return hk_fail(c, HK_E_ARG, "add_plain: level mismatch");
    if (pb != 1 && pb != B) return hk_fail(c, HK_E_LENGTH, "add_plain: plaintext batch");
    const long long BN = (long long)B * c->n;
    if (BN % 1024 == 0)
        k_add_plain4<<<dim3((unsigned)(BN / 1024), (unsigned)(la + 1), 2), 256, 0, c->stream>>>(
            (const ulonglong2 *)a, la, (const ulonglong2 *)pt, pb, negate, (ulonglong2 *)out, BN / 2, c->log_n,
            c->d_modq);
    else
        k_add_plain<<<egrid(BN, la + 1, 2), 256, 0, c->stream>>>(a, la, pt, pb, negate, out, BN, c->log_n, c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "add_plain");
    return HK_OK;
}

int hk_add_const(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *res, uint64_t *out, int32_t B) {
    if (la < 0 || la >= c->n_q) return hk_fail(c, HK_E_ARG, "add_const: level");
    Residues r;
    for (int l = 0; l <= la; ++l) r.v[l] = res[l];
    const long long BN = (long long)B * c->n;
    if (BN % 1024 == 0)
        k_add_const4<<<dim3((unsigned)(BN / 1024), (unsigned)(la + 1), 2), 256, 0, c->stream>>>(
            (const ulonglong2 *)a, la, r, (ulonglong2 *)out, BN / 2, c->d_modq);
    else
        k_add_const<<<egrid(BN, la + 1, 2), 256, 0, c->stream>>>(a, la, r, out, BN, c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "add_const");
    return HK_OK;
}

int hk_rescale(hk_ctx *c, const uint64_t *a, int32_t la, uint64_t *out, int32_t B) {
    if (la < 1 || la >= c->n_q) return hk_fail(c, HK_E_DEPTH, "rescale at level %d", la);
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * rs_scratch_words(c, la, B));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "rescale workspace");
    if (ntt16::fused(c)) return rescale_fused(c, make_src<SRC_PLAIN>(c, a, la, B), la, B, out, ws);
    return rescale_launch(c, a, la, B, out, ws);
}

int hk_mul_plain(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *pt, int32_t lp, int32_t pb,
                 uint64_t *out, int32_t B) {
    if (la < 0 || la >= c->n_q || lp < la) return hk_fail(c, HK_E_ARG, "mul_plain: level mismatch");
    if (la < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", la);
    if (pb != 1 && pb != B) return hk_fail(c, HK_E_LENGTH, "mul_plain: plaintext batch");
    const long long BN = (long long)B * c->n, tot = 2LL * (la + 1) * BN;
    if (ntt16::fused(c)) {
        uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * rs_scratch_words(c, la, B));
        if (!ws) return hk_fail(c, HK_E_NOMEM, "mul_plain workspace");
        RsSrc<SRC_MULPT> src = make_src<SRC_MULPT>(c, a, la, B);
        src.pt = pt;
        src.pb = pb;
        return rescale_fused(c, src, la, B, out, ws);
    }
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * (tot + rs_scratch_words(c, la, B)));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "mul_plain workspace");
    k_mul_plain<<<egrid(BN, la + 1, 2), 256, 0, c->stream>>>(a, la, pt, pb, ws, BN, c->log_n, c->d_modq); ++c->launches;
    HK_LAUNCH_CHECK(c, "mul_plain");
    return rescale_launch(c, ws, la, B, out, ws + tot);
}

int hk_mul_const(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *res, uint64_t *out, int32_t B) {
    if (la < 0 || la >= c->n_q) return hk_fail(c, HK_E_ARG, "mul_const: level");
    if (la < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", la);
    Residues r;
    for (int l = 0; l <= la; ++l) r.v[l] = res[l];
    const long long BN = (long long)B * c->n, tot = 2LL * (la + 1) * BN;
    if (ntt16::fused(c)) {
        uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * rs_scratch_words(c, la, B));
        if (!ws) return hk_fail(c, HK_E_NOMEM, "mul_const workspace");
        RsSrc<SRC_MULCONST> src = make_src<SRC_MULCONST>(c, a, la, B);
        src.k = r;
        for (int l = 0; l <= la; ++l) src.ksh.v[l] = (uint64_t)(((u128)r.v[l] << 64) / c->mod_h[l]);
        return rescale_fused(c, src, la, B, out, ws);
    }
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * (tot + rs_scratch_words(c, la, B)));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "mul_const workspace");
    k_mul_const<<<egrid(BN, la + 1, 2), 256, 0, c->stream>>>(a, la, r, ws, BN, c->d_modq); ++c->launches;
    HK_LAUNCH_CHECK(c, "mul_const");
    return rescale_launch(c, ws, la, B, out, ws + tot);
}

int hk_mac_plain(hk_ctx *c, const uint64_t *const *babies, const uint64_t *const *pts, int32_t n, int32_t la,
                 int32_t lp, int32_t pt_stride, uint64_t *out, int32_t B) {
    if (la < 0 || la >= c->n_q || lp < la || n < 1 || pt_stride < 1) return hk_fail(c, HK_E_ARG, "mac_plain: args");
    if (la < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", la);
    const long long BN = (long long)B * c->n, tot = 2LL * (la + 1) * BN;
    if (ntt16::fused(c) && n <= kMacMax) {
        uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * rs_scratch_words(c, la, B));
        if (!ws) return hk_fail(c, HK_E_NOMEM, "mac_plain workspace");
        RsSrc<SRC_MAC> src = make_src<SRC_MAC>(c, babies[0], la, B);
        src.n = n;
        src.ps = pt_stride;
        for (int i = 0; i < n; ++i) {
            src.babies.p[i] = babies[i];
            src.pts.p[i] = pts[i];
        }
        return rescale_fused(c, src, la, B, out, ws);
    }
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * (tot + rs_scratch_words(c, la, B)));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "mac_plain workspace");
    for (int s = 0; s < n; s += kMacMax) {
        const int cnt = std::min(kMacMax, n - s);
        PtrList bl, pl;
        for (int i = 0; i < cnt; ++i) {
            bl.p[i] = babies[s + i];
            pl.p[i] = pts[s + i];
        }
        k_mac<<<egrid(BN, la + 1, 2), 256, 0, c->stream>>>(bl, pl, cnt, la, pt_stride, ws, BN, c->log_n, s > 0,
                                                           c->d_modq);
        ++c->launches;
    }
    HK_LAUNCH_CHECK(c, "mac_plain");
    return rescale_launch(c, ws, la, B, out, ws + tot);
}

int hk_mac_plain_blocks(hk_ctx *c, const uint64_t *const *babies, int32_t n, int32_t la, const uint64_t *pt,
                        int32_t pt_count, int32_t nb, int32_t G, const int32_t *counts, uint64_t *const *outs,
                        int32_t B) {
    if (la < 0 || la >= c->n_q || n < 1 || n > kMacMax || G < 1 || G > 8 || nb < 1 || B < 1)
        return hk_fail(c, HK_E_ARG, "mac_plain_blocks: args");
    if (la < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", la);
    int need = 0;
    for (int g = 0; g < G; ++g) {
        if (counts[g] < 1 || counts[g] > n || counts[g] > nb) return hk_fail(c, HK_E_ARG, "mac_plain_blocks: count");
        need = std::max(need, g * nb + counts[g]);
    }
    if (need > pt_count) return hk_fail(c, HK_E_ARG, "mac_plain_blocks: plaintext count %d < %d", pt_count, need);
    if (c->n < kBlkK) return hk_fail(c, HK_E_ARG, "mac_plain_blocks: ring too small");
    const long long BN = (long long)B * c->n, tot = 2LL * (la + 1) * BN;
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * ((size_t)G * tot + rs_scratch_words(c, la, B)));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "mac_plain_blocks workspace");
    PtrList bl;
    for (int i = 0; i < n; ++i) bl.p[i] = babies[i];
    int cz[8] = {1, 1, 1, 1, 1, 1, 1, 1};
    for (int g = 0; g < G; ++g) cz[g] = counts[g];
    const int4 lo = make_int4(cz[0], cz[1], cz[2], cz[3]), hi = make_int4(cz[4], cz[5], cz[6], cz[7]);
    const size_t smem = sizeof(uint2) * (size_t)G * n * kBlkK;
    const dim3 grid((unsigned)(c->n / kBlkK), (unsigned)(la + 1));
#define HK_MACB(GV)                                                                                             \
    case GV:                                                                                                    \
        cudaFuncSetAttribute(k_mac_blocks<GV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
        k_mac_blocks<GV><<<grid, 256, smem, c->stream>>>(bl, n, nb, lo, hi, pt, pt_count, la, ws, BN, B,        \
                                                         c->log_n, c->d_modq);                                  \
        break;
    switch (G) {
        HK_MACB(1) HK_MACB(2) HK_MACB(3) HK_MACB(4) HK_MACB(5) HK_MACB(6) HK_MACB(7) HK_MACB(8)
        default: break;
    }
#undef HK_MACB
    ++c->launches;
    HK_LAUNCH_CHECK(c, "mac_plain_blocks");
    uint64_t *rs = ws + (size_t)G * tot;
    for (int g = 0; g < G; ++g) {
        int rc;
        if (ntt16::fused(c))
            rc = rescale_fused(c, make_src<SRC_PLAIN>(c, ws + (size_t)g * tot, la, B), la, B, outs[g], rs);
        else
            rc = rescale_launch(c, ws + (size_t)g * tot, la, B, outs[g], rs);
        if (rc) return rc;
    }
    return HK_OK;
}

static int mul_impl(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, uint64_t *out, int32_t B,
                    const LinTerm &lin, const Affine &aff, const Pair2 *pair2 = nullptr) {
    const int l = pair2 ? std::min(std::min(la, lb), std::min(pair2->la, pair2->lb)) : std::min(la, lb);
    const long long BN = (long long)B * c->n, pl = (long long)(l + 1) * BN;
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * (3 * pl + ks_words(c, l, B)));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "mul workspace");
    uint64_t *d = ws;
    const KsBufs kb = ks_bufs(c, l, B, ws + 3 * pl);
    if (ntt16::fused(c)) return mul_fused(c, a, la, b, lb, l, B, kb, out, lin, aff, pair2, d);
    k_tensor<<<egrid(BN, l + 1, 1), 256, 0, c->stream>>>(a, la, b, lb, l, d, BN, c->d_modq);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "tensor");
    if (pair2) {
        k_tensor_add<<<egrid(BN, l + 1, 1), 256, 0, c->stream>>>(pair2->a, pair2->la, pair2->b, pair2->lb, l, d, BN,
                                                                 c->d_modq);
        ++c->launches;
        HK_LAUNCH_CHECK(c, "tensor pair 2");
    }
    if (lin.x) {
        k_add_lin<<<egrid(BN, l + 1, 2), 256, 0, c->stream>>>(d, pl, lin, BN, c->d_modq);
        ++c->launches;
        HK_LAUNCH_CHECK(c, "linear term");
    }
    int rc = ks_modup(c, d + 2 * pl, l, B, kb);
    if (!rc) rc = ks_ip(c, d + 2 * pl, l, B, kb, KeyRef{c->d_relin, c->n_q - 1}, 1u);
    const int ne = l + 1 + c->n_p;
    if (!rc) rc = ks_moddown_rescale(c, kb.acc, d, l, B, kb, out);
    if (!rc) rc = ks_moddown_rescale(c, kb.acc + (size_t)ne * BN, d + pl, l, B, kb, out + (size_t)l * BN);
    if (!rc && (aff.dbl || aff.has_c)) {
        k_affine<<<egrid(BN, l, 2), 256, 0, c->stream>>>(out, (long long)l * BN, aff, BN, c->d_modq);
        ++c->launches;
        HK_LAUNCH_CHECK(c, "affine finish");
    }
    return rc;
}

int hk_mul(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, uint64_t *out, int32_t B) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (la < 0 || lb < 0 || la >= c->n_q || lb >= c->n_q) return hk_fail(c, HK_E_ARG, "mul: level");
    const int l = std::min(la, lb);
    if (l < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", l);
    LinTerm lin;
    memset(&lin, 0, sizeof lin);
    Affine aff;
    memset(&aff, 0, sizeof aff);
    return mul_impl(c, a, la, b, lb, out, B, lin, aff);
}

int hk_mul2(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, const uint64_t *a2, int32_t la2,
            const uint64_t *b2, int32_t lb2, uint64_t *out, int32_t B) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    const int lv[4] = {la, lb, la2, lb2};
    for (int i = 0; i < 4; ++i)
        if (lv[i] < 0 || lv[i] >= c->n_q) return hk_fail(c, HK_E_ARG, "mul2: level");
    const int l = std::min(std::min(la, lb), std::min(la2, lb2));
    if (l < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", l);
    LinTerm lin;
    memset(&lin, 0, sizeof lin);
    Affine aff;
    memset(&aff, 0, sizeof aff);
    const Pair2 p2{a2, b2, la2, lb2};
    return mul_impl(c, a, la, b, lb, out, B, lin, aff, &p2);
}

int hk_mul_affine(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, int32_t mult,
                  const uint64_t *res, uint64_t *out, int32_t B) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (la < 0 || lb < 0 || la >= c->n_q || lb >= c->n_q) return hk_fail(c, HK_E_ARG, "mul_affine: level");
    if (mult != 1 && mult != 2) return hk_fail(c, HK_E_ARG, "mul_affine: multiplier %d not 1 or 2", mult);
    const int l = std::min(la, lb);
    if (l < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", l);
    LinTerm lin;
    memset(&lin, 0, sizeof lin);
    Affine aff;
    memset(&aff, 0, sizeof aff);
    aff.dbl = mult == 2;
    aff.has_c = res != nullptr;
    if (res)
        for (int i = 0; i < l; ++i) aff.c.v[i] = res[i];
    return mul_impl(c, a, la, b, lb, out, B, lin, aff);
}

int hk_mul_lin(hk_ctx *c, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, const uint64_t *x,
               int32_t lx, const uint64_t *res, uint64_t *out, int32_t B) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (la < 0 || lb < 0 || la >= c->n_q || lb >= c->n_q || lx < 0 || lx >= c->n_q)
        return hk_fail(c, HK_E_ARG, "mul_lin: level");
    const int l = std::min(la, lb);
    if (l < 1) return hk_fail(c, HK_E_DEPTH, "multiplication at level %d", l);
    if (lx < l) return hk_fail(c, HK_E_ARG, "mul_lin: linear term at level %d below the product's %d", lx, l);
    LinTerm lin;
    memset(&lin, 0, sizeof lin);
    lin.x = x;
    lin.px = (long long)(lx + 1) * B * c->n;
    for (int i = 0; i <= l; ++i) {
        lin.k.v[i] = res[i];
        lin.ksh.v[i] = (uint64_t)(((u128)res[i] << 64) / c->mod_h[i]);
    }
    Affine aff;
    memset(&aff, 0, sizeof aff);
    return mul_impl(c, a, la, b, lb, out, B, lin, aff);
}

int hk_rotate_hoisted(hk_ctx *c, const uint64_t *a, int32_t la, const uint32_t *gs, int32_t n,
                      uint64_t *const *outs, int32_t B) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (la < 0 || la >= c->n_q) return hk_fail(c, HK_E_ARG, "rotate: level");
    if (n < 1) return HK_OK;
    std::vector<KeyRef> keys(n);
    std::vector<uint64_t *> o0(n), o1(n);
    const long long pl = (long long)(la + 1) * B * c->n;
    for (int i = 0; i < n; ++i) {
        auto it = c->gal.find(gs[i]);
        if (it == c->gal.end()) return hk_fail(c, HK_E_NOKEY, "no galois key for element %u", gs[i]);
        if (it->second.level < la)
            return hk_fail(c, HK_E_NOKEY, "galois key %u serves level %d < %d", gs[i], it->second.level, la);
        keys[i] = KeyRef{it->second.p, it->second.level};
        o0[i] = outs[i];
        o1[i] = outs[i] + pl;
    }
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * ks_words(c, la, B));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "rotate workspace");
    return keyswitch(c, a + pl, la, B, n, keys.data(), gs, o0.data(), o1.data(), a, ws);
}

// sum_i sigma_{g_i}(ct_i) with ONE ModDown (lazy BSGS giant steps): the key inner
// products of every term accumulate in the extended basis; sum_i sigma_{g_i}(c0_i)
// (and the c1 of identity terms, g_i = 1) join in the ModDown epilogues.
int hk_rotate_sum(hk_ctx *c, const uint64_t *const *cts, int32_t la, const uint32_t *gs, int32_t n, uint64_t *out,
                  int32_t B) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (la < 0 || la >= c->n_q || n < 1 || B < 1) return hk_fail(c, HK_E_ARG, "rotate_sum: args");
    const uint32_t M = 2u * (uint32_t)c->n;
    std::vector<KeyRef> keys(n);
    for (int i = 0; i < n; ++i) {
        if ((gs[i] & 1u) == 0 || gs[i] >= M) return hk_fail(c, HK_E_ARG, "galois element %u invalid", gs[i]);
        if (gs[i] == 1u) continue;
        auto it = c->gal.find(gs[i]);
        if (it == c->gal.end()) return hk_fail(c, HK_E_NOKEY, "no galois key for element %u", gs[i]);
        if (it->second.level < la)
            return hk_fail(c, HK_E_NOKEY, "galois key %u serves level %d < %d", gs[i], it->second.level, la);
        keys[i] = KeyRef{it->second.p, it->second.level};
    }
    const long long BN = (long long)B * c->n, pl = (long long)(la + 1) * BN;
    uint64_t *ws = (uint64_t *)hk_workspace(c, sizeof(uint64_t) * (ks_words(c, la, B) + 2 * pl));
    if (!ws) return hk_fail(c, HK_E_NOMEM, "rotate_sum workspace");
    uint64_t *c0sum = ws, *c1id = ws + pl;
    const KsBufs kb = ks_bufs(c, la, B, ws + 2 * pl);
    int n_id = 0, n_ks = 0, rc = HK_OK;
    for (int i = 0; i < n; ++i) {
        k_auto_acc<<<egrid(BN, la + 1, 1), 256, 0, c->stream>>>(cts[i], c0sum, gs[i], c->log_n, BN, i == 0,
                                                                c->d_modq);
        ++c->launches;
        if (gs[i] == 1u) {
            k_auto_acc<<<egrid(BN, la + 1, 1), 256, 0, c->stream>>>(cts[i] + pl, c1id, 1u, c->log_n, BN, n_id == 0,
                                                                    c->d_modq);
            ++c->launches;
            ++n_id;
        }
    }
    HK_LAUNCH_CHECK(c, "rotate_sum: automorphism sums");
    for (int i = 0; i < n && !rc; ++i) {
        if (gs[i] == 1u) continue;
        rc = ks_modup(c, cts[i] + pl, la, B, kb);
        if (!rc) rc = ks_ip(c, cts[i] + pl, la, B, kb, keys[i], gs[i], nullptr, n_ks > 0);
        ++n_ks;
    }
    if (rc) return rc;
    if (n_ks == 0) {
        HK_CUDA(c, cudaMemcpyAsync(out, c0sum, sizeof(uint64_t) * 2 * pl, cudaMemcpyDeviceToDevice, c->stream));
        return HK_OK;
    }
    const int ne = la + 1 + c->n_p;
    return ks_moddown2(c, la, B, kb, out, out + pl, c0sum, n_id ? c1id : nullptr, 1u);
}

int hk_rotate(hk_ctx *c, const uint64_t *a, int32_t la, uint32_t g, uint64_t *out, int32_t B) {
    uint64_t *outs[1] = {out};
    return hk_rotate_hoisted(c, a, la, &g, 1, outs, B);
}

}  // extern "C"
