// encode.cu — CKKS canonical-embedding encode/decode on the GPU.
//
// Replaces HeBackend.encode/_plain_slots (hekan/backend.py:149-158, :251-257)
// and the slot read-out of decrypt (:168-170). The special FFT runs in float64
// with FMA contraction disabled (__dmul_rn/__dadd_rn/__dsub_rn, and the TU is
// built with --fmad=false) so every rounding matches the oracle's restatement
// op for op; the resulting integer plaintexts are bit-identical.
#include <cmath>

#include "common.cuh"

namespace {

__global__ void load_slots(const double *__restrict__ slots, double2 *__restrict__ a, long long total) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) a[i] = make_double2(slots[i], 0.0);
}

// one stage of the inverse special FFT (len = S .. 2), B vectors of S points
__global__ void fft_inv_stage(double2 *__restrict__ a, int S, int len, int M, const double2 *__restrict__ zeta,
                              const uint32_t *__restrict__ rg, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int half = S >> 1;
    const long long v = gid / half;
    const int bi = (int)(gid - v * half);
    const int h = len >> 1, lq = len << 2, gap = M / lq;
    const int blk = bi / h, j = bi - blk * h, i = blk * len;
    const int idx = (int)(rg[j] % (uint32_t)lq) * gap;
    const double tr = zeta[idx].x, ti = zeta[idx].y;
    double2 *p = a + v * S;
    const double2 A = p[i + j], Bv = p[i + j + h];
    const double ur = __dadd_rn(A.x, Bv.x), ui = __dadd_rn(A.y, Bv.y);
    const double vr = __dsub_rn(A.x, Bv.x), vi = __dsub_rn(A.y, Bv.y);
    p[i + j] = make_double2(ur, ui);
    p[i + j + h] = make_double2(__dadd_rn(__dmul_rn(vr, tr), __dmul_rn(vi, ti)),
                                __dsub_rn(__dmul_rn(vi, tr), __dmul_rn(vr, ti)));
}

// one stage of the forward special FFT (len = 2 .. S)
__global__ void fft_fwd_stage(double2 *__restrict__ a, int S, int len, int M, const double2 *__restrict__ zeta,
                              const uint32_t *__restrict__ rg, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int half = S >> 1;
    const long long v = gid / half;
    const int bi = (int)(gid - v * half);
    const int h = len >> 1, lq = len << 2, gap = M / lq;
    const int blk = bi / h, j = bi - blk * h, i = blk * len;
    const int idx = (int)(rg[j] % (uint32_t)lq) * gap;
    const double tr = zeta[idx].x, ti = zeta[idx].y;
    double2 *p = a + v * S;
    const double2 A = p[i + j], Bv = p[i + j + h];
    const double vr = __dsub_rn(__dmul_rn(Bv.x, tr), __dmul_rn(Bv.y, ti));
    const double vi = __dadd_rn(__dmul_rn(Bv.x, ti), __dmul_rn(Bv.y, tr));
    p[i + j] = make_double2(__dadd_rn(A.x, vr), __dadd_rn(A.y, vi));
    p[i + j + h] = make_double2(__dsub_rn(A.x, vr), __dsub_rn(A.y, vi));
}

__global__ void bitrev_copy(const double2 *__restrict__ in, double2 *__restrict__ out, int S, int bits,
                            long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const long long v = gid / S;
    const int i = (int)(gid - v * S);
    out[v * S + (__brev((uint32_t)i) >> (32 - bits))] = in[gid];
}

// after the inverse FFT + bit reversal: coefficients c_i (re) and c_{i+S} (im),
// reduced into every limb: pt[l][b][k]
__global__ void round_to_limbs(const double2 *__restrict__ w, int S, int log_n, double inv_s, double scale,
                               int n_limbs, int B, const ModQ *__restrict__ mq, uint64_t *__restrict__ pt,
                               long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;  // total = B * S
    const long long b = gid / S;
    const int i = (int)(gid - b * S);
    const double2 x = w[gid];
    const long long cr = __double2ll_rn(__dmul_rn(__dmul_rn(x.x, inv_s), scale));
    const long long ci = __double2ll_rn(__dmul_rn(__dmul_rn(x.y, inv_s), scale));
    const int N = 1 << log_n;
    for (int l = 0; l < n_limbs; ++l) {
        const ModQ m = mq[l];
        uint64_t *dst = pt + ((size_t)l * B + b) * N;
        dst[i] = smod_q(cr, m);
        dst[i + S] = smod_q(ci, m);
    }
}

// BSGS diagonal base + v, rolled by its giant-step block's base (inference.py:172-176):
// slot s holds d[(s - rb) mod S] with rb = base + (v / nb) * nb and
// d[r] = W~[r][(r + base + v) mod m] for r < m, W~ = W (n_o x n_in, row-major)
// zero-padded to m x m
__global__ void gen_diagonals(const double *__restrict__ W, int n_o, int n_in, int m, int base, int nb, int S,
                              double2 *__restrict__ a, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const long long v = gid / S;
    const int s = (int)(gid - v * S);
    const int rb = base + (int)(v / nb) * nb;
    int r = s - rb % S;
    if (r < 0) r += S;
    double val = 0.0;
    if (r < m && r < n_o) {
        const int col = (int)(((long long)r + base + v) % m);
        if (col < n_in) val = W[(long long)r * n_in + col];
    }
    a[gid] = make_double2(val, 0.0);
}

}  // namespace

// slots already in a (B x S complex, real parts) -> pt [level+1][B][N], NTT domain
static int encode_loaded(hk_ctx *c, double2 *a, int B, int level, double scale, uint64_t *pt) {
    const int S = c->slots, M = 2 * c->n, bits = c->log_n - 1;
    const long long all = (long long)B * S, half = (long long)B * (S / 2);
    double2 *b2 = a + all;
    for (int len = S; len >= 2; len >>= 1) {
        fft_inv_stage<<<hk_grid(half, 256), 256, 0, c->stream>>>(a, S, len, M, c->d_zeta, c->d_rot_group, half);
        ++c->launches;
    }
    bitrev_copy<<<hk_grid(all, 256), 256, 0, c->stream>>>(a, b2, S, bits, all); ++c->launches;
    round_to_limbs<<<hk_grid(all, 256), 256, 0, c->stream>>>(b2, S, c->log_n, 1.0 / (double)S, scale, level + 1,
                                                             B, c->d_modq, pt, all); ++c->launches;
    HK_LAUNCH_CHECK(c, "encode");
    return ntt_fwd_launch(c, pt, 0, level + 1, B, 0);
}

// shared with crypt.cu: coefficient-domain values (as doubles / scale) -> slots
int hk_decode_launch(hk_ctx *c, double2 *w, double2 *tmp, int B, double *slots);

__global__ void store_re(const double2 *__restrict__ a, double *__restrict__ out, long long total) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) out[i] = a[i].x;
}

int hk_decode_launch(hk_ctx *c, double2 *w, double2 *tmp, int B, double *slots) {
    const int S = c->slots, M = 2 * c->n, bits = c->log_n - 1;
    const long long all = (long long)B * S, half = (long long)B * (S / 2);
    bitrev_copy<<<hk_grid(all, 256), 256, 0, c->stream>>>(w, tmp, S, bits, all); ++c->launches;
    for (int len = 2; len <= S; len <<= 1) {
        fft_fwd_stage<<<hk_grid(half, 256), 256, 0, c->stream>>>(tmp, S, len, M, c->d_zeta, c->d_rot_group,
                                                                half);
        ++c->launches;
    }
    store_re<<<hk_grid(all, 256), 256, 0, c->stream>>>(tmp, slots, all); ++c->launches;
    HK_LAUNCH_CHECK(c, "decode");
    return HK_OK;
}

extern "C" int hk_encode(hk_ctx *c, const double *slots, int32_t B, int32_t level, double scale, uint64_t *pt) {
    if (level < 0 || level >= c->n_q || B < 0) return hk_fail(c, HK_E_ARG, "encode: level %d out of range", level);
    if (B == 0) return HK_OK;
    const long long all = (long long)B * c->slots;
    double2 *a = (double2 *)hk_workspace(c, sizeof(double2) * 2 * all);
    if (!a) return hk_fail(c, HK_E_NOMEM, "encode workspace");
    load_slots<<<hk_grid(all, 256), 256, 0, c->stream>>>(slots, a, all); ++c->launches;
    return encode_loaded(c, a, B, level, scale, pt);
}

extern "C" int hk_encode_diagonals(hk_ctx *c, const double *W, int32_t n_o, int32_t n_in, int32_t m, int32_t base,
                                   int32_t count, int32_t nb, int32_t level, double scale, uint64_t *pt) {
    if (level < 0 || level >= c->n_q || count < 0) return hk_fail(c, HK_E_ARG, "encode_diagonals: level/count");
    if (n_o < 1 || n_in < 1 || m < n_o || m < n_in || m > c->slots || base < 0 || base + count > m || nb < 1)
        return hk_fail(c, HK_E_ARG, "encode_diagonals: shape (%d x %d, m %d, base %d, count %d)", n_o, n_in, m, base,
                       count);
    if (count == 0) return HK_OK;
    const long long all = (long long)count * c->slots;
    double2 *a = (double2 *)hk_workspace(c, sizeof(double2) * 2 * all);
    if (!a) return hk_fail(c, HK_E_NOMEM, "encode_diagonals workspace");
    gen_diagonals<<<hk_grid(all, 256), 256, 0, c->stream>>>(W, n_o, n_in, m, base, nb, c->slots, a, all);
    ++c->launches;
    return encode_loaded(c, a, count, level, scale, pt);
}

extern "C" int hk_encode_const(hk_ctx *c, double v, int32_t level, double scale, uint64_t *res) {
    // host-side scalar: residues of round(v * scale) (no device work)
    if (level < 0 || level >= c->n_q) return hk_fail(c, HK_E_ARG, "encode_const: level out of range");
    const double x = v * scale;
    if (!(std::fabs(x) < 9.0e18)) return hk_fail(c, HK_E_ARG, "encode_const: |c * scale| overflows 63 bits");
    const long long k = llrint(x);
    for (int l = 0; l <= level; ++l) {
        const uint64_t q = c->mod_h[l];
        res[l] = k >= 0 ? (uint64_t)k % q : q - 1 - ((uint64_t)(-(k + 1)) % q);
    }
    return HK_OK;
}
