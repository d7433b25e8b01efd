// common.cuh — shared device arithmetic and the engine context (sm_100a).
//
// All moduli are primes < 2^61 (the parameter generator keeps them < 2^50);
// residues are canonical in [0, q) at every kernel boundary so results are
// bit-identical to the CPU oracle (oracle/ckks_oracle.c).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/hekan.h"

typedef unsigned __int128 u128;

#define HK_MAX_MOD 128

// ---------------------------------------------------------------------------
// modular arithmetic
// ---------------------------------------------------------------------------
struct ModQ {
    uint64_t q;    // prime
    uint64_t mu;   // floor(2^(63+k) / q), k = bitlen(q)
    uint32_t k;    // bit length of q
};

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}
// Shoup: a * w mod q for any a < 2^64, wp = floor(w * 2^64 / q)
__device__ __forceinline__ uint64_t mul_shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t hi = __umul64hi(a, wp);
    uint64_t r = a * w - hi * q;
    return r >= q ? r - q : r;
}
// lazy Shoup: result in [0, 2q)
__device__ __forceinline__ uint64_t mul_shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    return a * w - __umul64hi(a, wp) * q;
}
// Barrett on a 128-bit value x = hi:lo < 2^(2k): one mulhi estimate, <= 2 corrections
__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo, const ModQ &m) {
    uint64_t t = (hi << (65 - m.k)) | (lo >> (m.k - 1));
    uint64_t q3 = __umul64hi(t, m.mu);
    uint64_t r = lo - q3 * m.q;
    if (r >= m.q) r -= m.q;
    if (r >= m.q) r -= m.q;
    return r;
}
__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const ModQ &m) {
    return reduce128(__umul64hi(a, b), a * b, m);
}
// any signed 64-bit value mod q (Barrett, no 64-bit division)
__device__ __forceinline__ uint64_t smod_q(int64_t v, const ModQ &m) {
    const uint64_t a = v < 0 ? 0ull - (uint64_t)v : (uint64_t)v;
    const uint64_t r = reduce128(0, a, m);
    return (v < 0 && r) ? m.q - r : r;
}
// 128-bit accumulate
__device__ __forceinline__ void mac128(uint64_t &hi, uint64_t &lo, uint64_t a, uint64_t b) {
    uint64_t l = a * b, h = __umul64hi(a, b);
    lo += l;
    hi += h + (lo < l);
}
// reduce an arbitrary 128-bit value (hi may exceed the < q^2 bound): fold hi first
__device__ __forceinline__ uint64_t reduce128_any(uint64_t hi, uint64_t lo, const ModQ &m,
                                                  uint64_t two64_mod_q, uint64_t two64_sh) {
    // hi*2^64 + lo = (hi mod q)*2^64 + lo  (mod q)
    uint64_t h = mul_shoup(hi, two64_mod_q, two64_sh, m.q);  // hi * 2^64 mod q
    uint64_t l = lo >= m.q ? lo % m.q : lo;
    return add_mod(h, l, m.q);
}

// 25-bit split multiply-accumulate (all primes are in (2^40, 2^50)): for
// x, y < 2^50, x*y = x1 y1 2^50 + (x1 y0 + x0 y1) 2^25 + x0 y0 with every
// partial product < 2^50; each term is one IMAD.WIDE.U32 with fused 64-bit
// accumulate. Sums of up to 64 products stay below 2^57 per accumulator.
#define HK_M25 0x1FFFFFFu
struct Acc3 {
    uint64_t s0, s1, s2;
};
__device__ __forceinline__ void acc3_zero(Acc3 &a) { a.s0 = a.s1 = a.s2 = 0; }
__device__ __forceinline__ void split25(uint64_t x, uint32_t &x0, uint32_t &x1) {
    x0 = (uint32_t)x & HK_M25;
    x1 = (uint32_t)(x >> 25);
}
__device__ __forceinline__ uint64_t mad_wide(uint32_t x, uint32_t y, uint64_t acc) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(x), "r"(y), "l"(acc));
    return r;
}
__device__ __forceinline__ void acc3_mac(Acc3 &a, uint32_t x0, uint32_t x1, uint32_t y0, uint32_t y1) {
    a.s0 = mad_wide(x0, y0, a.s0);
    a.s1 = mad_wide(x0, y1, a.s1);
    a.s1 = mad_wide(x1, y0, a.s1);
    a.s2 = mad_wide(x1, y1, a.s2);
}
__device__ __forceinline__ void acc3_mac(Acc3 &a, uint64_t x, uint64_t y) {
    uint32_t x0, x1, y0, y1;
    split25(x, x0, x1);
    split25(y, y0, y1);
    acc3_mac(a, x0, x1, y0, y1);
}
// X = s2 2^50 + s1 2^25 + s0 < 64 * 2^100 = 2^106 < 2^(63+k) for every prime
// (q > 2^44, so k >= 45): one Barrett step suffices.
__device__ __forceinline__ uint64_t acc3_reduce(const Acc3 &a, const ModQ &m) {
    uint64_t lo = a.s0, hi = 0;
    uint64_t t = a.s1 << 25;
    lo += t;
    hi += (lo < t) + (a.s1 >> 39);
    t = a.s2 << 50;
    lo += t;
    hi += (lo < t) + (a.s2 >> 14);
    return reduce128(hi, lo, m);
}
// Shoup multiply with a 3 x IMAD.WIDE quotient estimate (undershoot <= 2),
// canonical result. w < q < 2^50, wp = floor(w 2^64 / q), any y < 2^64.
__device__ __forceinline__ uint64_t mul_shoup_fast(uint64_t y, uint64_t w, uint64_t wp, uint64_t q) {
    const uint32_t y0 = (uint32_t)y, y1 = (uint32_t)(y >> 32);
    const uint32_t w0 = (uint32_t)wp, w1 = (uint32_t)(wp >> 32);
    const uint64_t Q = ((uint64_t)y1 * w1) + (((uint64_t)y1 * w0) >> 32) + (((uint64_t)y0 * w1) >> 32);
    uint64_t r = y * w - Q * q;  // [0, 4q)
    r = r >= 2 * q ? r - 2 * q : r;
    return r >= q ? r - q : r;
}

__device__ __forceinline__ uint32_t brev_bits(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

// Counter-mode randomness: ChaCha20 keyed by a 256-bit seed, 64-bit block
// counter (words 12-13) and the 64-bit stream id as the nonce (words 14-15).
// Word c of a stream is the 64-bit pair (2(c mod 8), 2(c mod 8)+1) of block
// c / 8 — identical to the oracle (oracle/ckks_oracle.c: rng64).
struct HkSeed {
    uint64_t w[4];
};
__device__ __forceinline__ uint32_t hk_rotl(uint32_t x, int r) { return __funnelshift_l(x, x, r); }
#define HK_QR(a, b, c, d)                                                              \
    a += b; d ^= a; d = hk_rotl(d, 16); c += d; b ^= c; b = hk_rotl(b, 12);            \
    a += b; d ^= a; d = hk_rotl(d, 8);  c += d; b ^= c; b = hk_rotl(b, 7);
// the 8 64-bit words of block `block` of `stream`
__device__ __forceinline__ void hk_chacha_block(const HkSeed &key, uint64_t block, uint64_t stream,
                                                uint64_t out[8]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                      (uint32_t)key.w[0], (uint32_t)(key.w[0] >> 32), (uint32_t)key.w[1], (uint32_t)(key.w[1] >> 32),
                      (uint32_t)key.w[2], (uint32_t)(key.w[2] >> 32), (uint32_t)key.w[3], (uint32_t)(key.w[3] >> 32),
                      (uint32_t)block, (uint32_t)(block >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = s[i];
#pragma unroll 1
    for (int r = 0; r < 10; ++r) {
        HK_QR(x[0], x[4], x[8], x[12]) HK_QR(x[1], x[5], x[9], x[13])
        HK_QR(x[2], x[6], x[10], x[14]) HK_QR(x[3], x[7], x[11], x[15])
        HK_QR(x[0], x[5], x[10], x[15]) HK_QR(x[1], x[6], x[11], x[12])
        HK_QR(x[2], x[7], x[8], x[13]) HK_QR(x[3], x[4], x[9], x[14])
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        out[j] = (uint64_t)(x[2 * j] + s[2 * j]) | ((uint64_t)(x[2 * j + 1] + s[2 * j + 1]) << 32);
}
__device__ __forceinline__ int64_t cbd21(uint64_t x) {
    return (int64_t)__popcll(x & 0x1FFFFFull) - (int64_t)__popcll((x >> 21) & 0x1FFFFFull);
}
__device__ __forceinline__ uint64_t smod_dev(int64_t v, uint64_t q) {  // |v| < q only (sampled noise)
    return v < 0 ? q - (uint64_t)(-v) : (uint64_t)v;
}
enum { ST_SECRET = 1, ST_ENC_A = 2, ST_ENC_E = 3, ST_KEY_A = 0x100, ST_KEY_E = 0x200 };

// ---------------------------------------------------------------------------
// basis-conversion tables for one (source set -> target set) conversion
// ---------------------------------------------------------------------------
struct ConvTable {
    int n_src, n_dst;
    uint64_t *d_inv;      // [n_src]  (Q_src/q_i)^-1 mod q_i
    uint64_t *d_inv_sh;   // [n_src]  Shoup companions
    uint64_t *d_hat;      // [n_dst][n_src] (Q_src/q_i) mod t
    int32_t *d_src_mod;   // [n_src]  chain index of each source prime
    int32_t *d_dst_mod;   // [n_dst]  chain index of each target prime
    // centred (exact) conversion: u = round(sum_i v_i / m_i) in float64, target t adds
    // u * (-M mod q_t), so the result is the centred remainder exactly (ModUp digits,
    // ModDown, merged ModDown + rescale); nullptr = plain fast conversion
    double *d_src_invd;   // [n_src]  1 / m_i
    uint64_t *d_neg_m;    // [n_dst]  -M mod q_t
    // tensor-core path (conv_tc.cu, <= 16 source slots): B[(t, b)][(i, a)] = byte b of
    // hat[t][i] 2^(8a) mod q_t (slot n_src: -M mod q_t), 8 rows per target, 128 bytes per
    // row, canonical no-swizzle UMMA layout
    uint8_t *d_bmat;
};

// A key-switching key truncated to `level`: digits 0..level/alpha, rows
// {q_0..q_level, p_0..p_{K-1}} ([digits][2][rows][N]); rows equal the full key's.
struct GalKey {
    uint64_t *p;
    int level;
    int rows;  // level + 1 + K
};

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct hk_ctx {
    int log_n, n, slots, n_q, n_p, dnum, alpha, n_digits, n_mod;
    int device;
    int n_sm;  // multiprocessors of the device (resident-grid sizing)
    cudaStream_t stream;
    std::vector<uint64_t> mod_h;
    std::vector<ModQ> modq_h;
    // device tables
    ModQ *d_modq;          // [n_mod]
    ulonglong2 *d_tw;      // [n_mod][N] {psi^brv(k), shoup}
    ulonglong2 *d_itw;     // [n_mod][N] {psi^-brv(k), shoup}
    ulonglong2 *d_ninv;    // [n_mod] {N^-1, shoup}
    // fused 2^16 kernels (ntt16.cuh), N = 2^16 (root psi) or 2^17 (root psi^2 per half); stride 2^16
    double2 *d_twf;        // [n_mod][2^16] {w^brv(k), w^brv(k)/q} as float64
    double2 *d_itwf;       // [n_mod][2^16] inverse twiddles, float64
    double2 *d_ninvf;      // [n_mod][2] {2^-16, 2^-16/q}, {2^-16 Ti[1], .../q} (inverse stage 0 fused)
    double2 *d_fmod;       // [n_mod] {q, 1/q} (every N)
    double *d_twist;       // [n_mod][256][256] w^(c (2 brv8(r) + 1 - 256)) as float64 (rows; w/q formed in-register)
    double *d_twistq;      // [n_mod][256][256] the correctly rounded w / q of d_twist (read for large primes only)
    double *d_itwist;      // [n_mod][256][256] inverse twist
    ulonglong2 *d_n17;     // N = 2^17: [n_mod][4][2^16] radix-2 pre/post twists (ntt.cu)
    ulonglong2 *d_n17w;    // N = 2^17: [n_mod][2] {psi^(2^16), inverse}
    double2 *d_zeta;       // [2N]
    uint32_t *d_rot_group; // [S]
    // rescale: qinv[l][i] = q_l^-1 mod q_i (i < l), Shoup pairs
    ulonglong2 *d_rs_qinv; // [n_q][n_q]
    // key switching: per (level, digit) ModUp tables; ModDown (P -> q) tables
    std::vector<std::vector<ConvTable>> modup;  // [level][digit]
    ConvTable moddown;                          // sources: specials, targets: q_0..q_{n_q-1}
    ulonglong2 *d_pinv;                         // [n_q] P^-1 mod q_i
    // ModDown merged with rescale (hk_mul): per level l >= 1, sources
    // {p_0..p_{K-1}, q_l} -> targets q_0..q_{l-1}
    std::vector<ConvTable> mdrs;                // [n_q] (entry 0 unused)
    ulonglong2 *d_pmod;                         // [n_q] P mod q_i (Shoup pairs)
    ulonglong2 *d_mqinv;                        // [n_q][n_q] (P q_l)^-1 mod q_t
    // keys
    uint64_t *d_sk;                 // [n_mod][N]
    uint64_t *d_relin;              // [n_digits][2][n_mod][N]
    std::map<uint32_t, GalKey> gal;
    bool have_keys;
    unsigned long long launches;    // kernels enqueued by this context (bench evidence)
    // scratch workspace (grown on demand, stream-ordered use only)
    void *ws;
    size_t ws_bytes;
    std::string err;
};

// error plumbing
int hk_fail(hk_ctx *c, int code, const char *fmt, ...);
int hk_cuda_check(hk_ctx *c, cudaError_t e, const char *what);
#define HK_CUDA(c, call)                                                  \
    do {                                                                  \
        cudaError_t _e = (call);                                          \
        if (_e != cudaSuccess) return hk_cuda_check((c), _e, #call);      \
    } while (0)
#define HK_LAUNCH_CHECK(c, what)                                          \
    do {                                                                  \
        cudaError_t _e = cudaGetLastError();                              \
        if (_e != cudaSuccess) return hk_cuda_check((c), _e, what);       \
    } while (0)

// workspace: returns a pointer to at least `bytes` bytes (reallocates)
void *hk_workspace(hk_ctx *c, size_t bytes);

// internal launchers (defined across translation units)
int ntt_fwd_launch(hk_ctx *c, uint64_t *buf, int limb0, int n_limbs, int batch, int limb_stride_polys);
int ntt_inv_launch(hk_ctx *c, uint64_t *buf, int limb0, int n_limbs, int batch, int limb_stride_polys);
int rescale_launch(hk_ctx *c, const uint64_t *in, int l, int batch, uint64_t *out, uint64_t *scratch);
bool conv_tc_ok(const hk_ctx *c, const ConvTable &T, int n_dst, long long BN, int prescaled);
int conv_tc_launch(hk_ctx *c, const ConvTable &T, const uint64_t *src, uint64_t *dst, int mode, int l, long long BN,
                   int n_dst);
int keyswitch_launch(hk_ctx *c, const uint64_t *d, int l, int batch, const uint64_t *const *keys,
                     const uint32_t *galois, int n_keys, uint64_t *const *outs_c0,
                     const uint64_t *c0_src, bool add_c0_auto);

static inline int hk_grid(long long work, int threads) {
    long long b = (work + threads - 1) / threads;
    if (b > (1ll << 30)) b = 1ll << 30;
    return (int)(b < 1 ? 1 : b);
}
