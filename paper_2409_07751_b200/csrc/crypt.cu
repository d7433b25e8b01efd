// crypt.cu — key generation, RLWE encryption and decryption on the GPU.
//
// Replaces HeBackend.encrypt/decrypt (hekan/backend.py:160-170), which in the
// reference copy slots. Randomness is counter-mode ChaCha20 (common.cuh:
// hk_chacha_block; seed, stream, counter) so the oracle reproduces every key
// and ciphertext bit for bit. Sampling kernels give each thread 8 consecutive
// coefficients: one ChaCha block per stream per thread (N >= 8).
#include "common.cuh"

int hk_decode_launch(hk_ctx *c, double2 *w, double2 *tmp, int B, double *slots);

namespace {

// residues of a ternary secret in every limb: s[m][k], 8 coefficients per thread
__global__ void sample_secret(uint64_t *__restrict__ s, HkSeed seed, int log_n, int nm,
                              const ModQ *__restrict__ mq) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int N = 1 << log_n;
    if (gid >= ((long long)nm * N) >> 3) return;
    const long long o = gid << 3;
    const int m = (int)(o >> log_n), k0 = (int)(o & (N - 1));
    uint64_t r[8];
    hk_chacha_block(seed, (uint64_t)k0 >> 3, ST_SECRET, r);
#pragma unroll
    for (int j = 0; j < 8; ++j) s[o + j] = smod_dev((int64_t)(r[j] % 3) - 1, mq[m].q);
}

__global__ void square_mod(const uint64_t *__restrict__ a, uint64_t *__restrict__ out, int log_n, int nm,
                           const ModQ *__restrict__ mq) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= ((long long)nm << log_n)) return;
    const ModQ m = mq[gid >> log_n];
    out[gid] = mul_mod(a[gid], a[gid], m);
}

// NTT-domain automorphism out[j] = in[src_g(j)], per polynomial of N
__device__ __forceinline__ uint32_t auto_src(uint32_t j, uint32_t g, int log_n) {
    const uint32_t M = 2u << log_n;
    const uint32_t e = 2u * brev_bits(j, log_n) + 1u;
    const uint32_t eg = (uint32_t)(((uint64_t)e * g) & (M - 1));
    return brev_bits((eg - 1u) >> 1, log_n);
}

__global__ void automorph_polys(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, uint32_t g,
                                int log_n, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int N = 1 << log_n;
    const long long poly = gid >> log_n;
    const uint32_t j = (uint32_t)(gid & (N - 1));
    out[gid] = in[(poly << log_n) + auto_src(j, g, log_n)];
}

// key digit j: a (uniform, NTT domain) and e (coefficient domain, reduced)
// key rows r < rows: modulus m = r <= top ? r : n_q + (r - top - 1) (top = key level)
__device__ __forceinline__ int key_row_mod(int r, int top, int n_q) { return r <= top ? r : n_q + (r - top - 1); }

__global__ void ks_sample(uint64_t *__restrict__ b, uint64_t *__restrict__ a, HkSeed seed, uint64_t stream_a,
                          uint64_t stream_e, int log_n, int rows, int top, int n_q, const ModQ *__restrict__ mq) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int N = 1 << log_n;
    if (gid >= ((long long)rows * N) >> 3) return;
    const long long o = gid << 3;
    const int r = (int)(o >> log_n), k0 = (int)(o & (N - 1));
    const int m = key_row_mod(r, top, n_q);
    const ModQ mm = mq[m];
    uint64_t ra[8], re[8];
    hk_chacha_block(seed, ((uint64_t)m * N + k0) >> 3, stream_a, ra);
    hk_chacha_block(seed, (uint64_t)k0 >> 3, stream_e, re);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a[o + j] = reduce128(0, ra[j], mm);  // == rng % q (exact Barrett)
        b[o + j] = smod_dev(cbd21(re[j]), mm.q);
    }
}

// b = e_ntt - a*s (+ P*s' on digit limbs); s, sp are full [n_mod][N]
__global__ void ks_finish(uint64_t *__restrict__ b, const uint64_t *__restrict__ a, const uint64_t *__restrict__ s,
                          const uint64_t *__restrict__ sp, const uint64_t *__restrict__ pmod, int d0, int d1,
                          int log_n, int rows, int top, int n_q, const ModQ *__restrict__ mq) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= ((long long)rows << log_n)) return;
    const int r = (int)(gid >> log_n), k = (int)(gid & ((1 << log_n) - 1));
    const int m = key_row_mod(r, top, n_q);
    const ModQ mm = mq[m];
    const long long o = ((long long)m << log_n) + k;
    uint64_t v = sub_mod(b[gid], mul_mod(a[gid], s[o], mm), mm.q);
    if (m >= d0 && m < d1) v = add_mod(v, mul_mod(pmod[m], sp[o], mm), mm.q);
    b[gid] = v;
}

// encryption: c1 = a (uniform), e (coefficient) into c0 temporarily
// sample index = first + b: a sharded batch encrypts exactly as the whole batch
__global__ void enc_sample(uint64_t *__restrict__ c0, uint64_t *__restrict__ c1, HkSeed seed, uint64_t first,
                           int log_n, int nl, int B, const ModQ *__restrict__ mq) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int N = 1 << log_n;
    if (gid >= ((long long)nl * B * N) >> 3) return;
    const long long o = gid << 3;
    const int k0 = (int)(o & (N - 1));
    const long long lb = o >> log_n;
    const int l = (int)(lb / B), b = (int)(lb - (long long)l * B);
    const ModQ mm = mq[l];
    const uint64_t smp = first + (uint64_t)b;
    uint64_t ra[8], re[8];
    hk_chacha_block(seed, ((smp * nl + l) * N + k0) >> 3, ST_ENC_A, ra);
    hk_chacha_block(seed, (smp * N + k0) >> 3, ST_ENC_E, re);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        c1[o + j] = reduce128(0, ra[j], mm);  // == rng % q
        c0[o + j] = smod_dev(cbd21(re[j]), mm.q);
    }
}

__global__ void enc_finish(uint64_t *__restrict__ c0, const uint64_t *__restrict__ c1,
                           const uint64_t *__restrict__ pt, const uint64_t *__restrict__ s, int log_n, int B,
                           const ModQ *__restrict__ mq, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int N = 1 << log_n;
    const int k = (int)(gid & (N - 1));
    const int l = (int)((gid >> log_n) / B);
    const ModQ m = mq[l];
    const uint64_t v = add_mod(pt[gid], c0[gid], m.q);
    c0[gid] = sub_mod(v, mul_mod(c1[gid], s[(size_t)l * N + k], m), m.q);
}

// m_l = c0_l + c1_l * s_l for limbs l < use
__global__ void dec_phase(const uint64_t *__restrict__ ct, int nl, int use, int B, const uint64_t *__restrict__ s,
                          int log_n, const ModQ *__restrict__ mq, uint64_t *__restrict__ m_out, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int N = 1 << log_n;
    const int k = (int)(gid & (N - 1));
    const int l = (int)((gid >> log_n) / B);
    const ModQ m = mq[l];
    const size_t poly = (size_t)nl * B * N;
    m_out[gid] = add_mod(ct[gid], mul_mod(ct[poly + gid], s[(size_t)l * N + k], m), m.q);
}

__device__ __forceinline__ double center_to_double(uint64_t x0, uint64_t x1, int use, uint64_t q0, uint64_t q1,
                                                   uint64_t i0, uint64_t i1, const ModQ &m0, const ModQ &m1) {
    if (use == 1) {
        const int64_t v = x0 > q0 / 2 ? -(int64_t)(q0 - x0) : (int64_t)x0;
        return (double)v;
    }
    const u128 Q = (u128)q0 * q1;
    u128 v = (u128)mul_mod(x0, i0, m0) * q1 + (u128)mul_mod(x1, i1, m1) * q0;
    if (v >= Q) v -= Q;
    const bool neg = v > Q / 2;
    const u128 mag = neg ? Q - v : v;
    const double d = __dadd_rn(__dmul_rn(__ull2double_rn((uint64_t)(mag >> 64)), 18446744073709551616.0),
                               __ull2double_rn((uint64_t)mag));
    return neg ? -d : d;
}

__global__ void dec_center(const uint64_t *__restrict__ m, int use, int B, int log_n, double scale,
                           const ModQ *__restrict__ mq, uint64_t i0, uint64_t i1, double2 *__restrict__ w,
                           long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;  // B * S
    const int N = 1 << log_n, S = N >> 1;
    const long long b = gid / S;
    const int i = (int)(gid - b * S);
    const ModQ m0 = mq[0], m1 = mq[use > 1 ? 1 : 0];
    const uint64_t *r0 = m + (size_t)b * N;
    const uint64_t *r1 = m + ((size_t)B + b) * N;
    const double a = center_to_double(r0[i], use > 1 ? r1[i] : 0, use, m0.q, m1.q, i0, i1, m0, m1);
    const double bb = center_to_double(r0[i + S], use > 1 ? r1[i + S] : 0, use, m0.q, m1.q, i0, i1, m0, m1);
    w[gid] = make_double2(__ddiv_rn(a, scale), __ddiv_rn(bb, scale));
}

uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
uint64_t h_inv(uint64_t a, uint64_t q) {
    uint64_t r = 1, e = q - 2;
    a %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, a, q);
        a = h_mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

// key-switching key for target s' (device [nm][N], NTT) into key [n_digits][2][nm][N]
int make_ks_key(hk_ctx *c, const HkSeed &seed, uint64_t tag, const uint64_t *sprime, uint64_t *key, int top) {
    const int N = c->n, nm = c->n_mod, rows = top + 1 + c->n_p, nd = top / c->alpha + 1;
    std::vector<uint64_t> pmod(nm, 0);
    for (int i = 0; i < c->n_q; ++i) {
        uint64_t acc = 1;
        for (int k = 0; k < c->n_p; ++k) acc = h_mulmod(acc, c->mod_h[c->n_q + k] % c->mod_h[i], c->mod_h[i]);
        pmod[i] = acc;
    }
    uint64_t *d_pmod = nullptr;
    HK_CUDA(c, cudaMalloc(&d_pmod, sizeof(uint64_t) * nm));
    HK_CUDA(c, cudaMemcpyAsync(d_pmod, pmod.data(), sizeof(uint64_t) * nm, cudaMemcpyHostToDevice, c->stream));
    const long long tot = (long long)rows * N;
    for (int j = 0; j < nd; ++j) {
        const int d0 = j * c->alpha, d1 = std::min((j + 1) * c->alpha, c->n_q);
        uint64_t *bj = key + ((size_t)j * 2 + 0) * rows * N;
        uint64_t *aj = key + ((size_t)j * 2 + 1) * rows * N;
        ks_sample<<<hk_grid(tot >> 3, 256), 256, 0, c->stream>>>(bj, aj, seed, ST_KEY_A + tag * 64 + j,
                                                              ST_KEY_E + tag * 64 + j, c->log_n, rows, top, c->n_q,
                                                              c->d_modq); ++c->launches;
        int rc = ntt_fwd_launch(c, bj, 0, top + 1, 1, 0);
        if (!rc) rc = ntt_fwd_launch(c, bj + (size_t)(top + 1) * N, c->n_q, c->n_p, 1, 0);
        if (rc) return rc;
        ks_finish<<<hk_grid(tot, 256), 256, 0, c->stream>>>(bj, aj, c->d_sk, sprime, d_pmod, d0, d1, c->log_n,
                                                              rows, top, c->n_q, c->d_modq); ++c->launches;
    }
    HK_LAUNCH_CHECK(c, "make_ks_key");
    HK_CUDA(c, cudaStreamSynchronize(c->stream));
    cudaFree(d_pmod);
    return HK_OK;
}

}  // namespace

int automorph_launch(hk_ctx *c, const uint64_t *in, uint64_t *out, uint32_t g, long long n_polys) {
    const long long total = n_polys << c->log_n;
    automorph_polys<<<hk_grid(total, 256), 256, 0, c->stream>>>(in, out, g, c->log_n, total); ++c->launches;
    HK_LAUNCH_CHECK(c, "automorph");
    return HK_OK;
}

extern "C" {

uint64_t hk_key_words(const hk_ctx *c, int32_t which) {
    const uint64_t nm = (uint64_t)c->n_mod, N = (uint64_t)c->n;
    if (which == 0) return nm * N;
    return (uint64_t)c->n_digits * 2 * nm * N;
}

static HkSeed to_seed(const uint64_t w[4]) { return HkSeed{{w[0], w[1], w[2], w[3]}}; }

int hk_keygen(hk_ctx *c, const uint64_t seed_words[4]) {
    const int N = c->n, nm = c->n_mod;
    if (!seed_words) return hk_fail(c, HK_E_ARG, "keygen: null seed");
    const HkSeed seed = to_seed(seed_words);
    cudaFree(c->d_sk);
    cudaFree(c->d_relin);
    for (auto &kv : c->gal) cudaFree(kv.second.p);
    c->gal.clear();
    c->d_sk = c->d_relin = nullptr;
    HK_CUDA(c, cudaMalloc(&c->d_sk, sizeof(uint64_t) * nm * N));
    HK_CUDA(c, cudaMalloc(&c->d_relin, sizeof(uint64_t) * hk_key_words(c, 1)));
    const long long tot = (long long)nm * N;
    sample_secret<<<hk_grid(tot >> 3, 256), 256, 0, c->stream>>>(c->d_sk, seed, c->log_n, nm, c->d_modq); ++c->launches;
    int rc = ntt_fwd_launch(c, c->d_sk, 0, nm, 1, 0);
    if (rc) return rc;
    uint64_t *s2 = nullptr;
    HK_CUDA(c, cudaMalloc(&s2, sizeof(uint64_t) * nm * N));
    square_mod<<<hk_grid(tot, 256), 256, 0, c->stream>>>(c->d_sk, s2, c->log_n, nm, c->d_modq); ++c->launches;
    rc = make_ks_key(c, seed, 0, s2, c->d_relin, c->n_q - 1);
    cudaFree(s2);
    if (rc) return rc;
    c->have_keys = true;
    return HK_OK;
}

int hk_has_galois_key(const hk_ctx *c, uint32_t g) {
    auto it = c->gal.find(g);
    return it == c->gal.end() ? 0 : it->second.level + 1;
}

int hk_add_galois_keys_level(hk_ctx *c, const uint64_t seed_words[4], const uint32_t *gs, int32_t n,
                             int32_t level) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (!seed_words) return hk_fail(c, HK_E_ARG, "galois keys: null seed");
    const HkSeed seed = to_seed(seed_words);
    if (level < 0 || level >= c->n_q) return hk_fail(c, HK_E_ARG, "galois key level %d out of range", level);
    const int N = c->n, nm = c->n_mod;
    const uint32_t M = 2u * (uint32_t)N;
    for (int i = 0; i < n; ++i) {
        const uint32_t g = gs[i];
        if ((g & 1u) == 0 || g >= M) return hk_fail(c, HK_E_ARG, "galois element %u invalid", g);
        auto it = c->gal.find(g);
        if (it != c->gal.end() && it->second.level >= level) continue;
        const int rows = level + 1 + c->n_p, nd = level / c->alpha + 1;
        uint64_t *sg = nullptr, *key = nullptr;
        HK_CUDA(c, cudaMalloc(&sg, sizeof(uint64_t) * nm * N));
        HK_CUDA(c, cudaMalloc(&key, sizeof(uint64_t) * (size_t)nd * 2 * rows * N));
        int rc = automorph_launch(c, c->d_sk, sg, g, nm);
        if (!rc) rc = make_ks_key(c, seed, 1 + (uint64_t)g, sg, key, level);
        cudaFree(sg);
        if (rc) {
            cudaFree(key);
            return rc;
        }
        if (it != c->gal.end()) cudaFree(it->second.p);  // grown to a higher level
        c->gal[g] = GalKey{key, level, rows};
    }
    return HK_OK;
}

int hk_add_galois_keys(hk_ctx *c, const uint64_t seed[4], const uint32_t *gs, int32_t n) {
    return hk_add_galois_keys_level(c, seed, gs, n, c->n_q - 1);
}

int hk_export_key(hk_ctx *c, int32_t which, uint32_t g, uint64_t *out) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "no keys");
    const uint64_t *src = nullptr;
    if (which == 0) src = c->d_sk;
    else if (which == 1) src = c->d_relin;
    else if (c->gal.count(g)) {
        if (c->gal[g].level != c->n_q - 1) return hk_fail(c, HK_E_ARG, "galois key %u is level-truncated", g);
        src = c->gal[g].p;
    }
    if (!src) return hk_fail(c, HK_E_NOKEY, "no galois key for %u", g);
    HK_CUDA(c, cudaMemcpyAsync(out, src, sizeof(uint64_t) * hk_key_words(c, which == 0 ? 0 : 1),
                               cudaMemcpyDeviceToDevice, c->stream));
    return HK_OK;
}

int hk_encrypt(hk_ctx *c, const uint64_t *pt, int32_t level, int32_t B, const uint64_t seed_words[4],
               uint64_t first_sample, uint64_t *ct) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (!seed_words) return hk_fail(c, HK_E_ARG, "encrypt: null seed");
    const HkSeed seed = to_seed(seed_words);
    if (level < 0 || level >= c->n_q || B < 0) return hk_fail(c, HK_E_ARG, "encrypt: level out of range");
    if (B == 0) return HK_OK;
    const int nl = level + 1;
    const long long tot = (long long)nl * B * c->n;
    uint64_t *c0 = ct, *c1 = ct + tot;
    enc_sample<<<hk_grid(tot >> 3, 256), 256, 0, c->stream>>>(c0, c1, seed, first_sample, c->log_n, nl, B,
                                                                   c->d_modq); ++c->launches;
    int rc = ntt_fwd_launch(c, c0, 0, nl, B, 0);
    if (rc) return rc;
    enc_finish<<<hk_grid(tot, 256), 256, 0, c->stream>>>(c0, c1, pt, c->d_sk, c->log_n, B, c->d_modq, tot); ++c->launches;
    HK_LAUNCH_CHECK(c, "encrypt");
    return HK_OK;
}

int hk_decrypt(hk_ctx *c, const uint64_t *ct, int32_t level, int32_t B, double scale, double *slots) {
    if (!c->have_keys) return hk_fail(c, HK_E_NOKEY, "keygen first");
    if (level < 0 || level >= c->n_q || B < 0) return hk_fail(c, HK_E_ARG, "decrypt: level out of range");
    if (B == 0) return HK_OK;
    const int N = c->n, S = c->slots, nl = level + 1, use = nl >= 2 ? 2 : 1;
    const size_t mwords = (size_t)2 * B * N;
    const size_t cwords = (size_t)B * S;
    char *ws = (char *)hk_workspace(c, sizeof(uint64_t) * mwords + 2 * sizeof(double2) * cwords);
    if (!ws) return hk_fail(c, HK_E_NOMEM, "decrypt workspace");
    uint64_t *m = (uint64_t *)ws;
    double2 *w = (double2 *)(ws + sizeof(uint64_t) * mwords);
    double2 *tmp = w + cwords;
    const long long tot = (long long)use * B * N;
    dec_phase<<<hk_grid(tot, 256), 256, 0, c->stream>>>(ct, nl, use, B, c->d_sk, c->log_n, c->d_modq, m, tot); ++c->launches;
    int rc = ntt_inv_launch(c, m, 0, use, B, 0);
    if (rc) return rc;
    uint64_t i0 = 0, i1 = 0;
    if (use == 2) {
        const uint64_t q0 = c->mod_h[0], q1 = c->mod_h[1];
        i0 = h_inv(q1 % q0, q0);
        i1 = h_inv(q0 % q1, q1);
    }
    dec_center<<<hk_grid((long long)cwords, 256), 256, 0, c->stream>>>(m, use, B, c->log_n, scale, c->d_modq, i0,
                                                                        i1, w, (long long)cwords); ++c->launches;
    HK_LAUNCH_CHECK(c, "decrypt");
    return hk_decode_launch(c, w, tmp, B, slots);
}

}  // extern "C"
