// ctx.cu — engine context: parameter tables in HBM, errors, workspace.
//
// Replaces BackendConfig + HeBackend.__init__ (hekan/backend.py:23-66,
// :140-143): everything the reference keeps as Python attributes becomes
// device-resident tables built once per context.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

static uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t h_powmod(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, b, q);
        b = h_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static uint64_t h_inv(uint64_t a, uint64_t q) { return h_powmod(a % q, q - 2, q); }
static uint64_t h_shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static uint32_t h_brv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

int hk_fail(hk_ctx *c, int code, const char *fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return code;
}

int hk_cuda_check(hk_ctx *c, cudaError_t e, const char *what) {
    return hk_fail(c, e == cudaErrorMemoryAllocation ? HK_E_NOMEM : HK_E_CUDA, "%s: %s", what,
                   cudaGetErrorString(e));
}

void *hk_workspace(hk_ctx *c, size_t bytes) {
    if (bytes <= c->ws_bytes) return c->ws;
    if (c->ws) {
        cudaStreamSynchronize(c->stream);
        cudaFree(c->ws);
        c->ws = nullptr;
        c->ws_bytes = 0;
    }
    size_t want = bytes + (bytes >> 3);
    if (cudaMalloc(&c->ws, want) != cudaSuccess) {
        cudaGetLastError();
        c->ws = nullptr;
        return nullptr;
    }
    c->ws_bytes = want;
    return c->ws;
}

template <typename T>
static T *upload(const std::vector<T> &v) {
    T *d = nullptr;
    if (v.empty()) return nullptr;
    if (cudaMalloc(&d, sizeof(T) * v.size()) != cudaSuccess) return nullptr;
    cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
    return d;
}

// fast basis conversion table: sources -> targets (chain indices)
static ConvTable make_conv(const std::vector<uint64_t> &mod, const std::vector<int> &src,
                           const std::vector<int> &dst, bool exact = false) {
    ConvTable t;
    t.n_src = (int)src.size();
    t.n_dst = (int)dst.size();
    std::vector<uint64_t> inv(src.size()), inv_sh(src.size()), hat(src.size() * dst.size());
    for (size_t i = 0; i < src.size(); ++i) {
        const uint64_t qi = mod[src[i]];
        uint64_t prod = 1;
        for (size_t k = 0; k < src.size(); ++k)
            if (k != i) prod = h_mulmod(prod, mod[src[k]] % qi, qi);
        inv[i] = h_inv(prod, qi);
        inv_sh[i] = h_shoup(inv[i], qi);
    }
    for (size_t d = 0; d < dst.size(); ++d) {
        const uint64_t qt = mod[dst[d]];
        for (size_t i = 0; i < src.size(); ++i) {
            uint64_t prod = 1;
            for (size_t k = 0; k < src.size(); ++k)
                if (k != i) prod = h_mulmod(prod, mod[src[k]] % qt, qt);
            hat[d * src.size() + i] = prod;
        }
    }
    t.d_inv = upload(inv);
    t.d_inv_sh = upload(inv_sh);
    t.d_hat = upload(hat);
    t.d_src_mod = upload(std::vector<int32_t>(src.begin(), src.end()));
    t.d_dst_mod = upload(std::vector<int32_t>(dst.begin(), dst.end()));
    t.d_src_invd = nullptr;
    t.d_neg_m = nullptr;
    t.d_bmat = nullptr;
    std::vector<uint64_t> negm;
    if (exact) {  // centred conversion: 1/m_i as float64, -M mod q_t (M = product of the sources)
        std::vector<double> invd(src.size());
        for (size_t i = 0; i < src.size(); ++i) invd[i] = 1.0 / (double)mod[src[i]];
        negm.resize(dst.size());
        for (size_t d = 0; d < dst.size(); ++d) {
            const uint64_t qt = mod[dst[d]];
            uint64_t M = 1;
            for (size_t k = 0; k < src.size(); ++k) M = h_mulmod(M, mod[src[k]] % qt, qt);
            negm[d] = (qt - M) % qt;
        }
        t.d_src_invd = upload(invd);
        t.d_neg_m = upload(negm);
    }
    // conv_tc.cu: B[(t, b)][(i, a)] = byte b of (hat[t][i] 2^(8a) mod q_t), one 8-row group
    // (7 bytes + a zero row) x 128 bytes per target in the no-swizzle K-major UMMA layout; a
    // centred conversion carries -M mod q_t as the constant of source slot n_src (the
    // overflow count u rides in the GEMM)
    bool below50 = true;  // 7-byte residues and constants (every generated prime is < 2^50)
    for (int m : src) below50 = below50 && mod[m] < (1ull << 50);
    for (int m : dst) below50 = below50 && mod[m] < (1ull << 50);
    const size_t slots = src.size() + (exact ? 1 : 0);
    if (below50 && slots <= 32) {
        const size_t kb = slots <= 16 ? 128 : 256, sbo = 8 * kb;  // bytes per row, per 8-row group (conv_tc.cu)
        std::vector<uint8_t> b(dst.size() * sbo, 0);
        for (size_t d = 0; d < dst.size(); ++d) {
            const uint64_t qt = mod[dst[d]];
            for (size_t i = 0; i < slots; ++i) {
                uint64_t cst = i < src.size() ? hat[d * src.size() + i] : negm[d];
                for (int a = 0; a < 8; ++a) {
                    for (int bb = 0; bb < 8; ++bb) {
                        const size_t n = d * 8 + bb, kk = i * 8 + a;
                        b[(n / 8) * sbo + (kk / 16) * 128 + (n % 8) * 16 + kk % 16] = (uint8_t)(cst >> (8 * bb));
                    }
                    cst = h_mulmod(cst, 256, qt);
                }
            }
        }
        t.d_bmat = upload(b);
    }
    return t;
}

static void free_conv(ConvTable &t) {
    cudaFree(t.d_inv);
    cudaFree(t.d_inv_sh);
    cudaFree(t.d_hat);
    cudaFree(t.d_src_mod);
    cudaFree(t.d_dst_mod);
    cudaFree(t.d_src_invd);
    cudaFree(t.d_neg_m);
    cudaFree(t.d_bmat);
}

extern "C" {

const char *hk_last_error(const hk_ctx *c) { return c ? c->err.c_str() : "null context"; }
int32_t hk_version(void) { return 1; }
uint64_t hk_launch_count(const hk_ctx *c) { return c ? c->launches : 0; }

int hk_set_stream(hk_ctx *c, void *s) {
    c->stream = (cudaStream_t)s;
    return HK_OK;
}

int hk_sync(hk_ctx *c) {
    HK_CUDA(c, cudaStreamSynchronize(c->stream));
    return HK_OK;
}

int hk_ctx_create(const hk_params *pr, int32_t device, hk_ctx **out) {
    if (!pr || !out || pr->log_n < 3 || pr->log_n > 17 || pr->n_q < 1 || pr->n_p < 1 || pr->dnum < 1 || pr->dnum > 8 ||
        pr->n_q + pr->n_p > HK_MAX_MOD)
        return HK_E_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return HK_E_CUDA;
    hk_ctx *c = new hk_ctx();
    c->device = device;
    c->n_sm = 148;
    cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
    c->stream = 0;
    c->log_n = pr->log_n;
    c->n = 1 << pr->log_n;
    c->slots = c->n / 2;
    c->n_q = pr->n_q;
    c->n_p = pr->n_p;
    c->dnum = pr->dnum;
    c->alpha = (pr->n_q + pr->dnum - 1) / pr->dnum;
    c->n_digits = (pr->n_q + c->alpha - 1) / c->alpha;
    c->n_mod = pr->n_q + pr->n_p;
    c->have_keys = false;
    c->ws = nullptr;
    c->ws_bytes = 0;
    c->launches = 0;
    c->d_sk = c->d_relin = nullptr;
    const int N = c->n, nm = c->n_mod;
    std::vector<uint64_t> psi(nm);
    c->mod_h.resize(nm);
    for (int i = 0; i < pr->n_q; ++i) { c->mod_h[i] = pr->q[i]; psi[i] = pr->psi_q[i]; }
    for (int i = 0; i < pr->n_p; ++i) { c->mod_h[pr->n_q + i] = pr->p[i]; psi[pr->n_q + i] = pr->psi_p[i]; }
    for (int i = 0; i < nm; ++i) {
        const uint64_t q = c->mod_h[i];
        if (q >= (1ull << 50) || q <= (1ull << 44) || (q - 1) % (2ull * N) != 0 || h_powmod(psi[i], N, q) != q - 1) {
            delete c;
            return HK_E_ARG;
        }
        ModQ m;
        m.q = q;
        m.k = 64 - __builtin_clzll(q);
        m.mu = (uint64_t)(((u128)1 << (63 + m.k)) / q);
        c->modq_h.push_back(m);
    }
    c->d_modq = upload(c->modq_h);
    // twiddles
    std::vector<ulonglong2> tw((size_t)nm * N), itw((size_t)nm * N), ninv(nm);
    for (int m = 0; m < nm; ++m) {
        const uint64_t q = c->mod_h[m], w = psi[m], iw = h_inv(psi[m], q);
        uint64_t pw = 1, ipw = 1;
        for (int k = 0; k < N; ++k) {
            const uint32_t r = h_brv((uint32_t)k, c->log_n);
            tw[(size_t)m * N + r] = make_ulonglong2(pw, h_shoup(pw, q));
            itw[(size_t)m * N + r] = make_ulonglong2(ipw, h_shoup(ipw, q));
            pw = h_mulmod(pw, w, q);
            ipw = h_mulmod(ipw, iw, q);
        }
        const uint64_t ni = h_inv((uint64_t)N % q, q);
        ninv[m] = make_ulonglong2(ni, h_shoup(ni, q));
    }
    c->d_tw = upload(tw);
    c->d_itw = upload(itw);
    c->d_ninv = upload(ninv);
    {
        std::vector<double2> fmod(nm);
        for (int m = 0; m < nm; ++m) fmod[m] = make_double2((double)c->mod_h[m], 1.0 / (double)c->mod_h[m]);
        c->d_fmod = upload(fmod);
    }
    // Tables of the fused 2^16 kernels (ntt16.cuh), float64 {w, w/q}, stride 2^16 per prime:
    // N = 2^16 uses root psi; N = 2^17 runs each half through the 2^16 kernel with root
    // psi^2 after one radix-2 stage and a pre-twist by psi^-+i (ntt.cu, ntt17_*).
    c->d_twf = c->d_itwf = c->d_ninvf = nullptr;
    c->d_twist = c->d_twistq = c->d_itwist = nullptr;
    c->d_n17 = nullptr;
    c->d_n17w = nullptr;
    if (c->log_n == 16 || c->log_n == 17) {
        const int H = 1 << 16;
        std::vector<double2> twf((size_t)nm * H), itwf((size_t)nm * H), ninvf(2 * (size_t)nm);
        std::vector<double> tws((size_t)nm * H), twsq((size_t)nm * H), itws((size_t)nm * H);
        const uint64_t M2 = 2ull * H;
        for (int m = 0; m < nm; ++m) {
            const uint64_t q = c->mod_h[m];
            const double qd = (double)q;
            const uint64_t w = c->log_n == 16 ? psi[m] : h_mulmod(psi[m], psi[m], q), iw = h_inv(w, q);
            uint64_t pw = 1, ipw = 1;
            for (int k = 0; k < H; ++k) {
                const size_t o = (size_t)m * H + h_brv((uint32_t)k, 16);
                twf[o] = make_double2((double)pw, (double)pw / qd);
                itwf[o] = make_double2((double)ipw, (double)ipw / qd);
                pw = h_mulmod(pw, w, q);
                ipw = h_mulmod(ipw, iw, q);
            }
            // T[1] = w^(2^15) (stage 0 of the 256-point sub-transforms) and its inverse, folded
            // into the twist tables (c >= 128) and the inverse scaling (ntt16.cuh)
            const uint64_t t1 = h_powmod(w, 1ull << 15, q), ti1 = h_inv(t1, q);
            const uint64_t ni = h_inv((uint64_t)H % q, q), niw = h_mulmod(ni, ti1, q);
            ninvf[2 * m] = make_double2((double)ni, (double)ni / qd);
            ninvf[2 * m + 1] = make_double2((double)niw, (double)niw / qd);
            // four-step twist for the 256 x 256 split: row r, column c
            for (int r = 0; r < 256; ++r) {
                const int64_t e = 2 * (int64_t)h_brv((uint32_t)r, 8) + 1 - 256;  // may be negative
                const uint64_t ep = (uint64_t)((e % (int64_t)M2 + (int64_t)M2) % (int64_t)M2);
                const uint64_t base = h_powmod(w, ep, q), ibase = h_inv(base, q);
                uint64_t t = 1, it = 1;
                for (int col = 0; col < 256; ++col) {
                    const size_t o = (size_t)m * H + (size_t)r * 256 + col;
                    const uint64_t tv = col < 128 ? t : h_mulmod(t, t1, q);
                    const uint64_t itv = col < 128 ? it : h_mulmod(it, ti1, q);
                    tws[o] = (double)tv;
                    twsq[o] = (double)tv / qd;
                    itws[o] = (double)itv;
                    t = h_mulmod(t, base, q);
                    it = h_mulmod(it, ibase, q);
                }
            }
        }
        c->d_twf = upload(twf);
        c->d_itwf = upload(itwf);
        c->d_ninvf = upload(ninvf);
        c->d_twist = upload(tws);
        c->d_twistq = upload(twsq);
        c->d_itwist = upload(itws);
        if (c->log_n == 17) {
            // [m][4][2^16] Shoup pairs: psi^-i, psi^i (forward pre-twist of halves 0 / 1),
            // psi^i / 2, psi^-i / 2 (inverse post-twist); [m][2]: w = psi^(2^16), w^-1
            std::vector<ulonglong2> t17((size_t)nm * 4 * H), w17((size_t)nm * 2);
            for (int m = 0; m < nm; ++m) {
                const uint64_t q = c->mod_h[m], ip = h_inv(psi[m], q), half = h_inv(2, q);
                uint64_t fw = 1, bw = 1;
                for (int i = 0; i < H; ++i) {
                    ulonglong2 *row = t17.data() + (size_t)m * 4 * H;
                    row[i] = make_ulonglong2(bw, h_shoup(bw, q));
                    row[H + i] = make_ulonglong2(fw, h_shoup(fw, q));
                    const uint64_t fh = h_mulmod(fw, half, q), bh = h_mulmod(bw, half, q);
                    row[2 * H + i] = make_ulonglong2(fh, h_shoup(fh, q));
                    row[3 * H + i] = make_ulonglong2(bh, h_shoup(bh, q));
                    fw = h_mulmod(fw, psi[m], q);
                    bw = h_mulmod(bw, ip, q);
                }
                const uint64_t w = h_powmod(psi[m], (uint64_t)H, q), wi = h_inv(w, q);
                w17[2 * m] = make_ulonglong2(w, h_shoup(w, q));
                w17[2 * m + 1] = make_ulonglong2(wi, h_shoup(wi, q));
            }
            c->d_n17 = upload(t17);
            c->d_n17w = upload(w17);
        }
    }
    // canonical-embedding tables (same formulas as the oracle)
    const int M = 2 * N;
    std::vector<double2> zeta(M);
    for (int k = 0; k < M; ++k) {
        const double ang = 2.0 * M_PI * (double)k / (double)M;
        zeta[k] = make_double2(cos(ang), sin(ang));
    }
    c->d_zeta = upload(zeta);
    std::vector<uint32_t> rg(c->slots);
    uint32_t g = 1;
    for (int j = 0; j < c->slots; ++j) { rg[j] = g; g = (uint32_t)(((uint64_t)g * 5) % (uint64_t)M); }
    c->d_rot_group = upload(rg);
    // rescale constants q_l^-1 mod q_i
    std::vector<ulonglong2> rs((size_t)c->n_q * c->n_q, make_ulonglong2(0, 0));
    for (int l = 1; l < c->n_q; ++l)
        for (int i = 0; i < l; ++i) {
            const uint64_t q = c->mod_h[i], v = h_inv(c->mod_h[l] % q, q);
            rs[(size_t)l * c->n_q + i] = make_ulonglong2(v, h_shoup(v, q));
        }
    c->d_rs_qinv = upload(rs);
    // ModUp tables per (level, digit): sources = digit primes <= level, targets = the rest
    c->modup.resize(c->n_q);
    for (int l = 0; l < c->n_q; ++l) {
        const int nd = l / c->alpha + 1;
        for (int j = 0; j < nd; ++j) {
            const int d0 = j * c->alpha, d1 = std::min((j + 1) * c->alpha, l + 1);
            std::vector<int> src, dst;
            for (int i = d0; i < d1; ++i) src.push_back(i);
            for (int t = 0; t <= l; ++t)
                if (t < d0 || t >= d1) dst.push_back(t);
            for (int k = 0; k < c->n_p; ++k) dst.push_back(c->n_q + k);
            c->modup[l].push_back(make_conv(c->mod_h, src, dst, true));
        }
    }
    // ModDown: specials -> all q primes (a level uses the first l+1 targets)
    {
        std::vector<int> src, dst;
        for (int k = 0; k < c->n_p; ++k) src.push_back(c->n_q + k);
        for (int i = 0; i < c->n_q; ++i) dst.push_back(i);
        c->moddown = make_conv(c->mod_h, src, dst, true);
        std::vector<ulonglong2> pinv(c->n_q);
        for (int i = 0; i < c->n_q; ++i) {
            const uint64_t q = c->mod_h[i];
            uint64_t P = 1;
            for (int k = 0; k < c->n_p; ++k) P = h_mulmod(P, c->mod_h[c->n_q + k] % q, q);
            const uint64_t v = h_inv(P, q);
            pinv[i] = make_ulonglong2(v, h_shoup(v, q));
        }
        c->d_pinv = upload(pinv);
        // merged ModDown + rescale tables
        c->mdrs.resize(c->n_q);
        std::vector<ulonglong2> pmod(c->n_q), mqinv((size_t)c->n_q * c->n_q, make_ulonglong2(0, 0));
        for (int i = 0; i < c->n_q; ++i) {
            const uint64_t q = c->mod_h[i];
            uint64_t P = 1;
            for (int k = 0; k < c->n_p; ++k) P = h_mulmod(P, c->mod_h[c->n_q + k] % q, q);
            pmod[i] = make_ulonglong2(P, h_shoup(P, q));
        }
        for (int l = 1; l < c->n_q; ++l) {
            std::vector<int> s2, d2;
            for (int k = 0; k < c->n_p; ++k) s2.push_back(c->n_q + k);
            s2.push_back(l);
            for (int t = 0; t < l; ++t) d2.push_back(t);
            c->mdrs[l] = make_conv(c->mod_h, s2, d2, true);
            for (int t = 0; t < l; ++t) {
                const uint64_t q = c->mod_h[t];
                const uint64_t v = h_inv(h_mulmod(pmod[t].x, c->mod_h[l] % q, q), q);
                mqinv[(size_t)l * c->n_q + t] = make_ulonglong2(v, h_shoup(v, q));
            }
        }
        c->d_pmod = upload(pmod);
        c->d_mqinv = upload(mqinv);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        delete c;
        return HK_E_CUDA;
    }
    *out = c;
    return HK_OK;
}

void hk_ctx_destroy(hk_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    cudaFree(c->d_modq);
    cudaFree(c->d_tw);
    cudaFree(c->d_itw);
    cudaFree(c->d_ninv);
    cudaFree(c->d_twf);
    cudaFree(c->d_itwf);
    cudaFree(c->d_ninvf);
    cudaFree(c->d_fmod);
    cudaFree(c->d_twist);
    cudaFree(c->d_twistq);
    cudaFree(c->d_itwist);
    cudaFree(c->d_n17);
    cudaFree(c->d_n17w);
    cudaFree(c->d_zeta);
    cudaFree(c->d_rot_group);
    cudaFree(c->d_rs_qinv);
    cudaFree(c->d_pinv);
    for (auto &lv : c->modup)
        for (auto &t : lv) free_conv(t);
    free_conv(c->moddown);
    for (size_t l = 1; l < c->mdrs.size(); ++l) free_conv(c->mdrs[l]);
    cudaFree(c->d_pmod);
    cudaFree(c->d_mqinv);
    cudaFree(c->d_sk);
    cudaFree(c->d_relin);
    for (auto &kv : c->gal) cudaFree(kv.second.p);
    cudaFree(c->ws);
    delete c;
}

}  // extern "C"
