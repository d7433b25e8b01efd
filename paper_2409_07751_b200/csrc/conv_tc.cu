// conv_tc.cu — fast basis conversion on the 5th-generation tensor cores.
//
// The conversion of key switching (ModUp per digit, ModDown, merged ModDown +
// rescale) is a contraction over the source limbs:
//
//   out[t][e] = (sum_i v[i][e] * hat[t][i] + u[e] * (-M mod q_t)) mod q_t
//
// with v < 2^50 the prescaled source residues and u = round(sum_i v_i / m_i)
// the overflow count of the centred conversion. Only the residue mod q_t
// matters, so the constants are reduced BEFORE the product: split v into bytes,
// v = sum_a 2^(8a) v_a, and let
//
//   c[t][i][a] = hat[t][i] * 2^(8a) mod q_t        (< 2^50, 7 bytes c_b)
//
// then  out = (sum_b 2^(8b) C_b) mod q_t  with
//
//   C_b[e][t] = sum_i sum_a v_a[i][e] * c_b[t][i][a],
//
// an unsigned 8-bit GEMM: A[e][(i, a)] are the little-endian bytes of the u64
// source words themselves (K = 8 bytes x 16 source slots = 128), and
// B[(t, b)][(i, a)] = byte b of c[t][i][a] (8 rows per target: 7 bytes and a
// zero row). The overflow term rides in the GEMM too: u is written into the
// first free source slot and that slot's constant is -M mod q_t. One
// tcgen05.mma.kind::i8 (M = 128 coefficients, N = 8 x up to 32 targets, K = 32)
// per 4 source slots accumulates int32 C in TMEM (every C_b < 2^23); the
// epilogue reads a coefficient's 8 sums of one target with one tcgen05.ld
// (32x32b.x8: TMEM lane = coefficient = thread), folds them into
// X = lo + 2^32 hi < 2^72 with five IMAD.WIDE, estimates X / q_t on the FP64 pipe
// (relative error 2^-51 on a quotient < 2^28: off by at most one) and takes the
// remainder in 64-bit wrapping arithmetic: the canonical residue, hence
// bit-identical to the IMAD kernel (ops.cu: k_conv) and to the oracle.
//
// Round-2 history: the first tensor-core version multiplied by the raw bytes of
// hat (13 byte-diagonals per target, 128-bit fold and Barrett step, ~50
// instructions per output and 16 TMEM columns per target); reducing the
// constants first halves the TMEM traffic and cuts the CUDA-core work per output
// to ~20 instructions (profiles/r2_notes.md §7).
//
// Layouts (no swizzle, K-major canonical UMMA layout): element (row r, byte k)
// of an operand lives at (r / 8) * 1024 + (k / 16) * 128 + (r % 8) * 16 + k % 16
// (8-row x 16-byte core matrices; LBO = 128 B between K-adjacent core matrices,
// SBO = 1024 B between 8-row groups). B is built on the host in exactly this
// layout (ctx.cu: ConvTable::d_bmat, one 1 KiB row group per target) and copied
// linearly into shared memory.
//
// Two instantiations: 16 source slots (K = 128 bytes per row, 4-deep TMA ring) and 32 slots
// (K = 256 bytes, 2-deep ring) for digits of up to 31 primes (c3's alpha = 19: 9.85 -> 11.67
// inferences/s against the IMAD kernel). When the B matrix of all targets does not fit the
// shared memory left, the launcher splits the targets into groups (one launch each).
//
// Data movement: the source words of a 128-coefficient tile ([slot][128] u64,
// 1 KiB contiguous per slot in HBM) arrive by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a 4-deep ring, issued by one
// lane several tiles ahead of the consumers; four transform warps turn a raw
// tile into the UMMA A layout (and compute u), double-buffered against the MMA.
#include "common.cuh"

#include "ntt16.cuh"

namespace {

constexpr int kTileM = 128;      // coefficients per tile (TMEM lanes)
constexpr int kKBytes = 128;     // 16 source slots x 8 bytes (kSlots = 16; 256 for kSlots = 32: c3's 19-prime digits)
constexpr int kRowsPerTarget = 8;
constexpr int kChunkTargets = 32;  // N <= 256 per MMA

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor: no swizzle, K-major
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t sbo_bytes) {
    const uint64_t lbo = 128 >> 4, sbo = sbo_bytes >> 4;
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

// instruction descriptor: kind::i8, u8 x u8 -> s32, K-major A and B, M = 128, N
__device__ __forceinline__ uint32_t umma_idesc(int n) {
    return (2u << 4)                      // D format: S32
           | (0u << 7) | (0u << 10)       // A, B: unsigned 8-bit
           | ((uint32_t)(n >> 3) << 17)   // N >> 3
           | ((uint32_t)(kTileM >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, int accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, 0x4000;\n\t"  // suspend-time hint: idle roles sleep instead of spinning
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// TMA bulk copy global -> shared, completion on an mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Power-of-two multipliers of the fold, kept opaque to ptxas (a literal is strength-
// reduced into shift / funnel-shift / carry sequences, 2-3 instructions per term
// instead of one IMAD.WIDE with a constant-bank operand).
__constant__ uint32_t kPow2[3] = {1u << 8, 1u << 16, 1u << 24};

struct TargetC {  // per-target constants of the epilogue (shared memory, broadcast reads)
    uint64_t q;     // prime
    double qi32;    // 2^32 / q
    uint64_t *out;  // row of this target in the output
};

// out = (sum_b C_b 2^(8b)) mod q from the 7 byte sums of the reduced constants
// (each C_b < 2^23, the sum X < 2^72). IMAD.WIDE chains build lo = C_0..C_3 (< 2^48)
// and Xh = floor(X / 2^32) = C_4 + (lo >> 32) + 2^8 C_5 + 2^16 C_6 (< 2^41), so
// X mod 2^64 = {lo.lo, Xh.lo}. t = round(Xh 2^32 / q) on the FP64 pipe (the integer
// sits in the low mantissa bits after adding 1.5 * 2^52): X / q < 2^28, dropping
// lo.lo costs < 2^-12 and the rounding of the estimate < 2^-20, so |X - t q| < q; the
// remainder in wrapping 64-bit arithmetic, one conditional add.
__device__ __forceinline__ uint64_t fold_reduce(const uint32_t (&C)[8], uint64_t q, double qi32, uint32_t p8,
                                                uint32_t p16, uint32_t p24) {
    const uint64_t lo = mad_wide(C[3], p24, mad_wide(C[2], p16, mad_wide(C[1], p8, C[0])));
    const uint64_t xh = mad_wide(C[6], p16, mad_wide(C[5], p8, (uint64_t)(C[4] + (uint32_t)(lo >> 32))));
    const uint32_t t = (uint32_t)__double_as_longlong(__fma_rn(ntt16::u2d(xh), qi32, ntt16::kMagic));
    const uint64_t x = (uint64_t)(uint32_t)lo | (xh << 32);
    const uint64_t tq = mad_wide(t, (uint32_t)q, (uint64_t)(t * (uint32_t)(q >> 32)) << 32);
    const int64_t r = (int64_t)(x - tq);
    return (uint64_t)(r < 0 ? r + (int64_t)q : r);
}

// Warp-specialised persistent kernel, one CTA per SM:
//   warp 0      TMA issuer (one lane): bulk copies of the source rows of a tile into
//               the raw ring, kRawStages tiles ahead;
//   warps 1-4   transform: raw tile -> UMMA A layout (+ the overflow count u in the
//               first free source slot), double-buffered;
//   warp 5      MMA issuer (one lane): per chunk of <= 32 targets, ksteps MMAs into
//               one of two 256-column TMEM accumulators;
//   warps 6-..  epilogue: kEpiWarps / 4 warps per TMEM lane quarter (warp % 4), each
//               taking every (kEpiWarps / 4)-th target of a chunk, four per TMEM wait.
// mbarriers: raw_full / raw_empty per ring stage, a_full / a_empty per A buffer,
// t_full / t_empty per TMEM buffer; "empty" waits start on parity 1 (the virtual
// previous phase).
constexpr int kXformWarp0 = 1, kXformWarps = 4, kMmaWarp = 5, kEpiWarp0 = 6;

// kSlots = 16 (K = 128 bytes per row, 4-deep raw ring) or 32 (K = 256 bytes, 2-deep ring: digits
// of up to 31 primes, e.g. c3's alpha = 19); d_off: position of target 0 of this launch in
// the conversion's target list (the launcher splits a conversion whose B matrix does not fit
// shared memory into target groups).
template <int kEpiWarps, int kSlots>
__global__ void __launch_bounds__((kEpiWarp0 + kEpiWarps) * 32, 1)
    k_conv_tc(const uint64_t *__restrict__ src, int n_src, const uint8_t *__restrict__ bmat,
              const int32_t *__restrict__ dst_mod, int n_dst, uint64_t *__restrict__ dst, int mode, int l, int n_q,
              long long BN, const double2 *__restrict__ fmod, const double *__restrict__ src_invd, int has_u,
              int d_off) {
    constexpr int kKBytes = kSlots * 8;                   // bytes per operand row
    constexpr int kTileBytes = kTileM * kKBytes;          // one A tile / one raw tile
    constexpr int kRawStages = kSlots == 16 ? 4 : 2;      // TMA ring depth (tiles)
    constexpr uint32_t kSbo = 8 * kKBytes;                // bytes between 8-row groups
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sa = smem;                                   // A: 2 tiles (UMMA layout)
    uint8_t *sraw = sa + 2 * kTileBytes;                  // raw ring: kRawStages x [kSlots][128] u64
    uint8_t *sb = sraw + kRawStages * kTileBytes;         // B: (n_dst + 1) row groups (one pad group)
    const int b_bytes = n_dst * kRowsPerTarget * kKBytes;
    TargetC *stc = reinterpret_cast<TargetC *>(sb + b_bytes + kRowsPerTarget * kKBytes);  // [n_dst]
    __shared__ __align__(8) uint64_t bars[2 * kRawStages + 8];
    __shared__ uint32_t tmem_base_s;
    constexpr int kThreadsWs = (kEpiWarp0 + kEpiWarps) * 32;
    constexpr int kPerQuarter = kEpiWarps / 4;  // epilogue warps sharing one TMEM lane quarter

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const uint4 *g = reinterpret_cast<const uint4 *>(bmat);
        uint4 *s = reinterpret_cast<uint4 *>(sb);
        for (int i = tid; i < b_bytes / 16; i += kThreadsWs) s[i] = g[i];
        for (int i = tid; i < kRowsPerTarget * kKBytes / 16; i += kThreadsWs)
            s[b_bytes / 16 + i] = make_uint4(0, 0, 0, 0);
        for (int d = tid; d < n_dst; d += kThreadsWs) {
            const int m = dst_mod[d];
            const double2 f = fmod[m];
            const int row = mode == 0 ? (m <= l ? m : l + 1 + m - n_q) : d_off + d;
            stc[d] = TargetC{(uint64_t)f.x, f.y * 4294967296.0, dst + (long long)row * BN};
        }
    }
    const uint32_t bar0 = smem_u32(&bars[0]);
    auto RAW_FULL = [&](int s) { return bar0 + 8u * s; };
    auto RAW_EMPTY = [&](int s) { return bar0 + 8u * (kRawStages + s); };
    auto A_FULL = [&](int s) { return bar0 + 8u * (2 * kRawStages + s); };
    auto A_EMPTY = [&](int s) { return bar0 + 8u * (2 * kRawStages + 2 + s); };
    auto T_FULL = [&](int s) { return bar0 + 8u * (2 * kRawStages + 4 + s); };
    auto T_EMPTY = [&](int s) { return bar0 + 8u * (2 * kRawStages + 6 + s); };
    if (warp == kMmaWarp) {  // TMEM: two 256-column int32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kRawStages; ++s) {
            mbar_init(RAW_FULL(s), 1);
            mbar_init(RAW_EMPTY(s), kXformWarps);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(A_FULL(s), kXformWarps);
            mbar_init(A_EMPTY(s), 1);
            mbar_init(T_FULL(s), 1);
            mbar_init(T_EMPTY(s), kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    const int n_slots = n_src + (has_u ? 1 : 0);
    const int ksteps = (n_slots + 3) >> 2;  // 4 source slots (32 bytes) per MMA
    const int n_chunks = (n_dst + kChunkTargets - 1) / kChunkTargets;
    const int chunk = (n_dst + n_chunks - 1) / n_chunks;  // balanced: 37 targets -> 19 + 18
    const long long tiles = BN / kTileM;

    if (warp == 0) {
        // ---------------------------------------------------------- TMA issuer
        if (lane == 0) {
            int i = 0;
            for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
                const int s = i % kRawStages, par = ((i / kRawStages) & 1) ^ 1;
                mbar_wait(RAW_EMPTY(s), par);
                mbar_expect_tx(RAW_FULL(s), (uint32_t)n_src * 1024u);
                const uint64_t *g = src + tile * kTileM;
                const uint32_t d0 = smem_u32(sraw + s * kTileBytes);
                for (int j = 0; j < n_src; ++j) bulk_g2s(d0 + j * 1024, g + (long long)j * BN, 1024, RAW_FULL(s));
            }
        }
    } else if (warp < kMmaWarp) {
        // ---------------------------------------------------------- transform
        const int r = tid - kXformWarp0 * 32;
        int i = 0;
        for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int rs = i % kRawStages;
            mbar_wait(RAW_FULL(rs), (i / kRawStages) & 1);
            const uint64_t *raw = reinterpret_cast<const uint64_t *>(sraw + rs * kTileBytes) + r;
            const int s = i & 1;
            uint8_t *row = sa + s * kTileBytes + (r >> 3) * kSbo + (r & 7) * 16;
            double frac = 0.0;  // sum_i v_i / m_i, fixed order, no contraction (as k_conv and the oracle)
#pragma unroll
            for (int h = 0; h < kSlots / 16; ++h) {  // 16 source slots at a time (register budget)
                uint64_t v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 16 * h + j < n_src ? raw[(16 * h + j) * kTileM] : 0;
                if (h == kSlots / 16 - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(RAW_EMPTY(rs));
                }
                if (has_u) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (16 * h + j < n_src) frac = __dadd_rn(frac, __dmul_rn(ntt16::u2d(v[j]), src_invd[16 * h + j]));
                }
                if (h == 0) mbar_wait(A_EMPTY(s), ((i >> 1) & 1) ^ 1);
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    *reinterpret_cast<uint4 *>(row + (8 * h + c) * 128) =
                        make_uint4((uint32_t)v[2 * c], (uint32_t)(v[2 * c] >> 32), (uint32_t)v[2 * c + 1],
                                   (uint32_t)(v[2 * c + 1] >> 32));
            }
            // the overflow count takes source slot n_src (zero so far)
            if (has_u)
                *reinterpret_cast<uint64_t *>(row + (n_src >> 1) * 128 + (n_src & 1) * 8) =
                    (uint64_t)floor(__dadd_rn(frac, 0.5));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(A_FULL(s));
        }
    } else if (warp == kMmaWarp) {
        // ---------------------------------------------------------- MMA issuer
        if (lane == 0) {
            int i = 0, g = 0;
            for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
                const int s = i & 1;
                mbar_wait(A_FULL(s), (i >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t a0 = smem_u32(sa + s * kTileBytes);
                for (int ch = 0; ch < n_chunks; ++ch, ++g) {
                    const int tb = g & 1;
                    mbar_wait(T_EMPTY(tb), ((g >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const int t0 = ch * chunk, nt = min(chunk, n_dst - t0);
                    // N is a multiple of 16: an odd target count also multiplies the next row
                    // group (the next target or the zero pad group), whose columns nobody reads
                    const uint32_t idesc = umma_idesc((nt * kRowsPerTarget + 15) & ~15);
                    const uint32_t b0 = smem_u32(sb + t0 * kRowsPerTarget * kKBytes);  // one row group per target
                    for (int k = 0; k < ksteps; ++k)
                        mma_i8(tmem + tb * 256, umma_desc(a0 + k * 256, kSbo), umma_desc(b0 + k * 256, kSbo), idesc, k);
                    umma_commit(T_FULL(tb));
                }
                umma_commit(A_EMPTY(s));  // every MMA reading this A buffer has completed
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        const int q = warp & 3, slot = (warp - kEpiWarp0) >> 2;
        const int row = q * 32 + lane;
        // read once: the "memory" clobbers of the TMEM waits would reload them per target
        const uint32_t p8 = kPow2[0], p16 = kPow2[1], p24 = kPow2[2];
        int g = 0;
        for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const long long e = tile * kTileM + row;
            for (int ch = 0; ch < n_chunks; ++ch, ++g) {
                const int tb = g & 1;
                mbar_wait(T_FULL(tb), (g >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const int t0 = ch * chunk, nt = min(chunk, n_dst - t0);
                const uint32_t tq = tmem + tb * 256 + ((uint32_t)(q * 32) << 16);
                // this warp's targets of the chunk: slot, slot + kPerQuarter, ... four per TMEM wait
                for (int tt = slot; tt < nt; tt += 4 * kPerQuarter) {
                    uint32_t C[4][8];
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        if (tt + w * kPerQuarter < nt)
                            tmem_ld8(tq + (uint32_t)((tt + w * kPerQuarter) * kRowsPerTarget), C[w]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        if (tt + w * kPerQuarter < nt) {
                            const TargetC tc = stc[t0 + tt + w * kPerQuarter];
                            tc.out[e] = fold_reduce(C[w], tc.q, tc.qi32, p8, p16, p24);
                        }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(T_EMPTY(tb));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

}  // namespace

// Usable for this table and launch: prescaled sources, at most 32 source slots (the
// overflow count of a centred conversion takes one), a built B matrix, whole
// 128-coefficient tiles.
bool conv_tc_ok(const hk_ctx *c, const ConvTable &T, int n_dst, long long BN, int prescaled) {
    static const bool off = getenv("HK_CONV_TC") && atoi(getenv("HK_CONV_TC")) == 0;  // A/B knob
    static const bool wide = !(getenv("HK_CONV_TC32") && atoi(getenv("HK_CONV_TC32")) == 0);  // A/B knob: 32-slot kernel
    const int slots = T.n_src + (T.d_neg_m ? 1 : 0);
    return !off && prescaled && T.d_bmat && (slots <= 16 || (wide && slots <= 32)) && n_dst <= T.n_dst &&
           BN % kTileM == 0 && c->log_n >= 7;
}

template <int kSlots>
static int conv_tc_launch_slots(hk_ctx *c, const ConvTable &T, const uint64_t *src, uint64_t *dst, int mode, int l,
                                long long BN, int n_dst) {
    constexpr int kKB = kSlots * 8, kStages = kSlots == 16 ? 4 : 2;
    const size_t fixed = (size_t)(2 + kStages) * kTileM * kKB + 64;
    const size_t per_target = (size_t)kRowsPerTarget * kKB + sizeof(TargetC);
    // targets per launch: the B matrix (one row group per target + one pad group) must fit
    const int cap = (int)((227 * 1024 - fixed - (size_t)kRowsPerTarget * kKB) / per_target);
    if (cap < 1) return hk_fail(c, HK_E_ARG, "conv_tc: no room for the B matrix");
    const int groups = (n_dst + cap - 1) / cap, per = (n_dst + groups - 1) / groups;
    static const int epi = getenv("HK_CONV_EPI") ? atoi(getenv("HK_CONV_EPI")) : 16;  // A/B knob: 8 / 12 / 16 warps
    const long long tiles = BN / kTileM;
    const unsigned grid = (unsigned)std::min<long long>(tiles, (long long)c->n_sm);  // one CTA per SM (512 TMEM columns)
    for (int d0 = 0; d0 < n_dst; d0 += per) {
        const int nd = std::min(per, n_dst - d0);
        const size_t smem = fixed + (size_t)(nd + 1) * kRowsPerTarget * kKB + (size_t)nd * sizeof(TargetC);
#define HK_CONV_TC(EW)                                                                                            \
    {                                                                                                             \
        static size_t attr = 0;                                                                                   \
        if (smem > attr) {                                                                                        \
            cudaFuncSetAttribute(k_conv_tc<EW, kSlots>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            attr = smem;                                                                                          \
        }                                                                                                         \
        k_conv_tc<EW, kSlots><<<grid, (kEpiWarp0 + EW) * 32, smem, c->stream>>>(                                  \
            src, T.n_src, T.d_bmat + (size_t)d0 * kRowsPerTarget * kKB, T.d_dst_mod + d0, nd, dst, mode, l,       \
            c->n_q, BN, c->d_fmod, T.d_src_invd, T.d_neg_m ? 1 : 0, d0);                                          \
    }
        if (epi == 16) HK_CONV_TC(16) else if (epi == 8) HK_CONV_TC(8) else HK_CONV_TC(12)
#undef HK_CONV_TC
        ++c->launches;
        HK_LAUNCH_CHECK(c, "basis conversion (tensor cores)");
    }
    return HK_OK;
}

int conv_tc_launch(hk_ctx *c, const ConvTable &T, const uint64_t *src, uint64_t *dst, int mode, int l, long long BN,
                   int n_dst) {
    if (T.n_src + (T.d_neg_m ? 1 : 0) <= 16) return conv_tc_launch_slots<16>(c, T, src, dst, mode, l, BN, n_dst);
    return conv_tc_launch_slots<32>(c, T, src, dst, mode, l, BN, n_dst);
}
