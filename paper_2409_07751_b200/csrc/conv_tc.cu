// conv_tc.cu — fast basis conversion on the 5th-generation tensor cores.
//
// The conversion of key switching (ModUp per digit, ModDown, merged ModDown +
// rescale) is a contraction over the source limbs:
//
//   X[e][t] = sum_i v[i][e] * hat[t][i]      (v < 2^50, hat < 2^50, exact)
//   out[t][e] = (X + u[e] * (-M mod q_t)) mod q_t
//
// Split both operands into bytes, v = sum_a 2^(8a) v_a and hat = sum_b 2^(8b)
// h_b. Then X = sum_d 2^(8d) C_d with
//
//   C_d[e][t] = sum_i sum_{a+b=d} v_a[i][e] h_b[t][i],
//
// an unsigned 8-bit GEMM: A[e][(i, a)] are the little-endian bytes of the u64
// source words themselves (K = 8 bytes x 16 source slots = 128), and
// B[(t, d)][(i, a)] = byte (d - a) of hat[t][i] (16 rows per target: the 13
// byte-diagonals d = 0..12 and three zero rows). One tcgen05.mma.kind::i8
// (M = 128 coefficients, N = 16 x 16 targets, K = 32) per 4 source slots
// accumulates int32 C in TMEM (every C_d < 2^23); the epilogue reads a
// coefficient's 16 diagonals of one target with a single tcgen05.ld
// (32x32b.x16: TMEM lane = coefficient = thread), folds them into the same
// three-limb integer s0 + s1 2^25 + s2 2^50 the IMAD kernel (ops.cu: k_conv)
// accumulates, and reduces it with the same Barrett step — so the output is
// bit-identical to k_conv and to the oracle. The k_conv IMAD formulation
// spends ~13 instructions per multiply-add on the FMA/ALU pipes (profiles/
// r2_notes.md); here the products run on the tensor pipe and the CUDA cores
// only do the ~50-instruction fold-and-reduce per output.
//
// Layouts (no swizzle, K-major canonical UMMA layout): element (row r, byte k)
// of an operand lives at (r / 8) * 1024 + (k / 16) * 128 + (r % 8) * 16 + k % 16
// (8-row x 16-byte core matrices; LBO = 128 B between K-adjacent core matrices,
// SBO = 1024 B between 8-row groups). B is built on the host in exactly this
// layout (ctx.cu: ConvTable::d_bmat) and copied linearly into shared memory.
#include "common.cuh"

#include "ntt16.cuh"

namespace {

constexpr int kTileM = 128;      // coefficients per tile (TMEM lanes)
constexpr int kKBytes = 128;     // 16 source slots x 8 bytes
constexpr int kRowsPerTarget = 16;
constexpr int kChunkTargets = 16;  // N = 256 per MMA

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor: no swizzle, K-major
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    const uint64_t lbo = 128 >> 4, sbo = 1024 >> 4;
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// out = (sum_d C_d 2^(8d) + u negM) mod q from the 13 byte-diagonal sums (each C_d
// < 2^23, the sum < 2^104): three 48-bit partial sums by IMAD.WIDE chains (weights
// 2^0, 2^32, 2^64), one 128-bit combine, one Barrett step (reduce128: X < 2^(63+k)).
// The same integer the IMAD kernel's three-limb accumulator holds, so the same result.
__device__ __forceinline__ uint64_t fold_reduce(const uint32_t (&C)[16], uint32_t u, uint64_t nm, const ModQ &q) {
    uint64_t lo = mad_wide(C[3], 1u << 24, mad_wide(C[2], 1u << 16, mad_wide(C[1], 1u << 8, C[0])));
    const uint64_t mid = mad_wide(C[7], 1u << 24, mad_wide(C[6], 1u << 16, mad_wide(C[5], 1u << 8, C[4])));
    uint64_t hi = mad_wide(C[11], 1u << 24, mad_wide(C[10], 1u << 16, mad_wide(C[9], 1u << 8, C[8]))) +
                  ((uint64_t)C[12] << 32);
    const uint64_t m32 = mid << 32;
    lo += m32;
    hi += (mid >> 32) + (lo < m32);
    const uint64_t un = mad_wide(u, (uint32_t)nm, (uint64_t)(u * (uint32_t)(nm >> 32)) << 32);  // u nm < 2^54
    lo += un;
    hi += lo < un;
    return reduce128(hi, lo, q);
}

// mbarrier helpers
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Warp-specialised persistent kernel, one CTA per SM, 13 warps:
//   warps 0-3   producers: A tile (the source words of 128 coefficients) and the
//               overflow counts u, double-buffered;
//   warp 4      MMA issuer (one lane): per 16-target chunk, ksteps MMAs into one
//               of two 256-column TMEM accumulators;
//   warps 5-12  epilogue: two warps per TMEM lane quarter (warp % 4), each taking
//               8 of a chunk's 16 targets.
// mbarriers: a_full / a_empty / u_empty per A buffer, t_full / t_empty per
// TMEM buffer; "empty" waits start on parity 1 (the virtual previous phase).
constexpr int kProducers = 4, kMmaWarp = 4, kEpiWarp0 = 5;

template <int kEpiWarps>
__global__ void __launch_bounds__((kEpiWarp0 + kEpiWarps) * 32, 1)
    k_conv_tc(const uint64_t *__restrict__ src, int n_src, const uint8_t *__restrict__ bmat,
              const int32_t *__restrict__ dst_mod, int n_dst, uint64_t *__restrict__ dst, int mode, int l, int n_q,
              long long BN, const ModQ *__restrict__ mq, const double *__restrict__ src_invd,
              const uint64_t *__restrict__ neg_m) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sa = smem;                                              // A: 2 x 128 x 128 bytes
    uint8_t *sb = smem + 2 * kTileM * kKBytes;                       // B: 16 n_dst x 128 bytes
    const int b_bytes = n_dst * kRowsPerTarget * kKBytes;
    uint64_t *su = reinterpret_cast<uint64_t *>(sb + b_bytes);      // u: 2 x 128
    ModQ *smq = reinterpret_cast<ModQ *>(su + 2 * kTileM);           // [n_dst]
    uint64_t *snm = reinterpret_cast<uint64_t *>(smq + n_dst);       // [n_dst]
    int *sidx = reinterpret_cast<int *>(snm + n_dst);                // [n_dst]
    __shared__ __align__(8) uint64_t bars[10];  // a_full[2] a_empty[2] u_empty[2] t_full[2] t_empty[2]
    __shared__ uint32_t tmem_base_s;
    constexpr int kThreadsWs = (kEpiWarp0 + kEpiWarps) * 32;
    constexpr int kPerQuarter = kEpiWarps / 4;  // epilogue warps sharing one TMEM lane quarter

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const uint4 *g = reinterpret_cast<const uint4 *>(bmat);
        uint4 *s = reinterpret_cast<uint4 *>(sb);
        for (int i = tid; i < b_bytes / 16; i += kThreadsWs) s[i] = g[i];
        for (int d = tid; d < n_dst; d += kThreadsWs) {
            const int m = dst_mod[d];
            smq[d] = mq[m];
            sidx[d] = mode == 0 ? (m <= l ? m : l + 1 + m - n_q) : d;
            snm[d] = neg_m ? neg_m[d] : 0;
        }
    }
    const uint32_t bar0 = smem_u32(&bars[0]);
    auto A_FULL = [&](int s) { return bar0 + 8u * (0 + s); };
    auto A_EMPTY = [&](int s) { return bar0 + 8u * (2 + s); };
    auto U_EMPTY = [&](int s) { return bar0 + 8u * (4 + s); };
    auto T_FULL = [&](int s) { return bar0 + 8u * (6 + s); };
    auto T_EMPTY = [&](int s) { return bar0 + 8u * (8 + s); };
    if (warp == kMmaWarp) {  // TMEM: two 256-column int32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(A_FULL(s), kProducers);
            mbar_init(A_EMPTY(s), 1);
            mbar_init(U_EMPTY(s), kEpiWarps);
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
    const int ksteps = (n_src + 3) >> 2;  // 4 source slots (32 bytes) per MMA
    const int n_chunks = (n_dst + kChunkTargets - 1) / kChunkTargets;
    const long long tiles = BN / kTileM;

    if (warp < kProducers) {
        // ---------------------------------------------------------- producers
        const int r = tid;
        int i = 0;
        for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int s = i & 1, par = ((i >> 1) & 1) ^ 1;
            mbar_wait(A_EMPTY(s), par);
            mbar_wait(U_EMPTY(s), par);
            const long long e0 = tile * kTileM;
            uint8_t *row = sa + s * (kTileM * kKBytes) + (r >> 3) * 1024 + (r & 7) * 16;
            uint64_t v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = j < n_src ? src[(long long)j * BN + e0 + r] : 0;
            double frac = 0.0;
            if (neg_m) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j < n_src) frac = __dadd_rn(frac, __dmul_rn(ntt16::u2d(v[j]), src_invd[j]));
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4 *>(row + c * 128) = make_uint4(
                    (uint32_t)v[2 * c], (uint32_t)(v[2 * c] >> 32), (uint32_t)v[2 * c + 1], (uint32_t)(v[2 * c + 1] >> 32));
            su[s * kTileM + r] = neg_m ? (uint64_t)floor(__dadd_rn(frac, 0.5)) : 0;
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
                const uint32_t a0 = smem_u32(sa + s * (kTileM * kKBytes));
                for (int ch = 0; ch < n_chunks; ++ch, ++g) {
                    const int tb = g & 1;
                    mbar_wait(T_EMPTY(tb), ((g >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const int t0 = ch * kChunkTargets, nt = min(kChunkTargets, n_dst - t0);
                    const uint32_t idesc = umma_idesc(nt * kRowsPerTarget);
                    const uint32_t b0 = smem_u32(sb + t0 * kRowsPerTarget * kKBytes);
                    for (int k = 0; k < ksteps; ++k)
                        mma_i8(tmem + tb * 256, umma_desc(a0 + k * 256), umma_desc(b0 + k * 256), idesc, k);
                    umma_commit(T_FULL(tb));
                }
                umma_commit(A_EMPTY(s));  // every MMA reading this A buffer has completed
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        const int q = warp & 3, slot = (warp - kEpiWarp0) >> 2;
        const int row = q * 32 + lane;
        int i = 0, g = 0;
        for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int s = i & 1;
            mbar_wait(A_FULL(s), (i >> 1) & 1);  // u of this tile is written
            const uint64_t u = su[s * kTileM + row];
            __syncwarp();
            if (lane == 0) mbar_arrive(U_EMPTY(s));
            const long long e = tile * kTileM + row;
            for (int ch = 0; ch < n_chunks; ++ch, ++g) {
                const int tb = g & 1;
                mbar_wait(T_FULL(tb), (g >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const int t0 = ch * kChunkTargets, nt = min(kChunkTargets, n_dst - t0);
                const uint32_t tq = tmem + tb * 256 + ((uint32_t)(q * 32) << 16);
                // this warp's targets of the chunk: slot, slot + kPerQuarter, ... two per TMEM wait
                for (int tt = slot; tt < nt; tt += 2 * kPerQuarter) {
                    const bool two = tt + kPerQuarter < nt;
                    uint32_t C0[16], C1[16];
                    tmem_ld16(tq + (uint32_t)(tt * kRowsPerTarget), C0);
                    if (two) tmem_ld16(tq + (uint32_t)((tt + kPerQuarter) * kRowsPerTarget), C1);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    {
                        const int d = t0 + tt;
                        dst[(long long)sidx[d] * BN + e] = fold_reduce(C0, (uint32_t)u, snm[d], smq[d]);
                    }
                    if (two) {
                        const int d = t0 + tt + kPerQuarter;
                        dst[(long long)sidx[d] * BN + e] = fold_reduce(C1, (uint32_t)u, snm[d], smq[d]);
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

// Usable for this table and launch: prescaled sources, at most 16 of them, a
// built B matrix, whole 128-coefficient tiles.
bool conv_tc_ok(const hk_ctx *c, const ConvTable &T, int n_dst, long long BN, int prescaled) {
    static const bool off = getenv("HK_CONV_TC") && atoi(getenv("HK_CONV_TC")) == 0;  // A/B knob
    return !off && prescaled && T.d_bmat && T.n_src <= 16 && n_dst <= T.n_dst && BN % kTileM == 0 &&
           c->log_n >= 7;
}

int conv_tc_launch(hk_ctx *c, const ConvTable &T, const uint64_t *src, uint64_t *dst, int mode, int l, long long BN,
                   int n_dst) {
    const size_t smem = 2 * (size_t)kTileM * kKBytes + (size_t)n_dst * kRowsPerTarget * kKBytes + 2 * kTileM * 8 +
                        n_dst * (sizeof(ModQ) + 8 + 4) + 64;
    if (smem > 227 * 1024) return hk_fail(c, HK_E_ARG, "conv_tc: %d targets exceed shared memory", n_dst);
    static const int epi = getenv("HK_CONV_EPI") ? atoi(getenv("HK_CONV_EPI")) : 16;  // A/B: 8 / 12 / 16 warps -> 26.8 / 27.3 / 27.3 c1 inf/s
    const long long tiles = BN / kTileM;
    const unsigned grid = (unsigned)std::min<long long>(tiles, (long long)c->n_sm);  // one CTA per SM (512 TMEM columns)
#define HK_CONV_TC(EW)                                                                                           \
    {                                                                                                            \
        static size_t attr = 0;                                                                                  \
        if (smem > attr) {                                                                                       \
            cudaFuncSetAttribute(k_conv_tc<EW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
            attr = smem;                                                                                         \
        }                                                                                                        \
        k_conv_tc<EW><<<grid, (kEpiWarp0 + EW) * 32, smem, c->stream>>>(src, T.n_src, T.d_bmat, T.d_dst_mod,     \
                                                                       n_dst, dst, mode, l, c->n_q, BN,         \
                                                                       c->d_modq, T.d_src_invd, T.d_neg_m);      \
    }
    if (epi == 16) HK_CONV_TC(16) else if (epi == 8) HK_CONV_TC(8) else HK_CONV_TC(12)
#undef HK_CONV_TC
    ++c->launches;
    HK_LAUNCH_CHECK(c, "basis conversion (tensor cores)");
    return HK_OK;
}
