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
constexpr int kThreads = 256;

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

// X = s0 + s1 2^25 + s2 2^50 from the 13 byte-diagonal sums C_d (X = sum C_d 2^(8d))
__device__ __forceinline__ Acc3 fold_diagonals(const uint32_t (&C)[16]) {
    Acc3 a;
    a.s0 = (uint64_t)C[0] + ((uint64_t)C[1] << 8) + ((uint64_t)C[2] << 16) + ((uint64_t)C[3] << 24);
    a.s1 = ((uint64_t)C[4] << 7) + ((uint64_t)C[5] << 15) + ((uint64_t)C[6] << 23);
    a.s2 = ((uint64_t)C[7] << 6) + ((uint64_t)C[8] << 14) + ((uint64_t)C[9] << 22) + ((uint64_t)C[10] << 30) +
           ((uint64_t)C[11] << 38) + ((uint64_t)C[12] << 46);
    return a;
}

// grid: persistent CTAs over tiles of 128 coefficients; all n_dst targets per tile
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_tc(const uint64_t *__restrict__ src, int n_src, const uint8_t *__restrict__ bmat,
              const int32_t *__restrict__ dst_mod, int n_dst, uint64_t *__restrict__ dst, int mode, int l, int n_q,
              long long BN, const ModQ *__restrict__ mq, const double *__restrict__ src_invd,
              const uint64_t *__restrict__ neg_m) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sa = smem;                                             // A: 128 x 128 bytes
    uint8_t *sb = smem + kTileM * kKBytes;                          // B: 16 n_dst x 128 bytes
    const int b_bytes = n_dst * kRowsPerTarget * kKBytes;
    uint64_t *su = reinterpret_cast<uint64_t *>(sb + b_bytes);     // u per row [128]
    ModQ *smq = reinterpret_cast<ModQ *>(su + kTileM);              // [n_dst]
    int *sidx = reinterpret_cast<int *>(smq + n_dst);               // [n_dst]
    uint64_t *snm = reinterpret_cast<uint64_t *>(sidx + ((n_dst + 1) & ~1));  // [n_dst]
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage B (constant for the launch) and the target tables
    {
        const uint4 *g = reinterpret_cast<const uint4 *>(bmat);
        uint4 *s = reinterpret_cast<uint4 *>(sb);
        for (int i = tid; i < b_bytes / 16; i += kThreads) s[i] = g[i];
        for (int d = tid; d < n_dst; d += kThreads) {
            const int m = dst_mod[d];
            smq[d] = mq[m];
            sidx[d] = mode == 0 ? (m <= l ? m : l + 1 + m - n_q) : d;
            snm[d] = neg_m ? neg_m[d] : 0;
        }
    }
    if (warp == 0) {  // TMEM: 256 columns (one 16-target chunk of int32 accumulators)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    const uint32_t bar = smem_u32(&mbar);
    uint32_t phase = 0;
    const int ksteps = (n_src + 3) >> 2;  // 4 source slots (32 bytes) per MMA
    const long long tiles = BN / kTileM;

    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long e0 = tile * kTileM;
        if (tid < kTileM) {  // A rows: the source words' bytes; u = round(sum v_i / m_i)
            const int r = tid;
            uint8_t *row = sa + (r >> 3) * 1024 + (r & 7) * 16;
            double frac = 0.0;
#pragma unroll 4
            for (int c = 0; c < 8; ++c) {
                uint64_t v0 = 0, v1 = 0;
                if (2 * c < n_src) v0 = src[(long long)(2 * c) * BN + e0 + r];
                if (2 * c + 1 < n_src) v1 = src[(long long)(2 * c + 1) * BN + e0 + r];
                if (neg_m) {
                    if (2 * c < n_src) frac = __dadd_rn(frac, __dmul_rn(ntt16::u2d(v0), src_invd[2 * c]));
                    if (2 * c + 1 < n_src) frac = __dadd_rn(frac, __dmul_rn(ntt16::u2d(v1), src_invd[2 * c + 1]));
                }
                *reinterpret_cast<uint4 *>(row + c * 128) =
                    make_uint4((uint32_t)v0, (uint32_t)(v0 >> 32), (uint32_t)v1, (uint32_t)(v1 >> 32));
            }
            su[r] = neg_m ? (uint64_t)floor(__dadd_rn(frac, 0.5)) : 0;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A visible to the tensor core
        __syncthreads();
        const int row = (warp & 3) * 32 + lane;  // TMEM lane quarter of this warp = coefficient
        const uint64_t u = su[row];
        for (int t0 = 0; t0 < n_dst; t0 += kChunkTargets) {
            const int nt = min(kChunkTargets, n_dst - t0);
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t idesc = umma_idesc(nt * kRowsPerTarget);
                const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb + t0 * kRowsPerTarget * kKBytes);
                for (int k = 0; k < ksteps; ++k)
                    mma_i8(tmem, umma_desc(a0 + k * 256), umma_desc(b0 + k * 256), idesc, k);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar));
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
            // warps 0-3: targets 0..7 of the chunk, warps 4-7: targets 8..15
            const int tb = (warp >> 2) * 8;
            for (int tt = tb; tt < min(tb + 8, nt); ++tt) {
                uint32_t C[16];
                tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(tt * kRowsPerTarget), C);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int d = t0 + tt;
                Acc3 A = fold_diagonals(C);
                A.s0 += u * snm[d];
                dst[(long long)sidx[d] * BN + e0 + row] = acc3_reduce(A, smq[d]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();  // TMEM and (after the last chunk) A are free again
        }
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
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
    const size_t smem = (size_t)kTileM * kKBytes + (size_t)n_dst * kRowsPerTarget * kKBytes + kTileM * 8 +
                        n_dst * (sizeof(ModQ) + 8 + 4) + 64;
    if (smem > 227 * 1024) return hk_fail(c, HK_E_ARG, "conv_tc: %d targets exceed shared memory", n_dst);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    const long long tiles = BN / kTileM;
    const int per_sm = smem <= 100 * 1024 ? 2 : 1;
    const unsigned grid = (unsigned)std::min<long long>(tiles, (long long)c->n_sm * per_sm);
    k_conv_tc<<<grid, kThreads, smem, c->stream>>>(src, T.n_src, T.d_bmat, T.d_dst_mod, n_dst, dst, mode, l, c->n_q,
                                                    BN, c->d_modq, T.d_src_invd, T.d_neg_m);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "basis conversion (tensor cores)");
    return HK_OK;
}
