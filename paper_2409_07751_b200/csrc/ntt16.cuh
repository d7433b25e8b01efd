// ntt16.cuh — fused N = 2^16 negacyclic NTT kernels with prologue/epilogue hooks.
//
// One cluster of 4 CTAs (256 threads each, four CTAs per SM) per
// polynomial; the polynomial is 16 column tiles / 16 row blocks of 16 (see
// ntt.cu for the stage split). The first phase reads its inputs through a prologue functor and the
// second phase hands canonical outputs to an epilogue functor, so element-wise
// work that surrounds an NTT in CKKS (basis conversion, the rescale
// remainder broadcast, plaintext products, the ModDown / rescale finish) runs
// inside the NTT's own global loads/stores instead of as separate passes.
//
//   Pro: __device__ uint64_t operator()(int l, long long P, int idx) const
//        canonical residue (mod the launch's prime l) of input element idx of
//        polynomial P (= l * B + b within the launch)
//   Epi: __device__ void operator()(int l, long long P, int idx, uint64_t v) const
//        consume canonical output v
// `inter` ([limbs][B][N] words) holds the between-phase data; it may alias the
// epilogue's output.
//
// Residues live in float64 registers as exact integers (|x| < 2^51): the
// DFMA/DMUL pipe (64/clk/SM on B200) carries the modular multiply as an exact
// two-product Shoup step. Small primes (q < 2^47) need no reduction inside a
// phase (8 stages from |x| < q stay below 13 q < 2^51); the phase boundary
// recentres. Large primes (q_0 ~ 2^50) recentre after every stage.
#pragma once

#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace ntt16 {

// Two-phase epilogues: an epilogue with a nested `Pre` type splits into
// `Pre prep(l, P, idx)` (every operand load; independent of the NTT output)
// and `fin(l, P, idx, pre, v)` (the arithmetic and the store). The row phase
// issues all 16 preps of a thread before its first store, so the operand
// loads of one row block are in flight together instead of one round trip per
// output (the functors' pointers may alias the output, so the compiler cannot
// hoist loads above earlier stores of a single-phase epilogue).
template <class E, class = void>
struct HasPrep : std::false_type {};
template <class E>
struct HasPrep<E, std::void_t<typename E::Pre>> : std::true_type {};

// Epilogues whose output is NOT the between-phase buffer declare
// `static constexpr bool kDiscardInter = true`: the row phase then drops each
// between-phase line from L2 once it has been read (discard.global.L2), so the dirty
// line is never written back to HBM. With an in-place epilogue the output
// overwrites the line instead and nothing is discarded.
template <class E, class = void>
struct DiscardInter : std::false_type {};
template <class E>
struct DiscardInter<E, std::enable_if_t<E::kDiscardInter>> : std::true_type {};

// Prologues may produce their value on the FP64 pipe: `dval(l, P, idx, m, big)` returns
// the input as an exact integer in a double, |x| <= 1.5 q for small primes and centred
// (|x| <= q/2) for the large one, instead of a canonical u64 that the kernel converts.
template <class Pr, class = void>
struct HasDval : std::false_type {};
template <class Pr>
struct HasDval<Pr, std::void_t<decltype(&Pr::dval)>> : std::true_type {};

constexpr int kLogN = 16;
constexpr int kN = 1 << kLogN;
constexpr int kCl = 16;                      // column tiles / row blocks of 16 per polynomial
constexpr int kTh = 256;                     // threads per CTA: 16 values each
constexpr int kTc = 256 / kCl;               // columns (column phase) / rows (row phase) per CTA
constexpr int kRowPad = 272;                 // 256 + 16: pad one element every 16
constexpr int kSmem = kTc * kRowPad * 8 + 256 * 16;  // data tile (>= 256*kTc*8) + 256-entry twiddle table
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;  // 2^52
constexpr uint64_t kSmallPrime = 1ull << 47;

struct FpMod {
    double q, qinv;
};

__device__ __forceinline__ int pad16(int c) { return c + (c >> 4); }

__device__ __forceinline__ double f_mulmod(double y, double w, double wq, double q) {
    const double h = __dmul_rn(y, w);
    const double l = __fma_rn(y, w, -h);
    const double t = __dsub_rn(__fma_rn(y, wq, kMagic), kMagic);
    return __dadd_rn(__fma_rn(-t, q, h), l);
}
__device__ __forceinline__ double f_center(double x, const FpMod &m) {
    const double t = __dsub_rn(__fma_rn(x, m.qinv, kMagic), kMagic);
    return __fma_rn(-t, m.q, x);
}
__device__ __forceinline__ double u2d(uint64_t x) {  // exact for x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), kTwo52);
}
// Canonical residue of the exact integer x (|x| < 2^51). The centred remainder c lies in
// [-q/2 - 1, q/2 + 1], so c + q is a positive integer below 2^52: adding 2^52 + q (exact:
// q < 2^51) leaves it in the low mantissa bits, and the final conditional subtraction
// runs on the integer pipe — four FP64-pipe operations instead of the eight of a
// compare-and-add chain in doubles (the FP64 pipe is what bounds the NTT).
__device__ __forceinline__ uint64_t d2canon(double x, const FpMod &m) {
    const double c = f_center(x, m);
    const uint64_t v =
        (uint64_t)__double_as_longlong(__dadd_rn(c, __dadd_rn(kTwo52, m.q))) & 0xFFFFFFFFFFFFFull;
    const uint64_t q = (uint64_t)__double_as_longlong(__dadd_rn(m.q, kTwo52)) & 0xFFFFFFFFFFFFFull;
    return v >= q ? v - q : v;
}

// Epilogues of the form out = (operand - v) * w (ModDown, rescale and their merged form)
// may finish on the FP64 pipe: with a nested `Pre`, `prep` as above and
//   uint64_t operand(const Pre &)        the canonical operand the output is subtracted from
//     (or double operand_d(const Pre &, int l, const FpMod &, bool big): the operand as an
//      exact integer in a double, |.| <= 2 q, centred when `big`)
//   double2 factor(int l)                {w, unused} as an exact integer in a double
//   void store(l, P, idx, pre, uint64_t) consume the canonical product
// the row phase forms (operand - x) * w from the UNCANONICALISED transform output x with
// one exact two-product Shoup step and canonicalises once — instead of canonicalising x
// and then spending ~25 integer instructions on a modular subtraction and a 64-bit Shoup
// multiply (profiles/r2_notes.md §13).
template <class E, class = void>
struct HasFactor : std::false_type {};
template <class E>
struct HasFactor<E, std::void_t<decltype(&E::factor)>> : std::true_type {};
template <class E, class = void>
struct HasOperandD : std::false_type {};
template <class E>
struct HasOperandD<E, std::void_t<decltype(&E::operand_d)>> : std::true_type {};

// Inverse-NTT epilogues that only multiply by a per-limb constant (the basis-conversion
// prescale) offer `uint64_t scale(int l)` and `store(l, P, idx, v)`: the kernel folds the
// constant into the N^-1 factors of its last stage, so the scaling costs nothing per
// element (it was a 64-bit integer Shoup multiply per output).
template <class E, class = void>
struct HasScale : std::false_type {};
template <class E>
struct HasScale<E, std::void_t<decltype(&E::scale)>> : std::true_type {};

template <bool kBig, class Pr>
__device__ __forceinline__ double pro_value(const Pr &pro, int l, long long P, int idx, const FpMod &m) {
    if constexpr (HasDval<Pr>::value) return pro.dval(l, P, idx, m, kBig);
    else return u2d(pro(l, P, idx));
}

// Cooley-Tukey butterfly. Large primes (2^47 <= q < 2^50) recentre after every SECOND
// stage (`cen`): |f_mulmod(y)| <= (1/2 + |y| 2^-53) q, so from |x| <= q/2 one stage gives
// |x| <= 1.07 q and the next |x| <= 1.7 q — still an exact integer in a double and, as
// the multiplicand of the following stage, below the 2^51 that keeps f_mulmod exact.
template <bool kBig>
__device__ __forceinline__ void ct_f(double &x, double &y, double2 w, const FpMod &m, bool cen = true) {
    const double r = f_mulmod(y, w.x, w.y, m.q);
    const double U = x;
    x = __dadd_rn(U, r);
    y = __dsub_rn(U, r);
    if (kBig && cen) {
        x = f_center(x, m);
        y = f_center(y, m);
    }
}
// Gentleman-Sande butterfly. The sum is recentred only when `center`: small primes
// (q < 2^47) recentre at stages 5 and 2 of each phase only. From inputs |x| <= 1.5 q the
// sums double per stage (3 q, 6 q, 12 q at stage 5: every difference stays below
// 2^51 > 16 q, the exact range of f_mulmod), a recentred stage returns to q / 2 and the
// products are below 0.75 q throughout.
// The large prime recentres sum and product after every second stage (`cen_big`, the
// odd stages): from |x| <= q/2 an uncentred stage leaves |x| <= q, so the next stage's
// difference stays below 2 q < 2^51.
template <bool kBig>
__device__ __forceinline__ void gs_f(double &x, double &y, double2 w, const FpMod &m, bool center = true,
                                     bool cen_big = true) {
    const double U = x, V = y;
    const double sum = __dadd_rn(U, V);
    x = (kBig ? cen_big : center) ? f_center(sum, m) : sum;
    y = f_mulmod(__dsub_rn(U, V), w.x, w.y, m.q);
    if (kBig && cen_big) y = f_center(y, m);
}

// The between-phase buffer is written once and read once by the cluster: its
// stores carry an L2 evict_last policy (keep it on chip until the other phase
// reads it) and its loads evict_first (dead after the read), so the streaming
// inputs and outputs do not push it out to HBM.
__device__ __forceinline__ void st_inter(double *p, double v) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_inter(const double *p) {
    uint64_t pol;
    double v;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// The shared 256-entry twiddle table is stored bank-conflict-free for the
// second half of each phase: stage s >= 5 reads entry 2^s + k 2^(s-4) + j in
// lane group k (16 row/column groups, j < 2^(s-4)), which in natural order puts
// the 16 lanes 2^(s-4) entries (>= 32 B) apart — an 8-way (s = 7) conflict per
// LDS.128 that kept the L1 data pipe at 93% (profiles/r2_ntt_notes.md). Stored
// at 2^s + 16 j + k instead, the 16 lanes read 16 consecutive entries.
__device__ __forceinline__ int tw_pos(int i) {  // storage slot of table entry i
    const int s = 31 - __clz(i | 1);
    if (s < 5) return i;
    const int m = i - (1 << s), sh = s - 4;
    return (1 << s) + ((m & ((1 << sh) - 1)) << 4) + (m >> sh);
}
// slot read by lane group k for element v (< 16) at stage s of a phase half
__device__ __forceinline__ int tw_idx(int s, int k, int v) {
    return s < 5 ? (1 << s) + ((16 * k + v) >> (8 - s)) : (1 << s) + ((v >> (8 - s)) << 4) + k;
}
// stage the shared 256-entry twiddle table of prime mi into shared memory
__device__ __forceinline__ void stage_table(double2 *st, const double2 *__restrict__ T) {
    for (int i = threadIdx.x; i < 256; i += kTh) st[tw_pos(i)] = T[i];
}

// ---------------------------------------------------------------- forward
// The column data is loaded before the twiddle table is staged (the table's
// load latency and the CTA barrier overlap the data loads).
template <bool kBig, class Pro>
__device__ __forceinline__ void fwd_cols(const Pro &pro, int l, long long P, double *inter, int tile,
                                         double2 *T, const double2 *__restrict__ Tg, const FpMod &m, double *sm,
                                         bool stage) {
    const int c = threadIdx.x % kTc, k = threadIdx.x / kTc, col = tile * kTc + c;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = pro_value<kBig>(pro, l, P, (k + 16 * u) * 256 + col, m);
    if (stage) {
        stage_table(T, Tg);
        __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int d = 8 >> s;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<kBig>(x[u], x[u + d], T[(1 << s) + (u >> (4 - s))], m, s & 1);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[(k + 16 * u) * kTc + c] = x[u];
    __syncthreads();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = sm[(16 * k + v) * kTc + c];
#pragma unroll
    for (int s = 4; s < 8; ++s) {
        const int d = 128 >> s;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) ct_f<kBig>(x[v], x[v + d], T[tw_idx(s, k, v)], m, (s & 1) && s != 7);
    }
#pragma unroll
    // no recentre for small primes: |x| < 13 q < 2^51 and the row phase starts with the
    // twist multiply (f_mulmod, exact for |x| < 2^51); the large prime leaves stage 7 with
    // |x| <= 1.7 q < 2^51 as well (its twist reads the correctly rounded w / q companion)
    for (int v = 0; v < 16; ++v) st_inter(inter + (16 * k + v) * 256 + col, x[v]);
}

// Row phase (four-step form): Z[r][c] = X[r][c] * tau(r, c) with
// tau(r, c) = psi^(c (2 brv8(r) + 1 - 256)); then the same 256-point negacyclic
// CT as the column phase (root psi^256, shared table T[1..255] held in shared
// memory `st`), output in bit-reversed order within the row. This is exactly
// stages 8..15 of the full transform; the twist replaces 255 row-specific
// twiddles per row by one coalesced table element per coefficient.
template <bool kBig, class Epi>
__device__ __forceinline__ void fwd_row(const Epi &epi, int l, long long P, const double *inter, int r,
                                        const double *__restrict__ tau, const double *__restrict__ tauq,
                                        const double2 *st, const FpMod &m, double *srow) {
    const int k = threadIdx.x & 15;
    const double *rd = inter + r * 256;
    const double *tr = tau + r * 256, *tq = tauq + r * 256;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = ld_inter(rd + k + 16 * u);
    // twist fused with stage 0 (pairs c, c+128, twiddle T[1]): the table holds
    // tau(r, c) for c < 128 and tau(r, c) * T[1] for c >= 128
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        // 8-byte table entries: w / q is one DMUL here instead of 8 more bytes per coefficient
        // through L1 (the L1 / LSU path ran at 77 % beside an FP64 pipe at 70 %)
        // (the large prime keeps the correctly rounded companion: its |x| <= 1.7 q multiplicand
        // leaves no room for the 1.5-ulp in-register estimate)
        const double ta = __ldg(tr + k + 16 * u), tb = __ldg(tr + k + 16 * (u + 8));
        const double aq = kBig ? __ldg(tq + k + 16 * u) : __dmul_rn(ta, m.qinv);
        const double bq = kBig ? __ldg(tq + k + 16 * (u + 8)) : __dmul_rn(tb, m.qinv);
        const double a = f_mulmod(x[u], ta, aq, m.q);
        const double b = f_mulmod(x[u + 8], tb, bq, m.q);
        x[u] = __dadd_rn(a, b);  // |a|, |b| <= 1.1 q (0.72 q for the large prime): an uncentred stage
        x[u + 8] = __dsub_rn(a, b);
    }
#pragma unroll
    for (int sp = 1; sp < 4; ++sp) {
        const int d = 8 >> sp;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) ct_f<kBig>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m, sp & 1);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = x[u];
    __syncwarp();
    // every lane's loads of this row have been consumed: drop its 16 lines (one per lane)
    if constexpr (DiscardInter<Epi>::value)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(rd + 16 * k) : "memory");
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
    for (int sp = 4; sp < 8; ++sp) {
        const int d = 128 >> sp;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) ct_f<kBig>(x[v], x[v + d], st[tw_idx(sp, k, v)], m, (sp & 1) && sp != 7);  // d2canon centres
    }
    __syncwarp();
    if constexpr (HasFactor<Epi>::value) {
        // |x| <= 13 q (small primes) or 1.7 q (the large prime, recentred here): the
        // difference from a canonical operand stays below 2^51
#pragma unroll
        for (int v = 0; v < 16; ++v) srow[pad16(16 * k + v)] = kBig ? f_center(x[v], m) : x[v];
        __syncwarp();
        const double w = epi.factor(l).x, wq = __dmul_rn(w, m.qinv);
        // operand loads in flight together: all 16 of the thread, or two groups of 8 when an
        // operand record is wider than one word (register budget: 64 per thread)
        constexpr int kG = sizeof(typename Epi::Pre) > 8 ? 8 : 16;
#pragma unroll
        for (int u0 = 0; u0 < 16; u0 += kG) {
            typename Epi::Pre pre[kG];
#pragma unroll
            for (int u = 0; u < kG; ++u) pre[u] = epi.prep(l, P, r * 256 + k + 16 * (u0 + u));
#pragma unroll
            for (int u = 0; u < kG; ++u) {
                double od;
                if constexpr (HasOperandD<Epi>::value) od = epi.operand_d(pre[u], l, m, kBig);
                else od = u2d(epi.operand(pre[u]));
                const double t = __dsub_rn(od, srow[pad16(k + 16 * (u0 + u))]);
                epi.store(l, P, r * 256 + k + 16 * (u0 + u), pre[u], d2canon(f_mulmod(t, w, wq, m.q), m));
            }
        }
    } else {
        uint64_t *su = reinterpret_cast<uint64_t *>(srow);
#pragma unroll
        for (int v = 0; v < 16; ++v) su[pad16(16 * k + v)] = d2canon(x[v], m);
        __syncwarp();
        if constexpr (HasPrep<Epi>::value) {
            typename Epi::Pre pre[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) pre[u] = epi.prep(l, P, r * 256 + k + 16 * u);
#pragma unroll
            for (int u = 0; u < 16; ++u) epi.fin(l, P, r * 256 + k + 16 * u, pre[u], su[pad16(k + 16 * u)]);
        } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) epi(l, P, r * 256 + k + 16 * u, su[pad16(k + 16 * u)]);
        }
    }
}

// One polynomial per cluster of CPP CTAs (launch attribute; CPP = 1: a lone CTA).
// Each CTA runs 16 / CPP column tiles, the cluster barrier, then 16 / CPP row
// blocks. Small clusters couple few CTAs at the phase barrier and pack every
// SM (16-CTA clusters at 4 CTAs/SM leave the SMs of a GPC beyond a multiple
// of four idle): 0.49-0.55 µs per limb-polynomial against 0.59 for one
// 16-CTA cluster per polynomial (tools/ntt_lab2.cu sweep, profiles/r1_notes.md).
template <class Pro, class Epi, int CPP>
__global__ void __launch_bounds__(kTh, 4)
    fwd_kernel(uint64_t *__restrict__ inter_base, int limb0, int B, const double2 *__restrict__ tw,
               const double *__restrict__ twist, const double *__restrict__ twistq, const FpMod *__restrict__ fm,
               Pro pro, Epi epi, int smaj) {
    constexpr int kT = kCl / CPP;
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % CPP;
    long long P = blockIdx.x / CPP;
    if (smaj) {  // sample-major launch order: the smaj limbs of one sample are adjacent
        const long long s = P / smaj;
        P = (P - s * smaj) * B + s;
    }
    const int l = (int)(P / B), mi = limb0 + l;
    const FpMod m = fm[mi];
    const double2 *T = tw + (size_t)mi * kN;
    const double *tau = twist + (size_t)mi * kN, *tauq = twistq + (size_t)mi * kN;
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    const int rs = threadIdx.x >> 4;
    if (m.q < (double)kSmallPrime) {
        for (int t = 0; t < kT; ++t) {
            if (t) __syncthreads();
            fwd_cols<false>(pro, l, P, inter, c * kT + t, st, T, m, smd, t == 0);
        }
        if (CPP > 1) cluster_sync_all();
        else __syncthreads();
        for (int t = 0; t < kT; ++t) {
            if (t) __syncwarp();
            fwd_row<false>(epi, l, P, inter, (c * kT + t) * kTc + rs, tau, tauq, st, m, smd + rs * kRowPad);
        }
    } else {
        for (int t = 0; t < kT; ++t) {
            if (t) __syncthreads();
            fwd_cols<true>(pro, l, P, inter, c * kT + t, st, T, m, smd, t == 0);
        }
        if (CPP > 1) cluster_sync_all();
        else __syncthreads();
        for (int t = 0; t < kT; ++t) {
            if (t) __syncwarp();
            fwd_row<true>(epi, l, P, inter, (c * kT + t) * kTc + rs, tau, tauq, st, m, smd + rs * kRowPad);
        }
    }
}

// ---------------------------------------------------------------- inverse
// Row phase, inverse (four-step form): the unscaled inverse of the twisted
// forward row phase is GS over the shared inverse table Ti[1..255] followed by
// multiplication with tau^-1(r, c).
template <bool kBig, class Pro>
__device__ __forceinline__ void inv_row(const Pro &pro, int l, long long P, double *inter, int r,
                                        const double *__restrict__ itau, const double2 *st, const FpMod &m,
                                        double *srow) {
    const int k = threadIdx.x & 15;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) srow[pad16(k + 16 * u)] = pro_value<kBig>(pro, l, P, r * 256 + k + 16 * u, m);
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = srow[pad16(16 * k + v)];
#pragma unroll
    for (int sp = 7; sp >= 4; --sp) {
        const int d = 128 >> sp;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) gs_f<kBig>(x[v], x[v + d], st[tw_idx(sp, k, v)], m, sp == 5, sp & 1);
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < 16; ++v) srow[pad16(16 * k + v)] = x[v];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = srow[pad16(k + 16 * u)];
#pragma unroll
    for (int sp = 3; sp >= 1; --sp) {
        const int d = 8 >> sp;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) gs_f<kBig>(x[u], x[u + d], st[(1 << sp) + (u >> (4 - sp))], m, sp == 2, sp & 1);
    }
    // stage 0 (pairs c, c+128, twiddle Ti[1]) fused with the untwist: the table holds
    // tau^-1(r, c) for c < 128 and tau^-1(r, c) * Ti[1] for c >= 128
    const double *tr = itau + r * 256;
    double *rd = inter + r * 256;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const double ta = __ldg(tr + k + 16 * u), tb = __ldg(tr + k + 16 * (u + 8));
        const double U = x[u], V = x[u + 8];
        // |f_mulmod| < 1.5 q: small primes skip the recentre (the column phase's first GS
        // stages keep |x| < 6 q); the large prime needs it for the next f_mulmod's range
        const double a = f_mulmod(__dadd_rn(U, V), ta, __dmul_rn(ta, m.qinv), m.q);
        const double b = f_mulmod(__dsub_rn(U, V), tb, __dmul_rn(tb, m.qinv), m.q);
        st_inter(rd + k + 16 * u, kBig ? f_center(a, m) : a);
        st_inter(rd + k + 16 * (u + 8), kBig ? f_center(b, m) : b);
    }
}

template <bool kBig, class Epi>
__device__ __forceinline__ void inv_cols(const Epi &epi, int l, long long P, const double *inter, int tile,
                                         const double2 *__restrict__ T, double2 ni, double2 niw, const FpMod &m,
                                         double *sm) {
    const int c = threadIdx.x % kTc, k = threadIdx.x / kTc, col = tile * kTc + c;
    double x[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = ld_inter(inter + (16 * k + v) * 256 + col);
#pragma unroll
    for (int s = 7; s >= 4; --s) {
        const int d = 128 >> s;
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (!(v & d)) gs_f<kBig>(x[v], x[v + d], T[tw_idx(s, k, v)], m, s == 5, s & 1);
    }
#pragma unroll
    for (int v = 0; v < 16; ++v) sm[(16 * k + v) * kTc + c] = x[v];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[(k + 16 * u) * kTc + c];
#pragma unroll
    for (int s = 3; s >= 1; --s) {
        const int d = 8 >> s;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (!(u & d)) gs_f<kBig>(x[u], x[u + d], T[(1 << s) + (u >> (4 - s))], m, s == 2, s & 1);
    }
    // stage 0 (twiddle Ti[1]) fused with the N^-1 scaling: niw = N^-1 * Ti[1]
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const double U = x[u], V = x[u + 8];
        x[u] = f_mulmod(__dadd_rn(U, V), ni.x, ni.y, m.q);
        x[u + 8] = f_mulmod(__dsub_rn(U, V), niw.x, niw.y, m.q);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        if constexpr (HasScale<Epi>::value) epi.store(l, P, (k + 16 * u) * 256 + col, d2canon(x[u], m));
        else epi(l, P, (k + 16 * u) * 256 + col, d2canon(x[u], m));
    }
}

template <class Pro, class Epi, int CPP>
__global__ void __launch_bounds__(kTh, 4)
    inv_kernel(uint64_t *__restrict__ inter_base, int limb0, int B, const double2 *__restrict__ itw,
               const double *__restrict__ itwist, const double2 *__restrict__ ninv, const FpMod *__restrict__ fm,
               Pro pro, Epi epi) {
    constexpr int kT = kCl / CPP;
    extern __shared__ double smd[];
    double2 *st = reinterpret_cast<double2 *>(smd + kTc * kRowPad);
    const int c = blockIdx.x % CPP;
    const long long P = blockIdx.x / CPP;
    const int l = (int)(P / B), mi = limb0 + l;
    const FpMod m = fm[mi];
    const double2 *T = itw + (size_t)mi * kN;
    const double *itau = itwist + (size_t)mi * kN;
    stage_table(st, T);
    __syncthreads();
    double *inter = reinterpret_cast<double *>(inter_base) + P * kN;
    const int rs = threadIdx.x >> 4;
    double2 ni = ninv[2 * mi], niw = ninv[2 * mi + 1];
    if constexpr (HasScale<Epi>::value) {  // N^-1 s and N^-1 Ti[1] s (|.| <= 0.75 q) with their /q companions
        const double sd = u2d(epi.scale(l)), sq = __dmul_rn(sd, m.qinv);
        ni.x = f_mulmod(ni.x, sd, sq, m.q);
        ni.y = __dmul_rn(ni.x, m.qinv);
        niw.x = f_mulmod(niw.x, sd, sq, m.q);
        niw.y = __dmul_rn(niw.x, m.qinv);
    }
    if (m.q < (double)kSmallPrime) {
        for (int t = 0; t < kT; ++t) {
            if (t) __syncwarp();
            inv_row<false>(pro, l, P, inter, (c * kT + t) * kTc + rs, itau, st, m, smd + rs * kRowPad);
        }
        if (CPP > 1) cluster_sync_all();
        else __syncthreads();
        for (int t = 0; t < kT; ++t) {
            if (t) __syncthreads();
            inv_cols<false>(epi, l, P, inter, c * kT + t, st, ni, niw, m, smd);
        }
    } else {
        for (int t = 0; t < kT; ++t) {
            if (t) __syncwarp();
            inv_row<true>(pro, l, P, inter, (c * kT + t) * kTc + rs, itau, st, m, smd + rs * kRowPad);
        }
        if (CPP > 1) cluster_sync_all();
        else __syncthreads();
        for (int t = 0; t < kT; ++t) {
            if (t) __syncthreads();
            inv_cols<true>(epi, l, P, inter, c * kT + t, st, ni, niw, m, smd);
        }
    }
}

// ---------------------------------------------------------------- functors
// (l, P, idx): limb l of the launch, polynomial P = l * B + b, coefficient idx < N
// of the context's ring (N = 2^16 or 2^17).
struct ProPlain {  // in[P][idx]
    const uint64_t *in;
    int log_n = kLogN;
    __device__ __forceinline__ uint64_t operator()(int, long long P, int idx) const { return in[(P << log_n) + idx]; }
};
struct EpiPlain {  // out[P][idx] = v
    uint64_t *out;
    int log_n = kLogN;
    __device__ __forceinline__ void operator()(int, long long P, int idx, uint64_t v) const {
        out[(P << log_n) + idx] = v;
    }
};

// ---------------------------------------------------------------- N = 2^17
// One radix-2 stage (pairs i, i + H, twiddle w = psi^H) plus a twist makes each
// half a 2^16 negacyclic transform with root psi^2 (half 0: (x_i + w x_{i+H}) psi^-i,
// half 1: (x_i - w x_{i+H}) psi^i), run by the kernels above as 2B sub-polynomials
// 2b + h of the same buffer; brv17(j) = 2 brv16(j) + h puts half h in positions
// [hH, (h+1)H) in exactly the 2^17 bit-reversed order. The inverse runs the 2^16
// inverse per half, then x_i = (z0 psi^i + z1 psi^-i) / 2, x_{i+H} = (z0 psi^i -
// z1 psi^-i) / (2w). Prologue / epilogue functors see the 2^17 indexing.
constexpr int kH17 = 1 << 16;

template <class Epi>
struct EpiHalf {  // sub-polynomial P2 = l * 2B + 2b + h, idx < 2^16 -> (l * B + b, h * H + idx)
    static constexpr bool kDiscardInter = DiscardInter<Epi>::value;
    Epi epi;
    int B;
    __device__ __forceinline__ void operator()(int l, long long P2, int idx, uint64_t v) const {
        const long long pb = P2 - (long long)l * 2 * B;
        epi(l, (long long)l * B + (pb >> 1), (int)((pb & 1) << 16) + idx, v);
    }
};
template <class Pro>
struct ProHalf {
    Pro pro;
    int B;
    __device__ __forceinline__ uint64_t operator()(int l, long long P2, int idx) const {
        const long long pb = P2 - (long long)l * 2 * B;
        return pro(l, (long long)l * B + (pb >> 1), (int)((pb & 1) << 16) + idx);
    }
};

template <class Pro>
__global__ void k17_pre(Pro pro, uint64_t *__restrict__ inter, int limb0, int B, const ulonglong2 *__restrict__ t17,
                        const ulonglong2 *__restrict__ w17, const ModQ *__restrict__ mq, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const long long P = gid >> 16;  // l * B + b
    const int i = (int)(gid & (kH17 - 1));
    const int l = (int)(P / B), m = limb0 + l;
    const uint64_t q = mq[m].q;
    const ulonglong2 w = w17[2 * m];
    const ulonglong2 *tm = t17 + (size_t)m * 4 * kH17;
    const uint64_t x = pro(l, P, i), t = mul_shoup(pro(l, P, i + kH17), w.x, w.y, q);
    const ulonglong2 pa = tm[i], pb = tm[kH17 + i];
    uint64_t *a = inter + (P << 17);
    a[i] = mul_shoup(add_mod(x, t, q), pa.x, pa.y, q);
    a[i + kH17] = mul_shoup(sub_mod(x, t, q), pb.x, pb.y, q);
}

template <class Epi>
__global__ void k17_post(Epi epi, const uint64_t *__restrict__ inter, int limb0, int B,
                         const ulonglong2 *__restrict__ t17, const ulonglong2 *__restrict__ w17,
                         const ModQ *__restrict__ mq, long long total) {
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const long long P = gid >> 16;
    const int i = (int)(gid & (kH17 - 1));
    const int l = (int)(P / B), m = limb0 + l;
    const uint64_t q = mq[m].q;
    const ulonglong2 wi = w17[2 * m + 1];
    const ulonglong2 *tm = t17 + (size_t)m * 4 * kH17;
    const ulonglong2 qa = tm[2 * kH17 + i], qb = tm[3 * kH17 + i];
    const uint64_t *a = inter + (P << 17);
    const uint64_t u0 = mul_shoup(a[i], qa.x, qa.y, q), u1 = mul_shoup(a[i + kH17], qb.x, qb.y, q);
    epi(l, P, i, add_mod(u0, u1, q));
    epi(l, P, i + kH17, mul_shoup(sub_mod(u0, u1, q), wi.x, wi.y, q));
}

// ---------------------------------------------------------------- launchers
// Forward / inverse NTT of n_limbs x B polynomials (primes limb0 ..) of the
// context's ring (2^16, or 2^17 via the radix-2 pass), input through `pro`,
// output through `epi`; `inter` ([n_limbs][B][N] words) may alias the output.
// CTAs per polynomial. The lab sweep (tools/ntt_lab2.cu) has 2 ahead by up to
// 4% on large isolated launches, but in the pipeline 4 is as fast on the
// device and 10% faster end to end: with 148 polynomials in flight the
// between-phase buffer (512 KiB each) stays in L2 instead of spilling to HBM
// (profiles/r1_notes.md).
constexpr int kCpp = 4;

template <class K, class... Args>
inline cudaError_t launch_clustered(K kern, int cpp, long long n_polys, cudaStream_t s, Args... args) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(cpp * n_polys));
    cfg.blockDim = dim3(kTh);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cpp;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <class Pro, class Epi>
inline int launch16_fwd(hk_ctx *c, uint64_t *inter, int limb0, int n_limbs, int B, const Pro &pro, const Epi &epi,
                        bool sample_major = false) {
    const long long n = (long long)n_limbs * B;
    const double2 *tw = (const double2 *)c->d_twf;
    const double *twist = c->d_twist, *twistq = c->d_twistq;
    const FpMod *fm = (const FpMod *)c->d_fmod;
    cudaError_t e;
    if constexpr (DiscardInter<Epi>::value) {
        // epilogues that stream operands and outputs past the between-phase buffer: fewer
        // polynomials in flight (8 CTAs each) keep that buffer in L2 (profiles/r2_notes.md §8)
        static const int cpp = getenv("HK_CPP_EPI") ? atoi(getenv("HK_CPP_EPI")) : 8;  // A/B knob: 4 -> 29.66, 8 -> 29.76 c1 inf/s
        if (cpp == 8)
            e = launch_clustered(fwd_kernel<Pro, Epi, 8>, 8, n, c->stream, inter, limb0, B, tw, twist, twistq, fm, pro, epi,
                                 sample_major ? n_limbs : 0);
        else
            e = launch_clustered(fwd_kernel<Pro, Epi, kCpp>, kCpp, n, c->stream, inter, limb0, B, tw, twist, twistq, fm, pro,
                                 epi, sample_major ? n_limbs : 0);
    } else {
        e = launch_clustered(fwd_kernel<Pro, Epi, kCpp>, kCpp, n, c->stream, inter, limb0, B, tw, twist, twistq, fm, pro, epi,
                             sample_major ? n_limbs : 0);
    }
    ++c->launches;
    if (e != cudaSuccess) return hk_fail(c, HK_E_CUDA, "ntt16 fwd launch: %s", cudaGetErrorString(e));
    HK_LAUNCH_CHECK(c, "ntt16 fwd");
    return HK_OK;
}

template <class Pro, class Epi>
inline int launch16_inv(hk_ctx *c, uint64_t *inter, int limb0, int n_limbs, int B, const Pro &pro, const Epi &epi) {
    const long long n = (long long)n_limbs * B;
    const double2 *itw = (const double2 *)c->d_itwf;
    const double *itwist = c->d_itwist;
    const double2 *ninv = (const double2 *)c->d_ninvf;
    const FpMod *fm = (const FpMod *)c->d_fmod;
    const cudaError_t e = launch_clustered(inv_kernel<Pro, Epi, kCpp>, kCpp, n, c->stream, inter, limb0, B, itw, itwist,
                                           ninv, fm, pro, epi);
    ++c->launches;
    if (e != cudaSuccess) return hk_fail(c, HK_E_CUDA, "ntt16 inv launch: %s", cudaGetErrorString(e));
    HK_LAUNCH_CHECK(c, "ntt16 inv");
    return HK_OK;
}

// rings served by the fused kernels
inline bool fused(const hk_ctx *c) { return c->log_n == kLogN || c->log_n == kLogN + 1; }

template <class Pro, class Epi>
// sample_major: launch the limbs of one sample next to each other (epilogues /
// prologues that read one per-sample operand for every limb, e.g. the rescale's
// broadcast remainder, then hit L2 instead of HBM)
inline int launch_fwd(hk_ctx *c, uint64_t *inter, int limb0, int n_limbs, int B, const Pro &pro, const Epi &epi,
                      bool sample_major = false) {
    if (n_limbs <= 0 || B <= 0) return HK_OK;
    if (c->log_n == kLogN) return launch16_fwd(c, inter, limb0, n_limbs, B, pro, epi, sample_major);
    const long long total = (long long)n_limbs * B * kH17;
    k17_pre<Pro><<<hk_grid(total, 256), 256, 0, c->stream>>>(pro, inter, limb0, B, c->d_n17, c->d_n17w, c->d_modq,
                                                             total);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "ntt17 pre");
    return launch16_fwd(c, inter, limb0, n_limbs, 2 * B, ProPlain{inter, kLogN}, EpiHalf<Epi>{epi, B}, sample_major);
}

template <class Pro, class Epi>
inline int launch_inv(hk_ctx *c, uint64_t *inter, int limb0, int n_limbs, int B, const Pro &pro, const Epi &epi) {
    if (n_limbs <= 0 || B <= 0) return HK_OK;
    if (c->log_n == kLogN) return launch16_inv(c, inter, limb0, n_limbs, B, pro, epi);
    int rc = launch16_inv(c, inter, limb0, n_limbs, 2 * B, ProHalf<Pro>{pro, B}, EpiPlain{inter, kLogN});
    if (rc) return rc;
    const long long total = (long long)n_limbs * B * kH17;
    k17_post<Epi><<<hk_grid(total, 256), 256, 0, c->stream>>>(epi, inter, limb0, B, c->d_n17, c->d_n17w, c->d_modq,
                                                              total);
    ++c->launches;
    HK_LAUNCH_CHECK(c, "ntt17 post");
    return HK_OK;
}

}  // namespace ntt16
