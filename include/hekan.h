/*
 * hekan.h — C ABI of the B200 RNS-CKKS engine behind the reference's
 * `HeBackend` plugin contract (/root/reference/pkg/src/hekan/backend.py:132-270).
 *
 * The reference is a pure-Python float64 slot simulator; this ABI is the
 * boundary a real scheme is substituted behind ("a swappable contract so a real
 * scheme can be substituted behind the same semantics", backend.py:6-7). Every
 * entry point below replaces one reference method; the Python host mirror
 * (paper_2409_07751_b200/backend.py) binds them with ctypes.
 *
 * Two libraries export this ABI:
 *   paper_2409_07751_b200/libhekan_gpu.so — the product (sm_100a CUDA); all
 *       buffer arguments are DEVICE pointers, work is enqueued on the stream set
 *       with hk_set_stream (default: the legacy stream).
 *   oracle/libckks_oracle.so — CPU restatement used only by tests/bench as the
 *       bit-exact checker; buffer arguments are HOST pointers.
 *
 * Conventions
 *   N = 2^log_n coefficients, S = N/2 complex slots (real payloads only).
 *   Every prime lies in (2^44, 2^50) and is 1 mod 2N (hk_ctx_create rejects others):
 *   the GPU keeps 25-bit limb splits and lazy NTT residues inside 64-bit words.
 *   A ciphertext at reference level l has l+1 RNS limbs (primes q_0..q_l) and
 *   layout u64 [2][l+1][B][N]  (poly, limb, batch, coefficient), NTT domain,
 *   canonical residues in [0, q_i). A plaintext at level l is u64 [l+1][Bp][N]
 *   with Bp = 1 (broadcast over the batch) or Bp = B.
 *   NTT domain order: position j holds a(psi^(2*brv(j)+1)) (bit-reversed).
 *   Slot j <-> root zeta^(5^j mod 2N); rotate-left by t <-> galois 5^t mod 2N.
 *   Levels passed as ints; an op on operands at different levels first drops
 *   the higher one to the lower (limbs beyond are ignored), as
 *   HeBackend.slotwise takes level = min(a.level, b.level) (backend.py:202-203).
 *
 * Status codes (every function returns int): HK_OK or one of HK_E_* below; a
 * message is available from hk_last_error(ctx). The Python mirror maps them to
 * the reference's exception taxonomy (errors.py:4-87).
 */
#ifndef HEKAN_H
#define HEKAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HK_OK 0
#define HK_E_ARG 1        /* ValueError: bad level/size/argument (backend.py:163-164, :240-241) */
#define HK_E_DEPTH 2      /* DepthExhausted: multiply at level < 1 (backend.py:216-217)          */
#define HK_E_LENGTH 3     /* LengthMismatch: wrong operand kind/size (backend.py:198-201, :253-255) */
#define HK_E_NOKEY 4      /* rotation/relin key missing for this galois element                  */
#define HK_E_CUDA 5       /* CUDA runtime error (product library only)                            */
#define HK_E_NOMEM 6      /* allocation failure                                                  */

typedef struct hk_ctx hk_ctx;

typedef struct hk_params {
    int32_t log_n;          /* N = 2^log_n                                            */
    int32_t n_q;            /* ciphertext primes q_0..q_{n_q-1}; depth budget = n_q-1 */
    int32_t n_p;            /* special primes for hybrid key switching                */
    int32_t dnum;           /* key-switching digits over the full q chain, 1..8       */
    const uint64_t *q;      /* [n_q]                                                  */
    const uint64_t *p;      /* [n_p]                                                  */
    const uint64_t *psi_q;  /* [n_q] primitive 2N-th roots                            */
    const uint64_t *psi_p;  /* [n_p]                                                  */
} hk_params;

/* ---- context (replaces BackendConfig + HeBackend.__init__, backend.py:23-66, :140-143) */
int hk_ctx_create(const hk_params *params, int32_t device, hk_ctx **out);
void hk_ctx_destroy(hk_ctx *ctx);
const char *hk_last_error(const hk_ctx *ctx);
int hk_set_stream(hk_ctx *ctx, void *cuda_stream);   /* oracle: no-op */
int hk_sync(hk_ctx *ctx);

/* ---- keys (client side; replaces nothing — the reference has no keys).
 * Randomness: ChaCha20 (20 rounds, 64-bit block counter + 64-bit stream as the
 * nonce) keyed by a 256-bit `seed` (4 words, HOST memory); 64-bit output word
 * c of stream s is words 2(c mod 8), 2(c mod 8)+1 of block c / 8. Identical in
 * oracle and GPU. Secret key, relinearisation key and one Galois key per element
 * come from one seed; callers draw it from the OS CSPRNG (the Python backend
 * does unless a test seeds it explicitly). */
int hk_keygen(hk_ctx *ctx, const uint64_t seed[4]);
int hk_add_galois_keys(hk_ctx *ctx, const uint64_t seed[4], const uint32_t *galois_elts, int32_t n);
/* Galois keys usable up to ciphertext `level` only: digits 0..level/alpha and the
 * rows of q_0..q_level plus the special primes (the same values as the full key's
 * rows, so results are identical). A key already present at a lower level is
 * regenerated at `level`; one at a higher level is kept. The oracle keeps full keys. */
int hk_add_galois_keys_level(hk_ctx *ctx, const uint64_t seed[4], const uint32_t *galois_elts, int32_t n,
                             int32_t level);
/* 0 if absent, else 1 + the highest ciphertext level the key serves. */
int hk_has_galois_key(const hk_ctx *ctx, uint32_t galois_elt);
/* copy key material out (parity tests): which = 0 secret [n_q+n_p][N];
 * 1 relin [n_digits][2][n_q+n_p][N]; 2 galois key for `galois_elt` (full-level
 * keys only, same layout as relin). */
int hk_export_key(hk_ctx *ctx, int32_t which, uint32_t galois_elt, uint64_t *out);
uint64_t hk_key_words(const hk_ctx *ctx, int32_t which);

/* ---- transforms on raw limb buffers [n_limbs][batch][N]; limb l uses prime
 * index limb0 + l in the concatenated chain (q_0..q_{n_q-1}, p_0..p_{n_p-1}). */
int hk_ntt_fwd(hk_ctx *ctx, uint64_t *buf, int32_t limb0, int32_t n_limbs, int32_t batch);
int hk_ntt_inv(hk_ctx *ctx, uint64_t *buf, int32_t limb0, int32_t n_limbs, int32_t batch);

/* ---- encode / decode (HeBackend.encode, backend.py:149-158; decrypt :168-170).
 * slots: f64 [batch][S] (real payloads). pt: u64 [level+1][batch][N], NTT. */
int hk_encode(hk_ctx *ctx, const double *slots, int32_t batch, int32_t level,
              double scale, uint64_t *pt);
/* BSGS diagonals of consecutive giant-step blocks of nb diagonals, generated and
 * encoded in one call (inference.py:166-176, the diagonal gather + np.roll + encode
 * per diagonal): diagonal v in [0, count) has slot s = W~[r][(r + base + v) mod m],
 * r = (s - rb) mod S with rb = base + (v / nb) * nb (its block's roll), zero for
 * r >= m, W~ the n_o x n_in row-major matrix `W` zero-padded to m x m (requires
 * base + count <= m <= S). W lives where the engine's buffers live (device for the
 * GPU, host for the oracle). pt: u64 [level+1][count][N], identical to hk_encode
 * of the same slot vectors. */
int hk_encode_diagonals(hk_ctx *ctx, const double *W, int32_t n_o, int32_t n_in, int32_t m, int32_t base,
                        int32_t count, int32_t nb, int32_t level, double scale, uint64_t *pt);
/* Constant c at scale: per-limb residues of round(c*scale) for limbs 0..level. */
int hk_encode_const(hk_ctx *ctx, double c, int32_t level, double scale, uint64_t *res);

/* ---- encrypt / decrypt (HeBackend.encrypt / decrypt, backend.py:160-170).
 * Secret-key RLWE encryption; randomness from (seed, sample, limb, coeff) with
 * sample = first_sample + batch index, so a batch sharded over ranks (rank r
 * passing its first global sample index) encrypts exactly as the whole batch
 * would in one call, and no (a, e) pair repeats across ranks. */
int hk_encrypt(hk_ctx *ctx, const uint64_t *pt, int32_t level, int32_t batch,
               const uint64_t seed[4], uint64_t first_sample, uint64_t *ct);
int hk_decrypt(hk_ctx *ctx, const uint64_t *ct, int32_t level, int32_t batch,
               double scale, double *slots);

/* ---- slot-wise arithmetic (HeBackend.slotwise add/sub, backend.py:192-214) */
int hk_add(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb,
           uint64_t *out, int32_t batch);
int hk_sub(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb,
           uint64_t *out, int32_t batch);
/* ct +/- plaintext; pt at level >= la (limbs beyond la ignored), pt_batch 1 or batch */
int hk_add_plain(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *pt, int32_t lp,
                 int32_t pt_batch, int32_t negate, uint64_t *out, int32_t batch);
/* ct + constant: res[l] = residue of the constant for limb l (hk_encode_const) */
/* res is a HOST array in both libraries */
int hk_add_const(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *res,
                 uint64_t *out, int32_t batch);

/* ---- multiplications (slotwise mul_pt / mul_ct, backend.py:215-224): each
 * consumes one level (rescale by q_la); out is at level la-1 (or min-1). */
int hk_mul_plain(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *pt, int32_t lp,
                 int32_t pt_batch, uint64_t *out, int32_t batch);
int hk_mul_const(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *res,
                 uint64_t *out, int32_t batch);
/* ct x ct: tensor product, relinearisation (hybrid key switch), rescale */
int hk_mul(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb,
           uint64_t *out, int32_t batch);
/* a x b + k x: a relinearised product and a constant multiple of a third
 * ciphertext x (level lx >= min(la, lb)) sharing one ModDown + rescale, the
 * Estrin / Chebyshev combine `hi * T + c * x` of approx.py:_combine
 * (reference approx.py:381-405: mul_ct, mul_pt by a scalar, add). res = HOST
 * residues of k for limbs 0..min(la, lb) (hk_encode_const at the scale that
 * puts k x / q_l on the product's scale). out is at level min(la, lb) - 1. */
int hk_mul_lin(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb,
               const uint64_t *x, int32_t lx, const uint64_t *res, uint64_t *out, int32_t batch);
/* a x b + a2 x b2: two products summed before one relinearisation and one
 * rescale (the Cox-de Boor step b = w1 b + w2 rot(b), reference
 * bspline.py:308-317 as two mul_ct and an add). out is at level
 * min(la, lb, la2, lb2) - 1. */
int hk_mul2(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, const uint64_t *a2,
            int32_t la2, const uint64_t *b2, int32_t lb2, uint64_t *out, int32_t batch);
/* mult * (a x b) + c: a relinearised product with the Chebyshev power step's
 * doubling and constant folded into its last epilogue (T_2k = 2 T_k^2 - 1,
 * reference approx.py:381-405 as mul_ct, add, add of a scalar); bit-identical
 * to hk_mul, hk_add(out, out), hk_add_const. mult is 1 or 2; res = HOST
 * residues of c for limbs 0..min(la, lb) - 1 (hk_encode_const at the output
 * level), or NULL for no constant. */
int hk_mul_affine(hk_ctx *ctx, const uint64_t *a, int32_t la, const uint64_t *b, int32_t lb, int32_t mult,
                  const uint64_t *res, uint64_t *out, int32_t batch);
/* rescale only (drop q_la): out level la-1 */
int hk_rescale(hk_ctx *ctx, const uint64_t *a, int32_t la, uint64_t *out, int32_t batch);

/* ---- rotation (HeBackend.rotate, backend.py:237-245): Galois automorphism
 * X -> X^g plus key switch back to s. Left rotation by t uses g = 5^t mod 2N. */
int hk_rotate(hk_ctx *ctx, const uint64_t *a, int32_t la, uint32_t galois_elt,
              uint64_t *out, int32_t batch);
/* Hoisted rotations of one source (baby steps of bsgs_matvec,
 * inference.py:161-162): one ModUp shared by all n outputs. outs[i] is a
 * ct at level la for galois_elts[i]. */
int hk_rotate_hoisted(hk_ctx *ctx, const uint64_t *a, int32_t la,
                      const uint32_t *galois_elts, int32_t n, uint64_t *const *outs,
                      int32_t batch);
/* sum_i sigma_{g_i}(ct_i) for n ciphertexts at level la (g_i = 1: identity, no key
 * switch): the BSGS giant-step accumulation of inference.py:177-180 with the key
 * inner products summed in the extended basis and ONE ModDown (lazy ModDown).
 * Logically n rotations (non-identity) + (n-1) adds; out [2][la+1][B][N]. */
int hk_rotate_sum(hk_ctx *ctx, const uint64_t *const *cts, int32_t la, const uint32_t *galois_elts, int32_t n,
                  uint64_t *out, int32_t batch);

/* ---- fused BSGS giant-step block (inference.py:166-178): for one giant step
 * out = sum_i pt_i (*) babies_i, accumulated lazily, then ONE rescale.
 * babies[i]: ct at level la; pts[i]: plaintext at level >= la (pt_batch 1) whose
 * limb l starts at pts[i] + l * pt_stride * N (1 for a plain [lp+1][1][N]
 * plaintext; `count` for diagonal v of hk_encode_diagonals, pts[v] = pt + v * N).
 * Logically this is n mul_pt + (n-1) add; out is at level la-1. */
int hk_mac_plain(hk_ctx *ctx, const uint64_t *const *babies, const uint64_t *const *pts,
                 int32_t n, int32_t la, int32_t lp, int32_t pt_stride, uint64_t *out, int32_t batch);

/* G <= 8 consecutive giant-step blocks sharing one set of n <= 192 babies, each
 * block exactly hk_mac_plain(babies[0..counts[g]), diagonals g*nb .. g*nb+counts[g]-1
 * of `pt` ([la+1][pt_count][N], hk_encode_diagonals), pt_stride = pt_count) into
 * outs[g] at level la-1. Every baby is read once for the group (c4/c5 BSGS). */
int hk_mac_plain_blocks(hk_ctx *ctx, const uint64_t *const *babies, int32_t n, int32_t la, const uint64_t *pt,
                        int32_t pt_count, int32_t nb, int32_t G, const int32_t *counts, uint64_t *const *outs,
                        int32_t batch);

/* ---- introspection */
int32_t hk_version(void);
/* kernels enqueued by this context so far (oracle: 0) — bench evidence */
uint64_t hk_launch_count(const hk_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* HEKAN_H */
