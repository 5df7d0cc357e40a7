/*
 * slotrank_b200.h -- C-ABI of the B200-native RNS-CKKS engine behind the
 * slotrank drop-in (paper_2412_15126_b200/engine.py).
 *
 * The reference's plug-in boundary is the duck-typed HESimulator method
 * surface (reference pkg/src/slotrank/engine.py:133-328); the algorithm
 * modules call nothing else.  Those methods are
 * realised by the Python engine on top of the entry points below, one group
 * per simulator method:
 *
 *   HESimulator.encrypt   engine.py:161-171  -> srk_encrypt (+ srk_small_to_ntt)
 *   HESimulator.decrypt   engine.py:173-175  -> srk_decrypt_limb0
 *   HESimulator.add/sub/negate engine.py:190-208 -> srk_addsub (+ level alignment:
 *                                               srk_mul_const_rescale)
 *   HESimulator.add_plain engine.py:209-213  -> srk_add_const / srk_add_plain
 *   HESimulator.mul       engine.py:215-223  -> srk_mul_relin_rescale
 *   HESimulator.mul_plain engine.py:225-232  -> srk_mul_const_rescale /
 *                                               srk_mul_plain_rescale (+ srk_encode_plain)
 *   HESimulator.rotate    engine.py:234-251  -> srk_rotate (+ srk_keygen for the
 *                                               Galois key of 5^k mod 2N)
 * and the finer primitives (srk_ntt*, srk_tensor, srk_rescale, srk_keyswitch,
 * srk_automorph, srk_mul_relin) are exported for bit-exact primitive parity
 * against oracle/ckks_oracle.c and for the config-2 microbenchmark.
 *
 * Conventions: every pointer argument named ct/a/b/out/pt/key is DEVICE
 * memory; k_res arrays are HOST arrays of per-limb residues.  A ciphertext at
 * level l is uint64[2][l+1][N] in NTT form (limb i under prime i).  Keys are
 * uint64[dnum][2][n_q+n_p][N] indexed by prime id.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  `ws` is a device workspace of
 * at least srk_workspace_bytes(ctx) bytes, 16-byte aligned, used stream-ordered.
 * Every function returns 0 on success or a negative code (SRK_E*) and sets a
 * thread-local message readable with srk_last_error(); nothing aborts.
 */
#ifndef SLOTRANK_B200_H
#define SLOTRANK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRK_OK 0
#define SRK_EINVAL -1
#define SRK_ENOMEM -2
#define SRK_ECUDA -3

typedef struct srk_ctx srk_ctx;

const char *srk_last_error(void);
int srk_version(void);
/* kernels launched by this library so far in this process (bench evidence) */
unsigned long long srk_kernel_launches(void);

/* measurement aid (bench.py's FP64 roof): launches one kernel of `ctas` CTAs x 256
 * threads in which every thread issues iters x 8 independent FP64 FMAs and nothing
 * else; the caller times it with events on `stream`.  sink: >= 1 device word. */
int srk_fp64_probe(int ctas, int iters, double *sink, void *stream);

/* context: primes[0..n_q) = Q chain, primes[n_q..n_q+n_p) = special primes;
 * roots[i] = primitive 2N-th root of unity mod primes[i] */
int srk_ctx_create(int device, int log_n, const uint64_t *primes, const uint64_t *roots, int n_q,
                   int n_p, int dnum, srk_ctx **out);
int srk_ctx_destroy(srk_ctx *ctx);
size_t srk_workspace_bytes(const srk_ctx *ctx);
/* Optional: the caller's second stream.  Two independent op sequences (the
 * ReplR and TransR+ReplC branches of the reference's rank_pipeline,
 * ranking.py:158-159) issued on the caller's main stream and on `stream`, each
 * with its own workspace, then run concurrently: ops on `stream` use the
 * context's second set of internal streams.  NULL unregisters. */
int srk_ctx_set_branch_stream(srk_ctx *ctx, void *stream);

/* batched NTT over n_polys polys of n_limbs limbs each (limb i under prime
 * first_prime + i; poly p at data + p * poly_stride words).  Inputs and
 * outputs are canonical residues in [0, q) (every entry point takes and returns
 * canonical limbs; the kernels' lazy / FP64 internal ranges depend on it). */
int srk_ntt(srk_ctx *ctx, uint64_t *data, int n_polys, long long poly_stride, int n_limbs,
            int first_prime, int inverse, void *stream);
/* NTT over extended polys at level l: limbs 0..l under Q primes, limbs
 * l+1..l+n_p under the special primes */
int srk_ntt_ext(srk_ctx *ctx, uint64_t *data, int n_polys, long long poly_stride, int level,
                int inverse, void *stream);

/* out = a (+|-) b, or -a (op 0 add, 1 sub, 2 negate) */
int srk_addsub(srk_ctx *ctx, const uint64_t *a, const uint64_t *b, uint64_t *out, int level,
               int op, void *stream);
/* out = a + constant (residues k_res[0..level]) in slot domain */
int srk_add_const(srk_ctx *ctx, const uint64_t *a, const uint64_t *k_res, uint64_t *out,
                  int level, void *stream);
/* out = a + pt (pt: uint64[level+1][N] NTT form) */
int srk_add_plain(srk_ctx *ctx, const uint64_t *a, const uint64_t *pt, uint64_t *out, int level,
                  void *stream);
/* out = a * k (no rescale); a read as a level-`level` view of a ciphertext
 * with src_limbs limbs per poly */
int srk_mul_const(srk_ctx *ctx, const uint64_t *a, int src_limbs, const uint64_t *k_res,
                  uint64_t *out, int level, void *stream);
int srk_mul_plain(srk_ctx *ctx, const uint64_t *a, const uint64_t *pt, uint64_t *out, int level,
                  void *stream);
/* d: uint64[3][level+1][N] */
int srk_tensor(srk_ctx *ctx, const uint64_t *a, const uint64_t *b, uint64_t *d, int level,
               void *stream);
/* level -> level-1, rounding division by q_level */
int srk_rescale(srk_ctx *ctx, const uint64_t *a, uint64_t *out, int level, void *ws,
                void *stream);
/* out(level-1) = rescale(view_level(a) * k) */
int srk_mul_const_rescale(srk_ctx *ctx, const uint64_t *a, int src_limbs, const uint64_t *k_res,
                          uint64_t *out, int level, void *ws, void *stream);
int srk_mul_plain_rescale(srk_ctx *ctx, const uint64_t *a, const uint64_t *pt, uint64_t *out,
                          int level, void *ws, void *stream);
/* hybrid key switching of d (uint64[level+1][N], NTT form) */
int srk_keyswitch(srk_ctx *ctx, const uint64_t *d, const uint64_t *key, uint64_t *out0,
                  uint64_t *out1, int level, void *ws, void *stream);
int srk_mul_relin(srk_ctx *ctx, const uint64_t *a, const uint64_t *b, const uint64_t *rlk,
                  uint64_t *out, int level, void *ws, void *stream);
int srk_mul_relin_rescale(srk_ctx *ctx, const uint64_t *a, const uint64_t *b,
                          const uint64_t *rlk, uint64_t *out, int level, void *ws, void *stream);
int srk_automorph(srk_ctx *ctx, const uint64_t *a, uint64_t *out, long long n_limbs_total,
                  uint64_t galois, void *stream);
int srk_rotate(srk_ctx *ctx, const uint64_t *a, const uint64_t *gkey, uint64_t *out, int level,
               uint64_t galois, void *ws, void *stream);

/* batched forms (the config-2 microbenchmark and multi-ciphertext
 * pipelines): `batch` ciphertexts at ct strides a_ct / out_ct (words) */
int srk_rescale_batch(srk_ctx *ctx, const uint64_t *a, long long a_ct, uint64_t *out,
                      long long out_ct, int batch, int level, void *ws, void *stream);
/* rescale != 0: relinearised product rescaled to level-1 */
int srk_mul_relin_batch(srk_ctx *ctx, const uint64_t *a, const uint64_t *b, long long ab_ct,
                        const uint64_t *rlk, uint64_t *out, long long out_ct, int batch, int level,
                        int rescale, void *ws, void *stream);
/* the same over a table of operand pairs: a[i] x b[i] for i < batch (HOST arrays of
 * DEVICE pointers to [2][level+1][N] ciphertexts; pairs may share operands -- the
 * composite polynomials' (y y, u3 y, u7 y) -- so no batch is copied together first);
 * out packed at ct stride out_ct.  HESimulator.mul on several pairs at once. */
int srk_mul_relin_ptrs(srk_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, int batch,
                       const uint64_t *rlk, uint64_t *out, long long out_ct, int level, int rescale,
                       void *ws, void *stream);
int srk_rotate_batch(srk_ctx *ctx, const uint64_t *a, long long a_ct, const uint64_t *gkey,
                     uint64_t *out, long long out_ct, int batch, int level, uint64_t galois,
                     void *ws, void *stream);
/* elementwise / plaintext ops over `batch` packed ciphertexts [batch][2][level+1][N] */
int srk_addsub_batch(srk_ctx *ctx, const uint64_t *a, const uint64_t *b, uint64_t *out, int batch,
                     int level, int op, void *stream);
/* pt != NULL: plaintexts at stride pt_ct words (0 = shared); else constant k_res */
int srk_add_plain_batch(srk_ctx *ctx, const uint64_t *a, const uint64_t *pt, long long pt_ct,
                        const uint64_t *k_res, uint64_t *out, int batch, int level, void *stream);
int srk_mul_const_rescale_batch(srk_ctx *ctx, const uint64_t *a, long long a_ct, int src_limbs,
                                const uint64_t *k_res, uint64_t *out, int batch, int level, void *ws,
                                void *stream);
int srk_mul_plain_rescale_batch(srk_ctx *ctx, const uint64_t *a, const uint64_t *pt, long long pt_ct,
                                uint64_t *out, int batch, int level, void *ws, void *stream);
/* n_rot rotations of each of `batch` ciphertexts sharing one base extension
 * per ciphertext (hoisting); gkeys / galois / outs are HOST arrays (of device
 * pointers); rotation r of ciphertext b lands at outs[r] + b * out_ct */
int srk_rotate_hoisted(srk_ctx *ctx, const uint64_t *a, long long a_ct, int batch, int n_rot,
                       const uint64_t *const *gkeys, const uint64_t *galois, uint64_t *const *outs,
                       long long out_ct, int level, void *ws, void *stream);

/* sampling / keys / encryption */
int srk_uniform(srk_ctx *ctx, uint64_t *a, int n_limbs, int first_prime, uint64_t seed,
                uint64_t stream_base, void *stream);
/* out[k] = NTT(v mod prime(first_prime + k)), v: int64[N] device */
int srk_small_to_ntt(srk_ctx *ctx, const int64_t *v, uint64_t *out, int n_limbs, int first_prime,
                     void *stream);
int srk_square(srk_ctx *ctx, const uint64_t *s, uint64_t *out, int n_limbs, void *stream);
/* switching key sfrom -> s; e: int64[dnum][N] device */
int srk_keygen(srk_ctx *ctx, const uint64_t *s_ntt, const uint64_t *sfrom_ntt, const int64_t *e,
               uint64_t seed, uint64_t key_id, uint64_t *key, void *ws, void *stream);
/* Rotation keys are consumed in "rotation layout": the switching key
 * sigma_g(s) -> s with every limb permuted by sigma_g^-1, so the key-switch
 * inner product streams coalesced and sigma_g is applied while ModDown reads
 * the accumulator.  srk_keygen_galois produces that layout directly;
 * srk_permute_key converts a standard-layout key in place (tmp: 2*n_primes
 * limbs of device scratch).  srk_rotate* expect rotation-layout keys. */
int srk_keygen_galois(srk_ctx *ctx, const uint64_t *s_ntt, const int64_t *e, uint64_t seed,
                      uint64_t key_id, uint64_t galois, uint64_t *key, void *ws, void *stream);
int srk_permute_key(srk_ctx *ctx, uint64_t *key, uint64_t galois, void *tmp, void *stream);
/* m, e: int64[N] device; out: uint64[2][level+1][N] */
int srk_encrypt(srk_ctx *ctx, const int64_t *m, const uint64_t *s_ntt, const int64_t *e,
                uint64_t seed, uint64_t seq, uint64_t *out, int level, void *ws, void *stream);
/* m_out: int64[N] device, centred coefficients of c0 + c1 s mod q_0 */
int srk_decrypt_limb0(srk_ctx *ctx, const uint64_t *ct, const uint64_t *s_ntt, int64_t *m_out,
                      int level, void *ws, void *stream);
/* BSGS leaf sum before its single rescale: out = sum_i k[i] * terms[i] over
 * limbs 0..level (terms: HOST array of device pointers, term_limbs: HOST
 * limbs per poly of each term, k: DEVICE residues [n_terms][level+1]) */
int srk_lincomb(srk_ctx *ctx, const uint64_t *const *terms, const int *term_limbs, int n_terms,
                const uint64_t *k, uint64_t *out, int batch, int level, void *stream);
/* n_out leaf sums over the SAME terms (every BSGS leaf of a polynomial shares the
 * baby-step ciphertexts, reference chebyshev.py:206-222): outs[l] = sum_i k[l][i] *
 * terms[i]; k: DEVICE residues [n_out][n_terms][level+1]; kf: DEVICE doubles k / q_j in
 * the same layout (limbs under primes < 2^41 then sum on the FP64 pipe, exactly) or
 * NULL; outs: HOST array of device pointers.  Each term word is read once per eight
 * outputs. */
int srk_lincomb_multi(srk_ctx *ctx, const uint64_t *const *terms, const int *term_limbs, int n_terms,
                      const uint64_t *k, const double *kf, uint64_t *const *outs, int n_out, int batch,
                      int level, void *stream);
/* multi-GPU fix-up after an int64 all-reduce of n_polys polys of level+1
 * limbs (values < 2^63): reduce every limb mod its prime in place */
int srk_reduce_mod(srk_ctx *ctx, uint64_t *data, int n_polys, int level, void *stream);
/* pt_out: uint64[level+1][N] = NTT(coeffs mod q_i) */
int srk_encode_plain(srk_ctx *ctx, const int64_t *coeffs, uint64_t *pt_out, int level,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif
