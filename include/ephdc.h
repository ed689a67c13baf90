/*
 * ephdc.h -- C ABI of libephdc.so, the B200 (sm_100a) hot path of EP-HDC's
 * client-side encrypted HDC inference (arXiv 2511.00737).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n
 * (both only on the build box), readings "#n" = DESIGN.md section "Readings".
 *
 * The problem: the server holds the secret key and encrypts the k
 * class hypervectors ONCE as D ciphertexts (slot i of ciphertext d holds
 * C[i mod k][d], P:650-653 / P:1471-1474); the client packs B = floor(N/k)
 * plaintext query hypervectors into D plaintexts (slot i of plaintext d holds
 * h[d][query i/k]) and evaluates sum_d CT_d (x) PT_d -- D ct*pt multiplies,
 * D-1 ct+ct adds, 0 rotations -- returning one scores
 * ciphertext per batch of B queries, which the server decrypts.
 *
 * Conventions (all entry points):
 *  - Return an ephdc_status; no exception crosses the ABI, nothing aborts.
 *  - Opaque handles (ctx, sk, model, workspace, ntt_plan) are owned by the
 *    library: create/free pairs; *_free(NULL) is a no-op.  Handles are
 *    immutable after creation except the workspace, which one stream at a
 *    time may use.
 *  - "d_" pointers are DEVICE pointers on the context's device, "h_" pointers
 *    are HOST pointers; both are caller-owned and only borrowed for the call.
 *  - Device work is enqueued asynchronously on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream); a launch failure returns
 *    EPHDC_ECUDA immediately.  Calls documented as "synchronous" finish all
 *    their device work before returning.
 *  - Layouts are C row-major, little-endian; residues are canonical in [0, p)
 *    at every boundary (reading #24).
 *  - Decryption failure (noise overflow) is NOT an error.
 *  - No CPU fallback: every compute entry point runs CUDA kernels; if no
 *    device is usable it returns EPHDC_ECUDA.
 */
#ifndef EPHDC_H
#define EPHDC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EPHDC_ABI_VERSION 4
#define EPHDC_MAX_PRIMES 16

typedef enum {
    EPHDC_OK = 0,
    EPHDC_EPARAM = 1,     /* bad N, t, q, sizes                      */
    EPHDC_ECONTEXT = 2,   /* handle from another context / host-only context       */
    EPHDC_EOVERFLOW = 3,  /* output capacity < ceil(nq / B) ciphertexts     */
    EPHDC_ERESOURCE = 4,  /* allocation failed                                     */
    EPHDC_ECUDA = 5,      /* CUDA error (no device, launch or copy failure)        */
    EPHDC_EDOMAIN = 6,    /* value outside its modular domain                      */
    EPHDC_ENULL = 7       /* required pointer is NULL                              */
} ephdc_status;

/* BFV + HDC parameter set (S8 of SURVEY.md; BASELINE.json configs). */
typedef struct {
    uint32_t log2N;          /* ring degree N = 2^log2N, 10 <= log2N <= 14        */
    uint32_t L;              /* number of RNS primes, 1..EPHDC_MAX_PRIMES         */
    const uint64_t *q;       /* [L] distinct primes = 1 mod 2N, < 2^60, != t      */
    uint64_t t;              /* plaintext modulus: prime = 1 mod 2N, < 2^30       */
    uint32_t k;              /* classes, 1 <= k <= N                              */
    uint32_t D_live;         /* hypervector dimension used by the model           */
    uint32_t D_stored;       /* rows of the projection base (>= D_live; padding)  */
    uint32_t F;              /* features per query, multiple of 4                 */
    uint32_t feat_unsigned;  /* 0: int8 features, 1: uint8 features               */
    uint32_t Qbits;          /* query HV width, 2..8 (reading #12)  */
    uint32_t Cbits;          /* class HV width, 2..8                              */
    uint32_t qshift;         /* query rounding shift s (reading #13)              */
    double sigma_e;          /* BFV error std-dev (3.2, BASELINE.json configs[0]) */
    uint32_t arith;          /* modular-arithmetic pipe of the fused NTT+MAC kernel:
                              * EPHDC_ARITH_AUTO (0): FP64 pipe when every q_j < 2^50
                              * and the value bounds of DESIGN.md "FP64 modular
                              * arithmetic" hold, else the integer pipe;
                              * EPHDC_ARITH_INT (1): integer pipe (u64 Shoup/Montgomery);
                              * EPHDC_ARITH_F64 (2): FP64 pipe, EPARAM if not eligible.
                              * Both give bit-identical results.                    */
    uint32_t encoder;        /* HDC encoding GEMM: EPHDC_ENCODER_AUTO (0): tcgen05
                              * kind::i8 tensor-core kernel fed by TMA when F % 16 == 0
                              * (else CUDA-core dp4a); EPHDC_ENCODER_DP4A (1): dp4a.
                              * Both are exact (int32).                              */
} ephdc_params;

#define EPHDC_ENCODER_AUTO 0u
#define EPHDC_ENCODER_DP4A 1u

#define EPHDC_ARITH_AUTO 0u
#define EPHDC_ARITH_INT 1u
#define EPHDC_ARITH_F64 2u

/* Derived values of a context (for tests and tooling). */
typedef struct {
    uint32_t N, L, B, k;     /* B = floor(N/k) queries per ciphertext     */
    uint64_t t, psi_t;       /* psi_t: minimal primitive 2N-th root mod t (#2)   */
    uint64_t q[EPHDC_MAX_PRIMES];
    uint64_t psi[EPHDC_MAX_PRIMES];    /* minimal primitive 2N-th roots mod q_j  */
    uint64_t delta[EPHDC_MAX_PRIMES];  /* floor(Q/t) mod q_j, Q = prod q_j (#4) */
    uint32_t fused_split;    /* S: CTAs per polynomial in the fused MAC kernel   */
    uint32_t fused_chunks;   /* dim chunks per batch in the fused MAC kernel     */
    int device;              /* CUDA device, -1 for a host-only context          */
    uint32_t arith;          /* selected pipe: EPHDC_ARITH_INT or EPHDC_ARITH_F64 */
    uint32_t f64_red_every;  /* FP64 path: accumulator reduction interval (dims) */
} ephdc_ctx_info;

/* TEST / PROFILING launch-plan overrides of a workspace (ephdc_workspace_create;
 * NULL or all zeros = the tuned plan).  Results are bit-identical for every value
 * (tests/test_gpu_variants.py); nothing else -- no environment variable -- changes a
 * launch plan. */
typedef struct {
    uint32_t flags;      /* FP64 fused kernel: bits 1-2 = 1/2/3 force the pass
                          * synchronisation WL = 0/2/1; bit 0 = no L2 prefetch of the
                          * model slice, bit 4 = prefetch; bit 3 = 32 elements per
                          * thread (NC = 2^13); bit 5 = the one-team kernel at NC =
                          * 2^13 with one slice (default there: two warp groups; bits
                          * 1-3 also select a one-team variant); bit 6 = the two-group
                          * kernel at N = 2^14 (default there: one team); bit 7 = the
                          * round-1 slot pack + INTT_t kernel (default at N >= 2^12:
                          * the ntt32_c5.cu passes); bit 8 = that kernel without the
                          * L1 prefetch of the next row's query bytes                 */
    uint32_t bg;         /* FP64 fused kernel: batches per group (0 = planner)       */
    uint32_t G;          /* FP64 fused kernel: dims per chunk (0 = planner)          */
    uint32_t m_batches;  /* batches of encoded plaintexts kept (0 = planner: all of
                          * max_nq, capped at 32 GB)                                 */
} ephdc_plan;

typedef struct ephdc_ctx ephdc_ctx;
typedef struct ephdc_sk ephdc_sk;
typedef struct ephdc_model ephdc_model;
typedef struct ephdc_workspace ephdc_workspace;
typedef struct ephdc_ntt_plan ephdc_ntt_plan;

/* Key of the random streams (reading #7): every secret-key coefficient, uniform a and
 * Gaussian e is a 64-bit word of a ChaCha20 block (RFC 8439 sec. 2.3) under this
 * 256-bit key, the block counter and nonce naming the value (tag, ciphertext index,
 * coefficient).  Threat model: c1 = a is published to the client, so the
 * generator must be a PRF under a key the client cannot guess -- a NULL seed pointer
 * (every entry point below that takes one) draws a fresh key from the OS CSPRNG.
 * Callers that need reproducible streams (parity tests, benchmarks) build a key with
 * ephdc_seed_u64: deterministic and GUESSABLE, never for real data. */
typedef struct {
    uint32_t key[8];
} ephdc_seed;
/* key <- 32 bytes of getrandom(2).  Errors: ENULL, ERESOURCE (no OS entropy). */
ephdc_status ephdc_seed_os(ephdc_seed *out);
/* TEST/BENCH ONLY: key = (lo32(v), hi32(v), 0, 0, 0, 0, 0, 0).  Errors: ENULL. */
ephdc_status ephdc_seed_u64(uint64_t v, ephdc_seed *out);
/* One ChaCha20 block (RFC 8439 sec. 2.3.1) of the library's generator, host side:
 * out[16] words for (key, counter, nonce[3]) -- exported so tests can pin it to the
 * RFC's known answers.  Errors: ENULL. */
ephdc_status ephdc_chacha20_block(const ephdc_seed *key, uint32_t counter, const uint32_t nonce[3],
                                  uint32_t out[16]);

const char *ephdc_status_string(ephdc_status s);
int ephdc_abi_version(void);

/* ---------------- host helpers (no device needed) ------------------------- */

/* Prime chain of BASELINE.json configs (reading #18): for each bound 2^bits[i],
 * the largest prime p < 2^bits[i] with p = 1 mod 2N that is not in exclude[]
 * and not already chosen.  out[count].  EPARAM if bits[i] > 62 or none exists. */
ephdc_status ephdc_find_ntt_primes(uint32_t log2N, const uint32_t *bits, uint32_t count,
                                   const uint64_t *exclude, uint32_t n_exclude, uint64_t *out);

/* Minimal primitive 2N-th root of unity mod prime p (reading #2). */
ephdc_status ephdc_min_psi(uint64_t p, uint32_t log2N, uint64_t *psi);

/* CDT thresholds of the discrete Gaussian sampler (reading #10): out[20]. */
ephdc_status ephdc_gaussian_cdt(double sigma, uint64_t *out20);

/* Query hypervector width (reading #12; the paper's Q bits): the largest
 * Q <= 8 with D_live * (2^(Q-1) - 1) * (2^(Cbits-1) - 1) <= (t-1)/2, so that no score
 * wraps mod t.  EPARAM if even Q = 2 wraps or Cbits is outside 2..8. */
ephdc_status ephdc_query_bits(uint32_t D_live, uint32_t Cbits, uint64_t t, uint32_t *Qbits);

/* Server model build (CS1; once, untimed): single-pass training and quantisation.
 * h_acc [D_live][n] int32: the raw projections of the n training samples
 * (ephdc_encode_raw); h_labels [n] in 0..k-1.
 *   class sums   v_c[d] = sum_{i: label i = c} acc[d][i]
 *   class HVs    C_c[d] = sign(v) floor((2|v| cmax + M_c) / (2 M_c)), M_c = max_d |v_c[d]|,
 *                cmax = 2^(Cbits-1) - 1 (round half away from zero, reading #14)
 *   query shift  *qshift = the smallest s >= 0 with max|acc| <= qmax 2^s, qmax =
 *                2^(Qbits-1) - 1 (max-abs calibration, reading #13)
 * h_class_hv [k][D_live] int8.  Host-only (no device needed).  Errors: ENULL, EPARAM
 * (k = 0, a label >= k, Cbits / Qbits outside 2..8). */
ephdc_status ephdc_train_model(uint32_t D_live, uint32_t n, uint32_t k, uint32_t Cbits, uint32_t Qbits,
                               const int32_t *h_acc, const int64_t *h_labels, int8_t *h_class_hv,
                               uint32_t *qshift);

/* Number of CUDA kernels this library has launched in this process (all
 * entry points).  Used by bench.py for the gpu_launches claim. */
uint64_t ephdc_launch_count(void);

/* ---------------- context ------------------------------------------------- */

/* Validates params, derives psi, Delta, B, builds the twiddle tables
 * (bit-reversed psi powers with Shoup companions) and, for device >= 0,
 * uploads them to that CUDA device.  device = -1 builds a HOST-ONLY context
 * usable by keygen, sk_export and decrypt_* (tests without a GPU).
 * Synchronous.  Errors: ENULL, EPARAM, ECUDA, ERESOURCE. */
ephdc_status ephdc_ctx_create(const ephdc_params *params, int device, ephdc_ctx **out);
void ephdc_ctx_free(ephdc_ctx *ctx);
ephdc_status ephdc_ctx_query(const ephdc_ctx *ctx, ephdc_ctx_info *info);

/* ---------------- server side (CS1) ---------------------------- */

/* Secret key: ternary s (reading #9) from the ChaCha20 stream of tag 2
 * (reading #7) under `seed` (NULL: a fresh OS key), and s_hat_j = NTT_j(s).
 * Host-only.  Errors: ENULL, ERESOURCE. */
ephdc_status ephdc_keygen(const ephdc_ctx *ctx, const ephdc_seed *seed, ephdc_sk **out);
void ephdc_sk_free(ephdc_sk *sk);
/* s_out[N] int8 in {-1,0,1}; s_hat_out[L][N] (may be NULL). */
ephdc_status ephdc_sk_export(const ephdc_sk *sk, int8_t *s_out, uint64_t *s_hat_out);

/* Encrypts the model ("encrypt the class hypervectors"): for
 * d < D_live, m_d = encode(tile_d), tile_d[i] = class_hv[i mod k][d] mod t for
 * i < k*B else 0; per prime: c1 = a (uniform in the NTT domain, #6, #8),
 * c0 = NTT_j([Delta*m_d + e_d]_{q_j}) - a (.) s_hat_j (secret-key BFV, #4, #5;
 * e_d CDT Gaussian, #10); a and e from the ChaCha20 streams of ciphertext index d
 * under `seed` (NULL: a fresh OS key, independent of the secret key's).
 * class_hv: HOST int8 [k][D_live] with |v| < t/2.  The model lives on the context's device: u64 [D_live][L][2][N].
 * Synchronous.  Errors: ENULL, ECONTEXT (host-only ctx), ECUDA, ERESOURCE. */
ephdc_status ephdc_encrypt_model(const ephdc_ctx *ctx, const ephdc_sk *sk, const int8_t *class_hv,
                                 const ephdc_seed *seed, ephdc_model **out);
void ephdc_model_free(ephdc_model *m);
/* Copies ciphertexts of dims [d0, d0+nd) to host_out [nd][L][2][N] (canonical).
 * Synchronous.  EPARAM if d0+nd > D_live. */
ephdc_status ephdc_model_export(const ephdc_model *m, uint32_t d0, uint32_t nd, uint64_t *host_out);

/* Accumulator scaling ("a scaling operation ... after every g HE
 * additions", g = 512): the client evaluation becomes
 *   acc <- (acc + sum_{d in group J} CT_d (x) PT_d) (x) s_J^-1   for J = 0, 1, ...
 * (groups of g consecutive dims, n_scales = ceil(D_live / g) scales, each s_J
 * invertible mod t; the plaintext constant s_J^-1 mod t acts on NTT-form residues as
 * its centered lift, reading #3).  Because ct (x) const distributes over the sum, this
 * call folds the schedule into the encrypted model once: the residues of dim d are
 * multiplied by prod_{J' >= J(d)} lift(s_J'^-1) mod q_j, after which ephdc_infer_batch
 * returns exactly the ciphertexts of the sequential scaled evaluation (no hot-path
 * cost).  The decrypted slot of (query, class) is then
 *   sum_J (sum_{d in J} h[d] C[d]) prod_{J' >= J} s_J'^-1  (mod t).
 * Mutates the model in place (do not run concurrently with infer on it).  Synchronous.
 * Errors: ENULL, ECONTEXT, EPARAM (g = 0, wrong n_scales, s = 0 mod t), ECUDA. */
ephdc_status ephdc_model_scale(const ephdc_ctx *ctx, ephdc_model *model, uint32_t g, const uint64_t *h_scales,
                               uint32_t n_scales);

/* ---------------- client side (the hot path; CS2) ---------------------------- */

/* Device scratch for up to max_nq queries: query/hypervector staging, the
 * encoded plaintexts (FP64 path: of every batch of the call, up to 32 GB) and the
 * scores buffers.  plan: launch-plan overrides for tests/profiling (ephdc_plan;
 * NULL = the tuned plan).  Synchronous.  Errors: ENULL, ECONTEXT (host-only
 * context), EPARAM (max_nq = 0), ERESOURCE. */
ephdc_status ephdc_workspace_create(const ephdc_ctx *ctx, uint32_t max_nq, const ephdc_plan *plan,
                                    ephdc_workspace **out);
void ephdc_workspace_free(ephdc_workspace *ws);
/* Per-kernel-class device time (ms, CUDA events on the launching stream) of
 * the calls since the last reset, when timing is enabled.  names/ms/launches
 * arrays of length *n (in: capacity, out: count).  Synchronises the workspace's
 * last stream.  Classes: "encode", "pack_intt", "ntt_mac", "finalize". */
ephdc_status ephdc_workspace_set_timing(ephdc_workspace *ws, int enable);
ephdc_status ephdc_workspace_timing(ephdc_workspace *ws, const char **names, double *ms,
                                    uint64_t *launches, uint32_t *n);

/* HDC encoding + quantisation (BASELINE.json subsystem (a)):
 * acc[d][q] = sum_f P[d][f] * X[q][f] (exact int32), h = clamp(floor((acc +
 * 2^(s-1)) / 2^s), +-(2^(Q-1)-1)) for d < D_live, q < nq.
 * d_X: [nq][F] int8 or uint8 (feat_unsigned); d_P: [D_stored][F] int8 (+-1, or 0);
 * d_H: [D_live][nq] int8 (dim-major: row d feeds plaintext d).  Async. */
ephdc_status ephdc_encode_queries(const ephdc_ctx *ctx, const void *d_X, const int8_t *d_P, uint32_t nq,
                                  int8_t *d_H, void *stream);

/* Unquantised projection acc[d][i] = sum_f P[d][f] X[i][f] (exact int32) for
 * d < D_live, i < n: the same kernel with a raw epilogue, used server-side to
 * encode training samples before bundling.  d_acc: [D_live][n]. Async. */
ephdc_status ephdc_encode_raw(const ephdc_ctx *ctx, const void *d_X, const int8_t *d_P, uint32_t n,
                              int32_t *d_acc, void *stream);

/* Client evaluation: for each batch b < nb = ceil(nq/B),
 * d_out[b] = sum_{d < D_live} CT_d (x) NTT(lift(encode(v_{b,d}))) where slot i of
 * v_{b,d} is h[d][b*B + i/k] mod t for i < k*n_b (n_b = queries in batch b),
 * else 0 (#19); lift is centered (#3).  d_H: [D_live][nq] int8; d_out:
 * [cap_ct][2][L][N] u64, canonical NTT form (slot order #1).  EOVERFLOW if
 * cap_ct < nb, EPARAM if nq > the workspace's max_nq.  Async. */
ephdc_status ephdc_infer_batch(const ephdc_ctx *ctx, const ephdc_model *model, ephdc_workspace *ws,
                               const int8_t *d_H, uint32_t nq, uint64_t *d_out, uint32_t cap_ct,
                               void *stream);

/* findDmax's evaluation (Algorithm 1 l.20: evalHEcomputation(N, T, D)):
 * ephdc_infer_batch where batch b sums only its first h_dims[b] dims (host array
 * [ceil(nq/B)], each <= D_live) -- the same kernels, so 1000 trials of different
 * lengths are one call.  Errors as ephdc_infer_batch, EPARAM if a count exceeds
 * D_live or nq exceeds the workspace.  Async (h_dims is consumed before return). */
ephdc_status ephdc_infer_batch_prefix(const ephdc_ctx *ctx, const ephdc_model *model, ephdc_workspace *ws,
                                      const int8_t *d_H, uint32_t nq, const uint32_t *h_dims, uint64_t *d_out,
                                      uint32_t cap_ct, void *stream);

/* Intermediate export for parity tests: the plaintext NTTs p_hat_{b,d,j} of
 * batch b for dims [d0, d0+nd): d_pt [nd][L][N] canonical.  Async. */
ephdc_status ephdc_encode_plaintexts(const ephdc_ctx *ctx, ephdc_workspace *ws, const int8_t *d_H,
                                     uint32_t nq, uint32_t b, uint32_t d0, uint32_t nd, uint64_t *d_pt,
                                     void *stream);

/* End-to-end client call with HOST buffers: copies h_X [nq][F] host->device,
 * runs encode_queries + infer_batch, copies the nb scores ciphertexts to
 * h_out [cap_ct][2][L][N].  d_P stays device-resident.  Synchronous on
 * `stream`.  h_X / h_out should be pinned for full copy bandwidth. */
ephdc_status ephdc_classify_host(const ephdc_ctx *ctx, const ephdc_model *model, ephdc_workspace *ws,
                                 const void *h_X, const int8_t *d_P, uint32_t nq, uint64_t *h_out,
                                 uint32_t cap_ct, void *stream);

/* ---------------- HE-HDC-SR: the server-side SIMD baseline -- */
/* P:257-265 / SPEC S:445-453: the CLIENT encrypts its query hypervectors in the same
 * interleave layout (slot i of ciphertext d = h[d][b*B + i/k], D_live ciphertexts per
 * batch of B queries) and uploads them; the SERVER multiplies them by the plaintext
 * class tiles (slot i = C[i mod k][d]) and sums over d -- the same arithmetic as
 * ephdc_infer_batch with the ct/pt roles of model and queries swapped (P:786 compares
 * the two: the client runtime is dominated by this encryption, the message is D_live
 * ciphertexts per batch instead of one). */

/* Client: batch b of d_H [D_live][nq] -> d_qct [D_live][L][2][N]: secret-key BFV with
 * the client's key (readings #4-#10), random streams of ciphertext index 2^32 + b*D_live + d (#25: disjoint from the model's
 * indices d < D_live, so query and model ciphertexts never share a or e) under `seed`
 * (NULL: a fresh OS key per call).  Uses the workspace's plaintext buffer.  Async. */
ephdc_status ephdc_sr_encrypt_queries(const ephdc_ctx *ctx, ephdc_sk *sk, ephdc_workspace *ws, const int8_t *d_H,
                                      uint32_t nq, uint32_t b, const ephdc_seed *seed, uint64_t *d_qct,
                                      void *stream);
/* Server, once: the plaintext class tiles in NTT form, d_pt [D_live][L][N] canonical:
 * NTT_j(centered lift(encode(tile_d))).  h_class_hv: HOST int8 [k][D_live].  Synchronous. */
ephdc_status ephdc_sr_model_plaintexts(const ephdc_ctx *ctx, const int8_t *h_class_hv, uint64_t *d_pt);
/* Server: d_out [2][L][N] = sum_d d_qct[d] (x) d_pt[d]: D_live MulCP, D_live-1 AddCC,
 * 0 rotations.  Decrypts with the client's key (ephdc_decrypt_scores).  Async. */
ephdc_status ephdc_sr_evaluate(const ephdc_ctx *ctx, const uint64_t *d_pt, const uint64_t *d_qct, uint64_t *d_out,
                               void *stream);

/* ---------------- scores message (client -> server) -------- */

/* The message the client sends per call: the nb scores ciphertexts ("only the
 * encrypted similarity scores") with the residues of prime j bit-packed at b_j =
 * bit_length(q_j) bits (little-endian bit order within a block), blocks in [nb][2][L]
 * order, each block N*b_j/8 bytes; no header (the parameters are the context's).
 * Size: nb * 2 * N * sum_j b_j / 8 bytes (c4: 1.77 MB per ciphertext vs 2.36 MB of
 * u64 words).  SURVEY NEXT #4. */
size_t ephdc_scores_message_bytes(const ephdc_ctx *ctx, uint32_t nb);
/* Device -> device packing of d_ct [nb][2][L][N] (canonical) into d_msg.  Async. */
ephdc_status ephdc_pack_scores(const ephdc_ctx *ctx, const uint64_t *d_ct, uint32_t nb, uint8_t *d_msg, void *stream);
/* Host unpacking (server side): h_msg -> h_ct [nb][2][L][N].  EDOMAIN if a residue
 * is >= its prime.  Synchronous. */
ephdc_status ephdc_unpack_scores(const ephdc_ctx *ctx, const uint8_t *h_msg, uint32_t nb, uint64_t *h_ct);
/* End-to-end client call producing the message: h_X -> device, encode_queries +
 * infer_batch + pack_scores, message -> h_msg (ephdc_scores_message_bytes(ctx, nb)
 * bytes; cap_bytes = capacity of h_msg, EOVERFLOW if smaller, nothing written).
 * Synchronous on `stream`. */
ephdc_status ephdc_classify_host_packed(const ephdc_ctx *ctx, const ephdc_model *model, ephdc_workspace *ws,
                                        const void *h_X, const int8_t *d_P, uint32_t nq, uint8_t *h_msg,
                                        size_t cap_bytes, void *stream);

/* ---------------- server decide (test-only host; CS3) ----------------------- */

/* Decrypts nb = ceil(nq/B) scores ciphertexts h_ct [nb][2][L][N]:
 * x = c0 + c1*s (CRT over the q_j, multi-precision), m = floor((t*x +
 * floor(Q/2)) / Q) mod t, slots = NTT_t(m), slot i -> (query b*B + i/k,
 * class i mod k), centered to (-t/2, t/2] (#20).  h_scores [nq][k] int64,
 * h_labels [nq] = lowest class attaining the max (may be NULL).
 * Host-only; works on a host-only context. */
ephdc_status ephdc_decrypt_scores(const ephdc_ctx *ctx, const ephdc_sk *sk, const uint64_t *h_ct,
                                  uint32_t nq, int64_t *h_scores, uint32_t *h_labels);
/* Decrypts one ciphertext h_ct [2][L][N] to its N slot values in [0, t). */
ephdc_status ephdc_decrypt_slots(const ephdc_ctx *ctx, const ephdc_sk *sk, const uint64_t *h_ct,
                                 uint64_t *h_slots);

/* Noise probe (findDmax, Algorithm 1 l.17-24; NEXT #2), on the GPU.
 * d_ct [nct][2][L][N]: device scores ciphertexts (NTT form, residues < q_j, e.g.
 * from ephdc_infer_batch).  For each: x = INTT(c0 + c1 s) mod Q, m = round(t x / Q)
 * mod t, e = x - floor(Q/t) m centered mod Q; h_bits[b] = EXACT bit length of
 * max_i |e_i| (0 for e = 0).  Decryption of the ciphertext is correct iff that noise
 * is below Delta/2; then e is the ciphertext noise (x - Delta m_expected).  h_flags[b]
 * (may be NULL) = 1 if some t x_i / Q lay within 2^-16 of a rounding boundary (the
 * decryption itself is ambiguous there), else 0.  h_log2[b] (may be NULL) = log2 of
 * that maximum from its top 128 bits (0 for e = 0).  Needs a device context; the
 * secret key's NTT form is uploaded per call.  Synchronous on `stream` (host
 * outputs).  Errors: ENULL, ECONTEXT (sk of another context, host-only context),
 * ERESOURCE, ECUDA. */
ephdc_status ephdc_noise_probe(const ephdc_ctx *ctx, const ephdc_sk *sk, const uint64_t *d_ct, uint32_t nct,
                               uint32_t *h_bits, uint32_t *h_flags, double *h_log2, void *stream);

/* ---------------- standalone kernels (c5 microbench; CS5) ------------------- */

/* Tables for L primes (each = 1 mod 2N, < 2^61) at ring degree N = 2^log2N,
 * 10 <= log2N <= 16, on `device`.  flags: 0 = the tuned kernels (FP64 pipe where
 * the bounds of DESIGN.md 5.1 hold, else the integer pipe); EPHDC_NTT_FORCE_INT =
 * the integer-pipe kernels everywhere; EPHDC_NTT_ALT_TEAMS = the alternative
 * layouts kept for A/B: at N = 2^13 the other warp layout of the c5 kernels (forward:
 * one 16-warp team instead of two 8-warp groups; inverse: two groups instead of one
 * team), the one-team cluster forward at 2^14-2^16, and the per-polynomial integer
 * kernels instead of the persistent ones; EPHDC_NTT_U32_GENERIC = the general u32
 * kernels (kernels.cu) instead of the persistent TMA-fed u32 kernels of ntt32_c5.cu at
 * N = 2^12 .. 2^14 (TEST/PROFILING only, all bit-identical).
 * Synchronous.  Errors: ENULL, EPARAM (sizes, a q_j that is not an NTT prime, unknown
 * flags), ECONTEXT (device < 0), ECUDA, ERESOURCE. */
#define EPHDC_NTT_FORCE_INT 1u
#define EPHDC_NTT_ALT_TEAMS 2u
#define EPHDC_NTT_U32_GENERIC 4u
ephdc_status ephdc_ntt_plan_create(const uint64_t *q, uint32_t L, uint32_t log2N, int device,
                                   uint32_t flags, ephdc_ntt_plan **out);
void ephdc_ntt_plan_free(ephdc_ntt_plan *p);
/* In-place negacyclic NTT of d_polys [batch][L][N] (residues < q_j), natural
 * coefficient order <-> bit-reversed evaluation order (#1).  Async. */
ephdc_status ephdc_ntt_fwd(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, void *stream);
ephdc_status ephdc_ntt_inv(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, void *stream);
/* Pointwise MAC: d_out[j][c][i] = sum_{d<D} d_ct[d][j][c][i] *
 * d_pt[d][j][i] mod q_j; d_ct [D][L][2][N], d_pt [D][L][N], d_out [L][2][N].
 * Exact modular products on the FP64 pipe when every q_j < 2^50, u64 Montgomery
 * otherwise.  Async (the call zeroes d_out itself). */
ephdc_status ephdc_mac(const ephdc_ntt_plan *p, const uint64_t *d_ct, const uint64_t *d_pt, uint32_t D,
                       uint64_t *d_out, void *stream);

/* The same three operations on 32-bit words (30-bit primes in u32): every
 * array is uint32 with the layouts above; the plan's primes must all be < 2^30
 * (EPARAM otherwise).  Integer-pipe u32 Shoup butterflies; MAC products accumulate
 * exactly in 64 bits (ephdc_mac32: d_ct and d_pt 16-byte aligned, else ECUDA).  Async. */
ephdc_status ephdc_ntt_fwd32(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, void *stream);
ephdc_status ephdc_ntt_inv32(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, void *stream);
ephdc_status ephdc_mac32(const ephdc_ntt_plan *p, const uint32_t *d_ct, const uint32_t *d_pt, uint32_t D,
                         uint32_t *d_out, void *stream);

/* Which kernels a plan runs (tests and the microbench report). */
#define EPHDC_NTT_KERNEL_INT 0u     /* integer pipe, u64 Shoup (any prime < 2^61)          */
#define EPHDC_NTT_KERNEL_F64 1u     /* FP64 pipe, per-polynomial CTAs (round-1 kernels)    */
#define EPHDC_NTT_KERNEL_C5_F64 2u  /* FP64 pipe, persistent TMA-fed kernels (ntt_c5.cu)   */
#define EPHDC_NTT_KERNEL_C5_U32 3u  /* integer pipe, persistent TMA-fed u32 kernels
                                       (ntt32_c5.cu; u32 words N = 2^12 .. 2^16 -- 2^15 /
                                       2^16 as global stages + 2^14 slices; u64 words
                                       with primes < 2^30 N = 2^12 .. 2^14)              */
typedef struct {
    uint32_t fwd_kernel, inv_kernel;  /* EPHDC_NTT_KERNEL_* of ephdc_ntt_fwd / _inv       */
    uint32_t u32_words;               /* 1 if the *32 entry points are available          */
    uint32_t u32_kernel;              /* EPHDC_NTT_KERNEL_* of ephdc_ntt_fwd32 / _inv32   */
} ephdc_ntt_plan_info;
ephdc_status ephdc_ntt_plan_query(const ephdc_ntt_plan *p, ephdc_ntt_plan_info *info);

#ifdef __cplusplus
}
#endif
#endif /* EPHDC_H */
