/*
 * oracle_core.c -- plain scalar C core of the CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs load this library.  It shares no code, header or table with the product
 * library (paper_2511_00737_b200/csrc); it is compiled by gcc, not nvcc.
 *
 * Everything follows the plain definitions:
 *   - modular product: (unsigned __int128)a*b % q                      (no Barrett/Shoup)
 *   - negacyclic NTT : the textbook Cooley-Tukey / Gentleman-Sande loops over
 *                      Z_q[X]/(X^N+1) (the BFV ring of PAPER.md l.135), output
 *                      index i = evaluation at psi^(2*brev(i)+1) (DESIGN.md
 *                      reading #1); pinned in tests against O(N^2) direct
 *                      evaluation and schoolbook negacyclic products.
 *   - slot encode    : inverse NTT mod t ("packing"; reading #1)
 *   - encryption     : symmetric BFV, c1 = a, c0 = NTT(Delta*m + e) - a*s
 *                      ("encrypted ... using a given secret key"; readings #4-#6)
 *   - client eval    : acc_j = sum_d c_{d,j} (.) NTT_j(lift_j(encode(v_{b,d})))
 *                      (D MulCP, D-1 AddCC, 0 Rot)
 *   - randomness     : ChaCha20 (RFC 8439) streams of DESIGN.md readings #7-#10.
 * OpenMP only splits independent dims d across threads; each thread runs the
 * same plain loop and the per-thread sums are added mod q at the end.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* plain modular arithmetic                                            */
/* ------------------------------------------------------------------ */
u64 or_mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
u64 or_addmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + b) % q); }
u64 or_submod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + q - b) % q); }

u64 or_powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = or_mulmod(r, a, q);
        a = or_mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

u32 or_brev(u32 i, int bits) {
    u32 r = 0;
    for (int b = 0; b < bits; ++b) { r = (r << 1) | (i & 1); i >>= 1; }
    return r;
}

/* table[i] = x^brev(i) mod q, i < N (x = psi for forward, psi^-1 for inverse) */
void or_pow_brev_table(u64 x, u64 q, int logN, u64 *table) {
    u32 N = 1u << logN;
    for (u32 i = 0; i < N; ++i) table[i] = or_powmod(x, or_brev(i, logN), q);
}

/* ------------------------------------------------------------------ */
/* textbook negacyclic NTT                                             */
/* ------------------------------------------------------------------ */
/* forward: natural-order coefficients -> a[i] = A(psi^(2 brev(i) + 1)) */
void or_ntt_fwd(u64 *a, int logN, u64 q, const u64 *psi_rev) {
    u32 N = 1u << logN;
    u32 t = N;
    for (u32 m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (u32 i = 0; i < m; ++i) {
            u64 w = psi_rev[m + i];
            u32 j1 = 2 * i * t;
            for (u32 j = j1; j < j1 + t; ++j) {
                u64 U = a[j];
                u64 V = or_mulmod(a[j + t], w, q);
                a[j] = or_addmod(U, V, q);
                a[j + t] = or_submod(U, V, q);
            }
        }
    }
}

/* inverse of or_ntt_fwd (Gentleman-Sande with psi^-1, then times N^-1) */
void or_ntt_inv(u64 *a, int logN, u64 q, const u64 *psiinv_rev) {
    u32 N = 1u << logN;
    u32 t = 1;
    for (u32 m = N; m > 1; m >>= 1) {
        u32 h = m >> 1;
        u32 j1 = 0;
        for (u32 i = 0; i < h; ++i) {
            u64 w = psiinv_rev[h + i];
            for (u32 j = j1; j < j1 + t; ++j) {
                u64 U = a[j];
                u64 V = a[j + t];
                a[j] = or_addmod(U, V, q);
                a[j + t] = or_mulmod(or_submod(U, V, q), w, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    u64 ninv = or_powmod(N, q - 2, q);
    for (u32 j = 0; j < N; ++j) a[j] = or_mulmod(a[j], ninv, q);
}

/* batched wrappers: polys[n][N] all mod q */
void or_ntt_fwd_many(u64 *polys, u64 n, int logN, u64 q, u64 psi) {
    u32 N = 1u << logN;
    u64 *tab = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(psi, q, logN, tab);
    #pragma omp parallel for schedule(static)
    for (long long p = 0; p < (long long)n; ++p) or_ntt_fwd(polys + (u64)p * N, logN, q, tab);
    free(tab);
}

void or_ntt_inv_many(u64 *polys, u64 n, int logN, u64 q, u64 psi) {
    u32 N = 1u << logN;
    u64 *tab = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(or_powmod(psi, q - 2, q), q, logN, tab);
    #pragma omp parallel for schedule(static)
    for (long long p = 0; p < (long long)n; ++p) or_ntt_inv(polys + (u64)p * N, logN, q, tab);
    free(tab);
}

/* Horner evaluation a(x) mod q: the definition of an NTT output point */
u64 or_eval(const u64 *a, u32 N, u64 q, u64 x) {
    u64 r = 0;
    for (u32 n = N; n-- > 0;) r = or_addmod(or_mulmod(r, x, q), a[n], q);
    return r;
}

/* schoolbook product in Z_q[X]/(X^N + 1) */
void or_negacyclic_mul(const u64 *a, const u64 *b, u64 *c, u32 N, u64 q) {
    for (u32 i = 0; i < N; ++i) c[i] = 0;
    for (u32 i = 0; i < N; ++i)
        for (u32 j = 0; j < N; ++j) {
            u64 p = or_mulmod(a[i], b[j], q);
            u32 k = i + j;
            if (k < N) c[k] = or_addmod(c[k], p, q);
            else c[k - N] = or_submod(c[k - N], p, q);
        }
}

/* ------------------------------------------------------------------ */
/* randomness: ChaCha20 streams (reading #7)                 */
/* ------------------------------------------------------------------ */
/* RFC 8439 sec. 2.1: the quarter round on four words of the state */
#define ROTL32(v, n) (((v) << (n)) | ((v) >> (32 - (n))))
static void quarter_round(u32 *s, int a, int b, int c, int d) {
    s[a] += s[b]; s[d] ^= s[a]; s[d] = ROTL32(s[d], 16);
    s[c] += s[d]; s[b] ^= s[c]; s[b] = ROTL32(s[b], 12);
    s[a] += s[b]; s[d] ^= s[a]; s[d] = ROTL32(s[d], 8);
    s[c] += s[d]; s[b] ^= s[c]; s[b] = ROTL32(s[b], 7);
}
/* RFC 8439 sec. 2.3: state = constants | key[8] | counter | nonce[3];
   10 x (4 column rounds + 4 diagonal rounds); out = state + working state */
void or_chacha20_block(const u32 *key, u32 counter, const u32 *nonce, u32 *out) {
    u32 st[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                  key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                  counter, nonce[0], nonce[1], nonce[2]};
    u32 w[16];
    memcpy(w, st, sizeof w);
    for (int r = 0; r < 10; ++r) {
        quarter_round(w, 0, 4, 8, 12);
        quarter_round(w, 1, 5, 9, 13);
        quarter_round(w, 2, 6, 10, 14);
        quarter_round(w, 3, 7, 11, 15);
        quarter_round(w, 0, 5, 10, 15);
        quarter_round(w, 1, 6, 11, 12);
        quarter_round(w, 2, 7, 8, 13);
        quarter_round(w, 3, 4, 9, 14);
    }
    for (int i = 0; i < 16; ++i) out[i] = w[i] + st[i];
}

enum { TAG_SK = 2, TAG_A = 3, TAG_E = 4, TAG_A_RETRY = 5 };

/* the generator's 64-bit word w (< 8) of block `ctr` of stream (tag, a) under the test
   key of a 64-bit seed: key = (lo32(seed), hi32(seed), 0, ..., 0), nonce = (tag,
   lo32(a), hi32(a)); word w = block bytes 8w..8w+7 little-endian */
u64 or_word64(u64 seed, u32 tag, u64 a, u32 ctr, u32 w) {
    u32 key[8] = {(u32)seed, (u32)(seed >> 32), 0, 0, 0, 0, 0, 0};
    u32 nonce[3] = {tag, (u32)a, (u32)(a >> 32)};
    u32 b[16];
    or_chacha20_block(key, ctr, nonce, b);
    return (u64)b[2 * w] | ((u64)b[2 * w + 1] << 32);
}

/* reading #9: s_i = (word i%8 of block i/8 of tag 2) mod 3 - 1 */
void or_sample_ternary(u64 seed, u32 N, int8_t *s) {
    for (u32 i = 0; i < N; ++i) s[i] = (int8_t)((int)(or_word64(seed, TAG_SK, 0, i / 8, i % 8) % 3) - 1);
}

static u64 bitmask_for(u64 q) {
    u64 m = 1;
    while (m < q) m = (m << 1) | 1;   /* 2^ceil(log2 q) - 1 (q is never a power of two) */
    return m;
}
/* reading #8: uniform mod q by rejection.  Draw 0 of coefficient i: word i%8 of block i/8
   of stream (tag 3, d*L + j); draw n >= 1: word (n-1)%8 of block i + ((n-1)/8)*2^16 of
   stream (tag 5, d*L + j)  (N <= 2^16) */
u64 or_uniform_mod(u64 seed, u64 d, u32 j, u32 L, u32 i, u64 q) {
    u64 a = d * L + j;
    u64 mask = bitmask_for(q);
    u64 u = or_word64(seed, TAG_A, a, i / 8, i % 8) & mask;
    for (u32 n = 1; u >= q; ++n) u = or_word64(seed, TAG_A_RETRY, a, i + ((n - 1) / 8) * 65536u, (n - 1) % 8) & mask;
    return u;
}
/* reading #10: CDT over magnitudes; block i/4 of stream (tag 4, d): magnitude from
   word 2(i%4) >> 1, sign = top bit of word 2(i%4)+1 */
long long or_gauss(u64 seed, u64 d, u32 i, const u64 *cdt, int ncdt) {
    u64 u = or_word64(seed, TAG_E, d, i / 4, 2 * (i % 4)) >> 1;
    int k = 0;
    while (k < ncdt - 1 && u >= cdt[k]) ++k;
    if (k == 0) return 0;
    return (or_word64(seed, TAG_E, d, i / 4, 2 * (i % 4) + 1) >> 63) ? -(long long)k : (long long)k;
}

/* whole polynomials: the same values as or_uniform_mod / or_gauss coefficient by
   coefficient, each block computed once for the 8 (uniform) or 4 (Gaussian)
   coefficients that read it (tests check the two forms agree) */
void or_sample_uniform_poly(u64 seed, u64 d, u32 j, u32 L, u64 q, u32 N, u64 *out) {
    u64 a = d * L + j;
    u64 mask = bitmask_for(q);
    u32 key[8] = {(u32)seed, (u32)(seed >> 32), 0, 0, 0, 0, 0, 0};
    u32 nonce[3] = {TAG_A, (u32)a, (u32)(a >> 32)};
    u32 b[16];
    for (u32 i = 0; i < N; ++i) {
        if (i % 8 == 0) or_chacha20_block(key, i / 8, nonce, b);
        u64 u = ((u64)b[2 * (i % 8)] | ((u64)b[2 * (i % 8) + 1] << 32)) & mask;
        for (u32 n = 1; u >= q; ++n) u = or_word64(seed, TAG_A_RETRY, a, i + ((n - 1) / 8) * 65536u, (n - 1) % 8) & mask;
        out[i] = u;
    }
}
void or_sample_gauss_poly(u64 seed, u64 d, u32 N, const u64 *cdt, int ncdt, long long *e) {
    u32 key[8] = {(u32)seed, (u32)(seed >> 32), 0, 0, 0, 0, 0, 0};
    u32 nonce[3] = {TAG_E, (u32)d, (u32)(d >> 32)};
    u32 b[16];
    for (u32 i = 0; i < N; ++i) {
        if (i % 4 == 0) or_chacha20_block(key, i / 4, nonce, b);
        u32 w = 2 * (i % 4);
        u64 u = ((u64)b[2 * w] | ((u64)b[2 * w + 1] << 32)) >> 1;
        int k = 0;
        while (k < ncdt - 1 && u >= cdt[k]) ++k;
        e[i] = k == 0 ? 0 : ((b[2 * w + 3] >> 31) ? -(long long)k : (long long)k);
    }
}

/* ------------------------------------------------------------------ */
/* BFV pieces of the method                                            */
/* ------------------------------------------------------------------ */
typedef struct {
    int logN;
    u32 L;
    const u64 *q;        /* [L] */
    const u64 *psi;      /* [L] */
    u64 t;
    u64 psi_t;
    u32 k;
    u32 D_live;
    const u64 *delta;    /* [L]  floor(Q/t) mod q_j */
    const u64 *s_hat;    /* [L][N] NTT_j(s) */
    u64 enc_seed;
    const u64 *cdt;
    int ncdt;
} or_bfv;

static u64 lift_centered(u64 m, u64 t, u64 q) {
    /* reading #3: m in [0,t) -> m if m <= (t-1)/2 else m - t + q (mod q) */
    if (m <= (t - 1) / 2) return m % q;
    return or_submod(m % q, t % q, q);
}

/* model tile of dim d: slot i <- C[i mod k][d] for i < k*floor(N/k), else 0
   (P:650-653 / P:1471-1474: k-fold interleave, B = floor(N/k)); returns m_d */
static void model_plaintext(const or_bfv *P, const int8_t *class_hv, u32 d, const u64 *tinv_tab, u64 *m) {
    u32 N = 1u << P->logN;
    u32 B = N / P->k;
    for (u32 i = 0; i < N; ++i) {
        long long v = (i < P->k * B) ? class_hv[(u64)(i % P->k) * P->D_live + d] : 0;
        m[i] = (u64)((v % (long long)P->t + (long long)P->t) % (long long)P->t);
    }
    or_ntt_inv(m, P->logN, P->t, tinv_tab);
}

/* secret-key encryption of the encoded message m ([0,t)) with the random streams of
   ciphertext index g: out[L][2][N] canonical NTT form */
static void encrypt_msg(const or_bfv *P, u64 g, const u64 *m, u64 *const *psi_tabs, long long *e, u64 *x,
                        u64 *out);

/* ciphertext of dim d, all primes: out[L][2][N] canonical NTT form */
static void encrypt_dim(const or_bfv *P, const int8_t *class_hv, u32 d, const u64 *tinv_tab,
                        u64 *const *psi_tabs, u64 *m, long long *e, u64 *x, u64 *out) {
    model_plaintext(P, class_hv, d, tinv_tab, m);
    encrypt_msg(P, d, m, psi_tabs, e, x, out);
}

static void encrypt_msg(const or_bfv *P, u64 g, const u64 *m, u64 *const *psi_tabs, long long *e, u64 *x,
                        u64 *out) {
    u32 N = 1u << P->logN;
    u64 d = g;
    or_sample_gauss_poly(P->enc_seed, d, N, P->cdt, P->ncdt, e);
    for (u32 j = 0; j < P->L; ++j) {
        u64 q = P->q[j];
        for (u32 i = 0; i < N; ++i) {
            u64 ei = e[i] >= 0 ? (u64)e[i] % q : or_submod(0, (u64)(-e[i]) % q, q);
            x[i] = or_addmod(or_mulmod(P->delta[j], m[i] % q, q), ei, q);   /* Delta*m + e, m in [0,t) */
        }
        or_ntt_fwd(x, P->logN, q, psi_tabs[j]);
        u64 *c0 = out + ((u64)j * 2 + 0) * N;
        u64 *c1 = out + ((u64)j * 2 + 1) * N;
        or_sample_uniform_poly(P->enc_seed, d, j, P->L, q, N, c1);   /* c1 = a */
        for (u32 i = 0; i < N; ++i) c0[i] = or_submod(x[i], or_mulmod(c1[i], P->s_hat[(u64)j * N + i], q), q);
    }
}

static u64 **make_psi_tabs(const or_bfv *P, int inverse) {
    u32 N = 1u << P->logN;
    u64 **tabs = (u64 **)malloc(sizeof(u64 *) * P->L);
    for (u32 j = 0; j < P->L; ++j) {
        tabs[j] = (u64 *)malloc(sizeof(u64) * N);
        u64 x = inverse ? or_powmod(P->psi[j], P->q[j] - 2, P->q[j]) : P->psi[j];
        or_pow_brev_table(x, P->q[j], P->logN, tabs[j]);
    }
    return tabs;
}
static void free_tabs(u64 **tabs, u32 L) { for (u32 j = 0; j < L; ++j) free(tabs[j]); free(tabs); }

/* model ciphertexts for dims [d0, d0+nd): out[nd][L][2][N] */
void or_encrypt_dims(const or_bfv *P, const int8_t *class_hv, u32 d0, u32 nd, u64 *out) {
    u32 N = 1u << P->logN;
    u64 *tinv = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(or_powmod(P->psi_t, P->t - 2, P->t), P->t, P->logN, tinv);
    u64 **fw = make_psi_tabs(P, 0);
    #pragma omp parallel
    {
        u64 *m = (u64 *)malloc(sizeof(u64) * N);
        u64 *x = (u64 *)malloc(sizeof(u64) * N);
        long long *e = (long long *)malloc(sizeof(long long) * N);
        #pragma omp for schedule(dynamic)
        for (long long dd = 0; dd < (long long)nd; ++dd)
            encrypt_dim(P, class_hv, d0 + (u32)dd, tinv, fw, m, e, x,
                        out + (u64)dd * P->L * 2 * N);
        free(m); free(x); free(e);
    }
    free(tinv);
    free_tabs(fw, P->L);
}

/* query slot vector of (batch b, dim d): slot i <- h[d][b*B + i/k] for i < k*n_b, else 0 */
static void query_plaintext(const or_bfv *P, const int8_t *H, u32 nq, u32 b, u32 d, const u64 *tinv, u64 *m) {
    u32 N = 1u << P->logN;
    u32 B = N / P->k;
    u32 nb = nq - b * B < B ? nq - b * B : B;
    for (u32 i = 0; i < N; ++i) {
        long long v = (i < P->k * nb) ? H[(u64)d * nq + (u64)b * B + i / P->k] : 0;
        m[i] = (u64)((v % (long long)P->t + (long long)P->t) % (long long)P->t);
    }
    or_ntt_inv(m, P->logN, P->t, tinv);      /* encode = INTT_t */
}

/* plaintext NTTs p_hat[b,d,j] for dims [d0,d0+nd): out[nd][L][N] */
void or_plaintext_ntts(const or_bfv *P, const int8_t *H, u32 nq, u32 b, u32 d0, u32 nd, u64 *out) {
    u32 N = 1u << P->logN;
    u64 *tinv = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(or_powmod(P->psi_t, P->t - 2, P->t), P->t, P->logN, tinv);
    u64 **fw = make_psi_tabs(P, 0);
    #pragma omp parallel
    {
        u64 *m = (u64 *)malloc(sizeof(u64) * N);
        #pragma omp for schedule(dynamic)
        for (long long dd = 0; dd < (long long)nd; ++dd) {
            query_plaintext(P, H, nq, b, d0 + (u32)dd, tinv, m);
            for (u32 j = 0; j < P->L; ++j) {
                u64 *p = out + ((u64)dd * P->L + j) * N;
                for (u32 i = 0; i < N; ++i) p[i] = lift_centered(m[i], P->t, P->q[j]);
                or_ntt_fwd(p, P->logN, P->q[j], fw[j]);
            }
        }
        free(m);
    }
    free(tinv);
    free_tabs(fw, P->L);
}

/* Client evaluation of batch b over dims [0, D_live):
   one MulCP per dim (ct_d (x) pt_{b,d}), D-1 AddCC, no rotation:
   acc[c][j][i] = sum_d ct_{d,j,c}[i] * p_hat_{b,d,j}[i]  (mod q_j), output [2][L][N].
   model == NULL: each dim's ciphertext is re-encrypted on the fly from class_hv
   (c4's model does not fit in host RAM); otherwise model is [D_live][L][2][N].
   counters (may be NULL): [0] MulCP, [1] AddCC, [2] rotations. */
void or_infer_batch_range(const or_bfv *P, const int8_t *H, u32 nq, u32 b, u32 d0, u32 d1,
                          const u64 *model, const int8_t *class_hv, u64 *acc, u64 *counters);

void or_infer_batch(const or_bfv *P, const int8_t *H, u32 nq, u32 b,
                    const u64 *model, const int8_t *class_hv, u64 *acc, u64 *counters) {
    or_infer_batch_range(P, H, nq, b, 0, P->D_live, model, class_hv, acc, counters);
}

/* The same sum over the dims [d0, d1) only (model, when given, is still indexed by the
   absolute dim); used by the scaled evaluation of oracle/bfv.py (groups of g dims). */
void or_infer_batch_range(const or_bfv *P, const int8_t *H, u32 nq, u32 b, u32 d0, u32 d1,
                          const u64 *model, const int8_t *class_hv, u64 *acc, u64 *counters) {
    u32 N = 1u << P->logN;
    u32 L = P->L;
    u64 *tinv = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(or_powmod(P->psi_t, P->t - 2, P->t), P->t, P->logN, tinv);
    u64 **fw = make_psi_tabs(P, 0);
    u64 n_mul = 0, n_add = 0;
    int first_global = 1;
    for (u64 x = 0; x < (u64)2 * L * N; ++x) acc[x] = 0;
    #pragma omp parallel reduction(+ : n_mul, n_add)
    {
        u64 *m = (u64 *)malloc(sizeof(u64) * N);
        u64 *p = (u64 *)malloc(sizeof(u64) * N);
        u64 *ct = (u64 *)malloc(sizeof(u64) * L * 2 * N);
        u64 *x = (u64 *)malloc(sizeof(u64) * N);
        long long *e = (long long *)malloc(sizeof(long long) * N);
        u64 *part = (u64 *)calloc((size_t)2 * L * N, sizeof(u64));
        int have = 0;
        #pragma omp for schedule(dynamic, 4)
        for (long long dd = d0; dd < (long long)d1; ++dd) {
            u32 d = (u32)dd;
            const u64 *c;
            if (model) c = model + (u64)d * L * 2 * N;
            else { encrypt_dim(P, class_hv, d, tinv, fw, m, e, x, ct); c = ct; }
            query_plaintext(P, H, nq, b, d, tinv, m);
            for (u32 j = 0; j < L; ++j) {
                u64 q = P->q[j];
                for (u32 i = 0; i < N; ++i) p[i] = lift_centered(m[i], P->t, q);
                or_ntt_fwd(p, P->logN, q, fw[j]);
                for (u32 cc = 0; cc < 2; ++cc) {
                    const u64 *cj = c + ((u64)j * 2 + cc) * N;
                    u64 *aj = part + ((u64)cc * L + j) * N;
                    for (u32 i = 0; i < N; ++i) aj[i] = or_addmod(aj[i], or_mulmod(cj[i], p[i], q), q);
                }
            }
            n_mul += 1;                 /* one ct x pt product (all primes, c0 and c1) */
            if (have) n_add += 1;       /* folding a product into a running sum */
            have = 1;
        }
        #pragma omp critical
        {
            if (have) {
                if (!first_global) n_add += 1;   /* merging two partial sums is one more AddCC */
                first_global = 0;
                for (u32 cc = 0; cc < 2; ++cc)
                    for (u32 j = 0; j < L; ++j)
                        for (u32 i = 0; i < N; ++i) {
                            u64 *a = acc + ((u64)cc * L + j) * N + i;
                            *a = or_addmod(*a, part[((u64)cc * L + j) * N + i], P->q[j]);
                        }
            }
        }
        free(m); free(p); free(ct); free(x); free(e); free(part);
    }
    if (counters) { counters[0] = n_mul; counters[1] = n_add; counters[2] = 0; }
    free(tinv);
    free_tabs(fw, L);
}

/* decryption helper (per prime, NTT domain): x_hat = c0 + c1 (.) s_hat, then INTT_j.
   ct: [2][L][N]; out: [L][N] coefficient form of the phase mod q_j */
void or_decrypt_phase(const or_bfv *P, const u64 *ct, u64 *out) {
    u32 N = 1u << P->logN;
    u64 **inv = make_psi_tabs(P, 1);
    for (u32 j = 0; j < P->L; ++j) {
        u64 q = P->q[j];
        const u64 *c0 = ct + ((u64)0 * P->L + j) * N;
        const u64 *c1 = ct + ((u64)1 * P->L + j) * N;
        u64 *o = out + (u64)j * N;
        for (u32 i = 0; i < N; ++i) o[i] = or_addmod(c0[i], or_mulmod(c1[i], P->s_hat[(u64)j * N + i], q), q);
        or_ntt_inv(o, P->logN, q, inv[j]);
    }
    free_tabs(inv, P->L);
}


/* ------------------------------------------------------------------ */
/* HE-HDC-SR, the server-side SIMD baseline (P:257-265;    */
/* SPEC S:445-453): the CLIENT encrypts its query hypervectors in the  */
/* interleave layout (D ciphertexts per batch of B queries), the       */
/* SERVER multiplies them by the plaintext class tiles.                */
/* ------------------------------------------------------------------ */

/* query ciphertexts of batch b, dims [d0, d0+nd): out[nd][L][2][N]; message = the query
   slot vector of (b, d) encoded mod t ([0,t), Delta*m as for the model, reading #4);
   random streams of ciphertext index g = 2^32 + b*D_live + d (DESIGN reading #25: an index
   space disjoint from the model's d < D_live). */
void or_encrypt_queries(const or_bfv *P, const int8_t *H, u32 nq, u32 b, u32 d0, u32 nd, u64 *out) {
    u32 N = 1u << P->logN;
    u64 *tinv = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(or_powmod(P->psi_t, P->t - 2, P->t), P->t, P->logN, tinv);
    u64 **fw = make_psi_tabs(P, 0);
    #pragma omp parallel
    {
        u64 *m = (u64 *)malloc(sizeof(u64) * N);
        u64 *x = (u64 *)malloc(sizeof(u64) * N);
        long long *e = (long long *)malloc(sizeof(long long) * N);
        #pragma omp for schedule(dynamic)
        for (long long dd = 0; dd < (long long)nd; ++dd) {
            u32 d = d0 + (u32)dd;
            query_plaintext(P, H, nq, b, d, tinv, m);
            encrypt_msg(P, (1ULL << 32) + (u64)b * P->D_live + d, m, fw, e, x, out + (u64)dd * P->L * 2 * N);
        }
        free(m); free(x); free(e);
    }
    free(tinv);
    free_tabs(fw, P->L);
}

/* server: acc[c][j] = sum_d qct_{d,j,c} (.) NTT_j(lift(encode(tile_d))), qct [D_live][L][2][N] */
void or_server_eval(const or_bfv *P, const int8_t *class_hv, const u64 *qct, u64 *acc) {
    u32 N = 1u << P->logN;
    u32 L = P->L;
    u64 *tinv = (u64 *)malloc(sizeof(u64) * N);
    or_pow_brev_table(or_powmod(P->psi_t, P->t - 2, P->t), P->t, P->logN, tinv);
    u64 **fw = make_psi_tabs(P, 0);
    u64 *m = (u64 *)malloc(sizeof(u64) * N);
    u64 *p = (u64 *)malloc(sizeof(u64) * N);
    for (u64 x = 0; x < (u64)2 * L * N; ++x) acc[x] = 0;
    for (u32 d = 0; d < P->D_live; ++d) {
        model_plaintext(P, class_hv, d, tinv, m);
        for (u32 j = 0; j < L; ++j) {
            u64 q = P->q[j];
            for (u32 i = 0; i < N; ++i) p[i] = lift_centered(m[i], P->t, q);
            or_ntt_fwd(p, P->logN, q, fw[j]);
            for (u32 cc = 0; cc < 2; ++cc) {
                const u64 *cj = qct + (((u64)d * L + j) * 2 + cc) * N;
                u64 *aj = acc + ((u64)cc * L + j) * N;
                for (u32 i = 0; i < N; ++i) aj[i] = or_addmod(aj[i], or_mulmod(cj[i], p[i], q), q);
            }
        }
    }
    free(m); free(p); free(tinv);
    free_tabs(fw, L);
}
