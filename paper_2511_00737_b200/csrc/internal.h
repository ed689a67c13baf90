// internal.h -- library-internal structures shared by api.cu and kernels.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <vector>

#include "../../include/ephdc.h"
#include "host_math.h"
#include "modarith.cuh"

namespace ephdc {

constexpr int kMaxL = EPHDC_MAX_PRIMES;

// Kernel arguments passed by value (fit in the 4 KB parameter space).
struct PrimeSet {
    u64 q[kMaxL];
    u64 qinv[kMaxL];   // q^-1 mod 2^64 (Montgomery)
    u64 r2[kMaxL];     // 2^128 mod q (undoes the 2^-64 of Montgomery sums)
    u64 qmt[kMaxL];    // q - t (centered lift, reading #3)
    u64 delta[kMaxL];  // floor(Q/t) mod q (reading #4)
    u64 delta_p[kMaxL];// Shoup companion of delta
    u64 mask[kMaxL];   // 2^ceil(log2 q) - 1 (rejection sampling, reading #8)
};

// Arguments of the FP64-pipe fused kernel (kernels_f64.cu).
struct F64MacArgs {
    double two52_plus_t;     // 2^52 + t (centered lift, modf64.cuh)
    const double2 *tw;       // [L][N] (psi_rev[i], fl(psi_rev[i]/q_j)); entry 0 = (q_j, fl(1/q_j))
    u32 half_t;              // (t-1)/2
    u32 L, D;                // primes, live dims
    u32 nb, bg;              // batches in the launch, batches per group (grid order)
    u32 chunks, G;           // dim chunks per batch, dims per chunk
    u32 red_every;           // accumulator reduction interval (dims)
    u32 flags;               // bit 0 = no explicit L2 prefetch of the model slice (launch plan)
    const u32 *dlim;         // [nb] dims summed per batch (ephdc_infer_batch_prefix), or null = D
};

// FP64 path plan: chosen at context creation when every q_j < 2^50 and the value
// bounds of DESIGN.md "FP64 modular arithmetic" hold.
struct F64Plan {
    bool enabled = false;
    u32 red_every = 1;       // accumulator reduction interval
};

struct ctxDev {
    double2 *tw_f64 = nullptr;     // [L][N] (w, w/q) for the FP64 path
    TwPair<u64> *tw_q = nullptr;   // [L][N] forward twiddles mod q_j
    TwPair<u32> *itw_t = nullptr;  // [N] inverse twiddles mod t
    u64 *cdt = nullptr;            // [20]
};

}  // namespace ephdc

struct ephdc_ctx {
    ephdc_params p{};
    std::vector<uint64_t> q;
    uint32_t N = 0, L = 0, B = 0;
    uint64_t t = 0, psi_t = 0;
    std::vector<uint64_t> psi, delta;
    uint32_t ninv_t = 0, ninv_t_p = 0;
    ephdc::PrimeSet ps{};
    uint64_t cdt[20]{};
    // host NTTs (keygen, decrypt)
    std::vector<ephdc_host::HostNtt> host_q;
    ephdc_host::HostNtt host_t;
    ephdc_host::CrtRound crt;
    // device
    int device = -1;
    ephdc::ctxDev dev;
    uint32_t fused_S = 1, fused_chunks = 1, fused_G = 1;
    ephdc::F64Plan f64;
    std::vector<uint32_t> qbits;   // bit_length(q_j): scores-message packing widths
};

struct ephdc_sk {
    const ephdc_ctx *ctx = nullptr;
    std::vector<int8_t> s;
    std::vector<uint64_t> s_hat;  // [L][N]
    uint64_t *d_shat_mont = nullptr;  // device copy of s_hat * 2^64 mod q_j (lazy, encryption)
};

struct ephdc_model {
    const ephdc_ctx *ctx = nullptr;
    uint64_t *d_ct = nullptr;     // [D_live][L][2][N]: u64 (integer path) or exact doubles (FP64 path)
    uint32_t D = 0;
    ephdc_model() = default;
    ephdc_model(const ephdc_model &) = delete;
    ephdc_model &operator=(const ephdc_model &) = delete;
    ~ephdc_model() {  // owns d_ct: every error path of ephdc_encrypt_model releases it
        if (d_ct) {
            cudaSetDevice(ctx->device);
            cudaFree(d_ct);
        }
    }
};

struct ephdc_workspace {
    const ephdc_ctx *ctx = nullptr;
    uint32_t max_nq = 0;
    uint32_t *d_M = nullptr;      // [m_batches][D_live][N] encoded plaintexts, centered int32 (#3)
    uint32_t m_batches = 1;       // batches d_M holds (FP64 path: all of max_nq, capped)
    void *d_X = nullptr;          // [max_nq][F]
    int8_t *d_H = nullptr;        // [D_live][max_nq]
    uint64_t *d_out = nullptr;    // [nb_max][2][L][N]
    uint8_t *d_msg = nullptr;     // packed scores message of nb_max ciphertexts
    uint32_t *d_dlim = nullptr;   // [nb_max] per-batch dim counts (ephdc_infer_batch_prefix)
    uint32_t nb_max = 0;
    ephdc_plan plan{};            // launch-plan overrides (tests/profiling; zeros = tuned)
    // timing
    bool timing = false;
    static constexpr int kClasses = 4;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_marks;  // (class, event index of start; end = +1)
    double ms[kClasses]{};
    uint64_t launches[kClasses]{};
    cudaStream_t last_stream = nullptr;
};

struct ephdc_ntt_plan {
    std::vector<uint64_t> q;
    uint32_t L = 0, log2N = 0, N = 0;
    int device = -1;
    ephdc::PrimeSet ps{};
    TwPair<u64> *tw = nullptr, *itw = nullptr;  // [L][N]
    uint64_t *ninv = nullptr;                            // [L][2] (N^-1, Shoup)
    // u32 words (every q_j < 2^30; ephdc_ntt_*32): the same tables in 32 bits
    TwPair<u32> *tw32 = nullptr, *itw32 = nullptr;  // [L][N]
    uint32_t *ninv32 = nullptr;                      // [L][2]
    // FP64 path (kernels_f64.cu k_ntt_std_f64) when the bounds allow it
    bool fwd_f64 = false, inv_f64 = false;
    bool inv_dit = false;   // FP64 inverse form: Cooley-Tukey DIT (true) or Gentleman-Sande
    // FP64 path: forward psi_rev table and the inverse's table -- GS: psi^-1_rev; DIT:
    // stage table (entry h + jj = omega^-(N/2h) jj) -- each [L][N] (w, w/q) with entry
    // 0 = (q, 1/q); the inverse's scaling: GS N^-1 [L], DIT N^-1 psi^-j [L][N] (w, w/q)
    double2 *tw_f64 = nullptr, *itw_f64 = nullptr;
    double2 *post_f64 = nullptr;
    // c5 kernels (ntt_c5.cu) when their bounds hold; c5_red: a cluster forward reduces
    // after its cross levels
    bool c5_fwd = false, c5_inv = false, c5_red = false;
    bool c5_alt_teams = false;   // EPHDC_NTT_ALT_TEAMS (A/B only)
    bool int_per_poly = false;   // EPHDC_NTT_ALT_TEAMS also selects the per-polynomial integer kernel (A/B)
    bool u32_generic = false;    // EPHDC_NTT_U32_GENERIC: the general u32 kernels instead of ntt32_c5.cu (A/B)
    // u64 words with every prime < 2^30 at N = 2^12 .. 2^14: the ntt32_c5.cu kernels on
    // the low words (unless EPHDC_NTT_U32_GENERIC / FORCE_INT)
    bool u32_for_u64 = false;
    // inverse: DIT table [L][N] (W[h + jj] = omega^-(N/2h) jj, entry 0 = (q, 1/q)), fused
    // level-12 scaling [L][NC/2][2] (sigma_r, sigma_r W[NC/2 + r]), sigma_r = N^-1 psi^-r;
    // c_loc = psi^-(NC/2); block constants c_k = psi^-(NC k) [L][8]
    double2 *c5_itw = nullptr, *c5_itail = nullptr, *c5_ck = nullptr;
    double2 c5_cinv[EPHDC_MAX_PRIMES]{};
};

namespace ephdc {

extern std::atomic<uint64_t> g_launches;

// ---- launchers (kernels.cu); all return cudaGetLastError() after the launch ----
cudaError_t launch_encode(const ephdc_ctx *c, const void *d_X, const int8_t *d_P, uint32_t nq, void *d_H, bool raw,
                          cudaStream_t st);
// slot pack + INTT_t of batches [b, b+nbat) x dims [d0, d0+nd) -> d_M [nbat][nd][N]
cudaError_t launch_pack_intt_queries(const ephdc_ctx *c, const int8_t *d_H, uint32_t nq, uint32_t b, uint32_t nbat,
                                     uint32_t d0, uint32_t nd, uint32_t *d_M, cudaStream_t st, uint32_t plan_flags = 0);
cudaError_t launch_pack_intt_model(const ephdc_ctx *c, const int8_t *d_C, uint32_t d0, uint32_t nd, uint32_t *d_M,
                                   cudaStream_t st);
cudaError_t launch_ntt_mac(const ephdc_ctx *c, const uint32_t *d_M, const uint64_t *d_model, uint64_t *d_out,
                           cudaStream_t st, uint32_t d_lim = 0xffffffffu);
cudaError_t launch_finalize(const ephdc_ctx *c, uint64_t *d_out, cudaStream_t st);
cudaError_t launch_plaintext_ntt(const ephdc_ctx *c, const uint32_t *d_M, uint32_t nd, uint64_t *d_pt,
                                 cudaStream_t st);
// secret-key encryption of nd encoded messages d_M ([0, t)): random streams g0 + dd
// under the ChaCha20 key (rng.cuh), output d_out [nd][L][2][N]
cudaError_t launch_encrypt(const ephdc_ctx *c, const uint32_t *d_M, uint64_t g0, uint32_t nd,
                           const uint64_t *d_shat_mont, const ephdc_seed &key, uint64_t *d_out, cudaStream_t st);
cudaError_t launch_pack_intt_sr(const ephdc_ctx *c, const int8_t *src, bool model, uint32_t nq, uint32_t b,
                                uint32_t d0, uint32_t nd, uint32_t *d_M, cudaStream_t st);
cudaError_t launch_mac_ctx(const ephdc_ctx *c, const uint64_t *d_ct, const uint64_t *d_pt, uint32_t D, uint64_t *d_out,
                           cudaStream_t st);
cudaError_t launch_ntt_batch(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, bool inverse,
                             cudaStream_t st);
cudaError_t launch_mac(const ephdc_ntt_plan *p, const uint64_t *d_ct, const uint64_t *d_pt, uint32_t D,
                       uint64_t *d_out, cudaStream_t st);
cudaError_t launch_ntt_batch32(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, bool inverse,
                               cudaStream_t st);
cudaError_t launch_mac32(const ephdc_ntt_plan *p, const uint32_t *d_ct, const uint32_t *d_pt, uint32_t D,
                         uint32_t *d_out, cudaStream_t st);
size_t ntt_mac_smem_bytes(uint32_t log2Nc);
// tcgen05 int8 encoder (encode_tc.cu)
bool encode_tc_supported(const ephdc_ctx *c);
cudaError_t launch_encode_tc(const ephdc_ctx *c, const void *d_X, const int8_t *d_P, uint32_t nq, void *d_H, bool raw,
                             cudaStream_t st);
// FP64-pipe path (kernels_f64.cu)
cudaError_t launch_ntt_mac_f64(const ephdc_ctx *c, const ephdc_plan &plan, const uint32_t *d_M, uint32_t nb,
                               const double *d_model, uint64_t *d_out, cudaStream_t st,
                               const uint32_t *d_dlim = nullptr);
cudaError_t launch_u64_to_f64(uint64_t *d, size_t n, cudaStream_t st);
// scores message layout (bit-packed residues, ephdc.h "scores message")
struct MsgLayout {
    u32 bits[kMaxL];     // bit_length(q_j)
    u64 prefix[kMaxL];   // byte offset of prime j inside a (batch, component) group
    u64 group_bytes;     // bytes of one (batch, component) group = N * sum_j bits / 8
};
MsgLayout msg_layout(const ephdc_ctx *c);
cudaError_t launch_pack_bits(const ephdc_ctx *c, const uint64_t *d_ct, uint32_t nb, uint8_t *d_msg, cudaStream_t st);
// model residues of dim d times fac[d / g][j] (ephdc_model_scale)
cudaError_t launch_model_scale(const ephdc_ctx *c, uint64_t *d_model, uint32_t D, uint32_t g, const uint64_t *d_fac,
                               cudaStream_t st);
cudaError_t launch_plaintext_ntt_f64(const ephdc_ctx *c, const uint32_t *d_M, uint32_t nd, uint64_t *d_pt,
                                     cudaStream_t st);
cudaError_t launch_reduce_out(const ephdc_ctx *c, uint64_t *d_out, uint32_t nb, cudaStream_t st);
int ntt_mac_f64_occupancy(uint32_t log2N);
struct StdF64Args {
    u32 L;
    const double2 *tw;     // [L][N] forward (psi_rev) or inverse (DIT stages) (w, w/q); entry 0 = (q, 1/q)
    const double2 *post;   // inverse scaling: GS [L] N^-1, DIT [L][N] N^-1 psi^-j (w, w/q)
};
cudaError_t launch_ntt_batch_f64(const ephdc_ntt_plan *pl, uint64_t *d_polys, uint32_t batch, bool inverse,
                                 cudaStream_t st);
void plan_ntt_f64(const std::vector<uint64_t> &q, uint32_t log2N, bool *fwd, bool *inv, bool *inv_dit);
// c5 standalone kernels (ntt_c5.cu)
struct C5Args {
    u64 *polys;            // [batch][L][N], in place
    const double2 *tw;     // forward: [L][N] (psi_rev[i], fl(psi_rev[i]/q_j)), entry 0 = (q_j, fl(1/q_j));
                           // inverse: the DIT table ephdc_ntt_plan::c5_itw
    const double2 *tail;   // inverse: ephdc_ntt_plan::c5_itail
    const double2 *ck;     // inverse: ephdc_ntt_plan::c5_ck
    u32 L, batch, items;   // items = L * batch (prime-major work order)
    u32 log2N;
    double2 cinv[kMaxL];   // inverse: c_loc = psi^-(NC/2) as (w, w/q)
};
cudaError_t plan_ntt_c5(ephdc_ntt_plan *p);
void ephdc_ntt_plan_c5_free(ephdc_ntt_plan *p);
cudaError_t launch_ntt_c5(const ephdc_ntt_plan *pl, uint64_t *d_polys, uint32_t batch, bool inverse, cudaStream_t st);
// query-path slot pack + INTT_t on the ntt32_c5.cu passes (N = 2^12 .. 2^14;
// cudaErrorNotSupported elsewhere)
cudaError_t launch_pack_intt_q32(const ephdc_ctx *c, const int8_t *d_H, uint32_t nq, uint32_t b0, uint32_t nbat,
                                 uint32_t *d_M, cudaStream_t st, bool no_prefetch = false);
cudaError_t launch_ntt32_c5_u64(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, bool inverse,
                                cudaStream_t st);
cudaError_t launch_ntt_global32(const ephdc_ntt_plan *p, uint32_t *polys, uint32_t batch, bool inverse,
                                cudaStream_t st);
// c5 u32 kernels (ntt32_c5.cu) at N = 2^12 .. 2^16 (2^15 / 2^16: global stages + 2^14
// slices); cudaErrorNotSupported elsewhere
cudaError_t launch_ntt32_c5(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, bool inverse,
                            cudaStream_t st);
bool plan_f64(const std::vector<uint64_t> &q, uint64_t t, uint32_t log2N, F64Plan *plan);
void f64_grid(const ephdc_ctx *c, uint32_t nb, uint32_t *bg, uint32_t *chunks, uint32_t *G);
int ntt_mac_occupancy(uint32_t log2N, uint32_t S);

}  // namespace ephdc
