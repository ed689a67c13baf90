// kernels_f64.cu -- the FP64-pipe variant of the dominant fused kernel (primes q < 2^50).
//
//  k_ntt_mac_f64   centered lift (#3) + forward NTT mod q_j + ct x pt MAC
//                  for ALL batches of a call in one launch; accumulators in registers
//  k_pt_ntt_f64    the same NTT, canonical outputs stored (parity export of p_hat)
//  k_reduce_out    out mod q_j (the atomically folded partial sums)
//
// Work item (one CTA) = (batch b, prime j, slice s of S, chunk of G dims).  Items are
// ordered [batch group][chunk][batch in group][prime][slice] so the ~148 CTAs resident
// at a time share their chunk's model tiles (read by every batch of the group) and
// encoded plaintexts (read by every prime and slice) through L2: the 23.6 GB model of
// c4 crosses HBM once per batch group instead of once per batch.  DESIGN.md "Kernels".
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "internal.h"
#include "modarith.cuh"
#include "ntt_f64.cuh"
#include "tmem.cuh"
#include "async_copy.cuh"

namespace ephdc {

using namespace ephdc_f64;

namespace {

EPHDC_D void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// model residue pairs: read by every batch of a group within a few microseconds, so
// they are loaded (and prefetched) with an L2 evict_last policy
EPHDC_D uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
EPHDC_D double2 ld_pair(const double *p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}
EPHDC_D void prefetch_l2_last(const void *p) { asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p)); }

inline cudaError_t counted(cudaError_t e) {
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

}  // namespace

// Occupancy: 512 threads x 128 registers per SM and 128 TMEM columns per warp of a lane
// quarter (512 per SM): one CTA at NC = 8192, two at 4096, four at <= 2048.
template <int LGC> constexpr int f64_ctas_per_sm() {
    constexpr int by_regs = (8192 >> LGC) > 1 ? (8192 >> LGC) : 1;
    return by_regs < 4 ? by_regs : 4;
}
#define EPHDC_F64_BOUNDS(LGC) __launch_bounds__((1 << (LGC)) / kE, f64_ctas_per_sm<LGC>())

// TMEM columns of one CTA: 128 per warp of a lane quarter (64 accumulator columns =
// 2 x 16 doubles, 32 last-stage twiddle columns = 8 x (w, w/q), 32 spare).
template <int LGC> constexpr uint32_t tmem_cols() {
    constexpr int warps = (1 << LGC) / kE / 32;
    return 128u * (uint32_t)((warps + 3) / 4);
}

// Dynamic shared memory of the fused kernel: head-stage twiddles [NC/2] double2, the
// NTT buffer, the staged plaintext row [S*NC] u32.
template <int LGC, int S> constexpr size_t mac_f64_smem() {
    constexpr size_t nc = (size_t)1 << LGC;
    return sizeof(double2) * (nc / 2) + sizeof(double) * (size_t)ephdc_f64::padded_len((int)nc) +
           sizeof(uint32_t) * nc * S;
}

// E = elements per thread (16: NC/16 threads x <= 128 registers; 32: NC/32 threads,
// twice the independent work per warp, up to 255 registers).
template <int LGC, int E> constexpr int mac_threads() { return (1 << LGC) / E; }
template <int LGC, int E> constexpr int mac_min_blocks() { return E == kE ? f64_ctas_per_sm<LGC>() : 1; }

// PREFIX (ephdc_infer_batch_prefix): batch b sums only its first dlim[b] dims.  A
// separate instantiation: even this one clamp reschedules the whole 128-register kernel
// (ptxas) and cost the default path 6% at c4 (r02: 260.4 vs 245 ms).
template <int LGC, int S, int WL, int E, bool PREFIX = false>
__global__ void __launch_bounds__(mac_threads<LGC, E>(), mac_min_blocks<LGC, E>())
    k_ntt_mac_f64(const u32 *__restrict__ M, const double *__restrict__ model, u64 *__restrict__ out, F64MacArgs a) {
    using namespace ephdc_async;
    constexpr int NC = 1 << LGC, N = NC * S;
    // TMEM: per thread 4E accumulator columns (E coefficients x 2 components x 2 words)
    // and 2E last-stage twiddle columns; warps of one lane quarter split the 512 columns
    constexpr int kWarps = NC / E / 32;
    constexpr uint32_t kWarpCols = kWarps >= 4 ? 512u / (uint32_t)(kWarps / 4) : 512u;
    static_assert(6 * E <= (int)kWarpCols, "TMEM columns per warp");
    constexpr uint32_t kCols = E == kE ? tmem_cols<LGC>() : 512u;
    constexpr uint32_t kColStride = E == kE ? 128u : kWarpCols;
    constexpr int NBLK = E / 4;                 // tail blocks of 2 coefficient pairs
    constexpr int PRE = E == kE ? 2 : 4;        // model blocks requested before the last head pass
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t mbar;
    double2 *tw = reinterpret_cast<double2 *>(smem_raw);                               // [NC/2]
    double *buf = reinterpret_cast<double *>(smem_raw + sizeof(double2) * (NC / 2));   // padded [NC]
    u32 *mst = reinterpret_cast<u32 *>(smem_raw + sizeof(double2) * (NC / 2) +
                                       sizeof(double) * padded_len(NC));               // [N]
    const int tid = threadIdx.x, warp = tid >> 5;
    // block order: batch fastest, then slice, prime, chunk, group -- the CTAs of a wave
    // cover bg batches x (a few primes and slices) of one chunk, so a model tile is
    // read by bg concurrent CTAs and a plaintext row by the slices/primes of the wave
    u32 x = blockIdx.x;
    const u32 bl = x % a.bg;
    x /= a.bg;
    const u32 s = x % S;
    x /= S;
    const u32 j = x % a.L;
    x /= a.L;
    const u32 chunk = x % a.chunks, grp = x / a.chunks;
    const u32 b = grp * a.bg + bl;
    if (b >= a.nb) return;
    const u32 d0 = chunk * a.G, d1 = PREFIX ? min(min(a.D, a.dlim[b]), d0 + a.G) : min(a.D, d0 + a.G);
    if (d0 >= d1) return;

    const u32 *Mb = M + (size_t)b * a.D * N;
    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, kCols);
    if (tid == 0) {
        mbar_init(&mbar, 1);
        // first plaintext row of the chunk -> shared memory (TMA bulk copy)
        mbar_arrive_expect_tx(&mbar, N * 4u);
#pragma unroll
        for (int c = 0; c < 4; ++c) bulk_g2s(mst + c * (N / 4), Mb + (size_t)d0 * N + c * (N / 4), N, &mbar);
    }
    const double2 *twg = a.tw + (size_t)j * N;
    const double2 qq = twg[0];  // slot 0 of the table holds (q_j, fl(1/q_j))
    const double q = qq.x, nq = -q, qinv = qq.y;
    load_twiddles<LGC, S, E>(tw, twg, (int)s, NC / 2);
    double2 w1 = make_double2(0.0, 0.0);
    if constexpr (S > 1) w1 = twg[1];
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    // this thread's TMEM columns: block c (pairs tail_pair(2c), tail_pair(2c+1)) keeps its
    // accumulators at 16c .. 16c+15 = (acc0[2u], acc0[2u+1], acc1[2u], acc1[2u+1]) x 2 words
    // and its last-stage twiddles at 4E + 8c .. 4E + 8c + 7 = (w, w/q) x 2 words x 2 pairs
    const uint32_t tacc = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * kColStride;
    const uint32_t ttw = tacc + 4u * E;
    {
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
        for (int c = 0; c < NBLK; ++c) ephdc_tmem::st16(tacc + 16 * c, z);
#pragma unroll
        for (int h = 0; h < E / 8; ++h) {
            uint32_t t[16];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double2 w = twg[tail_twiddle_index<LGC, S>((int)s, tail_pair<LGC, WL == 2, E>(4 * h + k))];
                t[4 * k] = (uint32_t)__double2loint(w.x);
                t[4 * k + 1] = (uint32_t)__double2hiint(w.x);
                t[4 * k + 2] = (uint32_t)__double2loint(w.y);
                t[4 * k + 3] = (uint32_t)__double2hiint(w.y);
            }
            ephdc_tmem::st16(ttw + 16 * h, t);
        }
    }

    u32 since_red = 0, phase = 0;
    const uint64_t pol = l2_evict_last_policy();
    for (u32 d = d0; d < d1; ++d) {
        const double *c0 = model + (((size_t)d * a.L + j) * 2) * N + (size_t)s * NC;
        const double *c1 = c0 + N;
        if (!(a.flags & 1u)) {
            prefetch_l2_last(c0 + 16 * tid);  // this dim's model slice, read by the last stage
            prefetch_l2_last(c1 + 16 * tid);
        }
        mbar_wait(&mbar, phase);     // plaintext row d is in mst
        phase ^= 1u;
        auto load = [&](int pos) -> double {
            const double U = from_i32((int)mst[pos]);
            if constexpr (S == 1) {
                return U;
            } else {
                // first global stage (half-size N/2) fused into the load: slice s keeps U +- w V
                const double V = from_i32((int)mst[pos + NC]);
                const double T = mul_tw(V, w1.x, w1.y, nq);
                return s == 0 ? __dadd_rn(U, T) : __dsub_rn(U, T);
            }
        };
        auto after_first = [&]() {  // mst consumed: fetch the next plaintext row
            if (tid == 0 && d + 1 < d1) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&mbar, N * 4u);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    bulk_g2s(mst + c * (N / 4), Mb + (size_t)(d + 1) * N + c * (N / 4), N, &mbar);
            }
        };
        // model pairs of the last stage: blocks 0, 1 (4 pairs each) are requested before the
        // last head pass, blocks 2, 3 when the last stage starts
        double2 mc[4][4];
        auto load_block = [&](int c, double2 (&dst)[4]) {
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
                const int g = tail_pair<LGC, WL == 2, E>(2 * c + uu);
                dst[2 * uu] = ld_pair(c0 + 2 * g, pol);
                dst[2 * uu + 1] = ld_pair(c1 + 2 * g, pol);
            }
        };
        auto before_last = [&]() {
#pragma unroll
            for (int c = 0; c < PRE; ++c) load_block(c, mc[c]);
        };
        fwd_ntt_head<LGC, WL, E>(buf, load, tw, nq, after_first, before_last);
        // last stage + MAC, one 16-column TMEM block (two coefficient pairs) at a time;
        // model blocks stream 4 ahead through mc[c % 4]
        const bool red = ++since_red >= a.red_every;
        if (red) since_red = 0;
        ephdc_tmem::wait_st();
#pragma unroll
        for (int c = PRE; c < 4 && c < NBLK; ++c) load_block(c, mc[c]);
#pragma unroll
        for (int c = 0; c < NBLK; ++c) {
            uint32_t r[16], t[8];
            ephdc_tmem::ld16(tacc + 16 * c, r);
            ephdc_tmem::ld8(ttw + 8 * c, t);
            ephdc_tmem::wait_ld(r);
            ephdc_tmem::after_wait(t);
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
                double x0, x1;
                fwd_ntt_tail<LGC, WL == 2, E>(buf, 2 * c + uu, __hiloint2double(t[4 * uu + 1], t[4 * uu]),
                                  __hiloint2double(t[4 * uu + 3], t[4 * uu + 2]), nq, x0, x1);
                const double2 m0v = mc[c % 4][2 * uu], m1v = mc[c % 4][2 * uu + 1];
                uint32_t *w = &r[uu * 8];
                double v[4] = {__hiloint2double(w[1], w[0]), __hiloint2double(w[3], w[2]),
                               __hiloint2double(w[5], w[4]), __hiloint2double(w[7], w[6])};
                v[0] = __dadd_rn(v[0], mul_rt(m0v.x, x0, qinv, nq));
                v[1] = __dadd_rn(v[1], mul_rt(m0v.y, x1, qinv, nq));
                v[2] = __dadd_rn(v[2], mul_rt(m1v.x, x0, qinv, nq));
                v[3] = __dadd_rn(v[3], mul_rt(m1v.y, x1, qinv, nq));
                if (red) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = reduce(v[e], qinv, nq);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    w[2 * e] = (uint32_t)__double2loint(v[e]);
                    w[2 * e + 1] = (uint32_t)__double2hiint(v[e]);
                }
            }
            ephdc_tmem::st16(tacc + 16 * c, r);
            if (c + 4 < NBLK) load_block(c + 4, mc[c % 4]);
        }
        __syncthreads();  // the next first pass overwrites buf
    }
    // fold this chunk's sum (canonical, < q) into the batch's scores ciphertext; the
    // sums of <= chunks values < q fit 64 bits (checked on the host) and integer
    // addition is order-independent, so the result is deterministic
    {
        uint32_t r[NBLK][16];
        ephdc_tmem::wait_st();
#pragma unroll
        for (int c = 0; c < NBLK; ++c) ephdc_tmem::ld16(tacc + 16 * c, r[c]);
        ephdc_tmem::wait_ld(r[0]);
#pragma unroll
        for (int c = 1; c < NBLK; ++c) ephdc_tmem::after_wait(r[c]);
        u64 *o0 = out + (((size_t)b * 2 + 0) * a.L + j) * N + (size_t)s * NC;
        u64 *o1 = out + (((size_t)b * 2 + 1) * a.L + j) * N + (size_t)s * NC;
#pragma unroll
        for (int u = 0; u < E / 2; ++u) {
            const int g = tail_pair<LGC, WL == 2, E>(u);
            const uint32_t *w = &r[u >> 1][(u & 1) * 8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double v = reduce(__hiloint2double(w[2 * e + 1], w[2 * e]), qinv, nq);
                u64 *o = (e < 2 ? o0 : o1) + 2 * g + (e & 1);
                atomicAdd(reinterpret_cast<unsigned long long *>(o), (unsigned long long)to_canonical_u64(v, q));
            }
        }
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_slot, kCols);
}

// ---------------------------------------------------------------------------------
// Two warp groups (NC = 2^13: c3, c4).  One CTA per work item as above, but its 16 warps
// form two 8-warp groups that take alternate dims of the chunk, each with its own NTT
// buffer (the TMA staging of the plaintext row is dropped: pass 1 reads the row from
// L2 directly, which frees the 64 KB).  Why: with one team every warp reaches the
// shared-memory phases of a pass together (barriers align them), so the ~3.5K clocks of
// shared-memory traffic per dim and the ~9.6K clocks of FP64 work serialise (measured
// 13.6K per dim); with the groups a pass apart, one group's loads and stores overlap the
// other's butterflies (the c5 forward gained 8% this way).  Each thread performs the
// one-team threads vt = t and t + 256 (same registers, same TMEM columns: warps w and
// w + 8 share a lane quarter), so both groups accumulate into the SAME TMEM accumulators;
// the read-modify-write of half h is serialised between the groups in dim order by a
// token per half (named barriers 4 + 2h: group 0 released it, 5 + 2h: group 1 did).
// ---------------------------------------------------------------------------------
EPHDC_D void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EPHDC_D void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int S> constexpr size_t mac_f64_2g_smem() {
    constexpr size_t nc = (size_t)1 << 13;
    return sizeof(double2) * (nc / 2) + 2 * sizeof(double) * (size_t)ephdc_f64::padded_len((int)nc);
}

template <int S>
__global__ void __launch_bounds__(512, 1)
    k_ntt_mac_f64_2g(const u32 *__restrict__ M, const double *__restrict__ model, u64 *__restrict__ out, F64MacArgs a) {
    constexpr int LGC = 13, E = kE, NC = 1 << LGC, N = NC * S, NT = NC / E;
    constexpr int NBLK = E / 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint32_t tmem_slot;
    double2 *tw = reinterpret_cast<double2 *>(smem_raw);                                  // [NC/2]
    const int tid = threadIdx.x, warp = tid >> 5, g = warp >> 3, gt = tid & 255;
    double *buf = reinterpret_cast<double *>(smem_raw + sizeof(double2) * (NC / 2)) + (size_t)g * padded_len(NC);
    u32 x = blockIdx.x;
    const u32 bl = x % a.bg;
    x /= a.bg;
    const u32 s = x % S;
    x /= S;
    const u32 j = x % a.L;
    x /= a.L;
    const u32 chunk = x % a.chunks, grp = x / a.chunks;
    const u32 b = grp * a.bg + bl;
    if (b >= a.nb) return;
    const u32 d0 = chunk * a.G, d1 = min(a.D, d0 + a.G);
    if (d0 >= d1) return;
    const u32 *Mb = M + (size_t)b * a.D * N;
    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, 512u);
    const double2 *twg = a.tw + (size_t)j * N;
    const double2 qq = twg[0];
    const double q = qq.x, nq = -q, qinv = qq.y;
    load_twiddles<LGC, S, E>(tw, twg, (int)s, NC / 2);
    double2 w1 = make_double2(0.0, 0.0);
    if constexpr (S > 1) w1 = twg[1];
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    // TMEM of one-team warp vw: accumulators at 128 (vw >> 2) + [0, 64), last-stage
    // twiddles at + [64, 96), lanes of quarter vw & 3 (= this warp's quarter)
    auto tacc_of = [&](int vw) {
        return tmem_slot + ((uint32_t)(32 * (vw & 3)) << 16) + (uint32_t)(vw >> 2) * 128u;
    };
    {   // each physical warp w initialises one-team warp w's columns (thread vt = tid)
        const uint32_t tacc = tacc_of(warp), ttw = tacc + 4u * E;
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
        for (int c = 0; c < NBLK; ++c) ephdc_tmem::st16(tacc + 16 * c, z);
#pragma unroll
        for (int h = 0; h < E / 8; ++h) {
            uint32_t t[16];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double2 w = twg[tail_twiddle_index<LGC, S>((int)s, tail_pair_vt<LGC>(4 * h + k, tid))];
                t[4 * k] = (uint32_t)__double2loint(w.x);
                t[4 * k + 1] = (uint32_t)__double2hiint(w.x);
                t[4 * k + 2] = (uint32_t)__double2loint(w.y);
                t[4 * k + 3] = (uint32_t)__double2hiint(w.y);
            }
            ephdc_tmem::st16(ttw + 16 * h, t);
        }
        ephdc_tmem::wait_st();
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    const uint64_t pol = l2_evict_last_policy();
    const bool pair = d0 + 1 < d1;
    if (g == 1 && pair) nbar_sync(3, 512);   // group 1 starts one pass behind group 0
    for (u32 d = d0 + (u32)g; d < d1; d += 2) {
        const u32 *row = Mb + (size_t)d * N;
        const double *c0 = model + (((size_t)d * a.L + j) * 2) * N + (size_t)s * NC;
        const double *c1 = c0 + N;
        auto load = [&](int pos) -> double {
            const double U = from_i32((int)__ldg(row + pos));
            if constexpr (S == 1) {
                return U;
            } else {
                const double V = from_i32((int)__ldg(row + pos + NC));
                const double T = mul_tw(V, w1.x, w1.y, nq);
                return s == 0 ? __dadd_rn(U, T) : __dsub_rn(U, T);
            }
        };
#pragma unroll 1
        for (int h = 0; h < 2; ++h) fwd_pass_vt<LGC, 12, 4, true>(buf, load, tw, nq, gt + 256 * h);
        nbar_sync(1 + g, 256);
        if (g == 0 && d == d0 && pair) nbar_arrive(3, 512);
        const bool red = (d - d0 + 1) % a.red_every == 0;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int vt = gt + 256 * h, vw = vt >> 5;
            fwd_pass_vt<LGC, 8, 4, false>(buf, load, tw, nq, vt);
            __syncwarp();
            double2 mc[4][4];
            auto load_block = [&](int c, double2 (&dst)[4]) {
#pragma unroll
                for (int uu = 0; uu < 2; ++uu) {
                    const int p = tail_pair_vt<LGC>(2 * c + uu, vt);
                    dst[2 * uu] = ld_pair(c0 + 2 * p, pol);
                    dst[2 * uu + 1] = ld_pair(c1 + 2 * p, pol);
                }
            };
#pragma unroll
            for (int c = 0; c < 2; ++c) load_block(c, mc[c]);
            fwd_pass_vt<LGC, 4, 4, false>(buf, load, tw, nq, vt);
            __syncwarp();
            // the token of half h: dims alternate between the groups
            if (g == 0 ? d >= d0 + 2 : true) nbar_sync(4 + 2 * h + (g == 0 ? 1 : 0), 512);
            ephdc_tmem::fence_after_sync();
            const uint32_t tacc = tacc_of(vw), ttw = tacc + 4u * E;
#pragma unroll
            for (int c = 2; c < 4; ++c) load_block(c, mc[c]);
#pragma unroll
            for (int c = 0; c < NBLK; ++c) {
                uint32_t r[16], t[8];
                ephdc_tmem::ld16(tacc + 16 * c, r);
                ephdc_tmem::ld8(ttw + 8 * c, t);
                ephdc_tmem::wait_ld(r);
                ephdc_tmem::after_wait(t);
#pragma unroll
                for (int uu = 0; uu < 2; ++uu) {
                    const int p = tail_pair_vt<LGC>(2 * c + uu, vt);
                    const int ad = pad(2 * p);
                    double x0 = buf[ad], x1 = buf[ad + 1];
                    ct_bfly(x0, x1, __hiloint2double(t[4 * uu + 1], t[4 * uu]), __hiloint2double(t[4 * uu + 3], t[4 * uu + 2]),
                            nq);
                    const double2 m0v = mc[c][2 * uu], m1v = mc[c][2 * uu + 1];
                    uint32_t *w = &r[uu * 8];
                    double v[4] = {__hiloint2double(w[1], w[0]), __hiloint2double(w[3], w[2]),
                                   __hiloint2double(w[5], w[4]), __hiloint2double(w[7], w[6])};
                    v[0] = __dadd_rn(v[0], mul_rt(m0v.x, x0, qinv, nq));
                    v[1] = __dadd_rn(v[1], mul_rt(m0v.y, x1, qinv, nq));
                    v[2] = __dadd_rn(v[2], mul_rt(m1v.x, x0, qinv, nq));
                    v[3] = __dadd_rn(v[3], mul_rt(m1v.y, x1, qinv, nq));
                    if (red) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) v[e] = reduce(v[e], qinv, nq);
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        w[2 * e] = (uint32_t)__double2loint(v[e]);
                        w[2 * e + 1] = (uint32_t)__double2hiint(v[e]);
                    }
                }
                ephdc_tmem::st16(tacc + 16 * c, r);
            }
            ephdc_tmem::wait_st();
            ephdc_tmem::fence_before_sync();
            if (d + 1 < d1) nbar_arrive(4 + 2 * h + (g == 0 ? 0 : 1), 512);   // pass the token on
        }
        nbar_sync(1 + g, 256);   // the next dim's first pass overwrites buf
    }
    // fold: each physical warp w folds one-team warp w's accumulators
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    {
        const uint32_t tacc = tacc_of(warp);
        uint32_t r[NBLK][16];
#pragma unroll
        for (int c = 0; c < NBLK; ++c) ephdc_tmem::ld16(tacc + 16 * c, r[c]);
        ephdc_tmem::wait_ld(r[0]);
#pragma unroll
        for (int c = 1; c < NBLK; ++c) ephdc_tmem::after_wait(r[c]);
        u64 *o0 = out + (((size_t)b * 2 + 0) * a.L + j) * N + (size_t)s * NC;
        u64 *o1 = out + (((size_t)b * 2 + 1) * a.L + j) * N + (size_t)s * NC;
#pragma unroll
        for (int u = 0; u < E / 2; ++u) {
            const int p = tail_pair_vt<LGC>(u, tid);
            const uint32_t *w = &r[u >> 1][(u & 1) * 8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double v = reduce(__hiloint2double(w[2 * e + 1], w[2 * e]), qinv, nq);
                u64 *o = (e < 2 ? o0 : o1) + 2 * p + (e & 1);
                atomicAdd(reinterpret_cast<unsigned long long *>(o), (unsigned long long)to_canonical_u64(v, q));
            }
        }
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_slot, 512u);
}

// Plaintext NTTs for the parity export: p_hat[dd][j] = NTT_j(lift(M[dd])), canonical.
// CTA = (dim dd, prime j, slice s); same passes as the fused kernel.
template <int LGC, int S>
__global__ void EPHDC_F64_BOUNDS(LGC)
    k_pt_ntt_f64(const u32 *__restrict__ M, u64 *__restrict__ pt, F64MacArgs a) {
    constexpr int NC = 1 << LGC, N = NC * S;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *tw = reinterpret_cast<double2 *>(smem_raw);
    double *buf = reinterpret_cast<double *>(smem_raw + sizeof(double2) * NC);
    u32 x = blockIdx.x;
    const u32 s = x % S;
    x /= S;
    const u32 j = x % a.L, dd = x / a.L;
    const double2 *twg = a.tw + (size_t)j * N;
    const double2 qq = twg[0];
    const double q = qq.x, nq = -q, qinv = qq.y;
    load_twiddles<LGC, S>(tw, twg, (int)s, NC);
    double2 w1 = make_double2(0.0, 0.0);
    if constexpr (S > 1) w1 = twg[1];
    __syncthreads();
    const u32 *m = M + (size_t)dd * N;
    auto load = [&](int pos) -> double {
        const double U = from_i32((int)m[pos]);
        if constexpr (S == 1) {
            return U;
        } else {
            const double V = from_i32((int)m[pos + NC]);
            const double T = mul_tw(V, w1.x, w1.y, nq);
            return s == 0 ? __dadd_rn(U, T) : __dsub_rn(U, T);
        }
    };
    auto none = [] {};
    fwd_ntt_head<LGC>(buf, load, tw, nq, none, none);
    u64 *o = pt + ((size_t)dd * a.L + j) * N + (size_t)s * NC;
#pragma unroll
    for (int u = 0; u < kE / 2; ++u) {
        const int g = tail_pair<LGC, false>(u);
        const double2 w = tw[NC / 2 + g];
        double x0, x1;
        fwd_ntt_tail<LGC, false>(buf, u, w.x, w.y, nq, x0, x1);
        ulonglong2 v;
        v.x = to_canonical_u64(reduce(x0, qinv, nq), q);
        v.y = to_canonical_u64(reduce(x1, qinv, nq), q);
        *reinterpret_cast<ulonglong2 *>(o + 2 * g) = v;
    }
}

// =====================================================================================
// Standalone negacyclic NTT on the FP64 pipe (c5 microbench; primes within the bounds
// of ephdc_ntt_plan_create).  In place on [batch][L][N] canonical u64.  CTA = (poly,
// prime, slice s of S = N/NC); forward at N = 2^14 runs as a 2-CTA cluster: each CTA
// computes the first stage for its output half while loading both halves, and a
// cluster barrier after the first pass keeps either CTA from overwriting input its
// partner still reads.  Inverse: S = 1 (N <= 2^13).
// =====================================================================================
// DIR: 0 forward, 1 inverse Gentleman-Sande (bound doubles per stage: small primes),
// 2 inverse Cooley-Tukey DIT (linear bound growth, per-coefficient N^-1 psi^-j)
template <int LGC, int S, int DIR>
__global__ void __launch_bounds__((1 << LGC) / kE, 1) k_ntt_std_f64(u64 *__restrict__ polys, u32 batch, StdF64Args a) {
    constexpr bool INV = DIR != 0;
    constexpr int NC = 1 << LGC, N = NC * S;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *tw = reinterpret_cast<double2 *>(smem_raw);
    double *buf = reinterpret_cast<double *>(smem_raw + sizeof(double2) * NC);
    const int tid = threadIdx.x;
    // persistent: CTA (worker w, prime j, slice s) transforms polys b = w, w + W, ... of prime j
    const u32 s = blockIdx.x % S, wj = blockIdx.x / S, j = wj % a.L, w0 = wj / a.L;
    const u32 W = gridDim.x / (S * a.L);
    const double2 *twg = a.tw + (size_t)j * N;
    const double2 qq = twg[0];
    const double q = qq.x, nq = -q, qinv = qq.y, half_q = 0.5 * q;
    if constexpr (DIR == 2) {
        for (int p = tid; p < NC; p += NC / kE) tw[p] = twg[p];   // DIT stage table, natural order
    } else if constexpr (DIR == 1) {
        load_inv_twiddles<LGC>(tw, twg);
    } else {
        load_twiddles<LGC, S>(tw, twg, (int)s, NC);
    }
    double2 w1 = make_double2(0.0, 0.0);
    if constexpr (S > 1) w1 = twg[1];
    const double2 *post = a.post + (size_t)j * N;   // inverse: N^-1 psi^-i (DIT), N^-1 at [0] (GS)
    const double2 ni = DIR == 1 ? post[0] : make_double2(0.0, 0.0);
    __syncthreads();
    auto centered = [&](u64 v) -> double {   // [0, q) -> (-q/2, q/2]
        const double x = from_u64(v);
        return x > half_q ? __dsub_rn(x, q) : x;
    };
    for (u32 b = w0; b < batch; b += W) {
        u64 *p = polys + ((size_t)b * a.L + j) * N;
        if (b + W < batch) {   // next polynomial of this CTA into L2 while this one computes
            const u64 *pn = polys + ((size_t)(b + W) * a.L + j) * N + (size_t)s * NC;
            for (int l = tid; l < (NC * 8) / 128; l += NC / kE) prefetch_l2(pn + 16 * l);
        }
        if constexpr (!INV) {
            auto load = [&](int pos) -> double {
                const double U = centered(__ldcs(reinterpret_cast<const unsigned long long *>(p + pos)));
                if constexpr (S == 1) {
                    return U;
                } else {
                    const double V = centered(__ldcs(reinterpret_cast<const unsigned long long *>(p + pos + NC)));
                    const double T = mul_tw(V, w1.x, w1.y, nq);
                    return s == 0 ? __dadd_rn(U, T) : __dsub_rn(U, T);
                }
            };
            auto after_first = [&]() {   // both halves consumed by both CTAs before any store
                if constexpr (S > 1) {
                    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
                    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
                }
            };
            auto none = [] {};
            // NC = 2^13: the windowed tail (WL 2: the last head pass ends with
            // __syncwarp); the lanes still store consecutive 16-byte pairs
            constexpr int WLS = LGC == 13 ? 2 : 1;
            fwd_ntt_head<LGC, WLS>(buf, load, tw, nq, after_first, none);
            u64 *o = p + (size_t)s * NC;
#pragma unroll
            for (int u = 0; u < kE / 2; ++u) {
                const int g = tail_pair<LGC, WLS == 2>(u);
                const double2 w = tw[NC / 2 + g];
                double x0, x1;
                fwd_ntt_tail<LGC, WLS == 2>(buf, u, w.x, w.y, nq, x0, x1);
                ulonglong2 v;
                v.x = to_canonical_u64(reduce(x0, qinv, nq), q);
                v.y = to_canonical_u64(reduce(x1, qinv, nq), q);
                __stcs(reinterpret_cast<ulonglong2 *>(o + 2 * g), v);
            }
        } else {
            // the first inverse pass groups 16 consecutive residues per thread (lanes 128 B
            // apart): stage the polynomial through shared memory with coalesced loads
            // instead (32x fewer L1 wavefronts than loading that pattern from global)
            {
                constexpr int NT = NC / kE;
#pragma unroll
                for (int e = 0; e < kE; ++e) {
                    const int pos = tid + e * NT;
                    buf[pad(pos)] = centered(__ldcs(reinterpret_cast<const unsigned long long *>(p + pos)));
                }
                __syncthreads();
            }
            auto load = [&](int pos) -> double { return buf[pad(pos)]; };
            // the last pass scales and stores straight to global memory (its lanes hold
            // consecutive positions: coalesced)
            auto sink = [&](int pos, double x) {
                const double2 c = DIR == 2 ? post[pos] : ni;
                const double y = reduce(mul_tw(x, c.x, c.y, nq), qinv, nq);
                __stcs(reinterpret_cast<unsigned long long *>(p + pos), (unsigned long long)to_canonical_u64(y, q));
            };
            if constexpr (DIR == 2) inv_dit_f64<LGC, 0, false>(buf, load, tw, nq, sink);
            else inv_ntt_f64<LGC, 0, false>(buf, load, tw, nq, sink);
        }
        __syncthreads();   // buf is rewritten by the next polynomial
    }
}

template <int LGC, int S, int DIR>
static cudaError_t std_f64_launch(const ephdc_ntt_plan *pl, u64 *polys, u32 batch, cudaStream_t st) {
    constexpr bool INV = DIR != 0;
    const size_t smem = sizeof(double2) * ((size_t)1 << LGC) + sizeof(double) * (size_t)padded_len(1 << LGC);
    auto kern = k_ntt_std_f64<LGC, S, DIR>;
    cudaError_t e = smem_attr(kern, smem);
    if (e != cudaSuccess) return e;
    StdF64Args a;
    a.L = pl->L;
    a.tw = INV ? pl->itw_f64 : pl->tw_f64;
    a.post = pl->post_f64;
    // workers per prime: fill the GPU (CTAs per SM from shared memory), at most batch
    const int per_sm = std::max<int>(1, (int)((228u << 10) / (smem + 1024)));
    const uint64_t ctas = 148ull * per_sm;
    const uint64_t W = std::max<uint64_t>(1, std::min<uint64_t>(batch, ctas / ((uint64_t)pl->L * S)));
    const uint64_t grid = W * pl->L * S;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((1 << LGC) / kE);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, polys, batch, a);
    return counted(e == cudaSuccess ? cudaGetLastError() : e);
}

// FP64 standalone NTT if the plan allows it for this direction and size; returns
// cudaErrorNotSupported otherwise (the caller then runs the integer kernels).
cudaError_t launch_ntt_batch_f64(const ephdc_ntt_plan *pl, uint64_t *d_polys, uint32_t batch, bool inverse,
                                 cudaStream_t st) {
    if (inverse ? !pl->inv_f64 : !pl->fwd_f64) return cudaErrorNotSupported;
    if (batch == 0) return cudaSuccess;
    if (!inverse) {
        switch (pl->log2N) {
            case 10: return std_f64_launch<10, 1, 0>(pl, d_polys, batch, st);
            case 11: return std_f64_launch<11, 1, 0>(pl, d_polys, batch, st);
            case 12: return std_f64_launch<12, 1, 0>(pl, d_polys, batch, st);
            case 13: return std_f64_launch<13, 1, 0>(pl, d_polys, batch, st);
            case 14: return std_f64_launch<13, 2, 0>(pl, d_polys, batch, st);
        }
    } else if (pl->inv_dit) {
        switch (pl->log2N) {
            case 10: return std_f64_launch<10, 1, 2>(pl, d_polys, batch, st);
            case 11: return std_f64_launch<11, 1, 2>(pl, d_polys, batch, st);
            case 12: return std_f64_launch<12, 1, 2>(pl, d_polys, batch, st);
            case 13: return std_f64_launch<13, 1, 2>(pl, d_polys, batch, st);
        }
    } else {
        switch (pl->log2N) {
            case 10: return std_f64_launch<10, 1, 1>(pl, d_polys, batch, st);
            case 11: return std_f64_launch<11, 1, 1>(pl, d_polys, batch, st);
            case 12: return std_f64_launch<12, 1, 1>(pl, d_polys, batch, st);
            case 13: return std_f64_launch<13, 1, 1>(pl, d_polys, batch, st);
        }
    }
    return cudaErrorNotSupported;
}

// Bounds of the standalone FP64 transforms: canonical inputs are
// centered (|x| <= q/2); forward CT stages and the inverse's CT DIT stages add
// <= (1/2 + B 2^-54) q each, inverse GS stages double the bound; every mul_tw input --
// for the inverse also the final scaling product -- must stay below 2^51.  The
// inverse uses GS where its bound allows (small primes: no per-coefficient scaling
// table to stream, measured faster), else DIT (profiles/r01/c5/ab_inv_dit.txt).
void plan_ntt_f64(const std::vector<uint64_t> &q, uint32_t log2N, bool *fwd, bool *inv, bool *inv_dit) {
    const double L51 = 0.98 * 2251799813685248.0, e54 = 1.0 / 18014398509481984.0;
    *fwd = log2N >= 10 && log2N <= 14;
    bool gs = log2N >= 10 && log2N <= 13, dit = gs;
    for (uint64_t qj : q) {
        if (qj >= (1ull << 50)) {
            *fwd = *inv = *inv_dit = false;
            return;
        }
        const double Q = (double)qj;
        double B = Q / 2 + 1;
        for (uint32_t st = 0; st < log2N; ++st) {
            if (B >= L51) *fwd = dit = false;
            B += (0.5 + B * e54) * Q + 2.0;
        }
        if (B >= L51) dit = false;
        double Bi = Q / 2 + 1;
        for (uint32_t st = 0; st < log2N; ++st) {
            if (2 * Bi >= L51) gs = false;
            Bi *= 2;
        }
    }
    *inv = gs || dit;
    *inv_dit = !gs && dit;
}

// model residues u64 -> exact doubles, in place (setup, once per model)
__global__ void k_u64_to_f64(u64 *__restrict__ d, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = (u64)__double_as_longlong(from_u64(d[i]));
}

cudaError_t launch_u64_to_f64(uint64_t *d, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_u64_to_f64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d, n);
    return counted(cudaGetLastError());
}

// model residue of (dim d, prime j) times fac[d / g][j] mod q_j (ephdc_model_scale):
// FP64 path (exact doubles, fac plain) or integer path (u64, fac in Montgomery form)
template <bool F64>
__global__ void k_model_scale(u64 *__restrict__ m, size_t n, u32 L, u32 N, u32 g, const u64 *__restrict__ fac,
                              PrimeSet ps) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t dj = i / ((size_t)2 * N);           // (d, j) of [D][L][2][N]
    const u32 j = (u32)(dj % L), d = (u32)(dj / L);
    const u64 q = ps.q[j], f = fac[(size_t)(d / g) * L + j];
    if constexpr (F64) {
        const double qd = (double)q;
        double r = mul_rt(__longlong_as_double((long long)m[i]), (double)f, 1.0 / qd, -qd);
        r = reduce(r, 1.0 / qd, -qd);
        if (r < 0) r = __dadd_rn(r, qd);
        m[i] = (u64)__double_as_longlong(r);
    } else {
        m[i] = mont_mul(m[i], f, q, ps.qinv[j]);
    }
}

cudaError_t launch_model_scale(const ephdc_ctx *c, uint64_t *d_model, uint32_t D, uint32_t g, const uint64_t *d_fac,
                               cudaStream_t st) {
    const size_t n = (size_t)D * c->L * 2 * c->N;
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (c->f64.enabled) k_model_scale<true><<<blocks, 256, 0, st>>>(d_model, n, c->L, c->N, g, d_fac, c->ps);
    else k_model_scale<false><<<blocks, 256, 0, st>>>(d_model, n, c->L, c->N, g, d_fac, c->ps);
    return counted(cudaGetLastError());
}

// Scores message: block (b, c, j) of N residues bit-packed at bits[j] bits; thread =
// 8 consecutive residues = bits[j] bytes.
__global__ void k_pack_bits(const u64 *__restrict__ ct, u32 nblocks, u32 L, u32 N, MsgLayout m,
                            uint8_t *__restrict__ msg) {
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const u32 per = N / 8;
    if (gid >= (size_t)nblocks * per) return;
    const u32 blk = (u32)(gid / per), g = (u32)(gid % per), j = blk % L, bc = blk / L, bj = m.bits[j];
    const u64 *x = ct + (size_t)blk * N + 8 * g;
    uint8_t *o = msg + (size_t)bc * m.group_bytes + m.prefix[j] + (size_t)g * bj;
    unsigned __int128 acc = 0;
    int have = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        acc |= (unsigned __int128)x[r] << have;
        have += (int)bj;
        while (have >= 8) {
            *o++ = (uint8_t)(acc & 0xFF);
            acc >>= 8;
            have -= 8;
        }
    }
}

MsgLayout msg_layout(const ephdc_ctx *c) {
    MsgLayout m{};
    u64 off = 0;
    for (u32 j = 0; j < c->L; ++j) {
        m.bits[j] = c->qbits[j];
        m.prefix[j] = off;
        off += (u64)c->N * c->qbits[j] / 8;
    }
    m.group_bytes = off;
    return m;
}

cudaError_t launch_pack_bits(const ephdc_ctx *c, const uint64_t *d_ct, uint32_t nb, uint8_t *d_msg, cudaStream_t st) {
    const u32 nblocks = nb * 2 * c->L;
    const size_t threads = (size_t)nblocks * (c->N / 8);
    if (threads == 0) return cudaSuccess;
    k_pack_bits<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(d_ct, nblocks, c->L, c->N, msg_layout(c), d_msg);
    return counted(cudaGetLastError());
}

// out[b][c][j][i] <- out mod q_j
__global__ void k_reduce_out(u64 *__restrict__ out, u32 L, u32 N, PrimeSet ps, size_t n_total) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_total) return;
    const u32 j = (u32)((i / N) % L);
    out[i] %= ps.q[j];
}

// ------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------
size_t ntt_f64_smem_bytes(uint32_t lgc) {
    const size_t nc = (size_t)1 << lgc;
    return sizeof(double2) * nc + sizeof(double) * (size_t)ephdc_f64::padded_len((int)nc);
}

static F64MacArgs f64_args(const ephdc_ctx *c) {
    F64MacArgs a{};
    a.half_t = (u32)((c->t - 1) / 2);
    a.two52_plus_t = 4503599627370496.0 + (double)c->t;
    a.L = c->L;
    a.D = c->p.D_live;
    a.red_every = c->f64.red_every;
    a.tw = c->dev.tw_f64;
    return a;
}

template <class K> static cudaError_t smem_attr(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int LGC, int S>
static cudaError_t mac_f64_launch(const ephdc_ctx *c, const ephdc_plan &plan, const u32 *M, uint32_t nb,
                                  const double *model, u64 *out, cudaStream_t st, const uint32_t *dlim) {
    // pad shared memory so that no more CTAs share an SM than its TMEM holds
    const size_t smem = std::max<size_t>(mac_f64_smem<LGC, S>(), (200u << 10) / f64_ctas_per_sm<LGC>());
    // Plan (profiles/r01/ab_wl2.txt): at NC = 2^13 the windowed tail (WL = 2: the last
    // head pass ends with __syncwarp, 2 CTA barriers per dim) without the explicit L2
    // prefetch of the model slice is fastest (c4 -5.5%, c3 -1.6%); smaller transforms
    // keep WL = 1 with the prefetch (c2: WL = 2 is 20% slower).
    // ephdc_plan.flags (workspace plan overrides, tests/profiling): bits 1-2 = 1/2/3 force
    // WL = 0/2/1; bit 0 forces the prefetch off, bit 4 on; bit 3 = 32 elements per
    // thread (LGC = 13 only; WL = 2 or 1); bit 5 = the one-team kernel at LGC = 13.
    u32 env = plan.flags;
    u32 wl = LGC >= 13 ? 2u : 1u;
    bool prefetch = LGC < 13;
    switch ((env >> 1) & 3u) {
        case 1: wl = 0; break;
        case 2: wl = 2; break;
        case 3: wl = 1; break;
        default: break;
    }
    if (env & 1u) prefetch = false;
    if (env & 16u) prefetch = true;
    const bool e32 = LGC == 13 && (env & 8u) != 0;
    // NC = 2^13, S = 1 (c3): the two-group kernel unless the plan asks for a one-team
    // variant (flags bits 1-3, or bit 5 = the one-team kernel with the default plan).
    // At S = 2 (c4) the one-team kernel stays the default: two groups measured 259.6 vs
    // 246.0 ms per c4 step (c3: 19.45 vs 19.95 ms; profiles/r02/ab/bench_*).  Plan bit 6
    // selects the two-group kernel at S = 2 (A/B).
    if constexpr (LGC == 13) {
        if (S == 2 && !(env & 64u)) env |= 32u;
        if (!dlim && (env & (32u | 14u)) == 0) {
            auto k2 = k_ntt_mac_f64_2g<S>;
            const size_t smem2 = mac_f64_2g_smem<S>();
            cudaError_t e2 = smem_attr(k2, smem2);
            if (e2 != cudaSuccess) return e2;
            F64MacArgs a = f64_args(c);
            a.nb = nb;
            f64_grid(c, nb, &a.bg, &a.chunks, &a.G);
            a.flags = 1u;
            if (plan.bg) a.bg = std::max<u32>(1, std::min<u32>(nb, plan.bg));
            if (plan.G) {
                const u32 gmin = (c->p.D_live + 1023) / 1024;
                a.G = std::max<u32>(gmin, std::min<u32>(c->p.D_live, plan.G));
                a.chunks = (c->p.D_live + a.G - 1) / a.G;
            }
            const uint64_t groups = (nb + a.bg - 1) / a.bg;
            const uint64_t grid = groups * a.chunks * a.bg * c->L * S;
            if (grid > 0x7fffffffull) return cudaErrorInvalidConfiguration;
            k2<<<(unsigned)grid, 512, smem2, st>>>(M, model, out, a);
            return counted(cudaGetLastError());
        }
    }
    auto kern = dlim ? (wl == 2 ? k_ntt_mac_f64<LGC, S, 2, kE, true> : k_ntt_mac_f64<LGC, S, 1, kE, true>)
                : e32 ? (wl == 2 ? k_ntt_mac_f64<LGC, S, 2, 32> : k_ntt_mac_f64<LGC, S, 1, 32>)
                      : wl == 0 ? k_ntt_mac_f64<LGC, S, 0, kE> : wl == 2 ? k_ntt_mac_f64<LGC, S, 2, kE> : k_ntt_mac_f64<LGC, S, 1, kE>;
    cudaError_t e = smem_attr(kern, smem);
    if (e != cudaSuccess) return e;
    F64MacArgs a = f64_args(c);
    a.nb = nb;
    f64_grid(c, nb, &a.bg, &a.chunks, &a.G);
    a.flags = prefetch ? 0u : 1u;  // bit 0: no explicit L2 prefetch of the model slice
    a.dlim = dlim;
    // plan overrides (ephdc_plan bg / G; tests and profiling only)
    if (plan.bg) a.bg = std::max<u32>(1, std::min<u32>(nb, plan.bg));
    if (plan.G) {  // <= 1024 chunks: the 64-bit fold of f64_grid
        const u32 gmin = (c->p.D_live + 1023) / 1024;
        a.G = std::max<u32>(gmin, std::min<u32>(c->p.D_live, plan.G));
        a.chunks = (c->p.D_live + a.G - 1) / a.G;
    }
    const uint64_t groups = (nb + a.bg - 1) / a.bg;
    const uint64_t grid = groups * a.chunks * a.bg * c->L * S;
    if (grid > 0x7fffffffull) return cudaErrorInvalidConfiguration;
    kern<<<(unsigned)grid, (1 << LGC) / (e32 && !dlim ? 32 : kE), smem, st>>>(M, model, out, a);
    return counted(cudaGetLastError());
}


cudaError_t launch_ntt_mac_f64(const ephdc_ctx *c, const ephdc_plan &plan, const uint32_t *d_M, uint32_t nb,
                               const double *d_model, uint64_t *d_out, cudaStream_t st, const uint32_t *d_dlim) {
    if (nb == 0) return cudaSuccess;
    switch (c->p.log2N) {
        case 10: return mac_f64_launch<10, 1>(c, plan, d_M, nb, d_model, d_out, st, d_dlim);
        case 11: return mac_f64_launch<11, 1>(c, plan, d_M, nb, d_model, d_out, st, d_dlim);
        case 12: return mac_f64_launch<12, 1>(c, plan, d_M, nb, d_model, d_out, st, d_dlim);
        case 13: return mac_f64_launch<13, 1>(c, plan, d_M, nb, d_model, d_out, st, d_dlim);
        case 14: return mac_f64_launch<13, 2>(c, plan, d_M, nb, d_model, d_out, st, d_dlim);
    }
    return cudaErrorInvalidValue;
}

template <int LGC, int S>
static cudaError_t pt_f64_launch(const ephdc_ctx *c, const u32 *M, uint32_t nd, u64 *pt, cudaStream_t st) {
    const size_t smem = ntt_f64_smem_bytes(LGC);
    auto kern = k_pt_ntt_f64<LGC, S>;
    cudaError_t e = smem_attr(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<nd * c->L * S, (1 << LGC) / kE, smem, st>>>(M, pt, f64_args(c));
    return counted(cudaGetLastError());
}


cudaError_t launch_plaintext_ntt_f64(const ephdc_ctx *c, const uint32_t *d_M, uint32_t nd, uint64_t *d_pt,
                                     cudaStream_t st) {
    if (nd == 0) return cudaSuccess;
    switch (c->p.log2N) {
        case 10: return pt_f64_launch<10, 1>(c, d_M, nd, d_pt, st);
        case 11: return pt_f64_launch<11, 1>(c, d_M, nd, d_pt, st);
        case 12: return pt_f64_launch<12, 1>(c, d_M, nd, d_pt, st);
        case 13: return pt_f64_launch<13, 1>(c, d_M, nd, d_pt, st);
        case 14: return pt_f64_launch<13, 2>(c, d_M, nd, d_pt, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce_out(const ephdc_ctx *c, uint64_t *d_out, uint32_t nb, cudaStream_t st) {
    const size_t n = (size_t)nb * 2 * c->L * c->N;
    if (n == 0) return cudaSuccess;
    k_reduce_out<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_out, c->L, c->N, c->ps, n);
    return counted(cudaGetLastError());
}

int ntt_mac_f64_occupancy(uint32_t log2N) {
    switch (log2N > 13 ? 13 : log2N) {
        case 13: return f64_ctas_per_sm<13>();
        case 12: return f64_ctas_per_sm<12>();
        case 11: return f64_ctas_per_sm<11>();
        default: return f64_ctas_per_sm<10>();
    }
}

// Value bounds of the FP64 path: every input of
// mul_tw below 2^51, every MAC operand |a b / q| below 2^51, accumulators below 2^53.
bool plan_f64(const std::vector<uint64_t> &q, uint64_t t, uint32_t log2N, F64Plan *plan) {
    *plan = F64Plan{};
    const double L51 = 0.98 * 2251799813685248.0, L53 = 0.98 * 9007199254740992.0, e54 = 1.0 / 18014398509481984.0;
    const uint32_t S = log2N >= 14 ? 2 : 1, lgc = log2N - (S - 1);
    u32 red_every = 1u << 20;
    for (uint64_t qj : q) {
        if (qj >= (1ull << 50)) return false;
        const double Q = (double)qj;
        auto rtw = [&](double X) { return (0.5 + X * e54) * Q + 2.0; };  // |mul_tw| bound
        double B = (double)((t - 1) / 2);                                // centered lift
        for (uint32_t st = 0; st < lgc + (S - 1); ++st) {                // every CT stage
            if (B >= L51) return false;
            B += rtw(B);
        }
        if (B >= L51) return false;                                      // MAC operand
        const double rmac = (0.5 + 2.0 * B * e54 * 2.0) * Q + 2.0;       // |mul_rt| bound
        const double n = std::floor((L53 - (Q / 2 + 2.0)) / rmac);
        if (n < 1) return false;
        red_every = std::min<u32>(red_every, (u32)std::min(n, 1048576.0));
    }
    plan->enabled = true;
    plan->red_every = red_every;
    return true;
}

// Grid of one fused launch over nb batches (profiles/r01/l2sched; ab_grid.txt).
//  * Block order batch-fastest, all batches in one group (bg = nb, at most one wave):
//    a wave covers the nb batches x W/nb (prime, slice) pairs of one dim chunk, so each
//    model tile is fetched about once per chunk by nb concurrent CTAs.  Measured at c4
//    (one launch): 115-122 GB of DRAM reads with bg = 29, 181 GB with 15, 636 GB with
//    the earlier prime/slice-fastest order (bg = 8, 589-dim chunks), ~10x the
//    algorithmic 62 GB.
//  * Dims per chunk G <= kMaxG, so the CTAs that share a tile start together and stay
//    within the L2 residency window over a chunk; among those chunkings the one
//    minimising waves x (G + 2) (two dims' worth of per-CTA setup and fold).
//  * At most 1024 chunks: the 64-bit atomic fold adds <= chunks values < q < 2^50.
void f64_grid(const ephdc_ctx *c, uint32_t nb, uint32_t *bg, uint32_t *chunks, uint32_t *G) {
    constexpr uint32_t kMaxG = 320;
    const uint32_t S = c->p.log2N >= 14 ? 2 : 1;
    const uint64_t W = 148ull * ntt_mac_f64_occupancy(c->p.log2N);
    const uint64_t LS = (uint64_t)c->L * S;
    const uint32_t D = c->p.D_live;
    *bg = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(nb, W));
    const uint64_t real = (uint64_t)nb * LS;
    const uint32_t cmax = std::min<uint32_t>(D, 1024);
    const uint32_t cmin = std::min<uint32_t>(cmax, (D + kMaxG - 1) / kMaxG);
    uint64_t best = ~0ull;
    uint32_t best_c = cmin;
    for (uint32_t ch = cmin; ch <= cmax; ++ch) {
        const uint64_t g = (D + ch - 1) / ch;
        const uint64_t waves = (real * ch + W - 1) / W;
        const uint64_t cost = waves * (g + 2);
        if (cost < best) {
            best = cost;
            best_c = ch;
        }
    }
    *G = (D + best_c - 1) / best_c;
    *chunks = (D + *G - 1) / *G;
}

}  // namespace ephdc
