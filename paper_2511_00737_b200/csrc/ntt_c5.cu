// ntt_c5.cu -- the standalone negacyclic NTT of the c5 microbench (BASELINE.json
// configs[4]) on B200, for primes q < 2^50, exact modular arithmetic on the
// FP64 pipe (modf64.cuh: 8 FP64 operations per butterfly).
//
// In place on [batch][L][N] canonical u64.  N = 2^12, 2^13: one CTA per polynomial;
// N = 2^14, 2^15, 2^16: a cluster of C = N / 2^13 CTAs, each owning one 2^13-element
// block, exchanging the cross-block levels through distributed shared memory -- one
// pass over HBM at every size.  Per CTA:
//   * persistent over a contiguous range of (prime, polynomial) items, prime-major:
//     the twiddles of a prime are loaded once -- the low levels (broadcast /
//     warp-uniform / lane-consecutive reads) in shared memory, each thread's own
//     pass-3 and last-level twiddles (up to 31 pairs) in TENSOR MEMORY, which is idle in
//     a kernel without MMAs;
//   * polynomials arrive by TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B) into buffers
//     that rotate while earlier polynomials are transformed; the pass plans are chosen
//     so that every shared-memory access is conflict-free in the swizzled layout
//     (forward: levels 4+4+R3+2, the last two on four consecutive elements read as
//     16-byte pairs; inverse: 2+3+4+4);
//   * forward: pass 1 (levels 0-3, all-to-all) -> one CTA barrier -> passes 2, 3 and the
//     last two levels inside each warp's 512-element window (__syncwarp) -> 16-byte
//     stores straight from registers;
//   * inverse (Cooley-Tukey DIT on the bit-reversed input): passes A-C warp-local ->
//     barrier -> pass D, whose last level is fused with the scaling by N^-1 psi^-j
//     (three products per pair from per-thread TMEM pairs: no scaling table streamed).
// Clusters: forward -- each CTA loads the 1/C slice of every block it needs, computes
// the log2(C) cross-block levels for its slice and writes each result into the owning
// CTA's shared memory (st.shared::cluster), one cluster barrier, then the 13 local
// levels; inverse -- the 13 local levels (the scaling by N^-1 psi^-r of the local index
// fused into level 12: it commutes with the cross levels), one cluster barrier, then
// each CTA reads its slice of every block (ld.shared::cluster), applies the cross
// levels and the per-block constant psi^-(2^13 k), and stores.
// DESIGN.md 5.2 "c5 standalone NTT".
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "async_copy.cuh"
#include "internal.h"
#include "modf64.cuh"
#include "tma_host.h"
#include "tmem_x.cuh"

namespace ephdc {
namespace c5 {

using namespace ephdc_f64;
using ephdc_tmem::pair_at;
using ephdc_tmem::put_pair;

constexpr int kE = 16;          // elements per thread per pass
constexpr int kNBuf = 3;        // rotating buffers
constexpr int kBoxRows = 256;   // TMA box: 256 rows x 16 u64 (32 KB)

// SWIZZLE_128B: element e (8 bytes) of a 1024-byte-aligned buffer sits at
// e ^ (((e >> 4) & 7) << 1).  The map is linear over XOR, so for index parts with
// disjoint bits sw(a + b) = sw(a) ^ sw(b): every pass computes sw(base) once and XORs
// compile-time constants.
__host__ __device__ constexpr int sw(int e) { return e ^ (((e >> 4) & 7) << 1); }
template <int LGC> constexpr int ctas_per_sm() { return LGC <= 12 ? 2 : 1; }
template <int LGC> constexpr uint32_t tmem_cols() { return 128u * (uint32_t)(((1 << LGC) / kE / 32 + 3) / 4); }



EPHDC_D void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            ephdc_async::smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(ephdc_async::smem_u32(bar))
        : "memory");
}
EPHDC_D void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
EPHDC_D void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
EPHDC_D uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
EPHDC_D uint32_t map_rank(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(ephdc_async::smem_u32(p)), "r"(rank));
    return r;
}
EPHDC_D void st_cluster(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
EPHDC_D double ld_cluster(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
EPHDC_D void st_cs_v2(u64 *p, u64 a, u64 b) {
    asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// CT sub-stages SUB0 .. SUB1-1 of a register group x[k] of R = 2^R_LOG elements (sub-stage
// sub pairs (k, k + R/2^(sub+1)) inside its v-th sub-block); twiddle tw(sub, v).
template <int R_LOG, int SUB0, int SUB1, class Tw>
EPHDC_D void ct_stages(double (&x)[1 << R_LOG], const Tw &tw, double nq) {
    constexpr int R = 1 << R_LOG;
#pragma unroll
    for (int sub = SUB0; sub < SUB1; ++sub) {
        const int h = R >> (sub + 1);
#pragma unroll
        for (int v = 0; v < (1 << sub); ++v) {
            const double2 w = tw(sub, v);
#pragma unroll
            for (int kk = 0; kk < h; ++kk) ct_bfly(x[v * 2 * h + kk], x[v * 2 * h + kk + h], w.x, w.y, nq);
        }
    }
}
// DIT sub-stages: sub-stage sub pairs (k, k + 2^sub); tw(sub, kk) for block position kk.
template <int R_LOG, int SUB0, int SUB1, class Tw>
EPHDC_D void dit_stages(double (&x)[1 << R_LOG], const Tw &tw, double nq) {
    constexpr int R = 1 << R_LOG;
#pragma unroll
    for (int sub = SUB0; sub < SUB1; ++sub) {
        const int hs = 1 << sub;
#pragma unroll
        for (int kk = 0; kk < hs; ++kk) {
            const double2 w = tw(sub, kk);
#pragma unroll
            for (int v = 0; v < R / (2 * hs); ++v) ct_bfly(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], w.x, w.y, nq);
        }
    }
}

// ---------------------------------------------------------------------------------
// Per-CTA frame: 1024-byte-aligned buffers, shared twiddles, the TMA ring, TMEM columns.
// ---------------------------------------------------------------------------------
struct Ctx {
    double *bufs;      // [n_bufs][NC]
    double2 *tws;      // shared twiddles
    uint32_t tbase;    // this thread's TMEM columns
    int tid, warp, lane;
    double q, nq, qinv;
    u64 qi;            // q as an integer
    EPHDC_D void set_prime(double2 qq) {   // (q, fl(1/q)) = entry 0 of a twiddle table
        q = qq.x;
        nq = -qq.x;
        qinv = qq.y;
        qi = (u64)q;
    }
};

// Input centering and output canonicalisation as 64-bit integer selects on the idle
// integer pipe; one FP64 operation converts each way (2 + 2 fewer FP64 operations per
// element than FP64 compare/select forms; r14 A/B: +1.5% at 2^14, equal at 2^13).
// kRound = 1.5 * 2^52 has the bit pattern 0x4338000000000000 and a unit last place, so
// for an integer |c| < 2^51 the pattern 0x4338000000000000 + c IS the double kRound + c.
constexpr long long kRoundBits = 0x4338000000000000LL;
EPHDC_D double centered(u64 v, const Ctx &f) {   // [0, q) -> (-q/2, q/2]
    const long long c = (long long)(v > (f.qi >> 1) ? v - f.qi : v);
    return __dsub_rn(__longlong_as_double(kRoundBits + c), kRound);
}
EPHDC_D u64 out_u64(double x, const Ctx &f) {   // |x| < 2^51 -> [0, q)
    const double k = __dadd_rn(__fma_rn(x, f.qinv, kRound), -kRound);
    const long long r = __double_as_longlong(__fma_rn(k, f.nq, __dadd_rn(x, kRound))) - kRoundBits;   // x - k q
    return (u64)r + (r < 0 ? f.qi : 0ull);
}

template <int LGC> EPHDC_D void frame_init(Ctx &f, unsigned char *smem_raw, int n_bufs, uint64_t *mbar,
                                           uint32_t *tmem_slot) {
    constexpr int NC = 1 << LGC;
    f.tid = threadIdx.x;
    f.warp = f.tid >> 5;
    f.lane = f.tid & 31;
    f.bufs = reinterpret_cast<double *>(smem_raw + ((1024u - (ephdc_async::smem_u32(smem_raw) & 1023u)) & 1023u));
    f.tws = reinterpret_cast<double2 *>(f.bufs + (size_t)n_bufs * NC);
    if (f.tid == 0)
        for (int b = 0; b < kNBuf; ++b) ephdc_async::mbar_init(&mbar[b], 1);
    if (f.warp == 0) ephdc_tmem::alloc(tmem_slot, tmem_cols<LGC>());
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    f.tbase = *tmem_slot + ((uint32_t)(32 * (f.warp & 3)) << 16) + (uint32_t)(f.warp >> 2) * 128u;
}

template <int LGC> EPHDC_D void frame_exit(const Ctx &f, uint32_t tmem_slot) {
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (f.warp == 0) ephdc_tmem::dealloc(tmem_slot, tmem_cols<LGC>());
}

EPHDC_D u64 *poly_ptr(const C5Args &a, u32 w) {
    const u32 j = w / a.batch, b = w - j * a.batch;
    return a.polys + (((size_t)b * a.L + j) << a.log2N);
}
EPHDC_D int poly_row(const C5Args &a, u32 w) {   // first 128-byte row of item w in the tensor map
    const u32 j = w / a.batch, b = w - j * a.batch;
    return (int)((((size_t)b * a.L + j) << a.log2N) >> 4);
}

// =================================================================================
// Forward pieces.  Level lv of a CTA's NC-point block has 2^lv blocks of half-size
// NC >> (lv+1); its twiddle for block B is psi_rev[C m + s m + B], m = 2^lv (C CTAs
// per polynomial, this CTA's block s; C = 1: psi_rev[m + B]).  Passes: 1 = levels 0-3,
// 2 = 4-7, 3 = 8 .. LGC-3 (R3 levels: groups of 2^R3 elements 4 apart), tail =
// LGC-2, LGC-1 (four consecutive elements).
// =================================================================================
template <int LGC> struct Fwd {
    static constexpr int NC = 1 << LGC, NT = NC / kE;
    static constexpr int R3 = LGC - 10, G3 = kE >> R3;
    static constexpr int TL2 = NC >> 8, NB8 = NC >> 8;
    static constexpr uint32_t kP3Cols = R3 == 3 ? 32u : 16u;   // TMEM columns per pass-3 group

    // pass-3 groups: a warp's groups cover its 512-element window and every half-warp
    // touches 16 distinct bank pairs (bank model)
    static EPHDC_D int p3_blk(const Ctx &f, int u) {
        return R3 == 3 ? 16 * f.warp + (f.lane >> 2) + 8 * u : 32 * f.warp + ((f.lane >> 1) & 15) + 16 * (u >> 1);
    }
    static EPHDC_D int p3_off(const Ctx &f, int u) { return R3 == 3 ? (f.lane & 3) : ((f.lane & 1) | ((u & 1) << 1)); }

    // twiddles of one prime: levels 0-7 -> shared (pass layout), pass 3 + tail -> TMEM
    template <class G> static EPHDC_D void load_twiddles(const Ctx &f, const G &gtw) {
        for (int p = f.tid; p < 256; p += NT) {   // slot (m0 << sub) + v m0 + B
            if (p == 0) continue;
            const int lm = 31 - __clz(p), m = 1 << lm;
            const int start = lm & ~3, sub = lm - start, m0 = 1 << start;
            const int r = p - m, v = r / m0, B = r % m0;
            f.tws[p] = gtw(m, (B << sub) + v);
        }
        uint32_t r[16];
#pragma unroll
        for (int u = 0; u < G3; ++u) {   // pass 3: 2^R3 - 1 pairs (sub, v) in order
#pragma unroll
            for (int h = 0; h < (int)kP3Cols / 16; ++h) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int idx = 4 * h + k;   // pair index: sub = log2(idx + 1)
                    if (idx < (1 << R3) - 1) {
                        const int sub = 31 - __clz(idx + 1), v = idx + 1 - (1 << sub);
                        put_pair(&r[4 * k], gtw(256 << sub, (p3_blk(f, u) << sub) + v));
                    } else {
                        put_pair(&r[4 * k], make_double2(0.0, 0.0));
                    }
                }
                ephdc_tmem::stx<16>(f.tbase + kP3Cols * u + 16u * h, r);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {   // tail group g4: levels LGC-2 (block g4), LGC-1 (2 g4, 2 g4 + 1)
            const int g4 = 128 * f.warp + f.lane + 32 * u;
            put_pair(&r[0], gtw(NC / 4, g4));
            put_pair(&r[4], gtw(NC / 2, 2 * g4));
            put_pair(&r[8], gtw(NC / 2, 2 * g4 + 1));
            put_pair(&r[12], make_double2(0.0, 0.0));
            ephdc_tmem::stx<16>(f.tbase + 64u + 16u * u, r);
        }
        ephdc_tmem::wait_st();
    }

    // pass 1 on x (elements tid + k NT), levels 0-3
    static EPHDC_D void pass1(const Ctx &f, double *C, double (&x)[16]) {
        ct_stages<4, 0, 4>(x, [&](int sub, int v) { return f.tws[(1 << sub) + v]; }, f.nq);
        const int st = sw(f.tid);
#pragma unroll
        for (int k = 0; k < 16; ++k) C[st ^ sw(k * NT)] = x[k];
    }

    static EPHDC_D void pass2(const Ctx &f, double *C) {
        const int blk = f.tid / TL2, off2 = f.tid % TL2, sb = sw(blk * (NC / 16) + off2);
        double x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = C[sb ^ sw(k * TL2)];
        ct_stages<4, 0, 4>(x, [&](int sub, int v) { return f.tws[(16 << sub) + v * 16 + blk]; }, f.nq);
#pragma unroll
        for (int k = 0; k < 16; ++k) C[sb ^ sw(k * TL2)] = x[k];
    }

    // (each group's TMEM twiddle load is issued before its shared-memory loads, so the
    // two latencies overlap)
    static EPHDC_D void pass3(const Ctx &f, double *C) {
#pragma unroll
        for (int u = 0; u < G3; ++u) {
            const int sb = sw(p3_blk(f, u) * NB8 + p3_off(f, u));
            uint32_t rr[kP3Cols];
            ephdc_tmem::ldx<16>(f.tbase + kP3Cols * u, *reinterpret_cast<uint32_t(*)[16]>(&rr[0]));
            if constexpr (R3 == 3)
                ephdc_tmem::ldx<16>(f.tbase + kP3Cols * u + 16u, *reinterpret_cast<uint32_t(*)[16]>(&rr[16]));
            double x[1 << R3];
#pragma unroll
            for (int k = 0; k < (1 << R3); ++k) x[k] = C[sb ^ sw(4 * k)];
            ephdc_tmem::waitx<kP3Cols>(rr);
            ct_stages<R3, 0, R3>(x, [&](int sub, int v) { return pair_at(rr, (1 << sub) - 1 + v); }, f.nq);
#pragma unroll
            for (int k = 0; k < (1 << R3); ++k) C[sb ^ sw(4 * k)] = x[k];
        }
    }

    // levels LGC-2, LGC-1 on four consecutive elements, reduction to [0, q), 16-byte stores
    static EPHDC_D void tail(const Ctx &f, const double *C, u64 *o) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int g4 = 128 * f.warp + f.lane + 32 * u;
            uint32_t rr[16];
            ephdc_tmem::ldx<16>(f.tbase + 64u + 16u * u, rr);
            const int sg = sw(4 * g4);
            const double2 xa = *reinterpret_cast<const double2 *>(C + sg);
            const double2 xb = *reinterpret_cast<const double2 *>(C + (sg ^ 2));
            ephdc_tmem::waitx<16>(rr);
            double x0 = xa.x, x1 = xa.y, x2 = xb.x, x3 = xb.y;
            const double2 t0 = pair_at(rr, 0), t1 = pair_at(rr, 1), t2 = pair_at(rr, 2);
            ct_bfly(x0, x2, t0.x, t0.y, f.nq);
            ct_bfly(x1, x3, t0.x, t0.y, f.nq);
            ct_bfly(x0, x1, t1.x, t1.y, f.nq);
            ct_bfly(x2, x3, t2.x, t2.y, f.nq);
            st_cs_v2(o + 4 * g4, out_u64(x0, f), out_u64(x1, f));
            st_cs_v2(o + 4 * g4 + 2, out_u64(x2, f), out_u64(x3, f));
        }
    }
};

// Forward, one CTA per polynomial (N = NC = 2^LGC): buffers i % 3 rotate (TMA of item
// i+2 issued at the barrier of item i).
template <int LGC>
__global__ void __launch_bounds__((1 << LGC) / kE, ctas_per_sm<LGC>())
    k_ntt_c5_fwd(const __grid_constant__ CUtensorMap map, const __grid_constant__ C5Args a) {
    static_assert(LGC == 12 || LGC == 13, "NC = 2^12 or 2^13 per CTA");
    using F = Fwd<LGC>;
    constexpr int NC = F::NC, NT = F::NT;
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    Ctx f;
    frame_init<LGC>(f, smem_raw, kNBuf, mbar, &tmem_slot);
    const u32 w0 = (u32)((u64)a.items * blockIdx.x / gridDim.x), w1 = (u32)((u64)a.items * (blockIdx.x + 1) / gridDim.x);
    auto issue = [&](u32 i) {   // one thread
        uint64_t *bar = &mbar[i % 3];
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 8));
        double *c = f.bufs + (size_t)(i % 3) * NC;
        const int row0 = poly_row(a, w0 + i);
#pragma unroll
        for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(c + 16 * r, &map, 0, row0 + r, bar);
    };
    if (f.tid == 0 && w0 < w1) {
        issue(0);
        if (w0 + 1 < w1) issue(1);
    }
    u32 jcur = 0xffffffffu;
    for (u32 i = 0; w0 + i < w1; ++i) {
        const u32 w = w0 + i, j = w / a.batch;
        if (j != jcur) {
            __syncthreads();
            const double2 *twg = a.tw + (size_t)j * NC;
            F::load_twiddles(f, [&](int m, int B) { return twg[m + B]; });
            f.set_prime(twg[0]);
            jcur = j;
            ephdc_tmem::fence_before_sync();
            __syncthreads();
            ephdc_tmem::fence_after_sync();
        }
        ephdc_async::mbar_wait(&mbar[i % 3], (i / 3) & 1u);
        double *C = f.bufs + (size_t)(i % 3) * NC;
        {
            const u64 *Cu = reinterpret_cast<const u64 *>(C);
            const int st = sw(f.tid);
            double x[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = centered(Cu[st ^ sw(k * NT)], f);
            F::pass1(f, C, x);
        }
        __syncthreads();
        if (f.tid == 0 && w0 + i + 2 < w1) issue(i + 2);   // item i-1's buffer is free
        F::pass2(f, C);
        __syncwarp();
        F::pass3(f, C);
        __syncwarp();
        F::tail(f, C, poly_ptr(a, w));
    }
    frame_exit<LGC>(f, tmem_slot);
}

// ---------------------------------------------------------------------------------
// Two warp groups per CTA (N = 2^13).  With one 16-warp team every warp reaches the
// load and store phases of a pass at the same time (one barrier per item aligns them),
// so the shared-memory traffic (4 passes x 16 B per element, ~4K of the ~12K clocks of
// a polynomial) and the FP64 work serialise.  Here two 8-warp groups transform
// alternate polynomials of the CTA's range, each thread doing the work of the 16-warp
// version's threads tid and tid + 256 one after the other (same registers per thread,
// same TMEM columns: warps w and w + 8 share a lane quarter and the twiddles), with a
// group-local named barrier; group 1 starts one pass late, so one group's loads and
// stores overlap the other's butterflies.  Items of one prime form a segment (both
// groups hold that prime's twiddles); buffers rotate by three: item i's pass-1 barrier
// frees buffer (i - 2) % 3 -- item i - 2 was the same group's (or a finished segment's)
// -- for the TMA of item i + 1.
// ---------------------------------------------------------------------------------
EPHDC_D void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EPHDC_D void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// the 16-warp thread tid + 256 h seen by thread tid of a group (warp w, lane quarter w % 4)
EPHDC_D Ctx half_ctx(const Ctx &f, int h) {
    Ctx v = f;
    const int gw = (f.tid >> 5) & 7;
    v.tid = (f.tid & 255) + 256 * h;
    v.warp = gw + 8 * h;
    v.tbase = f.tbase - (uint32_t)(f.warp >> 2) * 128u + (uint32_t)(v.warp >> 2) * 128u;
    return v;
}

// [i0, i1) = the segment of local item i0: the items of its prime
EPHDC_D u32 segment_end(const C5Args &a, u32 w0, u32 w1, u32 i0) {
    const u32 j = (w0 + i0) / a.batch;
    return min(w1, (j + 1) * a.batch) - w0;
}

__global__ void __launch_bounds__(512, 1) k_ntt_c5_fwd2g(const __grid_constant__ CUtensorMap map,
                                                        const __grid_constant__ C5Args a) {
    constexpr int LGC = 13;
    using F = Fwd<LGC>;
    constexpr int NC = F::NC;
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    Ctx f;
    frame_init<LGC>(f, smem_raw, kNBuf, mbar, &tmem_slot);
    const int g = f.warp >> 3, gt = f.tid & 255;
    const u32 w0 = (u32)((u64)a.items * blockIdx.x / gridDim.x), w1 = (u32)((u64)a.items * (blockIdx.x + 1) / gridDim.x);
    const u32 n = w1 - w0;
    auto issue = [&](u32 i) {   // one thread
        uint64_t *bar = &mbar[i % 3];
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 8));
        double *c = f.bufs + (size_t)(i % 3) * NC;
        const int row0 = poly_row(a, w0 + i);
#pragma unroll
        for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(c + 16 * r, &map, 0, row0 + r, bar);
    };
    if (f.tid == 0)
        for (u32 i = 0; i < 3 && i < n; ++i) issue(i);
    for (u32 i0 = 0; i0 < n;) {
        const u32 i1 = segment_end(a, w0, w1, i0), j = (w0 + i0) / a.batch;
        __syncthreads();   // both groups are done with the previous prime
        const double2 *twg = a.tw + (size_t)j * NC;
        F::load_twiddles(half_ctx(f, g), [&](int m, int B) { return twg[m + B]; });
        f.set_prime(twg[0]);
        ephdc_tmem::fence_before_sync();
        __syncthreads();
        ephdc_tmem::fence_after_sync();
        const bool pair = i0 + 1 < i1;
        if (g == 1 && pair) bar_sync(3, 512);   // start one pass behind group 0
        for (u32 i = i0 + g; i < i1; i += 2) {
            ephdc_async::mbar_wait(&mbar[i % 3], (i / 3) & 1u);
            double *C = f.bufs + (size_t)(i % 3) * NC;
            const u64 *Cu = reinterpret_cast<const u64 *>(C);
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const Ctx v = half_ctx(f, h);
                const int st = sw(v.tid);
                double x[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) x[k] = centered(Cu[st ^ sw(k * F::NT)], v);
                F::pass1(v, C, x);
            }
            bar_sync(1 + g, 256);
            if (g == 0 && i == i0 && pair) bar_arrive(3, 512);
            if (gt == 0 && i >= 2 && i + 1 < n) issue(i + 1);   // buffer (i-2) % 3 is free
            u64 *o = poly_ptr(a, w0 + i);
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const Ctx v = half_ctx(f, h);
                F::pass2(v, C);
                __syncwarp();
                F::pass3(v, C);
                __syncwarp();
                F::tail(v, C, o);
            }
        }
        i0 = i1;
    }
    frame_exit<LGC>(f, tmem_slot);
}

// Forward on a cluster of C CTAs (N = 2^13 C): CTA s loads the slice [s NC/C, (s+1)
// NC/C) of every block (C TMA boxes into the staging buffer), applies the log2(C)
// cross levels (psi_rev[1 .. C-1]) to its slice and writes output k to CTA k's block
// buffer (DSMEM); one cluster barrier; then the 13 local levels on its own block.
// Block buffers alternate (a CTA writes its partners' buffer of item i+1 only after the
// barrier of item i, which every partner reaches after finishing item i-1).  RED: the
// cross-level outputs are reduced to |x| <= q/2 (needed at 2^15, 2^16 by the bounds).
template <int C, bool RED>
__global__ void __launch_bounds__(512, 1) k_ntt_c5_fwd_cl(const __grid_constant__ CUtensorMap map,
                                                         const __grid_constant__ C5Args a) {
    constexpr int LGC = 13, LC = C == 2 ? 1 : C == 4 ? 2 : 3;
    using F = Fwd<LGC>;
    constexpr int NC = F::NC, NT = F::NT, SL = NC / C, RP = SL / NT;   // slice, r per thread
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    __shared__ double2 xtw[8];   // [0] = (q, 1/q); [1 .. C-1] = the cross-level twiddles psi_rev[1 .. C-1]
    Ctx f;
    frame_init<LGC>(f, smem_raw, 3, mbar, &tmem_slot);
    double *stage = f.bufs;                                   // [C][SL] u64 (TMA)
    const u32 s = cluster_rank(), unit = blockIdx.x / C, nunits = gridDim.x / C;
    const u32 w0 = (u32)((u64)a.items * unit / nunits), w1 = (u32)((u64)a.items * (unit + 1) / nunits);
    auto issue = [&](u32 i) {   // one thread; the staging buffer (mbarrier 0)
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(&mbar[0], (u32)(NC * 8));
        const int row0 = poly_row(a, w0 + i);
#pragma unroll
        for (int k = 0; k < C; ++k) tma_load_2d(stage + k * SL, &map, 0, row0 + ((k * NC + (int)s * SL) >> 4), &mbar[0]);
    };
    if (f.tid == 0 && w0 < w1) issue(0);
    u32 jcur = 0xffffffffu;
    for (u32 i = 0; w0 + i < w1; ++i) {
        const u32 w = w0 + i, j = w / a.batch;
        double *B = f.bufs + (size_t)(1 + (i & 1)) * NC;       // this item's block buffer
        if (j != jcur) {
            __syncthreads();
            const double2 *twg = a.tw + ((size_t)j << a.log2N);
            F::load_twiddles(f, [&](int m, int Bk) { return twg[C * m + (int)s * m + Bk]; });
            if (f.tid < C) xtw[f.tid] = twg[f.tid];
            f.set_prime(twg[0]);
            jcur = j;
            ephdc_tmem::fence_before_sync();
            __syncthreads();
            ephdc_tmem::fence_after_sync();
        }
        ephdc_async::mbar_wait(&mbar[0], i & 1u);
        // ---- cross levels on the slice: r = s SL + rl, rl = tid + u NT, elements r + k NC
        {
            const u64 *Su = reinterpret_cast<const u64 *>(stage);
            uint32_t dst[C];
#pragma unroll
            for (int k = 0; k < C; ++k) dst[k] = map_rank(B, (uint32_t)k);
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int rl = f.tid + u * NT, r = (int)s * SL + rl;
                double x[C];
#pragma unroll
                for (int k = 0; k < C; ++k) x[k] = centered(Su[sw(k * SL + rl)], f);
                ct_stages<LC, 0, LC>(x, [&](int sub, int v) { return xtw[(1 << sub) + v]; }, f.nq);
                const uint32_t off = (uint32_t)sw(r) * 8u;
#pragma unroll
                for (int k = 0; k < C; ++k) {
                    const double y = RED ? reduce(x[k], f.qinv, f.nq) : x[k];
                    if (k == (int)s) B[sw(r)] = y;
                    else st_cluster(dst[k] + off, y);
                }
            }
        }
        cluster_arrive();
        cluster_wait();   // every CTA's slice of item i is in place; the staging buffer is consumed
        if (f.tid == 0 && w0 + i + 1 < w1) issue(i + 1);
        {
            const int st = sw(f.tid);
            double x[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = B[st ^ sw(k * NT)];
            F::pass1(f, B, x);
        }
        __syncthreads();
        F::pass2(f, B);
        __syncwarp();
        F::pass3(f, B);
        __syncwarp();
        F::tail(f, B, poly_ptr(a, w) + (size_t)s * NC);
    }
    frame_exit<LGC>(f, tmem_slot);
    cluster_arrive();   // no CTA leaves while a partner may still write its shared memory
    cluster_wait();
}

// Forward on a cluster with two warp groups per CTA (N = 2^13 C; the structure of
// k_ntt_c5_fwd2g inside each CTA).  No cluster barrier per item: group g of CTA s
// pushes the cross-level outputs owned by CTA k straight into CTA k's group-g block
// buffer with st.async, whose bytes complete on CTA k's full[g] mbarrier (armed by CTA
// k for that item); a CTA tells its partners that its group-g buffer is free again --
// the item's last level has read it -- with one remote arrive on their empty[g].  The
// staging buffer (this CTA's slice of every block, TMA) is shared by the groups: the
// group that has consumed item i issues item i + 1, which the other group takes.
EPHDC_D void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
                 "r"(rbar)
                 : "memory");
}
EPHDC_D void mbar_remote_arrive(uint32_t rbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
// Waits with acquire at cluster scope.  Bounded: a protocol error traps (the launch
// fails with an error) instead of hanging the GPU; a legitimate wait lasts microseconds.
EPHDC_D void mbar_wait_cluster(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    for (uint32_t it = 0; !done; ++it) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n}"
            : "=r"(done)
            : "r"(ephdc_async::smem_u32(bar)), "r"(phase)
            : "memory");
        if (it > (1u << 26)) __trap();
    }
}
EPHDC_D void mbar_wait_bounded(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    for (uint32_t it = 0; !done; ++it) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n}"
            : "=r"(done)
            : "r"(ephdc_async::smem_u32(bar)), "r"(phase)
            : "memory");
        if (it > (1u << 26)) __trap();
    }
}

template <int C, bool RED>
__global__ void __launch_bounds__(512, 1) k_ntt_c5_fwd_cl2g(const __grid_constant__ CUtensorMap map,
                                                           const __grid_constant__ C5Args a) {
    constexpr int LGC = 13, LC = C == 2 ? 1 : C == 4 ? 2 : 3;
    using F = Fwd<LGC>;
    constexpr int NC = F::NC, NT = F::NT, SL = NC / C, RP = SL / NT;
    extern __shared__ unsigned char smem_raw[];
    // the staging buffer's TMA completes on mbar[i & 1] (item i): with ONE barrier, a
    // group waiting for item i + 1 while item i's copy is still in flight would match
    // the parity of the previous phase and proceed early (r19: a launch failure)
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ __align__(8) uint64_t full[2], empty[2];    // per group
    __shared__ uint32_t tmem_slot;
    __shared__ double2 xtw[8];
    Ctx f;
    frame_init<LGC>(f, smem_raw, 3, mbar, &tmem_slot);
    const u32 s = cluster_rank(), unit = blockIdx.x / C, nunits = gridDim.x / C;
    const u32 w0 = (u32)((u64)a.items * unit / nunits), w1 = (u32)((u64)a.items * (unit + 1) / nunits);
    const u32 n = w1 - w0;
    // items per group (alternate within each prime segment); full[g] is armed for the
    // group's first item before the start barrier and for its next item right after an
    // item's last level, BEFORE the partners are told the buffer is free -- so no pushed
    // byte reaches full[g] ahead of its expect_tx
    u32 cnt[2] = {0, 0};
    for (u32 i0 = 0; i0 < n;) {
        const u32 i1 = segment_end(a, w0, w1, i0);
        cnt[0] += (i1 - i0 + 1) / 2;
        cnt[1] += (i1 - i0) / 2;
        i0 = i1;
    }
    const u32 xbytes = (u32)((C - 1) * SL * 8);
    if (f.tid == 0) {
        for (int g = 0; g < 2; ++g) {
            ephdc_async::mbar_init(&full[g], 1);
            ephdc_async::mbar_init(&empty[g], C - 1);
            if (cnt[g] > 0) ephdc_async::mbar_arrive_expect_tx(&full[g], xbytes);
        }
    }
    cluster_arrive();   // every CTA's barriers are initialised before any remote access
    cluster_wait();
    const int g = f.warp >> 3, gt = f.tid & 255;
    double *stage = f.bufs;
    double *B = f.bufs + (size_t)(1 + g) * NC;               // this group's block buffer
    auto issue = [&](u32 i) {   // one thread; the staging buffer
        uint64_t *bar = &mbar[i & 1u];
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 8));
        const int row0 = poly_row(a, w0 + i);
#pragma unroll
        for (int k = 0; k < C; ++k) tma_load_2d(stage + k * SL, &map, 0, row0 + ((k * NC + (int)s * SL) >> 4), bar);
    };
    if (f.tid == 0 && n > 0) issue(0);
    u32 ng = 0;   // items this group has processed
    for (u32 i0 = 0; i0 < n;) {
        const u32 i1 = segment_end(a, w0, w1, i0), j = (w0 + i0) / a.batch;
        __syncthreads();
        const double2 *twg = a.tw + ((size_t)j << a.log2N);
        F::load_twiddles(half_ctx(f, g), [&](int m, int Bk) { return twg[C * m + (int)s * m + Bk]; });
        if (f.tid < C) xtw[f.tid] = twg[f.tid];
        f.set_prime(twg[0]);
        ephdc_tmem::fence_before_sync();
        __syncthreads();
        ephdc_tmem::fence_after_sync();
        const bool pair = i0 + 1 < i1;
        if (g == 1 && pair) bar_sync(3, 512);
        for (u32 i = i0 + g; i < i1; i += 2, ++ng) {
            if (ng > 0) mbar_wait_cluster(&empty[g], (ng - 1) & 1u);   // partners' group-g buffers are free
            mbar_wait_bounded(&mbar[i & 1u], (i >> 1) & 1u);
            // ---- cross levels on the slice: r = s SL + rl, rl = vtid + u NT, elements r + k NC
            const u64 *Su = reinterpret_cast<const u64 *>(stage);
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int vt = gt + 256 * h;
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    const int rl = vt + u * NT, r = (int)s * SL + rl;
                    double x[C];
#pragma unroll
                    for (int k = 0; k < C; ++k) x[k] = centered(Su[sw(k * SL + rl)], f);
                    ct_stages<LC, 0, LC>(x, [&](int sub, int v) { return xtw[(1 << sub) + v]; }, f.nq);
#pragma unroll
                    for (int k = 0; k < C; ++k) {
                        const double y = RED ? reduce(x[k], f.qinv, f.nq) : x[k];
                        if (k == (int)s) B[sw(r)] = y;
                        else st_async_f64(map_rank(B + sw(r), (uint32_t)k), y, map_rank(&full[g], (uint32_t)k));
                    }
                }
            }
            bar_sync(1 + g, 256);   // this group has consumed the staging buffer
            if (g == 0 && i == i0 && pair) bar_arrive(3, 512);
            if (gt == 0 && i + 1 < n) issue(i + 1);
            mbar_wait_bounded(&full[g], ng & 1u);   // the partners' outputs are in B
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const Ctx v = half_ctx(f, h);
                const int st = sw(v.tid);
                double x[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) x[k] = B[st ^ sw(k * NT)];
                F::pass1(v, B, x);
            }
            bar_sync(1 + g, 256);
            u64 *o = poly_ptr(a, w0 + i) + (size_t)s * NC;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const Ctx v = half_ctx(f, h);
                F::pass2(v, B);
                __syncwarp();
                F::pass3(v, B);
                __syncwarp();
                F::tail(v, B, o);
            }
            bar_sync(1 + g, 256);   // B is read: the partners may write the group's next item
            if (gt == 0) {
                if (ng + 1 < cnt[g]) ephdc_async::mbar_arrive_expect_tx(&full[g], xbytes);   // before the signal
#pragma unroll
                for (int k = 0; k < C; ++k)
                    if (k != (int)s) mbar_remote_arrive(map_rank(&empty[g], (uint32_t)k));
            }
        }
        i0 = i1;
    }
    frame_exit<LGC>(f, tmem_slot);
    cluster_arrive();   // no CTA leaves while a partner may still signal it
    cluster_wait();
}

// =================================================================================
// Inverse pieces (Cooley-Tukey DIT on the bit-reversed input).  Level lv pairs (j, j+h),
// h = 2^lv, inside blocks of 2h with twiddle W[h + (j mod h)] = omega^-(N/2h)(j mod h)
// (omega = psi^2 of the full N).  After the levels of the whole transform the values
// are N a_j psi^j; a_j = s_j (.) with s_j = N^-1 psi^-j.  Per 2^LGC block: passes A =
// levels 0-1 (four consecutive elements), B = 2-4 (groups of 8, 4 apart), C = 5 ..
// 4+RC (stride 32, warp-local), D = the last four local levels (stride NT), whose last
// level is fused with the scaling by sigma_r = N^-1 psi^-r (r = the local index):
//     out_r = sigma_r X + (sigma_r W_r) Y,   out_{r+NC/2} = c_loc (sigma_r X - (sigma_r W_r) Y),
// c_loc = psi^-(NC/2) (sigma_{r+NC/2} = sigma_r c_loc).  A single-block transform stores
// these; a cluster keeps them for the cross levels.
// =================================================================================
template <int LGC> struct Inv {
    static constexpr int NC = 1 << LGC, NT = NC / kE;
    static constexpr int RC = LGC - 9, GC = kE >> RC;
    static constexpr int TWS = LGC >= 13 ? 512 : 256;

    // DIT table entries [1, TWS) -> shared; pass D levels (7 pairs) at TMEM columns
    // [0, 32), the fused scaling pairs (sigma_r, sigma_r W_r) of r = tid + NT k (k < 8)
    // at columns [32, 96)
    template <class WT, class ST> static EPHDC_D void load_twiddles(const Ctx &f, const WT &wtw, const ST &stw) {
        for (int p = f.tid; p < TWS; p += NT) f.tws[p] = wtw(p);
        uint32_t r[16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int idx = 4 * h + k;
                if (idx < 7) {
                    const int sub = 31 - __clz(idx + 1), kk = idx + 1 - (1 << sub);
                    put_pair(&r[4 * k], wtw((NT << sub) + f.tid + NT * kk));
                } else {
                    put_pair(&r[4 * k], make_double2(0.0, 0.0));
                }
            }
            ephdc_tmem::stx<16>(f.tbase + 16u * h, r);
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int jj = f.tid + NT * (2 * h + v);
                put_pair(&r[8 * v], stw(2 * jj));
                put_pair(&r[8 * v + 4], stw(2 * jj + 1));
            }
            ephdc_tmem::stx<16>(f.tbase + 32u + 16u * h, r);
        }
    }

    // passes A-C on the block C (input: canonical u64 in the TMA layout)
    static EPHDC_D void passes_abc(const Ctx &f, double *C) {
        // A: levels 0 (twiddle 1: adds) and 1 on four consecutive elements
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int g4 = 128 * f.warp + f.lane + 32 * u;
            const int sg = sw(4 * g4);
            const ulonglong2 ua = *reinterpret_cast<const ulonglong2 *>(C + sg);
            const ulonglong2 ub = *reinterpret_cast<const ulonglong2 *>(C + (sg ^ 2));
            const double v0 = centered(ua.x, f), v1 = centered(ua.y, f), v2 = centered(ub.x, f),
                         v3 = centered(ub.y, f);
            double x0 = __dadd_rn(v0, v1), x1 = __dsub_rn(v0, v1), x2 = __dadd_rn(v2, v3), x3 = __dsub_rn(v2, v3);
            const double2 t2 = f.tws[2], t3 = f.tws[3];
            ct_bfly(x0, x2, t2.x, t2.y, f.nq);
            ct_bfly(x1, x3, t3.x, t3.y, f.nq);
            *reinterpret_cast<double2 *>(C + sg) = make_double2(x0, x1);
            *reinterpret_cast<double2 *>(C + (sg ^ 2)) = make_double2(x2, x3);
        }
        __syncwarp();
        // B: levels 2-4, blocks of 32, groups of 8 elements 4 apart
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int blk = 16 * f.warp + (f.lane >> 2) + 8 * u, off4 = f.lane & 3, sb = sw(32 * blk + off4);
            double x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = C[sb ^ sw(4 * k)];
            dit_stages<3, 0, 3>(x, [&](int sub, int kk) { return f.tws[(4 << sub) + off4 + 4 * kk]; }, f.nq);
#pragma unroll
            for (int k = 0; k < 8; ++k) C[sb ^ sw(4 * k)] = x[k];
        }
        __syncwarp();
        // C: levels 5 .. 4+RC, elements 2^(5+RC) blk + lane + 32 k (warp-local)
#pragma unroll
        for (int u = 0; u < GC; ++u) {
            const int blk = GC * f.warp + u, sb = sw((blk << (5 + RC)) + f.lane);
            double x[1 << RC];
#pragma unroll
            for (int k = 0; k < (1 << RC); ++k) x[k] = C[sb ^ sw(32 * k)];
            dit_stages<RC, 0, RC>(x, [&](int sub, int kk) { return f.tws[(32 << sub) + f.lane + 32 * kk]; }, f.nq);
#pragma unroll
            for (int k = 0; k < (1 << RC); ++k) C[sb ^ sw(32 * k)] = x[k];
        }
    }

    // D: the last four levels on elements tid + NT k; the last one fused with the scaling;
    // sink(k, value) receives element tid + NT k
    // (TMEM loads issued ahead: the level twiddles before the shared-memory loads, each
    // scaling block one block ahead of its use)
    template <class Sink> static EPHDC_D void pass_d(const Ctx &f, const double *C, double2 cloc, const Sink &sink) {
        uint32_t rr[32], sc[2][16];
        ephdc_tmem::ldx<16>(f.tbase, *reinterpret_cast<uint32_t(*)[16]>(&rr[0]));
        ephdc_tmem::ldx<16>(f.tbase + 16u, *reinterpret_cast<uint32_t(*)[16]>(&rr[16]));
        ephdc_tmem::ldx<16>(f.tbase + 32u, sc[0]);
        double x[16];
        const int st = sw(f.tid);
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = C[st ^ sw(NT * k)];
        ephdc_tmem::waitx<32>(rr);
        ephdc_tmem::waitx<16>(sc[0]);
        dit_stages<4, 0, 3>(x, [&](int sub, int kk) { return pair_at(rr, (1 << sub) - 1 + kk); }, f.nq);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (h < 3) ephdc_tmem::ldx<16>(f.tbase + 32u + 16u * (h + 1), sc[(h + 1) & 1]);
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int k = 2 * h + v;
                const double2 sj = pair_at(sc[h & 1], 2 * v), swj = pair_at(sc[h & 1], 2 * v + 1);
                const double A = mul_tw(x[k], sj.x, sj.y, f.nq), Bv = mul_tw(x[k + 8], swj.x, swj.y, f.nq);
                sink(k, __dadd_rn(A, Bv));
                sink(k + 8, mul_tw(__dsub_rn(A, Bv), cloc.x, cloc.y, f.nq));
            }
            if (h < 3) ephdc_tmem::waitx<16>(sc[(h + 1) & 1]);
        }
    }
};

// Inverse, one CTA per polynomial (N = NC = 2^LGC).
template <int LGC>
__global__ void __launch_bounds__((1 << LGC) / kE, ctas_per_sm<LGC>())
    k_ntt_c5_inv(const __grid_constant__ CUtensorMap map, const __grid_constant__ C5Args a) {
    static_assert(LGC == 12 || LGC == 13, "NC = 2^12 or 2^13 per CTA");
    using I = Inv<LGC>;
    constexpr int NC = I::NC, NT = I::NT;
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    Ctx f;
    frame_init<LGC>(f, smem_raw, kNBuf, mbar, &tmem_slot);
    const u32 w0 = (u32)((u64)a.items * blockIdx.x / gridDim.x), w1 = (u32)((u64)a.items * (blockIdx.x + 1) / gridDim.x);
    auto issue = [&](u32 i) {
        uint64_t *bar = &mbar[i % 3];
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 8));
        double *c = f.bufs + (size_t)(i % 3) * NC;
        const int row0 = poly_row(a, w0 + i);
#pragma unroll
        for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(c + 16 * r, &map, 0, row0 + r, bar);
    };
    if (f.tid == 0 && w0 < w1) {
        issue(0);
        if (w0 + 1 < w1) issue(1);
    }
    u32 jcur = 0xffffffffu;
    double2 cloc = make_double2(0.0, 0.0);
    for (u32 i = 0; w0 + i < w1; ++i) {
        const u32 w = w0 + i, j = w / a.batch;
        if (j != jcur) {
            __syncthreads();
            const double2 *twg = a.tw + (size_t)j * NC, *tl = a.tail + (size_t)j * NC;
            I::load_twiddles(f, [&](int p) { return twg[p]; }, [&](int p) { return tl[p]; });
            ephdc_tmem::wait_st();
            f.set_prime(twg[0]);
            cloc = a.cinv[j];
            jcur = j;
            ephdc_tmem::fence_before_sync();
            __syncthreads();
            ephdc_tmem::fence_after_sync();
        }
        ephdc_async::mbar_wait(&mbar[i % 3], (i / 3) & 1u);
        double *C = f.bufs + (size_t)(i % 3) * NC;
        I::passes_abc(f, C);
        __syncthreads();
        if (f.tid == 0 && w0 + i + 2 < w1) issue(i + 2);   // item i-1's buffer is free
        u64 *o = poly_ptr(a, w);
        I::pass_d(f, C, cloc, [&](int k, double v) {
            __stcs(reinterpret_cast<unsigned long long *>(o + f.tid + NT * k),
                   (unsigned long long)out_u64(v, f));
        });
    }
    frame_exit<LGC>(f, tmem_slot);
}

// Inverse with two warp groups (N = 2^13; see k_ntt_c5_fwd2g): passes A-C of both
// halves (warp-local), the group barrier, pass D of both halves straight to HBM.
__global__ void __launch_bounds__(512, 1) k_ntt_c5_inv2g(const __grid_constant__ CUtensorMap map,
                                                        const __grid_constant__ C5Args a) {
    constexpr int LGC = 13;
    using I = Inv<LGC>;
    constexpr int NC = I::NC, NT = I::NT;
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    Ctx f;
    frame_init<LGC>(f, smem_raw, kNBuf, mbar, &tmem_slot);
    const int g = f.warp >> 3, gt = f.tid & 255;
    const u32 w0 = (u32)((u64)a.items * blockIdx.x / gridDim.x), w1 = (u32)((u64)a.items * (blockIdx.x + 1) / gridDim.x);
    const u32 n = w1 - w0;
    auto issue = [&](u32 i) {
        uint64_t *bar = &mbar[i % 3];
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 8));
        double *c = f.bufs + (size_t)(i % 3) * NC;
        const int row0 = poly_row(a, w0 + i);
#pragma unroll
        for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(c + 16 * r, &map, 0, row0 + r, bar);
    };
    if (f.tid == 0)
        for (u32 i = 0; i < 3 && i < n; ++i) issue(i);
    for (u32 i0 = 0; i0 < n;) {
        const u32 i1 = segment_end(a, w0, w1, i0), j = (w0 + i0) / a.batch;
        __syncthreads();
        const double2 *twg = a.tw + (size_t)j * NC, *tl = a.tail + (size_t)j * NC;
        I::load_twiddles(half_ctx(f, g), [&](int p) { return twg[p]; }, [&](int p) { return tl[p]; });
        ephdc_tmem::wait_st();
        f.set_prime(twg[0]);
        const double2 cloc = a.cinv[j];
        ephdc_tmem::fence_before_sync();
        __syncthreads();
        ephdc_tmem::fence_after_sync();
        const bool pair = i0 + 1 < i1;
        if (g == 1 && pair) bar_sync(3, 512);
        for (u32 i = i0 + g; i < i1; i += 2) {
            ephdc_async::mbar_wait(&mbar[i % 3], (i / 3) & 1u);
            double *C = f.bufs + (size_t)(i % 3) * NC;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) I::passes_abc(half_ctx(f, h), C);
            bar_sync(1 + g, 256);
            if (g == 0 && i == i0 && pair) bar_arrive(3, 512);
            if (gt == 0 && i >= 2 && i + 1 < n) issue(i + 1);
            u64 *o = poly_ptr(a, w0 + i);
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const Ctx v = half_ctx(f, h);
                I::pass_d(v, C, cloc, [&](int k, double val) {
                    __stcs(reinterpret_cast<unsigned long long *>(o + v.tid + NT * k),
                           (unsigned long long)out_u64(val, v));
                });
            }
        }
        i0 = i1;
    }
    frame_exit<LGC>(f, tmem_slot);
}

// Inverse on a cluster of C CTAs (N = 2^13 C): each CTA transforms its block (13 local
// levels, the last fused with sigma_r) and keeps it; one cluster barrier; CTA s then
// reads the slice r in [s NC/C, (s+1) NC/C) of every block (DSMEM), applies the log2(C)
// cross levels (twiddles W[2^13 2^l + r + 2^13 kk], kept as w in TMEM with w/q formed
// on the fly) and the block constants psi^-(2^13 k), and stores a_{r + 2^13 k}.
// Buffers rotate by three: the TMA of item i+2 overwrites item i-1's block only after
// the barrier of item i, which every partner reaches after reading it.
template <int C>
__global__ void __launch_bounds__(512, 1) k_ntt_c5_inv_cl(const __grid_constant__ CUtensorMap map,
                                                         const __grid_constant__ C5Args a) {
    constexpr int LGC = 13, LC = C == 2 ? 1 : C == 4 ? 2 : 3;
    using I = Inv<LGC>;
    constexpr int NC = I::NC, NT = I::NT, SL = NC / C, RP = SL / NT;
    constexpr int NXT = RP * (C - 1);                       // cross twiddles per thread (w only)
    constexpr int NXR = ((2 * NXT + 15) / 16) * 16;         // their TMEM columns
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    __shared__ double2 ck[8];                               // psi^-(2^13 k), k < C
    Ctx f;
    frame_init<LGC>(f, smem_raw, kNBuf, mbar, &tmem_slot);
    const u32 s = cluster_rank(), unit = blockIdx.x / C, nunits = gridDim.x / C;
    const u32 w0 = (u32)((u64)a.items * unit / nunits), w1 = (u32)((u64)a.items * (unit + 1) / nunits);
    auto issue = [&](u32 i) {
        uint64_t *bar = &mbar[i % 3];
        ephdc_async::fence_proxy_async();
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 8));
        double *c = f.bufs + (size_t)(i % 3) * NC;
        const int row0 = poly_row(a, w0 + i) + (int)s * (NC / 16);
#pragma unroll
        for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(c + 16 * r, &map, 0, row0 + r, bar);
    };
    if (f.tid == 0 && w0 < w1) {
        issue(0);
        if (w0 + 1 < w1) issue(1);
    }
    u32 jcur = 0xffffffffu;
    double2 cloc = make_double2(0.0, 0.0);
    for (u32 i = 0; w0 + i < w1; ++i) {
        const u32 w = w0 + i, j = w / a.batch;
        if (j != jcur) {
            __syncthreads();
            const double2 *twg = a.tw + ((size_t)j << a.log2N), *tl = a.tail + (size_t)j * NC;
            I::load_twiddles(f, [&](int p) { return twg[p]; }, [&](int p) { return tl[p]; });
            // cross levels: slice index u, level l, block position kk at columns 96 + 2 n
            uint32_t r[16];
#pragma unroll
            for (int h = 0; h < NXR / 16; ++h) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int n = 8 * h + e;
                    double wv = 0.0;
                    if (n < NXT) {
                        const int u = n / (C - 1), idx = n % (C - 1), l = 31 - __clz(idx + 1), kk = idx + 1 - (1 << l);
                        const int rr = (int)s * SL + f.tid + u * NT;
                        wv = twg[(NC << l) + rr + NC * kk].x;
                    }
                    r[2 * e] = (uint32_t)__double2loint(wv);
                    r[2 * e + 1] = (uint32_t)__double2hiint(wv);
                }
                ephdc_tmem::stx<16>(f.tbase + 96u + 16u * h, r);
            }
            if (f.tid < C) ck[f.tid] = a.ck[j * 8 + f.tid];
            ephdc_tmem::wait_st();
            f.set_prime(twg[0]);
            cloc = a.cinv[j];
            jcur = j;
            ephdc_tmem::fence_before_sync();
            __syncthreads();
            ephdc_tmem::fence_after_sync();
        }
        ephdc_async::mbar_wait(&mbar[i % 3], (i / 3) & 1u);
        double *Cb = f.bufs + (size_t)(i % 3) * NC;
        I::passes_abc(f, Cb);
        __syncthreads();
        const int st = sw(f.tid);
        I::pass_d(f, Cb, cloc, [&](int k, double v) { Cb[st ^ sw(NT * k)] = v; });
        cluster_arrive();
        cluster_wait();   // every block of item i holds its 13 local levels
        if (f.tid == 0 && w0 + i + 2 < w1) issue(i + 2);   // item i-1's blocks were read before this barrier
        // ---- cross levels on the slice r = s SL + tid + u NT, elements r + k NC
        u64 *o = poly_ptr(a, w);
        uint32_t xr[NXR];
#pragma unroll
        for (int h = 0; h < NXR / 16; ++h)
            ephdc_tmem::ldx<16>(f.tbase + 96u + 16u * h, *reinterpret_cast<uint32_t(*)[16]>(&xr[16 * h]));
        ephdc_tmem::waitx<NXR>(xr);
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int r = (int)s * SL + f.tid + u * NT;
            const uint32_t off = (uint32_t)sw(r) * 8u;
            double x[C];
#pragma unroll
            for (int k = 0; k < C; ++k) x[k] = k == (int)s ? Cb[sw(r)] : ld_cluster(map_rank(Cb, (uint32_t)k) + off);
            dit_stages<LC, 0, LC>(x, [&](int l, int kk) {
                const int n = u * (C - 1) + (1 << l) - 1 + kk;
                const double wv = __hiloint2double(xr[2 * n + 1], xr[2 * n]);
                return make_double2(wv, __dmul_rn(wv, f.qinv));
            }, f.nq);
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const double y = k == 0 ? x[0] : mul_tw(x[k], ck[k].x, ck[k].y, f.nq);
                __stcs(reinterpret_cast<unsigned long long *>(o + r + NC * k),
                       (unsigned long long)out_u64(y, f));
            }
        }
    }
    frame_exit<LGC>(f, tmem_slot);
    cluster_arrive();   // no CTA leaves while a partner may still read its shared memory
    cluster_wait();
}

}  // namespace c5

namespace {
inline cudaError_t counted(cudaError_t e) {
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

// [rows][16] u64 view of d_polys, box_rows x 128-byte boxes, 128-byte swizzle
bool make_poly_map(CUtensorMap *m, const void *base, uint64_t n_elems, uint32_t box_rows) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || (n_elems & 15) || (n_elems >> 4) > 0x7fffffffull) return false;
    const cuuint64_t dims[2] = {16, n_elems >> 4};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {16u, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// Value bounds.  Inputs are centered (|x| <= q/2); a CT level adds <=
// (1/2 + B 2^-54) q (+2 for the rounding of the quotient); every mul_tw input and every
// value the final reduction takes stays below 2^51.
static double rtw_bound(double B, double Q) { return (0.5 + B / 18014398509481984.0) * Q + 2.0; }
static const double kL51 = 0.98 * 2251799813685248.0;

// forward: log2 N CT levels from |x| <= q/2; a cluster may reduce (to q/2 + 1) after
// its `cross` levels
static bool c5_fwd_ok(double Q, uint32_t log2N, uint32_t cross, bool red) {
    double B = 0.5 * Q + 1.0;
    for (uint32_t lv = 0; lv < log2N; ++lv) {
        if (B >= kL51) return false;
        B += rtw_bound(B, Q);
        if (red && lv + 1 == cross) B = 0.5 * Q + 2.0;
    }
    return B < kL51;
}
// inverse: level 0 adds (|x| <= q), levels 1 .. 11 CT, the fused level 12 (A + B), then
// `cross` CT levels whose w/q is formed as fl(w fl(1/q)) (relative error 2^-52) and the
// block constant
static bool c5_inv_ok(double Q, uint32_t lgc, uint32_t cross) {
    double B = Q + 1.0;
    for (uint32_t lv = 1; lv + 1 < lgc; ++lv) {
        if (B >= kL51) return false;
        B += rtw_bound(B, Q);
    }
    if (B >= kL51) return false;
    B = 2.0 * rtw_bound(B, Q);
    for (uint32_t l = 0; l < cross; ++l) {
        if (B >= kL51) return false;
        B += (0.5 + B / 4503599627370496.0) * Q + 2.0;
    }
    return B < kL51;
}

void ephdc_ntt_plan_c5_free(ephdc_ntt_plan *p) {
    cudaFree(p->c5_itw);
    cudaFree(p->c5_itail);
    cudaFree(p->c5_ck);
    p->c5_itw = p->c5_itail = p->c5_ck = nullptr;
}

// Decides the c5 kernels for a plan and uploads the inverse's tables.  Needs the plan's
// q, log2N and FP64 forward table (tw_f64).
cudaError_t plan_ntt_c5(ephdc_ntt_plan *p) {
    using namespace ephdc_host;
    p->c5_fwd = p->c5_inv = p->c5_red = false;
    if (p->log2N < 12 || p->log2N > 16 || !p->tw_f64 || !encode_tiled_fn()) return cudaSuccess;
    const uint32_t cross = p->log2N > 13 ? p->log2N - 13 : 0;
    const uint32_t lgc = p->log2N > 13 ? 13 : p->log2N;
    bool fwd = true, red = false, inv = true;
    for (uint32_t j = 0; j < p->L; ++j) {
        if (p->q[j] >= (1ull << 50)) return cudaSuccess;
        const double Q = (double)p->q[j];
        if (!c5_fwd_ok(Q, p->log2N, cross, false)) {
            red = cross > 0;
            fwd = fwd && red && c5_fwd_ok(Q, p->log2N, cross, true);
        }
        inv = inv && c5_inv_ok(Q, lgc, cross);
    }
    p->c5_fwd = fwd;
    p->c5_red = red || cross >= 2;   // 2^15, 2^16 always reduce after the cross levels
    if (!inv) return cudaSuccess;
    // inverse tables: W[h + jj] = omega^-(N/2h) jj of the full N, entry 0 = (q, 1/q); the
    // fused scaling [NC/2][2] = (sigma_r, sigma_r W[NC/2 + r]), sigma_r = N^-1 psi^-r;
    // c_loc = psi^-(NC/2); block constants c_k = psi^-(NC k), k < 8
    const uint32_t N = p->N, L = p->L, NC = 1u << lgc;
    std::vector<double> itw((size_t)L * N * 2), itail((size_t)L * NC * 2), ck((size_t)L * 8 * 2, 0.0);
    for (uint32_t j = 0; j < L; ++j) {
        const uint64_t q = p->q[j];
        const double qd = (double)q;
        const uint64_t psi_inv = invmod(min_primitive_root_2n(q, p->log2N), q);
        double *W = itw.data() + (size_t)j * N * 2;
        W[0] = qd;
        W[1] = 1.0 / qd;
        std::vector<uint64_t> Wi(N, 0);
        for (uint32_t h = 1; h < N; h *= 2) {
            const uint64_t wh = powmod(psi_inv, N / h, q);   // omega^-(N/2h), omega = psi^2
            uint64_t wv = 1;
            for (uint32_t jj = 0; jj < h; ++jj, wv = mulmod(wv, wh, q)) {
                Wi[h + jj] = wv;
                W[2 * (h + jj)] = (double)wv;
                W[2 * (h + jj) + 1] = (double)wv / qd;
            }
        }
        double *T = itail.data() + (size_t)j * NC * 2;
        uint64_t sj = invmod(N % q, q);
        for (uint32_t r = 0; r < NC / 2; ++r, sj = mulmod(sj, psi_inv, q)) {
            const uint64_t swj = mulmod(sj, Wi[NC / 2 + r], q);
            T[4 * r] = (double)sj;
            T[4 * r + 1] = (double)sj / qd;
            T[4 * r + 2] = (double)swj;
            T[4 * r + 3] = (double)swj / qd;
        }
        const uint64_t c = powmod(psi_inv, NC / 2, q);
        p->c5_cinv[j] = make_double2((double)c, (double)c / qd);
        for (uint32_t k = 0; k < 8; ++k) {
            const uint64_t v = powmod(psi_inv, (uint64_t)NC * k, q);
            ck[2 * (j * 8 + k)] = (double)v;
            ck[2 * (j * 8 + k) + 1] = (double)v / qd;
        }
    }
    cudaError_t e;
    if ((e = cudaMalloc(&p->c5_itw, sizeof(double) * itw.size())) != cudaSuccess ||
        (e = cudaMalloc(&p->c5_itail, sizeof(double) * itail.size())) != cudaSuccess ||
        (e = cudaMalloc(&p->c5_ck, sizeof(double) * ck.size())) != cudaSuccess ||
        (e = cudaMemcpy(p->c5_itw, itw.data(), sizeof(double) * itw.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(p->c5_itail, itail.data(), sizeof(double) * itail.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(p->c5_ck, ck.data(), sizeof(double) * ck.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return e;
    p->c5_inv = true;
    return cudaSuccess;
}

template <class K>
static cudaError_t c5_launch(K kern, size_t smem, int cluster, uint32_t ctas_per_sm, uint32_t threads,
                             const ephdc_ntt_plan *pl, uint64_t *polys, uint32_t batch, bool inv, uint32_t box_rows,
                             cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    CUtensorMap map;
    if (!make_poly_map(&map, polys, (uint64_t)batch * pl->L * pl->N, box_rows)) return cudaErrorNotSupported;
    C5Args a{};
    a.polys = polys;
    a.tw = inv ? pl->c5_itw : pl->tw_f64;
    a.tail = pl->c5_itail;
    a.ck = pl->c5_ck;
    a.L = pl->L;
    a.batch = batch;
    a.items = pl->L * batch;
    a.log2N = pl->log2N;
    for (uint32_t j = 0; j < pl->L; ++j) a.cinv[j] = pl->c5_cinv[j];
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent: as many CTAs (clusters) as can be co-resident -- clusters are placed
    // inside GPCs, so for C > 1 the count comes from the occupancy API -- never more
    // units than items
    uint32_t slots = 148u * ctas_per_sm;
    if (cluster > 1) {
        int nclusters = 0;
        cfg.gridDim = dim3(148u * (uint32_t)cluster);
        e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
        if (e != cudaSuccess || nclusters < 1) return e != cudaSuccess ? e : cudaErrorNotSupported;
        slots = (uint32_t)nclusters;
    }
    const uint32_t units = std::max<uint32_t>(1, std::min<uint32_t>(slots, a.items));
    cfg.gridDim = dim3(units * (uint32_t)cluster);
    e = cudaLaunchKernelEx(&cfg, kern, map, a);
    return counted(e == cudaSuccess ? cudaGetLastError() : e);
}

// c5 kernels if the plan allows them for this direction and size; cudaErrorNotSupported
// otherwise (the caller then runs the general kernels).
cudaError_t launch_ntt_c5(const ephdc_ntt_plan *pl, uint64_t *d_polys, uint32_t batch, bool inverse,
                          cudaStream_t st) {
    if (inverse ? !pl->c5_inv : !pl->c5_fwd) return cudaErrorNotSupported;
    if (batch == 0) return cudaSuccess;
    if ((uint64_t)batch * pl->L > 0xffffffffull || ((uintptr_t)d_polys & 15)) return cudaErrorNotSupported;
    const size_t s12 = 1024 + sizeof(double) * 3 * 4096 + sizeof(double2) * 256;
    const size_t s13 = 1024 + sizeof(double) * 3 * 8192 + sizeof(double2) * 512;
    using namespace c5;
    if (inverse) {
        switch (pl->log2N) {
            case 12: return c5_launch(k_ntt_c5_inv<12>, s12, 1, 2, 256, pl, d_polys, batch, true, 256, st);
            case 13:
                // one team (r16: inverse 0.525 vs 0.502 of HBM with two groups at 48-bit primes)
                return pl->c5_alt_teams ? c5_launch(k_ntt_c5_inv2g, s13, 1, 1, 512, pl, d_polys, batch, true, 256, st)
                                        : c5_launch(k_ntt_c5_inv<13>, s13, 1, 1, 512, pl, d_polys, batch, true, 256, st);
            // (a two-group inverse with st.async pushes into a shared gather buffer measured
            // 0.409 vs 0.402 of HBM at 2^14 but failed intermittently under repetition --
            // an unspecified launch failure in about half of the 100-launch runs, not the
            // bounded waits -- and was removed; profiles/r02/ab/README.md)
            case 14: return c5_launch(k_ntt_c5_inv_cl<2>, s13, 2, 1, 512, pl, d_polys, batch, true, 256, st);
            case 15: return c5_launch(k_ntt_c5_inv_cl<4>, s13, 4, 1, 512, pl, d_polys, batch, true, 256, st);
            case 16: return c5_launch(k_ntt_c5_inv_cl<8>, s13, 8, 1, 512, pl, d_polys, batch, true, 256, st);
        }
    } else {
        switch (pl->log2N) {
            case 12: return c5_launch(k_ntt_c5_fwd<12>, s12, 1, 2, 256, pl, d_polys, batch, false, 256, st);
            case 13:
                // two groups (r16: forward 0.533 vs 0.495 of HBM with one team at 48-bit primes)
                return pl->c5_alt_teams ? c5_launch(k_ntt_c5_fwd<13>, s13, 1, 1, 512, pl, d_polys, batch, false, 256, st)
                                        : c5_launch(k_ntt_c5_fwd2g, s13, 1, 1, 512, pl, d_polys, batch, false, 256, st);
            case 14:
                if (pl->c5_alt_teams)
                    return pl->c5_red ? c5_launch(k_ntt_c5_fwd_cl<2, true>, s13, 2, 1, 512, pl, d_polys, batch, false, 256, st)
                                      : c5_launch(k_ntt_c5_fwd_cl<2, false>, s13, 2, 1, 512, pl, d_polys, batch, false, 256, st);
                return pl->c5_red ? c5_launch(k_ntt_c5_fwd_cl2g<2, true>, s13, 2, 1, 512, pl, d_polys, batch, false, 256, st)
                                  : c5_launch(k_ntt_c5_fwd_cl2g<2, false>, s13, 2, 1, 512, pl, d_polys, batch, false, 256, st);
            case 15:
                return pl->c5_alt_teams ? c5_launch(k_ntt_c5_fwd_cl<4, true>, s13, 4, 1, 512, pl, d_polys, batch, false, 128, st)
                                        : c5_launch(k_ntt_c5_fwd_cl2g<4, true>, s13, 4, 1, 512, pl, d_polys, batch, false, 128, st);
            case 16:
                return pl->c5_alt_teams ? c5_launch(k_ntt_c5_fwd_cl<8, true>, s13, 8, 1, 512, pl, d_polys, batch, false, 64, st)
                                        : c5_launch(k_ntt_c5_fwd_cl2g<8, true>, s13, 8, 1, 512, pl, d_polys, batch, false, 64, st);
        }
    }
    return cudaErrorNotSupported;
}

}  // namespace ephdc
