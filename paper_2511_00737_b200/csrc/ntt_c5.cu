// ntt_c5.cu -- the standalone negacyclic NTT of the c5 microbench (BASELINE.json
// configs[4]) on B200, for primes q < 2^50: FP64 pipe + integer pipe.
//
// Forward N = 2^12, 2^13 (one CTA per polynomial) and 2^14 (a 2-CTA cluster, one output
// half per CTA); inverse N = 2^12, 2^13.  In place on [batch][L][N] canonical u64.
// Per CTA:
//   * persistent over a contiguous range of (prime, polynomial) items, prime-major: the
//     twiddles of a prime are loaded once -- the low levels (broadcast / warp-uniform /
//     lane-consecutive reads) in shared memory, the thread's own pass-3 and last-level
//     twiddles (23-26 (w, w/q) pairs) in TENSOR MEMORY, idle in a kernel without MMAs;
//   * three 64 KB buffers: polynomial i+2 arrives by TMA (cp.async.bulk.tensor.2d,
//     SWIZZLE_128B, 32 KB boxes: two copies per polynomial) while polynomial i is
//     transformed.  The passes are chosen so that every access is conflict-free in the
//     swizzled layout: forward 4+4+R3+2 levels (the last two as radix-4 groups of four
//     consecutive elements read as 16-byte pairs), inverse 2+3+4+4;
//   * the cheap levels on the INTEGER pipe (forward level 0: u64 Shoup product; inverse
//     level 0: twiddle 1, adds only) and the reduction to [0, q) (Barrett), the rest on
//     the FP64 pipe with the exact double arithmetic of modf64.cuh (8 FP64 ops per
//     butterfly) -- the FP64 pipe, which bounds these kernels, does the butterflies and
//     two exact conversions per element (the 1.5*2^52 bias);
//   * one CTA barrier per polynomial: forward pass 1 (levels 0-3, all-to-all) -> barrier
//     -> passes 2, 3, tail inside each warp's 512-element window (__syncwarp) -> 16-byte
//     stores straight from registers; inverse passes A-C warp-local -> barrier -> pass D
//     with the last level fused with the scaling by N^-1 psi^-j.
// Forward N = 2^14: both CTAs of the cluster read both input halves and compute global
// level 0 redundantly on the integer pipe; a split cluster barrier (arrive after pass 1,
// wait before the stores) keeps either CTA from overwriting input its partner has not
// consumed.  DESIGN.md 5.2 "c5 standalone NTT".
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

constexpr int kE = 16;      // elements per thread per pass
constexpr int kNBuf = 3;    // data buffers per CTA
constexpr int kBoxRows = 256;   // TMA box: 256 rows x 16 u64 (32 KB)
#ifndef EPHDC_C5_L0F
#define EPHDC_C5_L0F 1
#endif
#ifndef EPHDC_C5_OUTF
#define EPHDC_C5_OUTF 1
#endif
constexpr bool kL0F = EPHDC_C5_L0F != 0;    // A/B build switches (tools/ab_c5.sh), not runtime knobs:
constexpr bool kOUTF = EPHDC_C5_OUTF != 0;  // level 0 / the final reduction on the FP64 pipe

// SWIZZLE_128B: element e (8 bytes) of a 1024-byte-aligned buffer sits at e ^ (((e >> 4) & 7) << 1)
// The map is linear over XOR, so for index parts with disjoint bits sw(a + b) =
// sw(a) ^ sw(b): every pass computes sw(base) once and XORs compile-time constants.
__host__ __device__ constexpr int sw(int e) { return e ^ (((e >> 4) & 7) << 1); }
template <int LGC> constexpr int ctas_per_sm() { return LGC <= 12 ? 2 : 1; }
template <int LGC> constexpr int tw_smem(bool inv) { return inv && LGC >= 13 ? 512 : 256; }
template <int LGC, bool INV> constexpr size_t smem_bytes() {
    return 1024 + sizeof(double) * kNBuf * (1 << LGC) + sizeof(double2) * tw_smem<LGC>(INV);
}
template <int LGC> constexpr uint32_t tmem_cols() { return 128u * (uint32_t)(((1 << LGC) / kE / 32 + 3) / 4); }

// exact int64 <-> double for |v| < 2^51 (1.5 * 2^52 bias: one DADD each way)
EPHDC_D double i2d(long long v) {
    return __dsub_rn(__longlong_as_double(v + 0x4338000000000000LL), 6755399441055744.0);
}
EPHDC_D long long d2i(double x) {
    return __double_as_longlong(__dadd_rn(x, 6755399441055744.0)) - 0x4338000000000000LL;
}
// y * w mod q in [0, 2q) (Shoup, wp = floor(w 2^64 / q)), any y < 2^64
EPHDC_D u64 shoup(u64 y, u64 w, u64 wp, u64 q) { return y * w - __umul64hi(y, wp) * q; }
// v in [0, 2q) -> the centered representative in (-q/2, q/2] (hq = (q-1)/2)
EPHDC_D long long center2(u64 v, u64 q, u64 hq) {
    const u64 r = v >= q ? v - q : v;
    return r > hq ? (long long)r - (long long)q : (long long)r;
}
// x -> x mod q in [0, q) for |x| < off = K q, y = x + off < 2^53: Barrett with
// bm = floor(2^64 / q).  BIGQ (q > 2^32, so bm < 2^32): floor(y bm / 2^64) =
// (hi32(y) bm + mulhi32(lo32(y), bm)) >> 32 exactly (the dropped fraction is < 1 and
// the sum is an integer), three integer multiplies instead of a 64x64 high product.
template <bool BIGQ> EPHDC_D u64 canon(long long x, u64 q, u64 bm, u64 off) {
    const u64 y = (u64)(x + (long long)off);
    u64 k;
    if constexpr (BIGQ) k = ((y >> 32) * bm + __umulhi((u32)y, (u32)bm)) >> 32;
    else k = __umul64hi(y, bm);
    const u64 r = y - k * q;
    return r >= q ? r - q : r;
}

// final value (|x| < off) -> canonical u64: FP64 reduction or integer Barrett (A/B switch)
template <bool BIGQ>
EPHDC_D u64 out_u64(double x, double q, double nq, double qinv, u64 qi, u64 bm, u64 off) {
    if constexpr (kOUTF) return to_canonical_u64(reduce(x, qinv, nq), q);
    else return canon<BIGQ>(d2i(x), qi, bm, off);
}

EPHDC_D void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            ephdc_async::smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(ephdc_async::smem_u32(bar))
        : "memory");
}
EPHDC_D void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
EPHDC_D void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
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

// Shared frame of both kernels: buffers, the TMA ring, the item range.
template <int LGC, int S> struct Frame {
    static constexpr int NC = 1 << LGC, N = NC * S, NT = NC / kE;
    double *bufs;      // [3][NC], 1024-byte aligned
    double2 *tws;      // [tw_smem]
    uint64_t *mbar;    // [3]
    u32 s, w0, w1;

    EPHDC_D double *buf(u32 b) const { return bufs + (size_t)b * NC; }
    EPHDC_D u64 *poly(const C5Args &a, u32 w) const {
        const u32 j = w / a.batch, b = w - j * a.batch;
        return a.polys + ((size_t)b * a.L + j) * N;
    }
    // one thread: the TMA copies of item i (S = 1: into buffer i % 3; S = 2: the half H0
    // into buffer 2 (i & 1), H1 into buffer 1)
    EPHDC_D void issue(const C5Args &a, const CUtensorMap *map, u32 i) const {
        using namespace ephdc_async;
        const u32 w = w0 + i, j = w / a.batch, b = w - j * a.batch;
        const int row0 = (int)((((size_t)b * a.L + j) * N) >> 4);
        uint64_t *bar = &mbar[S == 1 ? i % 3 : (i & 1)];
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, (u32)(S * NC * 8));
        double *c = buf(S == 1 ? i % 3 : 2 * (i & 1));
#pragma unroll
        for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(c + 16 * r, map, 0, row0 + r, bar);
        if constexpr (S == 2) {
#pragma unroll
            for (int r = 0; r < NC / 16; r += kBoxRows) tma_load_2d(buf(1) + 16 * r, map, 0, row0 + NC / 16 + r, bar);
        }
    }
    EPHDC_D void wait(u32 i) const {
        if constexpr (S == 1) ephdc_async::mbar_wait(&mbar[i % 3], (i / 3) & 1u);
        else ephdc_async::mbar_wait(&mbar[i & 1], (i >> 1) & 1u);
    }
};

// ---------------------------------------------------------------------------------
// Forward.  Level lv of the CTA's NC-point transform has 2^lv blocks of half-size
// NC >> (lv+1); its twiddle for block B is psi_rev[S m + s m + B], m = 2^lv (S = 2: the
// CTA owns blocks [s m, (s+1) m) of global level lv+1; global level 0 is the redundant
// integer stage).  Passes: 1 = levels 0-3, 2 = 4-7, 3 = 8 .. LGC-3 (R3 levels, groups of
// 2^R3 elements 4 apart), tail = LGC-2, LGC-1 (four consecutive elements).
// ---------------------------------------------------------------------------------
template <int LGC, int S, bool BIGQ>
__global__ void __launch_bounds__((1 << LGC) / kE, ctas_per_sm<LGC>())
    k_ntt_c5_fwd(const __grid_constant__ CUtensorMap map, const __grid_constant__ C5Args a) {
    static_assert(LGC == 12 || LGC == 13, "NC = 2^12 or 2^13 per CTA");
    using F = Frame<LGC, S>;
    constexpr int NC = F::NC, N = F::N, NT = F::NT;
    constexpr int R3 = LGC - 10, G3 = kE >> R3;   // pass 3: levels, groups per thread
    constexpr int TL2 = NC >> 8, NB8 = NC >> 8;    // pass 2 stride, level-8 block size
    constexpr uint32_t kCols = tmem_cols<LGC>();
    constexpr uint32_t kP3Cols = R3 == 3 ? 32u : 16u;   // TMEM columns per pass-3 group
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    F f;
    f.bufs = reinterpret_cast<double *>(smem_raw + ((1024u - (ephdc_async::smem_u32(smem_raw) & 1023u)) & 1023u));
    f.tws = reinterpret_cast<double2 *>(f.bufs + kNBuf * NC);
    f.mbar = mbar;
    f.s = blockIdx.x % S;
    const u32 unit = blockIdx.x / S, nunits = gridDim.x / S;
    f.w0 = (u32)((u64)a.items * unit / nunits);
    f.w1 = (u32)((u64)a.items * (unit + 1) / nunits);
    const u32 s = f.s, w0 = f.w0, w1 = f.w1;

    if (tid == 0)
        for (int b = 0; b < kNBuf; ++b) ephdc_async::mbar_init(&mbar[b], 1);
    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, kCols);
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    const uint32_t tbase = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 128u;
    if (tid == 0 && w0 < w1) {
        f.issue(a, &map, 0);
        if (S == 1 && w0 + 1 < w1) f.issue(a, &map, 1);
    }
    // pass-3 groups: a warp's groups cover its 512-element window and every half-warp
    // touches 16 distinct bank pairs (the bank model in DESIGN.md 5.2)
    auto p3_blk = [&](int u) -> int {
        return R3 == 3 ? 16 * warp + (lane >> 2) + 8 * u : 32 * warp + ((lane >> 1) & 15) + 16 * (u >> 1);
    };
    auto p3_off = [&](int u) -> int { return R3 == 3 ? (lane & 3) : ((lane & 1) | ((u & 1) << 1)); };

    u32 jcur = 0xffffffffu;
    double nq = 0.0;
    u64 qi = 0, hq = 0, wi = 0, wip = 0, bm = 0, off = 0;
    double qinv = 0.0;
    for (u32 i = 0; w0 + i < w1; ++i) {
        const u32 w = w0 + i, j = w / a.batch;
        if (j != jcur) {   // twiddles of prime j: levels 0-7 -> shared, pass 3 + tail -> TMEM
            __syncthreads();
            const double2 *twg = a.tw + (size_t)j * N;
            auto gtw = [&](int m, int B) { return twg[S * m + (int)s * m + B]; };
            for (int p = tid; p < 256; p += NT) {   // pass layout: slot (m0 << sub) + v m0 + B
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
                            put_pair(&r[4 * k], gtw(256 << sub, (p3_blk(u) << sub) + v));
                        } else {
                            put_pair(&r[4 * k], make_double2(0.0, 0.0));
                        }
                    }
                    ephdc_tmem::stx<16>(tbase + kP3Cols * u + 16u * h, r);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {   // tail group g4: levels LGC-2 (block g4), LGC-1 (2 g4, 2 g4 + 1)
                const int g4 = 128 * warp + lane + 32 * u;
                put_pair(&r[0], gtw(NC / 4, g4));
                put_pair(&r[4], gtw(NC / 2, 2 * g4));
                put_pair(&r[8], gtw(NC / 2, 2 * g4 + 1));
                put_pair(&r[12], make_double2(0.0, 0.0));
                ephdc_tmem::stx<16>(tbase + 64u + 16u * u, r);
            }
            ephdc_tmem::wait_st();
            nq = -twg[0].x;
            qinv = twg[0].y;
            qi = a.q[j];
            hq = (qi - 1) / 2;
            wi = a.w1[j];
            wip = a.w1p[j];
            bm = a.bm[j];
            off = a.off[j];
            jcur = j;
            ephdc_tmem::fence_before_sync();
            __syncthreads();
            ephdc_tmem::fence_after_sync();
        }
        f.wait(i);
        double *C = f.buf(S == 1 ? i % 3 : 2 * (i & 1));

        // ---- pass 1: levels 0-3 (level 0 on the integer pipe), elements tid + k NT
        {
            const u64 *Cu = reinterpret_cast<const u64 *>(C);
            const int st = sw(tid);
            double x[16];
            if constexpr (S == 1 && kL0F) {   // A/B variant: level 0 on the FP64 pipe
                const double q = -nq, hqd = 0.5 * q;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double v = from_u64(Cu[st ^ sw(k * NT)]);
                    x[k] = v > hqd ? __dsub_rn(v, q) : v;
                }
                ct_stages<4, 0, 4>(x, [&](int sub, int v) { return f.tws[(1 << sub) + v]; }, nq);
            } else if constexpr (S == 1) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const u64 u0 = Cu[st ^ sw(k * NT)], u1 = Cu[st ^ sw((k + 8) * NT)];
                    u64 t = shoup(u1, wi, wip, qi);
                    t = t >= qi ? t - qi : t;                                      // [0, q)
                    x[k] = i2d(center2(u0 + t, qi, hq));                           // (-q/2, q/2]
                    x[k + 8] = i2d(center2(u0 + qi - t, qi, hq));
                }
                ct_stages<4, 1, 4>(x, [&](int sub, int v) { return f.tws[(1 << sub) + v]; }, nq);
            } else {
                const u64 *Au = reinterpret_cast<const u64 *>(f.buf(1));
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int e = st ^ sw(k * NT);
                    u64 t = shoup(Au[e], wi, wip, qi);
                    t = t >= qi ? t - qi : t;
                    const u64 u0 = Cu[e];
                    x[k] = i2d(center2(s == 0 ? u0 + t : u0 + qi - t, qi, hq));   // (-q/2, q/2]
                }
                ct_stages<4, 0, 4>(x, [&](int sub, int v) { return f.tws[(1 << sub) + v]; }, nq);
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) C[st ^ sw(k * NT)] = x[k];
        }
        __syncthreads();
        if (tid == 0) {   // the buffer pass 1 freed (S = 2) / the previous item's (S = 1)
            if constexpr (S == 1) {
                if (w0 + i + 2 < w1) f.issue(a, &map, i + 2);
            } else {
                if (w0 + i + 1 < w1) f.issue(a, &map, i + 1);
            }
        }
        if constexpr (S == 2) cluster_arrive();   // this CTA consumed item i's input

        // ---- pass 2: levels 4-7; a warp's groups lie in its 512-element window
        {
            const int blk = tid / TL2, off2 = tid % TL2, sb = sw(blk * (NC / 16) + off2);
            double x[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = C[sb ^ sw(k * TL2)];
            ct_stages<4, 0, 4>(x, [&](int sub, int v) { return f.tws[(16 << sub) + v * 16 + blk]; }, nq);
#pragma unroll
            for (int k = 0; k < 16; ++k) C[sb ^ sw(k * TL2)] = x[k];
        }
        __syncwarp();
        // ---- pass 3: levels 8 .. LGC-3, groups of 2^R3 elements 4 apart, twiddles from TMEM
#pragma unroll
        for (int u = 0; u < G3; ++u) {
            const int sb = sw(p3_blk(u) * NB8 + p3_off(u));
            double x[1 << R3];
#pragma unroll
            for (int k = 0; k < (1 << R3); ++k) x[k] = C[sb ^ sw(4 * k)];
            if constexpr (R3 == 3) {
                uint32_t rr[32];
                ephdc_tmem::ldx<16>(tbase + kP3Cols * u, *reinterpret_cast<uint32_t(*)[16]>(&rr[0]));
                ephdc_tmem::ldx<16>(tbase + kP3Cols * u + 16u, *reinterpret_cast<uint32_t(*)[16]>(&rr[16]));
                ephdc_tmem::waitx<32>(rr);
                ct_stages<R3, 0, R3>(x, [&](int sub, int v) { return pair_at(rr, (1 << sub) - 1 + v); }, nq);
            } else {
                uint32_t rr[16];
                ephdc_tmem::ldx<16>(tbase + kP3Cols * u, rr);
                ephdc_tmem::waitx<16>(rr);
                ct_stages<R3, 0, R3>(x, [&](int sub, int v) { return pair_at(rr, (1 << sub) - 1 + v); }, nq);
            }
#pragma unroll
            for (int k = 0; k < (1 << R3); ++k) C[sb ^ sw(4 * k)] = x[k];
        }
        __syncwarp();
        if constexpr (S == 2) cluster_wait();     // the partner consumed item i's input
        // ---- tail: levels LGC-2, LGC-1 on four consecutive elements, reduction to [0, q),
        //      16-byte stores
        {
            u64 *o = f.poly(a, w) + (size_t)s * NC;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int g4 = 128 * warp + lane + 32 * u;
                uint32_t rr[16];
                ephdc_tmem::ldx<16>(tbase + 64u + 16u * u, rr);
                const int sg = sw(4 * g4);
                const double2 xa = *reinterpret_cast<const double2 *>(C + sg);
                const double2 xb = *reinterpret_cast<const double2 *>(C + (sg ^ 2));
                ephdc_tmem::waitx<16>(rr);
                double x0 = xa.x, x1 = xa.y, x2 = xb.x, x3 = xb.y;
                const double2 t0 = pair_at(rr, 0), t1 = pair_at(rr, 1), t2 = pair_at(rr, 2);
                ct_bfly(x0, x2, t0.x, t0.y, nq);
                ct_bfly(x1, x3, t0.x, t0.y, nq);
                ct_bfly(x0, x1, t1.x, t1.y, nq);
                ct_bfly(x2, x3, t2.x, t2.y, nq);
                auto oc = [&](double v) { return out_u64<BIGQ>(v, -nq, nq, qinv, qi, bm, off); };
                st_cs_v2(o + 4 * g4, oc(x0), oc(x1));
                st_cs_v2(o + 4 * g4 + 2, oc(x2), oc(x3));
            }
        }
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_slot, kCols);
    if constexpr (S == 2) {   // no CTA of the pair may exit while its partner can still arrive
        cluster_arrive();
        cluster_wait();
    }
}

// ---------------------------------------------------------------------------------
// Inverse (N = 2^12, 2^13).  Cooley-Tukey DIT on the bit-reversed input: level lv pairs
// (j, j + h), h = 2^lv, inside blocks of 2h with twiddle W[h + (j mod h)] =
// omega^-(N/2h)(j mod h) (omega = psi^2); after all levels the values are N a_j psi^j.
// The last level is fused with the scaling by s_j = N^-1 psi^-j:
//     a_j = s_j X + (s_j W_j) Y,   a_{j+N/2} = c (s_j X - (s_j W_j) Y),   c = psi^-N/2
// (s_{j+N/2} = s_j c): three products per pair with the thread's pairs (s_j, s_j W_j) in
// TMEM -- no scaling table streamed.  Level 0 (twiddle 1: adds only) on the integer
// pipe.  Passes: A = levels 0-1 (four consecutive elements), B = 2-4 (groups of 8, 4
// apart), C = 5 .. LGC-5 (stride 32, warp-local), D = the last four (stride NT).
// ---------------------------------------------------------------------------------
template <int LGC, bool BIGQ>
__global__ void __launch_bounds__((1 << LGC) / kE, ctas_per_sm<LGC>())
    k_ntt_c5_inv(const __grid_constant__ CUtensorMap map, const __grid_constant__ C5Args a) {
    static_assert(LGC == 12 || LGC == 13, "NC = 2^12 or 2^13 per CTA");
    using F = Frame<LGC, 1>;
    constexpr int NC = F::NC, N = F::N, NT = F::NT;
    constexpr int RC = LGC - 9, GC = kE >> RC;   // pass C: levels 5 .. 4+RC, groups per thread
    constexpr uint32_t kCols = tmem_cols<LGC>();
    constexpr int TWS = tw_smem<LGC>(true);
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    F f;
    f.bufs = reinterpret_cast<double *>(smem_raw + ((1024u - (ephdc_async::smem_u32(smem_raw) & 1023u)) & 1023u));
    f.tws = reinterpret_cast<double2 *>(f.bufs + kNBuf * NC);
    f.mbar = mbar;
    f.s = 0;
    f.w0 = (u32)((u64)a.items * blockIdx.x / gridDim.x);
    f.w1 = (u32)((u64)a.items * (blockIdx.x + 1) / gridDim.x);
    const u32 w0 = f.w0, w1 = f.w1;

    if (tid == 0)
        for (int b = 0; b < kNBuf; ++b) ephdc_async::mbar_init(&mbar[b], 1);
    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, kCols);
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    const uint32_t tbase = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 128u;
    if (tid == 0 && w0 < w1) {
        f.issue(a, &map, 0);
        if (w0 + 1 < w1) f.issue(a, &map, 1);
    }

    u32 jcur = 0xffffffffu;
    double nq = 0.0;
    double2 cc = make_double2(0.0, 0.0);
    u64 qi = 0, hq = 0, bm = 0, off = 0;
    double qinv = 0.0;
    for (u32 i = 0; w0 + i < w1; ++i) {
        const u32 w = w0 + i, j = w / a.batch;
        if (j != jcur) {   // DIT table of prime j: [1, TWS) -> shared; pass D + scaling -> TMEM
            __syncthreads();
            const double2 *twg = a.tw + (size_t)j * N;
            const double2 *tl = a.tail + (size_t)j * N;   // [N/2][2] (s_j, s_j W_j)
            for (int p = tid; p < TWS; p += NT) f.tws[p] = twg[p];
            uint32_t r[16];
            // pass D levels LGC-4 .. LGC-2: sub-stage sub, block position kk at pair
            // index 2^sub - 1 + kk: W[NT 2^sub + tid + NT kk]; columns [0, 32)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int idx = 4 * h + k;
                    if (idx < 7) {
                        const int sub = 31 - __clz(idx + 1), kk = idx + 1 - (1 << sub);
                        put_pair(&r[4 * k], twg[(NT << sub) + tid + NT * kk]);
                    } else {
                        put_pair(&r[4 * k], make_double2(0.0, 0.0));
                    }
                }
                ephdc_tmem::stx<16>(tbase + 16u * h, r);
            }
            // last level: j = tid + NT k (k < 8), (s_j, s_j W_j) at columns 32 + 8k
#pragma unroll
            for (int h = 0; h < 4; ++h) {
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int jj = tid + NT * (2 * h + v);
                    put_pair(&r[8 * v], tl[2 * jj]);
                    put_pair(&r[8 * v + 4], tl[2 * jj + 1]);
                }
                ephdc_tmem::stx<16>(tbase + 32u + 16u * h, r);
            }
            ephdc_tmem::wait_st();
            nq = -twg[0].x;
            qinv = twg[0].y;
            cc = a.cinv[j];
            qi = a.q[j];
            hq = (qi - 1) / 2;
            bm = a.bm[j];
            off = a.off[j];
            jcur = j;
            ephdc_tmem::fence_before_sync();
            __syncthreads();
            ephdc_tmem::fence_after_sync();
        }
        f.wait(i);
        double *C = f.buf(i % 3);

        // ---- pass A: levels 0 (integer pipe: twiddle 1) and 1 on four consecutive elements
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int g4 = 128 * warp + lane + 32 * u;
            const int sg = sw(4 * g4);
            const ulonglong2 ua = *reinterpret_cast<const ulonglong2 *>(C + sg);
            const ulonglong2 ub = *reinterpret_cast<const ulonglong2 *>(C + (sg ^ 2));
            double x0, x1, x2, x3;
            if constexpr (kL0F) {   // A/B variant: centered doubles, level 0 as FP64 adds
                const double q = -nq, hqd = 0.5 * q;
                auto cv = [&](u64 u) { const double v = from_u64(u); return v > hqd ? __dsub_rn(v, q) : v; };
                const double v0 = cv(ua.x), v1 = cv(ua.y), v2 = cv(ub.x), v3 = cv(ub.y);
                x0 = __dadd_rn(v0, v1), x1 = __dsub_rn(v0, v1), x2 = __dadd_rn(v2, v3), x3 = __dsub_rn(v2, v3);
            } else {
                x0 = i2d(center2(ua.x + ua.y, qi, hq)), x1 = i2d(center2(ua.x + qi - ua.y, qi, hq));
                x2 = i2d(center2(ub.x + ub.y, qi, hq)), x3 = i2d(center2(ub.x + qi - ub.y, qi, hq));
            }
            const double2 t2 = f.tws[2], t3 = f.tws[3];
            ct_bfly(x0, x2, t2.x, t2.y, nq);
            ct_bfly(x1, x3, t3.x, t3.y, nq);
            *reinterpret_cast<double2 *>(C + sg) = make_double2(x0, x1);
            *reinterpret_cast<double2 *>(C + (sg ^ 2)) = make_double2(x2, x3);
        }
        __syncwarp();
        // ---- pass B: levels 2-4, blocks of 32, groups of 8 elements 4 apart
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int blk = 16 * warp + (lane >> 2) + 8 * u, off4 = lane & 3, sb = sw(32 * blk + off4);
            double x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = C[sb ^ sw(4 * k)];
            dit_stages<3, 0, 3>(x, [&](int sub, int kk) { return f.tws[(4 << sub) + off4 + 4 * kk]; }, nq);
#pragma unroll
            for (int k = 0; k < 8; ++k) C[sb ^ sw(4 * k)] = x[k];
        }
        __syncwarp();
        // ---- pass C: levels 5 .. 4+RC, elements 2^(5+RC) blk + lane + 32 k (warp-local)
#pragma unroll
        for (int u = 0; u < GC; ++u) {
            const int blk = GC * warp + u, sb = sw((blk << (5 + RC)) + lane);
            double x[1 << RC];
#pragma unroll
            for (int k = 0; k < (1 << RC); ++k) x[k] = C[sb ^ sw(32 * k)];
            dit_stages<RC, 0, RC>(x, [&](int sub, int kk) { return f.tws[(32 << sub) + lane + 32 * kk]; }, nq);
#pragma unroll
            for (int k = 0; k < (1 << RC); ++k) C[sb ^ sw(32 * k)] = x[k];
        }
        __syncthreads();
        if (tid == 0 && w0 + i + 2 < w1) f.issue(a, &map, i + 2);   // item i-1's buffer is free
        // ---- pass D: the last four levels, elements tid + NT k; the last fused with the scaling
        {
            double x[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = C[sw(tid) ^ sw(NT * k)];
            {
                uint32_t rr[32];
                ephdc_tmem::ldx<16>(tbase, *reinterpret_cast<uint32_t(*)[16]>(&rr[0]));
                ephdc_tmem::ldx<16>(tbase + 16u, *reinterpret_cast<uint32_t(*)[16]>(&rr[16]));
                ephdc_tmem::waitx<32>(rr);
                dit_stages<4, 0, 3>(x, [&](int sub, int kk) { return pair_at(rr, (1 << sub) - 1 + kk); }, nq);
            }
            u64 *o = f.poly(a, w);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                uint32_t rr[16];
                ephdc_tmem::ldx<16>(tbase + 32u + 16u * h, rr);
                ephdc_tmem::waitx<16>(rr);
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int k = 2 * h + v, jj = tid + NT * k;
                    const double2 sj = pair_at(rr, 2 * v), swj = pair_at(rr, 2 * v + 1);
                    const double A = mul_tw(x[k], sj.x, sj.y, nq), Bv = mul_tw(x[k + 8], swj.x, swj.y, nq);
                    const double lo = __dadd_rn(A, Bv), hi = mul_tw(__dsub_rn(A, Bv), cc.x, cc.y, nq);
                    __stcs(reinterpret_cast<unsigned long long *>(o + jj),
                           (unsigned long long)out_u64<BIGQ>(lo, -nq, nq, qinv, qi, bm, off));
                    __stcs(reinterpret_cast<unsigned long long *>(o + jj + NC / 2),
                           (unsigned long long)out_u64<BIGQ>(hi, -nq, nq, qinv, qi, bm, off));
                }
            }
        }
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_slot, kCols);
}

}  // namespace c5

namespace {
inline cudaError_t counted(cudaError_t e) {
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

// [rows][16] u64 view of d_polys, 256-row x 128-byte boxes, 128-byte swizzle
bool make_poly_map(CUtensorMap *m, const void *base, uint64_t n_elems) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || (n_elems & 15) || (n_elems >> 4) > 0x7fffffffull) return false;
    const cuuint64_t dims[2] = {16, n_elems >> 4};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {16u, (cuuint32_t)c5::kBoxRows};
    const cuuint32_t estr[2] = {1u, 1u};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// Value bounds of the c5 kernels: after the integer level 0 every value
// is centered, |x| <= q/2; each FP64 CT level adds <= (1/2 + B 2^-54) q (+2 for the rounding of the
// quotient); every mul_tw input and the final values (converted through the 1.5*2^52
// bias) stay below 2^51.  off = K q exceeds the final bound (Barrett input).
static bool c5_bound(uint64_t qj, double start, uint32_t fp64_levels, bool fused_scaling, uint64_t *off) {
    const double L51 = 0.98 * 2251799813685248.0, e54 = 1.0 / 18014398509481984.0, Q = (double)qj;
    if (qj >= (1ull << 50)) return false;
    auto rtw = [&](double X) { return (0.5 + X * e54) * Q + 2.0; };
    double B = start * Q + 1.0;
    for (uint32_t lv = 0; lv < fp64_levels; ++lv) {
        if (B >= L51) return false;
        B += rtw(B);
    }
    if (B >= L51) return false;
    if (fused_scaling) B = 2.0 * rtw(B);   // a_j = A + Bv; a_{j+N/2} = c (A - Bv) is smaller
    if (B >= L51) return false;
    *off = (uint64_t)(std::ceil(B / Q) + 1.0) * qj;
    return true;
}

void ephdc_ntt_plan_c5_free(ephdc_ntt_plan *p) {
    cudaFree(p->c5_itw);
    cudaFree(p->c5_itail);
    p->c5_itw = p->c5_itail = nullptr;
}

// Decides the c5 kernels for a plan and uploads the inverse's tables.  Needs the plan's
// q, log2N, FP64 forward table (tw_f64) and the Shoup level-0 twiddles (c5_w1/_w1p).
cudaError_t plan_ntt_c5(ephdc_ntt_plan *p) {
    using namespace ephdc_host;
    p->c5_fwd = p->c5_inv = false;
    if (p->log2N < 12 || p->log2N > 14 || !p->tw_f64 || !encode_tiled_fn()) return cudaSuccess;
    bool fwd = true, inv = p->log2N <= 13;
    for (uint32_t j = 0; j < p->L; ++j) {
        uint64_t off_f = 0, off_i = 0;
        fwd = fwd && c5_bound(p->q[j], 0.5, p->log2N - (c5::kL0F && p->log2N <= 13 ? 0 : 1), false, &off_f);
        inv = inv && c5_bound(p->q[j], c5::kL0F ? 1.0 : 0.5, p->log2N - 2, true, &off_i);   // level 1 .. LGC-2
        p->c5_off[j] = std::max(off_f, off_i);
        p->c5_bm[j] = ~0ull / p->q[j];   // floor((2^64 - 1) / q) = floor(2^64 / q): q odd
    }
    p->c5_fwd = fwd;
    if (!inv) return cudaSuccess;
    // inverse tables: W[h + jj] = omega^-(N/2h) jj, entry 0 = (q, 1/q); tail [N/2][2] =
    // (s_j, s_j W[N/2 + j]) with s_j = N^-1 psi^-j; c = psi^-N/2
    const uint32_t N = p->N, L = p->L;
    std::vector<double> itw((size_t)L * N * 2), itail((size_t)L * N * 2);
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
        double *T = itail.data() + (size_t)j * N * 2;
        uint64_t sj = invmod(N % q, q);
        for (uint32_t jj = 0; jj < N / 2; ++jj, sj = mulmod(sj, psi_inv, q)) {
            const uint64_t swj = mulmod(sj, Wi[N / 2 + jj], q);
            T[4 * jj] = (double)sj;
            T[4 * jj + 1] = (double)sj / qd;
            T[4 * jj + 2] = (double)swj;
            T[4 * jj + 3] = (double)swj / qd;
        }
        const uint64_t c = powmod(psi_inv, N / 2, q);
        p->c5_cinv[j] = make_double2((double)c, (double)c / qd);
    }
    cudaError_t e;
    if ((e = cudaMalloc(&p->c5_itw, sizeof(double) * itw.size())) != cudaSuccess ||
        (e = cudaMalloc(&p->c5_itail, sizeof(double) * itail.size())) != cudaSuccess ||
        (e = cudaMemcpy(p->c5_itw, itw.data(), sizeof(double) * itw.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(p->c5_itail, itail.data(), sizeof(double) * itail.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return e;
    p->c5_inv = true;
    return cudaSuccess;
}

template <int LGC, int S, bool INV>
static cudaError_t c5_launch(const ephdc_ntt_plan *pl, uint64_t *polys, uint32_t batch, cudaStream_t st) {
    constexpr size_t smem = c5::smem_bytes<LGC, INV>();
    bool bigq = true;   // every q_j > 2^32: the short Barrett quotient
    for (uint32_t j = 0; j < pl->L; ++j) bigq = bigq && pl->q[j] > (1ull << 32);
    void (*kern)(const CUtensorMap, const C5Args);
    if constexpr (INV) kern = bigq ? c5::k_ntt_c5_inv<LGC, true> : c5::k_ntt_c5_inv<LGC, false>;
    else kern = bigq ? c5::k_ntt_c5_fwd<LGC, S, true> : c5::k_ntt_c5_fwd<LGC, S, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    CUtensorMap map;
    if (!make_poly_map(&map, polys, (uint64_t)batch * pl->L * pl->N)) return cudaErrorNotSupported;
    C5Args a{};
    a.polys = polys;
    a.tw = INV ? pl->c5_itw : pl->tw_f64;
    a.tail = pl->c5_itail;
    a.L = pl->L;
    a.batch = batch;
    a.items = pl->L * batch;
    for (uint32_t j = 0; j < pl->L; ++j) {
        a.q[j] = pl->q[j];
        a.w1[j] = pl->c5_w1[j];
        a.w1p[j] = pl->c5_w1p[j];
        a.bm[j] = pl->c5_bm[j];
        a.off[j] = pl->c5_off[j];
        a.cinv[j] = pl->c5_cinv[j];
    }
    // persistent: one CTA (pair) per SM slot, never more units than items
    const uint32_t slots = 148u * c5::ctas_per_sm<LGC>() / S;
    const uint32_t units = std::max<uint32_t>(1, std::min<uint32_t>(slots, a.items));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units * S);
    cfg.blockDim = dim3((1 << LGC) / c5::kE);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
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
    if (inverse) {
        switch (pl->log2N) {
            case 12: return c5_launch<12, 1, true>(pl, d_polys, batch, st);
            case 13: return c5_launch<13, 1, true>(pl, d_polys, batch, st);
        }
    } else {
        switch (pl->log2N) {
            case 12: return c5_launch<12, 1, false>(pl, d_polys, batch, st);
            case 13: return c5_launch<13, 1, false>(pl, d_polys, batch, st);
            case 14: return c5_launch<13, 2, false>(pl, d_polys, batch, st);
        }
    }
    return cudaErrorNotSupported;
}

}  // namespace ephdc
