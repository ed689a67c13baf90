// ntt32_c5.cu -- the c5 standalone negacyclic NTT on u32 words (every prime < 2^30;
// BASELINE.json configs[4], SURVEY 8(d) "30-bit primes in u32"), integer pipe.
//
// The textbook loops of oracle/oracle_core.c (forward Cooley-Tukey over psi_rev, inverse
// Gentleman-Sande over psiinv_rev then N^-1; P:1458-1459 counts one forward NTT per
// plaintext), with u32 Shoup products and Harvey's lazy ranges (modarith.cuh: forward
// values in [0, 4q), inverse in [0, 2q); 4q < 2^32 because q < 2^30).
//
// In place on [batch][L][N] canonical u32, N = NC = 2^12, 2^13, 2^14 (one CTA per
// polynomial; 2^15 / 2^16 keep the general kernels).  Per CTA, NT = NC/32 threads with
// 32 elements each, persistent over a contiguous range of prime-major items:
//   * polynomials arrive by TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B: word e of a
//     1024-byte-aligned buffer sits at sw(e) = e ^ (((e >> 5) & 7) << 2)) into a ring
//     of three buffers -- the load of item i+3 is issued once item i has been stored;
//     results leave by a TMA store of the same buffer (cp.async.bulk.tensor ...
//     bulk_group);
//   * forward levels in three register passes, all conflict-free in the swizzled
//     layout and all with compile-time offsets from per-group bases:
//       A  levels 0 .. LG-10:  groups {g + 512k} (lanes consecutive),
//       B  levels LG-9 .. LG-6: groups {512 blk + off + 32k}, off = lane (a 32-word row
//          holds one k, so the XOR term depends on k & 7 only: 8 bases),
//       C  levels LG-5 .. LG-1: one 32-word row per thread, read and written as eight
//          16-byte chunks (chunk m of row g sits at m ^ (g & 7): a quarter warp touches 8
//          distinct chunks);
//     the inverse runs C (half-sizes 1..16), B (32..256), A (512..NC/2) with the
//     scaling by N^-1 fused into the last level: (X + Y) N^-1 and (X - Y) (w N^-1);
//   * twiddles: the levels of A and B are warp-uniform (broadcast reads of the first
//     NC/32 table entries in shared memory); the 31 (w, w') pairs of a thread's row in
//     pass C live in TENSOR MEMORY (64 columns per thread), loaded once per prime.
// DESIGN.md 5.2 "c5 u32 kernels".
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "async_copy.cuh"
#include "internal.h"
#include "modarith.cuh"
#include "tma_host.h"
#include "tmem_x.cuh"

namespace ephdc {
namespace c5u32 {

constexpr int kE = 32;      // elements per thread
constexpr int kNBuf = 3;    // rotating polynomial buffers

template <int LG> __host__ __device__ constexpr int nthreads() { return (1 << LG) / kE; }
template <int LG> __host__ __device__ constexpr int ctas_per_sm() { return LG == 12 ? 4 : LG == 13 ? 2 : 1; }
// OCC (A/B): two buffers per CTA, so that 6 / 3 CTAs fit an SM at 2^12 / 2^13 (<= 80 registers)
template <int LG, bool OCC> __host__ __device__ constexpr int nbuf() { return OCC && LG <= 13 ? 2 : kNBuf; }
template <int LG, bool OCC> __host__ __device__ constexpr int cps() {
    return OCC && LG <= 13 ? (LG == 12 ? 6 : 3) : ctas_per_sm<LG>();
}
// 64 TMEM columns per thread (31 pairs); warps w and w + 4 share a lane quarter
template <int LG> __host__ __device__ constexpr uint32_t tmem_cols() { return 64u * (uint32_t)((nthreads<LG>() / 32 + 3) / 4); }
template <int LG> __host__ __device__ constexpr int box_rows() { return (1 << LG) / 32 > 256 ? 256 : (1 << LG) / 32; }
template <int LG, bool OCC> __host__ __device__ constexpr size_t smem_bytes() {
    return 1024 + sizeof(u32) * nbuf<LG, OCC>() * ((size_t)1 << LG) + sizeof(TwPair<u32>) * (((size_t)1 << LG) >> 5);
}

struct Args {
    u32 L, batch, items;
    const TwPair<u32> *tw;   // [L][N] psi_rev (forward) or psiinv_rev (inverse), Shoup pairs
    const u32 *ninv;         // [L][2] (N^-1, Shoup)
    u32 q[kMaxL];
    u32 zero;                // 0: a runtime addend that keeps the butterfly sums 3-input IADD3s
    u64 *polys64;            // IO64: [batch][L][N] u64 words (residues < 2^30)
    u32 *polys32;            // DOUT: the u32 words (results stored from the last pass)
    u32 slog;                // log2 of the slices per polynomial (N = NC << slog): items (prime, slice, poly)
};

EPHDC_D void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ephdc_async::smem_u32(dst)), "l"(src) : "memory");
}
// arrives on *bar once all of this thread's earlier cp.async copies have landed
EPHDC_D void cp_async_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ephdc_async::smem_u32(bar)) : "memory");
}

EPHDC_D int sw(int e) { return e ^ (((e >> 5) & 7) << 2); }

EPHDC_D void tma_load(void *dst, const CUtensorMap *map, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            ephdc_async::smem_u32(dst)),
        "l"(map), "r"(0), "r"(y), "r"(ephdc_async::smem_u32(bar))
        : "memory");
}
EPHDC_D void tma_store(const CUtensorMap *map, int y, const void *src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(0), "r"(y),
                 "r"(ephdc_async::smem_u32(src))
                 : "memory");
}
EPHDC_D void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
EPHDC_D void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
EPHDC_D void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct Prime {
    u32 q, two_q, z;
    TwPair<u32> ninv, wn;   // inverse: N^-1 and w N^-1 (w = psiinv_rev[1]) for the last level
};

// Register sub-stages with compile-time trip counts (template recursion: ptxas keeps
// x[] in registers).  CT sub-stage sub pairs (k, k + R/2^(sub+1)) of sub-block v, twiddle
// tw(sub, v); GS sub-stage sub pairs (k, k + 2^sub) of block v = k >> (sub+1).
template <int R_LOG, int SUB, int END, class Tw, class Bf>
EPHDC_D void ct_subs(u32 (&x)[1 << R_LOG], const Tw &tw, const Bf &bf) {
    if constexpr (SUB < END) {
        constexpr int R = 1 << R_LOG, h = R >> (SUB + 1);
#pragma unroll
        for (int v = 0; v < (1 << SUB); ++v) {
            const auto t = tw(SUB, v);
#pragma unroll
            for (int kk = 0; kk < h; ++kk) bf(x[v * 2 * h + kk], x[v * 2 * h + kk + h], t);
        }
        ct_subs<R_LOG, SUB + 1, END>(x, tw, bf);
    }
}
template <int R_LOG, int SUB, int END, class Tw, class Bf>
EPHDC_D void gs_subs(u32 (&x)[1 << R_LOG], const Tw &tw, const Bf &bf) {
    if constexpr (SUB < END) {
        constexpr int R = 1 << R_LOG, hs = 1 << SUB;
#pragma unroll
        for (int v = 0; v < R / (2 * hs); ++v) {
            const auto t = tw(SUB, v);
#pragma unroll
            for (int kk = 0; kk < hs; ++kk) bf(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], t);
        }
        gs_subs<R_LOG, SUB + 1, END>(x, tw, bf);
    }
}

// Shared-memory twiddle of passes A and B (a Shoup pair).
typedef TwPair<u32> TwH;

// butterfly functors: Shoup pairs (pass C, TMEM) and the shared TwH entries (A, B)
// Harvey butterflies (modarith.cuh ct_bfly / gs_bfly) with the two-input sums written
// as three-input sums with a runtime zero: ptxas then issues IADD3 on the ALU pipe
// instead of IMAD.IADD on the IMAD pipe, which the Shoup products already load.
EPHDC_D auto ct_shoup(const Prime &pr) {
    return [&pr](u32 &X, u32 &Y, const TwPair<u32> &t) {
        const u32 x = csub(X, pr.two_q), r = mul_shoup_lazy<u32>(Y, t.w, t.wp, pr.q);
        X = x + r + pr.z;
        Y = x - r + pr.two_q;
    };
}
EPHDC_D auto gs_shoup(const Prime &pr) {
    return [&pr](u32 &X, u32 &Y, const TwPair<u32> &t) {
        const u32 x = X, y = Y;
        X = csub(x + y + pr.z, pr.two_q);
        Y = mul_shoup_lazy<u32>(x - y + pr.two_q, t.w, t.wp, pr.q);
    };
}
EPHDC_D auto ct_ab(const Prime &pr) { return ct_shoup(pr); }
EPHDC_D auto gs_ab(const Prime &pr) { return gs_shoup(pr); }

// ---- pass A: R = 2^(LG-9) elements {g + 512k} per group, 32/R groups per thread ----
struct ToSmem {
    EPHDC_D void operator()(int, u32) const {}
};
// (Out: the inverse's output element e goes to out(e, value) instead of B)
template <int LG, bool INV, bool FUSE = true, class Out = ToSmem>
EPHDC_D void pass_a(u32 *B, const TwH *tws, const Prime &pr, int tid, const Out &out = Out()) {
    constexpr bool kOut = !std::is_same<Out, ToSmem>::value;
    constexpr int NC = 1 << LG, NT = NC / kE, RA = LG - 9, R = 1 << RA, GA = kE / R;
#pragma unroll
    for (int u = 0; u < GA; ++u) {
        u32 *P = B + sw(tid + u * NT);   // sw(g + 512k) = sw(g) + 512k (g < 512)
        u32 x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = P[512 * k];
        if constexpr (!INV) {   // levels 0 .. RA-1: psi_rev[2^sub + v]
            ct_subs<RA, 0, RA>(x, [&](int sub, int v) { return tws[(1 << sub) + v]; }, ct_ab(pr));
        } else {   // half-sizes 2^(9+sub): psiinv_rev[NC/2^(10+sub) + v]; the last one fused with N^-1
            gs_subs<RA, 0, RA - 1>(x, [&](int sub, int v) { return tws[(NC >> (10 + sub)) + v]; }, gs_ab(pr));
            constexpr int hs = R / 2;
            if constexpr (FUSE) {
#pragma unroll
                for (int kk = 0; kk < hs; ++kk) {
                    const u32 X = x[kk], Y = x[kk + hs];
                    x[kk] = csub(mul_shoup_lazy<u32>(X + Y, pr.ninv.w, pr.ninv.wp, pr.q), pr.q);
                    x[kk + hs] = csub(mul_shoup_lazy<u32>(X - Y + pr.two_q, pr.wn.w, pr.wn.wp, pr.q), pr.q);
                }
            } else {   // a slice: the last local level is a plain GS level (lazy [0, 2q) out)
                const TwPair<u32> t = tws[1];
#pragma unroll
                for (int kk = 0; kk < hs; ++kk) gs_ab(pr)(x[kk], x[kk + hs], t);
            }
        }
        if constexpr (kOut) {
#pragma unroll
            for (int k = 0; k < R; ++k) out(tid + u * NT + 512 * k, x[k]);
        } else {
#pragma unroll
            for (int k = 0; k < R; ++k) P[512 * k] = x[k];
        }
    }
}

// ---- pass B: 16 elements {512 blk + off + 32k} per group, two groups per thread ----
template <int LG, bool INV> EPHDC_D void pass_b(u32 *B, const TwH *tws, const Prime &pr, int tid) {
    constexpr int NC = 1 << LG, NT = NC / kE;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int g = tid + u * NT, blk = g >> 5, off = g & 31;
        u32 *P = B + blk * 512;
        int o[8];   // row k holds word off at off ^ ((k & 7) << 2)
#pragma unroll
        for (int c = 0; c < 8; ++c) o[c] = off ^ (c << 2);
        u32 x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = P[o[k & 7] + 32 * k];
        if constexpr (!INV)   // level LG-9+sub, block blk 2^sub + v
            ct_subs<4, 0, 4>(x, [&](int sub, int v) { return tws[((NC >> 9) << sub) + (blk << sub) + v]; }, ct_ab(pr));
        else                  // half-size 2^(5+sub): psiinv_rev[NC/2^(6+sub) + blk 2^(3-sub) + v]
            gs_subs<4, 0, 4>(x, [&](int sub, int v) { return tws[(NC >> (6 + sub)) + (blk << (3 - sub)) + v]; },
                             gs_ab(pr));
#pragma unroll
        for (int k = 0; k < 16; ++k) P[o[k & 7] + 32 * k] = x[k];
    }
}

EPHDC_D TwPair<u32> tpair(const uint32_t (&r0)[32], const uint32_t (&r1)[32], int p) {
    return p < 16 ? TwPair<u32>{r0[2 * p], r0[2 * p + 1]} : TwPair<u32>{r1[2 * p - 32], r1[2 * p - 31]};
}

// ---- pass C: the thread's 32-word row, 16-byte chunks; twiddle pairs from TMEM ----
struct FromSmem {
    EPHDC_D u32 operator()(int) const { return 0u; }
};
// (Load: the inverse's input element i of the row comes from load(i) instead of B --
// the slot pack of the query path)
struct RowToSmem {
    EPHDC_D void operator()(const u32 (&)[32]) const {}
};
// (RowOut: the row's 32 results go to out(x) instead of back to B)
template <int LG, bool INV, class Load = FromSmem, class RowOut = RowToSmem>
EPHDC_D void pass_c(u32 *B, uint32_t tbase, const Prime &pr, int tid, const Load &load = Load(),
                    const RowOut &rout = RowOut()) {
    constexpr bool kLoad = !std::is_same<Load, FromSmem>::value;
    constexpr bool kRowOut = !std::is_same<RowOut, RowToSmem>::value;
    uint32_t r0[32], r1[32];
    ephdc_tmem::ldx<32>(tbase, r0);
    ephdc_tmem::ldx<32>(tbase + 32u, r1);
    u32 *P = B + 32 * tid;
    const int g7 = tid & 7;
    u32 x[32];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        if constexpr (kLoad) {
#pragma unroll
            for (int c = 0; c < 4; ++c) x[4 * m + c] = load(32 * tid + 4 * m + c);
        } else {
            const uint4 v = *reinterpret_cast<const uint4 *>(P + 4 * (m ^ g7));
            x[4 * m] = v.x;
            x[4 * m + 1] = v.y;
            x[4 * m + 2] = v.z;
            x[4 * m + 3] = v.w;
        }
    }
    ephdc_tmem::waitx<32>(r0);
    ephdc_tmem::waitx<32>(r1);
    if constexpr (!INV) {   // level LG-5+sub, pair (2^sub - 1) + v
        ct_subs<5, 0, 5>(x, [&](int sub, int v) { return tpair(r0, r1, (1 << sub) - 1 + v); }, ct_shoup(pr));
#pragma unroll
        for (int k = 0; k < 32; ++k) x[k] = reduce4<u32>(x[k], pr.q, pr.two_q);
    } else {   // half-size 2^s, pair 32 - 2^(5-s) + v
        gs_subs<5, 0, 5>(x, [&](int s, int v) { return tpair(r0, r1, 32 - (32 >> s) + v); }, gs_shoup(pr));
    }
    if constexpr (kRowOut) {
        rout(x);
    } else {
#pragma unroll
        for (int m = 0; m < 8; ++m)
            *reinterpret_cast<uint4 *>(P + 4 * (m ^ g7)) = make_uint4(x[4 * m], x[4 * m + 1], x[4 * m + 2], x[4 * m + 3]);
    }
}

// IO64: u64 words (every residue < 2^30).  TMA cannot drop the high words into the
// 128-byte swizzled rows, so every thread copies the low words of 32 elements with
// 4-byte cp.async (lanes on consecutive elements) into the same swizzled u32 layout,
// signalling the buffer's mbarrier (NT arrivals) -- issued two items ahead, after the
// first barrier of the current item -- and results leave as zero-extended u64 with
// lanes on consecutive elements: the inverse straight from pass A's registers, the
// forward from B after pass C (storing each thread's 256-byte row from registers
// measured 0.45 vs 0.54 of HBM at 2^13: uncoalesced).
// DOUT (u32 words): TMA in, but results stored by the threads -- the inverse from pass
// A's registers (lanes on consecutive elements), the forward by each warp from its own
// rows after pass C (16-byte stores, lanes on consecutive chunks) -- so no item ends with
// a CTA barrier; the load of item i + kNB - 1 is issued after item i's first barrier.
// SLC: the CTA transforms 2^LG-point slices of a 2^(LG + slog)-point transform whose
// global stages run in k_ntt_global (N^-1 applied there, not in pass A).
template <int LG, bool INV, bool OCC, bool IO64 = false, bool DOUT = false, bool SLC = false>
__global__ void __launch_bounds__(nthreads<LG>(), cps<LG, OCC>())
    k_ntt32_c5(const __grid_constant__ CUtensorMap map, const __grid_constant__ Args a) {
    constexpr int NC = 1 << LG, NT = NC / kE, NTW = NC >> 5, kNB = nbuf<LG, OCC>();
    constexpr int kBox = box_rows<LG>(), kBoxes = NC / 32 / kBox;
    static_assert(LG >= 12 && LG <= 14, "one CTA per polynomial, 2^12 .. 2^14");
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kNB];
    __shared__ uint32_t tmem_slot;
    u32 *bufs = reinterpret_cast<u32 *>(smem_raw + ((1024u - (ephdc_async::smem_u32(smem_raw) & 1023u)) & 1023u));
    TwH *tws = reinterpret_cast<TwH *>(bufs + kNB * NC);
    const int tid = threadIdx.x, warp = tid >> 5;
    const u32 slog_ = SLC ? a.slog : 0u;
    if (tid == 0)
        for (int b = 0; b < kNB; ++b) ephdc_async::mbar_init(&mbar[b], IO64 ? NT : 1);
    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, tmem_cols<LG>());
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    const uint32_t tbase = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 64u;
    // items are (prime j, slice s, polynomial b), b fastest: segment js = j 2^slog + s
    auto elem_off = [&](u32 w) -> size_t {   // first element of item w
        const u32 js = w / a.batch, b = w - js * a.batch;
        const u32 j = js >> slog_, sl = js & ((1u << slog_) - 1u);
        return ((((size_t)b * a.L + j) << slog_) + sl) << LG;
    };
    auto poly64 = [&](u32 w) -> u64 * { return a.polys64 + elem_off(w); };

    const u32 w0 = (u32)((u64)a.items * blockIdx.x / gridDim.x), w1 = (u32)((u64)a.items * (blockIdx.x + 1) / gridDim.x);
    const u32 n = w1 - w0;
    auto row_of = [&](u32 w) -> int { return (int)(elem_off(w) >> 5); };   // first 128-byte row
    auto issue = [&](u32 i) {   // one thread
        uint64_t *bar = &mbar[i % kNB];
        u32 *dst = bufs + (i % kNB) * NC;
        ephdc_async::mbar_arrive_expect_tx(bar, (u32)(NC * 4));
        const int y = row_of(w0 + i);
#pragma unroll
        for (int k = 0; k < kBoxes; ++k) tma_load(dst + k * kBox * 32, &map, y + k * kBox, bar);
    };
    auto issue64 = [&](u32 i) {   // every thread: the low words of elements tid + NT k
        u32 *dst = bufs + (i % kNB) * NC;
        const u32 *src = reinterpret_cast<const u32 *>(poly64(w0 + i));
#pragma unroll
        for (int k = 0; k < kE; ++k) cp_async4(dst + sw(tid + NT * k), src + 2 * (tid + NT * k));
        cp_async_arrive(&mbar[i % kNB]);
    };
    if constexpr (IO64) {
        for (u32 i = 0; i + 1 < (u32)kNB && i < n; ++i) issue64(i);
    } else if constexpr (DOUT) {
        if (tid == 0)
            for (u32 i = 0; i + 1 < (u32)kNB && i < n; ++i) issue(i);
    } else {
        if (tid == 0)
            for (u32 i = 0; i < (u32)kNB && i < n; ++i) issue(i);
    }

    u32 jcur = 0xffffffffu;
    Prime pr{0, 0, a.zero, {0, 0}, {0, 0}};
    for (u32 i = 0; i < n; ++i) {
        const u32 w = w0 + i, js = w / a.batch, j = js >> slog_;
        if (js != jcur) {   // the previous item's last barrier freed the twiddles
            if constexpr (IO64 || DOUT) __syncthreads();   // (these items end without one)
            const TwPair<u32> *gt = a.tw + ((size_t)j << (LG + slog_));
            // slice sl of S = 2^slog: the local table entry m + B (m a power of two) is the
            // global entry (S + sl) m + B (S = 1: the identity)
            const u32 ssl = (1u << slog_) + (js & ((1u << slog_) - 1u));
            auto glob = [&](int idx) -> int {
                const int m = 1 << (31 - __clz(idx));
                return (int)ssl * m + (idx - m);
            };
            for (int p = tid; p < NTW; p += NT)
                if (p > 0) tws[p] = gt[glob(p)];
            uint32_t r[16];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int p = 8 * h + c;
                    TwPair<u32> t{0, 0};
                    if (p < 31) {
                        int idx;
                        if constexpr (!INV) {   // level LG-5+sub, block tid 2^sub + v: psi_rev[NC/32 2^sub + ...]
                            const int sub = 31 - __clz(p + 1), v = p + 1 - (1 << sub);
                            idx = ((NC >> 5) << sub) + (tid << sub) + v;
                        } else {                // half-size 2^s: psiinv_rev[NC/2^(s+1) + tid 2^(4-s) + v]
                            const int s = p < 16 ? 0 : p < 24 ? 1 : p < 28 ? 2 : p < 30 ? 3 : 4;
                            const int v = p - (32 - (32 >> s));
                            idx = (NC >> (s + 1)) + (tid << (4 - s)) + v;
                        }
                        t = gt[glob(idx)];
                    }
                    r[2 * c] = t.w;
                    r[2 * c + 1] = t.wp;
                }
                ephdc_tmem::stx<16>(tbase + 16u * h, r);
            }
            ephdc_tmem::wait_st();
            pr.q = a.q[j];
            pr.two_q = 2 * pr.q;
            if constexpr (INV) {
                pr.ninv = TwPair<u32>{a.ninv[2 * j], a.ninv[2 * j + 1]};
                const u32 wv = (u32)(((u64)gt[1].w * pr.ninv.w) % pr.q);
                pr.wn = TwPair<u32>{wv, (u32)(((u64)wv << 32) / pr.q)};
            }
            jcur = js;
            __syncthreads();
        }
        u32 *B = bufs + (i % kNB) * NC;
        ephdc_async::mbar_wait(&mbar[i % kNB], (i / kNB) & 1);
        if constexpr (IO64) {
            // the buffer of item i + kNB - 1 was last read by item i - 1, which every thread
            // has left once the first barrier of item i is passed
            u64 *o = poly64(w);
            if constexpr (!INV) {
                pass_a<LG, false>(B, tws, pr, tid);
                __syncthreads();
                if (i + kNB - 1 < n) issue64(i + kNB - 1);
                pass_b<LG, false>(B, tws, pr, tid);
                __syncthreads();
                pass_c<LG, false>(B, tbase, pr, tid);
                // rows back in B; warp w's rows are elements [1024 w, 1024 w + 1024), stored
                // by the same warp with lanes on consecutive pairs: a warp barrier suffices
                __syncwarp();
                const int eb = 1024 * warp + 2 * (tid & 31);
#pragma unroll
                for (int k = 0; k < kE / 2; ++k) {   // pairs (e, e + 1): sw keeps them adjacent
                    const int e = eb + 64 * k;
                    const uint2 v = *reinterpret_cast<const uint2 *>(B + sw(e));
                    __stcs(reinterpret_cast<ulonglong2 *>(o + e), make_ulonglong2(v.x, v.y));
                }
            } else {
                pass_c<LG, true>(B, tbase, pr, tid);
                __syncthreads();
                if (i + kNB - 1 < n) issue64(i + kNB - 1);
                pass_b<LG, true>(B, tws, pr, tid);
                __syncthreads();
                pass_a<LG, true>(B, tws, pr, tid, [&](int e, u32 y) { __stcs(o + e, (unsigned long long)y); });
            }
            continue;
        }
        if constexpr (DOUT) {
            u32 *o = a.polys32 + elem_off(w);
            auto reissue = [&]() {   // item i - 1's buffer is free behind item i's first barrier
                if (tid == 0 && i + kNB - 1 < n) {
                    ephdc_async::fence_proxy_async();
                    issue(i + kNB - 1);
                }
            };
            if constexpr (!INV) {
                pass_a<LG, false>(B, tws, pr, tid);
                __syncthreads();
                reissue();
                pass_b<LG, false>(B, tws, pr, tid);
                __syncthreads();
                pass_c<LG, false>(B, tbase, pr, tid);
                __syncwarp();   // warp w's rows = words [1024 w, 1024 w + 1024)
                const int eb = 1024 * warp + 4 * (tid & 31);
#pragma unroll
                for (int k = 0; k < kE / 4; ++k) {
                    const int e = eb + 128 * k;
                    __stcs(reinterpret_cast<uint4 *>(o + e), *reinterpret_cast<const uint4 *>(B + sw(e)));
                }
            } else {
                pass_c<LG, true>(B, tbase, pr, tid);
                __syncthreads();
                reissue();
                pass_b<LG, true>(B, tws, pr, tid);
                __syncthreads();
                pass_a<LG, true, !SLC>(B, tws, pr, tid, [&](int e, u32 y) { __stcs(o + e, y); });
            }
            continue;
        }
        if constexpr (!INV) {
            pass_a<LG, false>(B, tws, pr, tid);
            __syncthreads();
            pass_b<LG, false>(B, tws, pr, tid);
            __syncthreads();
            pass_c<LG, false>(B, tbase, pr, tid);
        } else {
            pass_c<LG, true>(B, tbase, pr, tid);
            __syncthreads();
            pass_b<LG, true>(B, tws, pr, tid);
            __syncthreads();
            pass_a<LG, true, !SLC>(B, tws, pr, tid);
        }
        ephdc_async::fence_proxy_async();   // this thread's writes -> the TMA store
        __syncthreads();
        if (tid == 0) {
            const int y = row_of(w);
#pragma unroll
            for (int k = 0; k < kBoxes; ++k) tma_store(&map, y + k * kBox, B + k * kBox * 32);
            bulk_commit();
            if (i + kNB < n) {
                bulk_wait_read0();   // the store has read the buffer
                issue(i + kNB);
            }
        }
    }
    if (!IO64 && !DOUT && tid == 0) bulk_wait0();
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_slot, tmem_cols<LG>());
}

// =====================================================================================
// The query path's slot pack + INTT mod t ("EncPt"; K2 of DESIGN.md) on the same
// passes: row (b, d) of M [nbat][D][N] = centered lift of INTT_t(slots), slot i holding
// h[d][b B + i/k] for i < k n_b (reading #1), 0 beyond.  Pass C reads the
// slots of its row straight from H (int8 [D][nq]) instead of shared memory, pass A
// writes the centered int32 results straight to M (lanes consecutive: coalesced).  Two
// row buffers alternate, so a row costs two CTA barriers.  Persistent over rows.
// =====================================================================================
struct PackArgs32 {
    u32 t, ninv, ninv_p, k, B, D, nq, b0, nbat, kmagic, zero;
    const TwPair<u32> *itw;   // [N] psiinv_rev mod t, Shoup pairs
};

template <int LG, bool PF = true>
__global__ void __launch_bounds__(nthreads<LG>(), ctas_per_sm<LG>())
    k_pack_intt32(const int8_t *__restrict__ H, PackArgs32 a, u32 *__restrict__ M) {
    constexpr int NC = 1 << LG, NT = NC / kE, NTW = NC >> 5;
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint32_t tmem_slot;
    u32 *bufs = reinterpret_cast<u32 *>(smem_raw + ((1024u - (ephdc_async::smem_u32(smem_raw) & 1023u)) & 1023u));
    TwH *tws = reinterpret_cast<TwH *>(bufs + 2 * NC);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, tmem_cols<LG>());
    for (int p = tid; p < NTW; p += NT) tws[p] = a.itw[p];
    {   // this thread's row twiddles (inverse order, as in k_ntt32_c5)
        uint32_t r[16];
        ephdc_tmem::fence_before_sync();
        __syncthreads();
        ephdc_tmem::fence_after_sync();
        const uint32_t tb = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 64u;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int p = 8 * h + c;
                TwPair<u32> t{0, 0};
                if (p < 31) {
                    const int s = p < 16 ? 0 : p < 24 ? 1 : p < 28 ? 2 : p < 30 ? 3 : 4;
                    t = a.itw[(NC >> (s + 1)) + (tid << (4 - s)) + (p - (32 - (32 >> s)))];
                }
                r[2 * c] = t.w;
                r[2 * c + 1] = t.wp;
            }
            ephdc_tmem::stx<16>(tb + 16u * h, r);
        }
        ephdc_tmem::wait_st();
    }
    const uint32_t tbase = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 64u;
    Prime pr{a.t, 2 * a.t, a.zero, {a.ninv, a.ninv_p}, {0, 0}};
    {
        const u32 wv = (u32)(((u64)a.itw[1].w * a.ninv) % a.t);
        pr.wn = TwPair<u32>{wv, (u32)(((u64)wv << 32) / a.t)};
    }
    const u32 half_t = (a.t - 1) / 2;
    __syncthreads();
    const u32 rows = a.nbat * a.D;
    u32 par = 0;
    for (u32 row = blockIdx.x; row < rows; row += gridDim.x, par ^= 1u) {
        const u32 bb = row / a.D, d = row - bb * a.D, b = a.b0 + bb;
        const u32 lim = a.k * min(a.B, a.nq - b * a.B);
        const int8_t *src = H + (size_t)d * a.nq + (size_t)b * a.B;
        u32 *B = bufs + par * NC;
        auto load = [&](int i) -> u32 {   // slot i -> h[d][b B + i/k] mod t
            if ((u32)i >= lim) return 0u;
            const int v = __ldg(src + (a.k == 1u ? (u32)i : __umulhi((u32)i, a.kmagic)));
            return v < 0 ? (u32)((int)a.t + v) : (u32)v;
        };
        pass_c<LG, true>(B, tbase, pr, tid, load);
        __syncthreads();
        if constexpr (PF) {   // the next row's H bytes of this thread's slots toward L2 / L1
            const u32 rn = row + gridDim.x;
            if (rn < rows) {
                const u32 bbn = rn / a.D, dn = rn - bbn * a.D, bn = a.b0 + bbn;
                const u32 q0 = a.k == 1u ? 32u * tid : __umulhi(32u * tid, a.kmagic);
                if (q0 < min(a.B, a.nq - bn * a.B))   // only bytes the row reads (never past H)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(H + (size_t)dn * a.nq + (size_t)bn * a.B + q0));
            }
        }
        pass_b<LG, true>(B, tws, pr, tid);
        __syncthreads();
        u32 *o = M + (size_t)row * NC;
        pass_a<LG, true>(B, tws, pr, tid, [&](int e, u32 y) {
            o[e] = y <= half_t ? y : (u32)((int)y - (int)a.t);   // centered lift (reading #3)
        });
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_slot, tmem_cols<LG>());
}

inline cudaError_t counted(cudaError_t e) {
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

// [n_words / 32] rows of 128 bytes, box box_rows x 128 bytes, 128-byte swizzle
bool make_map32(CUtensorMap *m, const void *base, uint64_t n_words, uint32_t box_rows) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || (n_words & 31) || (n_words >> 5) > 0x7fffffffull) return false;
    const cuuint64_t dims[2] = {32, n_words >> 5};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {32u, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LG, bool INV>
cudaError_t launch(const ephdc_ntt_plan *p, void *polys, uint32_t batch, cudaStream_t st, bool u64_words = false,
                   uint32_t slog = 0) {
    // inverse: the OCC form (two buffers, 3 / 6 CTAs per SM at 2^13 / 2^12: 0.546 vs
    // 0.531 of HBM at 2^13); forward: three buffers (0.525 vs 0.526; r47).
    // EPHDC_NTT_ALT_TEAMS swaps the forms (A/B).
    // u64 words: the IO64 form (three buffers, cp.async in, u64 stores out)
    // u32 words: the inverse stores from pass A's registers (DOUT: 0.551 / 0.511 vs 0.547
    // / 0.494 of HBM with the TMA store at 2^13 / 2^14), the forward keeps the TMA store
    // (0.527 / 0.498 vs 0.511 / 0.472 with per-warp 16-byte stores; r57).
    // EPHDC_NTT_ALT_TEAMS swaps the forms (A/B).
    const bool occ = !u64_words && INV;
    const bool dout = INV != p->c5_alt_teams;
    auto kern = u64_words ? k_ntt32_c5<LG, INV, false, true>
                : slog    ? (dout ? k_ntt32_c5<LG, INV, false, false, true, true> : k_ntt32_c5<LG, INV, false, false, false, true>)
                : occ     ? (dout ? k_ntt32_c5<LG, INV, true, false, true> : k_ntt32_c5<LG, INV, true>)
                          : (dout ? k_ntt32_c5<LG, INV, false, false, true> : k_ntt32_c5<LG, INV, false>);
    const size_t smem = occ ? smem_bytes<LG, true>() : smem_bytes<LG, false>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    CUtensorMap map{};
    const uint64_t n = (uint64_t)batch * p->L * p->N;
    if (!u64_words && !make_map32(&map, polys, n, (uint32_t)box_rows<LG>())) return cudaErrorNotSupported;
    Args a{};
    a.L = p->L;
    a.batch = batch;
    a.items = (p->L << slog) * batch;
    a.slog = slog;
    a.tw = INV ? p->itw32 : p->tw32;
    a.ninv = p->ninv32;
    for (uint32_t j = 0; j < p->L; ++j) a.q[j] = (u32)p->q[j];
    a.zero = 0;
    a.polys64 = u64_words ? static_cast<u64 *>(polys) : nullptr;
    a.polys32 = u64_words ? nullptr : static_cast<u32 *>(polys);
    const uint32_t units = std::max<uint32_t>(1, std::min<uint32_t>(148u * (occ ? cps<LG, true>() : cps<LG, false>()), a.items));
    kern<<<units, nthreads<LG>(), smem, st>>>(map, a);
    return counted(cudaGetLastError());
}

}  // namespace c5u32

// The c5 u32 kernels where they apply (N = 2^12 .. 2^14, unless the plan asks for the
// general kernels); cudaErrorNotSupported otherwise (the caller runs the general ones).
cudaError_t launch_ntt32_c5(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, bool inverse,
                            cudaStream_t st) {
    if (p->u32_generic || !p->tw32) return cudaErrorNotSupported;
    if (batch == 0) return cudaSuccess;
    if ((uint64_t)batch * p->L > 0xffffffffull || ((uintptr_t)d_polys & 15)) return cudaErrorNotSupported;
    using namespace c5u32;
    switch (p->log2N) {
        case 12: return inverse ? launch<12, true>(p, d_polys, batch, st) : launch<12, false>(p, d_polys, batch, st);
        case 13: return inverse ? launch<13, true>(p, d_polys, batch, st) : launch<13, false>(p, d_polys, batch, st);
        case 14: return inverse ? launch<14, true>(p, d_polys, batch, st) : launch<14, false>(p, d_polys, batch, st);
        case 15:
        case 16: {   // log2(N) - 14 global stages (one HBM pass) + 2^14-point slices
            if (((uint64_t)batch * p->L << (p->log2N - 14)) > 0xffffffffull) return cudaErrorNotSupported;
            const uint32_t slog = p->log2N - 14;
            cudaError_t e;
            if (!inverse) {
                if ((e = launch_ntt_global32(p, d_polys, batch, false, st)) != cudaSuccess) return e;
                return launch<14, false>(p, d_polys, batch, st, false, slog);
            }
            if ((e = launch<14, true>(p, d_polys, batch, st, false, slog)) != cudaSuccess) return e;
            return launch_ntt_global32(p, d_polys, batch, true, st);
        }
    }
    return cudaErrorNotSupported;
}

// u64 words, every prime < 2^30 (residues < q: the high words are zero and stay zero)
cudaError_t launch_ntt32_c5_u64(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, bool inverse,
                                cudaStream_t st) {
    if (!p->u32_for_u64 || !p->tw32) return cudaErrorNotSupported;
    if (batch == 0) return cudaSuccess;
    if ((uint64_t)batch * p->L > 0xffffffffull || ((uintptr_t)d_polys & 15)) return cudaErrorNotSupported;
    using namespace c5u32;
    switch (p->log2N) {
        case 12: return inverse ? launch<12, true>(p, d_polys, batch, st, true) : launch<12, false>(p, d_polys, batch, st, true);
        case 13: return inverse ? launch<13, true>(p, d_polys, batch, st, true) : launch<13, false>(p, d_polys, batch, st, true);
        case 14: return inverse ? launch<14, true>(p, d_polys, batch, st, true) : launch<14, false>(p, d_polys, batch, st, true);
    }
    return cudaErrorNotSupported;
}

// Slot pack + INTT_t of the query path at N = 2^12 .. 2^14 (cudaErrorNotSupported below).
cudaError_t launch_pack_intt_q32(const ephdc_ctx *c, const int8_t *d_H, uint32_t nq, uint32_t b0, uint32_t nbat,
                                 uint32_t *d_M, cudaStream_t st, bool no_prefetch) {
    using namespace c5u32;
    PackArgs32 a{};
    a.t = (u32)c->t;
    a.ninv = c->ninv_t;
    a.ninv_p = c->ninv_t_p;
    a.k = c->p.k;
    a.B = c->B;
    a.D = c->p.D_live;
    a.nq = nq;
    a.b0 = b0;
    a.nbat = nbat;
    a.kmagic = c->p.k > 1 ? (u32)((1ull << 32) / c->p.k + 1) : 0u;   // k = 1: identity
    a.zero = 0;
    a.itw = c->dev.itw_t;
    const uint64_t rows = (uint64_t)nbat * a.D;
    if (rows == 0) return cudaSuccess;
    auto go = [&](auto kern, int lg) -> cudaError_t {
        const u32 grid = (u32)std::min<uint64_t>(rows, 148ull * (lg == 12 ? 4 : lg == 13 ? 2 : 1));
        const size_t smem = 1024 + sizeof(u32) * 2 * ((size_t)1 << lg) + sizeof(TwPair<u32>) * (((size_t)1 << lg) >> 5);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, (1u << lg) / kE, smem, st>>>(d_H, a, d_M);
        return counted(cudaGetLastError());
    };
    switch (c->p.log2N) {
        case 12: return no_prefetch ? go(k_pack_intt32<12, false>, 12) : go(k_pack_intt32<12, true>, 12);
        case 13: return no_prefetch ? go(k_pack_intt32<13, false>, 13) : go(k_pack_intt32<13, true>, 13);
        case 14: return no_prefetch ? go(k_pack_intt32<14, false>, 14) : go(k_pack_intt32<14, true>, 14);
    }
    return cudaErrorNotSupported;
}

}  // namespace ephdc
