// kernels.cu -- sm_100a kernels of the EP-HDC client hot path and their launchers.
//
//  K1 k_encode        HDC encoding GEMM + quantisation          [int8 dp4a]
//  K2 k_pack_intt     slot pack + inverse NTT mod t ("EncPt")
//  K3+K4 k_ntt_mac    centered lift (#3) + forward NTT mod q_j + ct x pt MAC over a
//                     chunk of dims, atomically folded into the scores
//  k_finalize         canonical scores ciphertext (undo the Montgomery 2^-64)
//  k_encrypt          model encryption c0 = NTT(Delta m + e) - a s, c1 = a
//  k_ntt_batch / k_mac  standalone kernels of the c5 microbench
// DESIGN.md "Kernels" gives each kernel's roofline and algorithmic bytes/ops.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "internal.h"
#include "modf64.cuh"
#include "ntt_dev.cuh"
#include "rng.cuh"

namespace ephdc {

std::atomic<uint64_t> g_launches{0};

using namespace ephdc_ntt;

constexpr int kE = 16;  // elements per thread in every NTT pass
// one CTA per 2^14-coefficient polynomial: 32 elements per thread (512 threads keep 128
// registers each; 1024 threads x 64 registers spilled)
template <int LG> constexpr int batch_E() { return LG >= 14 ? 32 : kE; }

// streaming (evict-first) 64-bit load for data read once
EPHDC_D u64 ldcs64(const u64 *p) { return (u64)__ldcs(reinterpret_cast<const unsigned long long *>(p)); }

// =====================================================================================
// K1: encoder  acc[d][q] = sum_f P[d][f] X[q][f];  h = clamp((acc + 2^(s-1)) >> s)
// =====================================================================================
template <bool UNSIGNED_X>
__device__ __forceinline__ int dot4(int a, int b, int c) {
    int r;
    if constexpr (UNSIGNED_X) asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    else asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

template <bool UNSIGNED_X, bool RAW>
__global__ void __launch_bounds__(256) k_encode(const uint8_t *__restrict__ X, const int8_t *__restrict__ P, u32 nq,
                                                u32 F, u32 D_live, u32 shift, int qmax, void *__restrict__ Hout) {
    constexpr int TD = 64, TQ = 64, KW = 16;  // tile 64 dims x 64 queries, 64-byte K step
    __shared__ int Ps[TD][KW + 1];
    __shared__ int Xs[TQ][KW + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const u32 d0 = blockIdx.y * TD, q0 = blockIdx.x * TQ;
    int acc[4][4] = {};
    const u32 FW = F >> 2;
    for (u32 k0 = 0; k0 < FW; k0 += KW) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int idx = threadIdx.x + r * 256;
            const int row = idx >> 4, w = idx & 15;
            const u32 kw = k0 + w;
            int pv = 0, xv = 0;
            if (kw < FW) {
                if (d0 + row < D_live) pv = *reinterpret_cast<const int *>(P + (size_t)(d0 + row) * F + 4 * kw);
                if (q0 + row < nq) xv = *reinterpret_cast<const int *>(X + (size_t)(q0 + row) * F + 4 * kw);
            }
            Ps[row][w] = pv;
            Xs[row][w] = xv;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            int a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = Ps[ty * 4 + i][w];
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = Xs[tx * 4 + i][w];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) acc[i][jj] = dot4<UNSIGNED_X>(a[i], b[jj], acc[i][jj]);
        }
        __syncthreads();
    }
    const int rnd = shift ? (1 << (shift - 1)) : 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const u32 d = d0 + ty * 4 + i;
        if (d >= D_live) continue;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const u32 q = q0 + tx * 4 + jj;
            if (q >= nq) continue;
            if constexpr (RAW) {
                reinterpret_cast<int *>(Hout)[(size_t)d * nq + q] = acc[i][jj];
            } else {
                int h = (acc[i][jj] + rnd) >> shift;   // arithmetic shift = floor division
                h = max(-qmax, min(qmax, h));
                reinterpret_cast<int8_t *>(Hout)[(size_t)d * nq + q] = (int8_t)h;
            }
        }
    }
}

// =====================================================================================
// K2: slot pack + INTT mod t.  One CTA per dim; output M[d][N] (u32, canonical).
// =====================================================================================
struct PackArgs {
    u32 t, two_t, ninv, ninv_p;
    u32 k, B, D_live;
    const TwPair<u32> *itw;
};

template <int LG, bool MODEL, bool CENTER>
__global__ void __launch_bounds__((1 << LG) / kE)
    k_pack_intt(const int8_t *__restrict__ src, u32 nq, u32 b, u32 d0, PackArgs a, u32 *__restrict__ M) {
    constexpr int N = 1 << LG, NT = N / kE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    u32 *buf = reinterpret_cast<u32 *>(smem_raw);
    const u32 d = d0 + blockIdx.x;
    b += blockIdx.y;  // grid.y = consecutive batches, written to M[blockIdx.y][blockIdx.x]
    u32 lim;
    const int8_t *row;
    if constexpr (MODEL) {
        lim = a.k * a.B;                 // model tile: slot i <- C[i mod k][d], i < k*B
        row = src + d;                   // src = class_hv [k][D_live]
    } else {
        const u32 nb = min(a.B, nq - b * a.B);
        lim = a.k * nb;                  // query slots: slot i <- h[d][b*B + i/k], i < k*n_b
        row = src + (size_t)d * nq + (size_t)b * a.B;
    }
    const u32 k = a.k, t = a.t;
    auto load = [&](int i) -> u32 {
        if ((u32)i >= lim) return 0u;
        int v;
        if constexpr (MODEL) v = row[(size_t)((u32)i % k) * a.D_live];
        else v = row[(u32)i / k];
        return v < 0 ? (u32)((int)t + v) : (u32)v;
    };
    inv_ntt<u32, LG, kE>(buf, load, a.itw, t);
    u32 *out = M + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * N;
    const u32 half_t = (t - 1) / 2;
    const int stid = sidx<u32>(threadIdx.x);
#pragma unroll
    for (int e = 0; e < kE; ++e) {
        const int pos = threadIdx.x + e * NT;
        const u32 y = csub(mul_shoup_lazy<u32>(buf[sidx_at<u32>(stid, e * NT)], a.ninv, a.ninv_p, t), t);
        // encryption inputs stay in [0, t) (Delta * m, reading #4); plaintexts that are
        // multiplied into ciphertexts are stored as their centered lift (reading #3), a
        // signed int32 (|m| < t/2 < 2^29)
        if constexpr (!CENTER) out[pos] = y;
        else out[pos] = y <= half_t ? y : (u32)((int)y - (int)t);
    }
}

// Inverse (Gentleman-Sande) passes over a twiddle table held in shared memory in the
// pass-major layout: the twiddle of (sub-stage sub, block-group blk, v) sits at slot
// N/2^(T0+sub+1) + v*nblk + blk, so a warp's lanes (consecutive blk) read consecutive
// pairs.  Same arithmetic as ntt_dev.cuh inv_pass (u32, lazy [0, 2t)).
// one Gentleman-Sande sub-stage (compile-time trip counts, so x[] stays in registers)
template <int N_, int T0_LOG, int R_LOG, int SUB>
EPHDC_D void gs_substages(u32 (&x)[1 << R_LOG], const TwPair<u32> *tw, int blk, u32 t, u32 two_t) {
    if constexpr (SUB < R_LOG) {
        constexpr int R = 1 << R_LOG, hs = 1 << SUB, nv = R / (2 * hs), nblk = N_ >> (T0_LOG + R_LOG);
#pragma unroll
        for (int v = 0; v < nv; ++v) {
            const TwPair<u32> w = tw[(N_ >> (T0_LOG + SUB + 1)) + v * nblk + blk];
#pragma unroll
            for (int kk = 0; kk < hs; ++kk) gs_bfly<u32>(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], w, t, two_t);
        }
        gs_substages<N_, T0_LOG, R_LOG, SUB + 1>(x, tw, blk, t, two_t);
    }
}

template <int LG, int T0_LOG, int R_LOG, bool FIRST, class Load>
EPHDC_D void inv_pass_perm(u32 *buf, const Load &load, const TwPair<u32> *tw, u32 t, u32 two_t) {
    constexpr int N = 1 << LG, NT = N / kE;
    constexpr int R = 1 << R_LOG, T0 = 1 << T0_LOG;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < kE / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> T0_LOG, off = g & (T0 - 1);
        const int base = blk * (T0 * R) + off;
        const int sb = sidx<u32>(base);
        u32 x[R];
#pragma unroll
        for (int kk = 0; kk < R; ++kk) {
            if constexpr (FIRST) x[kk] = load(base + kk * T0);
            else x[kk] = buf[sidx_at<u32>(sb, kk * T0)];
        }
        gs_substages<N, T0_LOG, R_LOG, 0>(x, tw, blk, t, two_t);
#pragma unroll
        for (int kk = 0; kk < R; ++kk) buf[sidx_at<u32>(sb, kk * T0)] = x[kk];
    }
    __syncthreads();
}

template <int LG, int DONE, bool FIRST, class Load>
EPHDC_D void inv_passes_perm(u32 *buf, const Load &load, const TwPair<u32> *tw, u32 t, u32 two_t) {
    if constexpr (DONE < LG) {
        constexpr int R_LOG = (LG - DONE) >= 4 ? 4 : (LG - DONE);
        inv_pass_perm<LG, DONE, R_LOG, FIRST>(buf, load, tw, t, two_t);
        inv_passes_perm<LG, DONE + R_LOG, false>(buf, load, tw, t, two_t);
    }
}

// =====================================================================================
// K2 (query path, persistent): slot pack + INTT mod t for a range of (batch, dim) rows.
// A CTA keeps the whole psi_t^-1 table in shared memory in the pass-major layout (the
// lanes of a warp read consecutive 8-byte pairs: conflict-free) and loops over rows
// with stride gridDim.x; the slot -> query division i / k is a multiply-high by
// m = floor(2^32 / k) + 1 (exact for i < 2^16, 2 <= k <= 2^16; k = 1 is the identity,
// whose multiplier 2^32 + 1 does not fit 32 bits).  Output: centered int32.
// =====================================================================================
template <int LG>
__global__ void __launch_bounds__((1 << LG) / kE, (LG >= 14) ? 1 : (16384 >> LG))
    k_pack_intt_q(const int8_t *__restrict__ H, u32 nq, u32 b0, u32 nbat, u32 D, PackArgs a, u32 kmagic,
                  u32 *__restrict__ M) {
    constexpr int N = 1 << LG, NT = N / kE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TwPair<u32> *tw = reinterpret_cast<TwPair<u32> *>(smem_raw);         // [N]
    u32 *buf = reinterpret_cast<u32 *>(smem_raw + sizeof(TwPair<u32>) * N);
    const int tid = threadIdx.x;
    for (int p = tid; p < N; p += NT) {
        if (p == 0) continue;
        const int lsb = 31 - __clz(p), sb = 1 << lsb;       // stage with sb blocks, half-size N/(2 sb)
        const int st = LG - 1 - lsb;                        // log2 of the half-size
        const int done = st & ~3, sub = st - done;
        const int rlog = (LG - done) < 4 ? (LG - done) : 4;
        const int nblk = N >> (done + rlog);
        const int r = p - sb, v = r / nblk, blk = r % nblk;
        tw[p] = a.itw[sb + blk * ((1 << rlog) >> (sub + 1)) + v];
    }
    __syncthreads();
    const u32 k = a.k, t = a.t, two_t = 2 * t, half_t = (t - 1) / 2;
    const u32 rows = nbat * D;
    for (u32 row = blockIdx.x; row < rows; row += gridDim.x) {
        const u32 bb = row / D, d = row - bb * D, b = b0 + bb;
        const u32 nb = min(a.B, nq - b * a.B);
        const u32 lim = k * nb;                 // query slots: slot i <- h[d][b*B + i/k], i < k*n_b
        const int8_t *src = H + (size_t)d * nq + (size_t)b * a.B;
        auto load = [&](int i) -> u32 {
            if ((u32)i >= lim) return 0u;
            const int v = src[k == 1u ? (u32)i : __umulhi((u32)i, kmagic)];
            return v < 0 ? (u32)((int)t + v) : (u32)v;
        };
        inv_passes_perm<LG, 0, true>(buf, load, tw, t, two_t);
        u32 *out = M + (size_t)row * N;
        const int stid = sidx<u32>(tid);
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const int pos = tid + e * NT;
            const u32 y = csub(mul_shoup_lazy<u32>(buf[sidx_at<u32>(stid, e * NT)], a.ninv, a.ninv_p, t), t);
            out[pos] = y <= half_t ? y : (u32)((int)y - (int)t);   // centered lift (reading #3)
        }
        __syncthreads();   // buf is rewritten by the next row's first pass
    }
}

// =====================================================================================
// K3+K4: centered lift + forward NTT mod q_j + MAC over a chunk of dims.
// CTA = (prime j, slice s of S, dim chunk); NC = N/S coefficients per CTA.
// =====================================================================================
struct MacArgs {
    PrimeSet ps;
    u32 t, half_t;       // lift threshold (t-1)/2
    u32 L, D_live, G;    // G = dims per chunk
    const TwPair<u64> *tw;  // [L][N]
};

template <int LGC, int S>
__global__ void __launch_bounds__((1 << LGC) / kE)
    k_ntt_mac(const u32 *__restrict__ M, const u64 *__restrict__ model, u64 *__restrict__ out, MacArgs a) {
    constexpr int NC = 1 << LGC, NT = NC / kE, N = NC * S;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    u64 *buf = reinterpret_cast<u64 *>(smem_raw);
    u64 *acc = buf + padded_len(NC);  // [2][kE][NT], thread-private columns
    const int tid = threadIdx.x;
    const u32 x = blockIdx.x;
    const u32 js = x % (a.L * S), chunk = x / (a.L * S);
    const u32 j = js / S, s = js % S;
    const u64 q = a.ps.q[j], qinv = a.ps.qinv[j], two_q = 2 * q;
    const TwPair<u64> *tw = a.tw + (size_t)j * N;
    const u32 d0 = chunk * a.G, d1 = min(a.D_live, d0 + a.G);
#pragma unroll
    for (int e = 0; e < 2 * kE; ++e) acc[e * NT + tid] = 0;
    TwPair<u64> w1{0, 0};
    if constexpr (S > 1) w1 = tw[1];
    for (u32 d = d0; d < d1; ++d) {
        const u32 *m = M + (size_t)d * N;
        auto lift = [&](u32 v) -> u64 { return (int)v >= 0 ? (u64)v : (u64)(int64_t)(int)v + q; };
        auto load = [&](int pos) -> u64 {
            const u64 U = lift(__ldg(m + pos));
            if constexpr (S == 1) {
                return U;
            } else {
                // first global stage (half-size N/2) fused into the load: slice s keeps U +- w V
                const u64 V = lift(__ldg(m + pos + NC));
                const u64 T = mul_shoup_lazy<u64>(V, w1.w, w1.wp, q);
                return s == 0 ? U + T : U + two_q - T;
            }
        };
        fwd_ntt<u64, LGC, kE>(buf, load, tw, (u32)(N + s * NC), q);
        const u64 *c0 = model + (((size_t)d * a.L + j) * 2) * N + (size_t)s * NC;
        const u64 *c1 = c0 + N;
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const int pos = tid + e * NT;
            const u64 p = reduce4<u64>(buf[pad(pos)], q, two_q);
            const u64 r0 = mont_mul(ldcs64(c0 + pos), p, q, qinv);
            const u64 r1 = mont_mul(ldcs64(c1 + pos), p, q, qinv);
            acc[e * NT + tid] = csub(acc[e * NT + tid] + r0, q);
            acc[(kE + e) * NT + tid] = csub(acc[(kE + e) * NT + tid] + r1, q);
        }
        __syncthreads();
    }
    u64 *o0 = out + ((size_t)0 * a.L + j) * N + (size_t)s * NC;
    u64 *o1 = out + ((size_t)1 * a.L + j) * N + (size_t)s * NC;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
        const int pos = tid + e * NT;
        atomicAdd(reinterpret_cast<unsigned long long *>(o0 + pos), acc[e * NT + tid]);
        atomicAdd(reinterpret_cast<unsigned long long *>(o1 + pos), acc[(kE + e) * NT + tid]);
    }
}

// out[c][j][i] <- (out mod q_j) * 2^64 mod q_j  (undo the 2^-64 of the Montgomery products)
__global__ void k_finalize(u64 *__restrict__ out, u32 L, u32 N, PrimeSet ps, u32 n_total) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_total) return;
    const u32 j = (i / N) % L;
    const u64 q = ps.q[j];
    out[i] = mont_mul(out[i] % q, ps.r2[j], q, ps.qinv[j]);
}

// Plaintext NTTs for parity export: p_hat[dd][j] = NTT_j(lift(M[dd])) (full N, one CTA per (dd, j)).
template <int LG>
__global__ void __launch_bounds__((1 << LG) / batch_E<LG>())
    k_plaintext_ntt(const u32 *__restrict__ M, u64 *__restrict__ pt, MacArgs a) {
    constexpr int E = batch_E<LG>();
    constexpr int N = 1 << LG, NT = N / E;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    u64 *buf = reinterpret_cast<u64 *>(smem_raw);
    const u32 j = blockIdx.x % a.L, dd = blockIdx.x / a.L;
    const u64 q = a.ps.q[j];
    const u32 *m = M + (size_t)dd * N;
    auto load = [&](int pos) -> u64 {
        const u32 v = m[pos];
        return (int)v >= 0 ? (u64)v : (u64)(int64_t)(int)v + q;
    };
    fwd_ntt<u64, LG, E>(buf, load, a.tw + (size_t)j * N, (u32)N, q);
    u64 *o = pt + ((size_t)dd * a.L + j) * N;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int pos = threadIdx.x + e * NT;
        o[pos] = reduce4<u64>(buf[pad(pos)], q, 2 * q);
    }
}

// =====================================================================================
// Model encryption: per (dim d, prime j): x = [Delta m_d + e_d]_q, c1 = a, c0 = NTT(x) - a s
// =====================================================================================
struct EncArgs {
    PrimeSet ps;
    u32 L;
    ephdc_rng::Key key;
    const u64 *cdt;
    const u64 *shat_mont;   // [L][N], s_hat * 2^64 mod q
    const TwPair<u64> *tw;  // [L][N]
};

template <int LG>
__global__ void __launch_bounds__((1 << LG) / batch_E<LG>())
    k_encrypt(const u32 *__restrict__ M, u64 g0, EncArgs a, u64 *__restrict__ out) {
    constexpr int E = batch_E<LG>();
    constexpr int N = 1 << LG, NT = N / E;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    u64 *buf = reinterpret_cast<u64 *>(smem_raw);
    __shared__ u64 cdt[ephdc_rng::kCdtLen];
    if (threadIdx.x < ephdc_rng::kCdtLen) cdt[threadIdx.x] = a.cdt[threadIdx.x];
    __syncthreads();
    const u32 j = blockIdx.x % a.L, dd = blockIdx.x / a.L;
    const u64 d = g0 + dd;   // random-stream index (model: d; HE-HDC-SR queries: 2^32 + b D + d)
    const u64 q = a.ps.q[j], delta = a.ps.delta[j], delta_p = a.ps.delta_p[j];
    const u32 *m = M + (size_t)dd * N;
    const ephdc_rng::Key &key = a.key;
    auto load = [&](int pos) -> u64 {
        const u64 x = mul_shoup_lazy<u64>((u64)m[pos], delta, delta_p, q);  // Delta*m in [0, 2q)
        const int e = ephdc_rng::gaussian(key, d, (u32)pos, cdt);
        return e >= 0 ? x + (u64)e : x + q - (u64)(-e);                     // [0, 4q)
    };
    fwd_ntt<u64, LG, E>(buf, load, a.tw + (size_t)j * N, (u32)N, q);
    u64 *c0 = out + (((size_t)dd * a.L + j) * 2) * N;
    u64 *c1 = c0 + N;
    const u64 *sh = a.shat_mont + (size_t)j * N;
    const u64 mask = a.ps.mask[j];
#pragma unroll 4
    for (int e = 0; e < E; ++e) {
        const int pos = threadIdx.x + e * NT;
        const u64 xh = reduce4<u64>(buf[pad(pos)], q, 2 * q);
        const u64 av = ephdc_rng::uniform_mod(key, d, j, a.L, (u32)pos, q, mask);
        const u64 as = mont_mul(av, sh[pos], q, a.ps.qinv[j]);
        c0[pos] = xh >= as ? xh - as : xh + q - as;
        c1[pos] = av;
    }
}

// =====================================================================================
// Standalone batched NTT (c5): CTA per (poly, prime, slice), in place on [batch][L][N].
// N <= 2^14: one CTA holds the whole polynomial.  N = 2^15, 2^16: the first (forward)
// or last (inverse) log2(N) - 14 stages run in k_ntt_global (one radix-2^GS butterfly
// group per thread, straight from/to HBM) and S = N / 2^14 CTAs each transform one
// slice of 2^14 coefficients in shared memory.
// =====================================================================================
// Word type W: u64 residues (any prime < 2^61) or u32 residues (primes < 2^30: the lazy
// [0, 4q) range fits 32 bits) -- the c5 sweep's two word classes.
template <typename W> struct NttArgsW {
    PrimeSet ps;
    u32 L;
    u32 log2N;               // full transform size (slices: LG < log2N)
    const TwPair<W> *tw;     // [L][N]
    const W *ninv;           // [L][2]
};
using NttArgs = NttArgsW<u64>;

template <typename W> EPHDC_D W ld_stream(const W *p) {
    if constexpr (sizeof(W) == 8) return (W)__ldcs(reinterpret_cast<const unsigned long long *>(p));
    else return (W)__ldcs(reinterpret_cast<const unsigned int *>(p));
}
template <typename W> EPHDC_D void st_stream(W *p, W v) {
    if constexpr (sizeof(W) == 8) __stcs(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
    else __stcs(reinterpret_cast<unsigned int *>(p), (unsigned int)v);
}

// elements per thread: 16, or 32 at 2^14 points (512 threads x 128 registers: no spills)
template <int LG, bool INV, typename W = u64>
__global__ void __launch_bounds__((1 << LG) / batch_E<LG>()) k_ntt_batch(W *__restrict__ polys, NttArgsW<W> a) {
    constexpr int E = batch_E<LG>();
    constexpr int NC = 1 << LG, NT = NC / E;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W *buf = reinterpret_cast<W *>(smem_raw);
    const u32 S = 1u << (a.log2N - LG), N = 1u << a.log2N;
    const u32 s = blockIdx.x % S, pj = blockIdx.x / S;   // pj = poly * L + j
    const u32 j = pj % a.L;
    W *p = polys + (size_t)pj * N + (size_t)s * NC;
    const W q = (W)a.ps.q[j];
    const TwPair<W> *tw = a.tw + (size_t)j * N;
    auto load = [&](int pos) -> W { return p[pos]; };
    if constexpr (!INV) {
        fwd_ntt<W, LG, E>(buf, load, tw, N + s * NC, q);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = threadIdx.x + e * NT;
            p[pos] = reduce4<W>(buf[sidx<W>(pos)], q, (W)(2 * q));
        }
    } else {
        // the first inverse pass groups E consecutive residues per thread: stage the
        // slice through shared memory with coalesced loads instead of reading that
        // pattern from global memory (32x the L1 wavefronts); the pass then reads and
        // rewrites only its own positions
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = threadIdx.x + e * NT;
            buf[sidx<W>(pos)] = p[pos];
        }
        __syncthreads();
        auto sload = [&](int pos) -> W { return buf[sidx<W>(pos)]; };
        inv_ntt<W, LG, E>(buf, sload, tw, q, N + s * NC);
        if (S == 1) {
            const W ni = a.ninv[2 * j], nip = a.ninv[2 * j + 1];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = threadIdx.x + e * NT;
                p[pos] = csub(mul_shoup_lazy<W>(buf[sidx<W>(pos)], ni, nip, q), q);
            }
        } else {  // lazy [0, 2q): the global stages and N^-1 follow in k_ntt_global
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = threadIdx.x + e * NT;
                p[pos] = buf[sidx<W>(pos)];
            }
        }
    }
}

// Persistent form of k_ntt_batch for one-CTA transforms (S = 1): a CTA walks a
// contiguous range of (prime, polynomial) items, prime-major, with the prime's whole
// twiddle table staged in shared memory once (the per-polynomial kernel reads it from
// L1/L2 in every pass).  u32 words: up to 2^14 (table + buffer 192 KB); u64: up to 2^13.
template <int LG, bool INV, typename W> constexpr size_t nttp_smem() {
    return sizeof(TwPair<W>) * ((size_t)1 << LG) + sizeof(W) * (size_t)padded_len(1 << LG);
}
template <int LG, typename W> constexpr int nttp_ctas_per_sm() {
    constexpr int by_smem = (int)((200u << 10) / nttp_smem<LG, false, W>());
    return by_smem < 1 ? 1 : by_smem > 4 ? 4 : by_smem;
}

template <int LG, bool INV, typename W>
__global__ void __launch_bounds__((1 << LG) / batch_E<LG>(), nttp_ctas_per_sm<LG, W>())
    k_ntt_batch_p(W *__restrict__ polys, NttArgsW<W> a, u32 batch) {
    constexpr int E = batch_E<LG>();
    constexpr int NC = 1 << LG, NT = NC / E;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TwPair<W> *tws = reinterpret_cast<TwPair<W> *>(smem_raw);
    W *buf = reinterpret_cast<W *>(smem_raw + sizeof(TwPair<W>) * NC);
    const u32 items = batch * a.L;
    const u32 w0 = (u32)((u64)items * blockIdx.x / gridDim.x), w1 = (u32)((u64)items * (blockIdx.x + 1) / gridDim.x);
    u32 jcur = 0xffffffffu;
    W q = 0, ni = 0, nip = 0;
    for (u32 w = w0; w < w1; ++w) {
        const u32 j = w / batch, b = w - j * batch;
        if (j != jcur) {
            __syncthreads();
            const TwPair<W> *tw = a.tw + (size_t)j * NC;
            for (int i = threadIdx.x; i < NC; i += NT) tws[i] = tw[i];
            q = (W)a.ps.q[j];
            if constexpr (INV) {
                ni = a.ninv[2 * j];
                nip = a.ninv[2 * j + 1];
            }
            jcur = j;
            __syncthreads();
        }
        W *p = polys + ((size_t)b * a.L + j) * NC;
        if constexpr (!INV) {
            auto load = [&](int pos) -> W { return ld_stream<W>(p + pos); };
            fwd_ntt<W, LG, E>(buf, load, tws, NC, q);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = threadIdx.x + e * NT;
                st_stream<W>(p + pos, reduce4<W>(buf[sidx<W>(pos)], q, (W)(2 * q)));
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = threadIdx.x + e * NT;
                buf[sidx<W>(pos)] = ld_stream<W>(p + pos);
            }
            __syncthreads();
            auto sload = [&](int pos) -> W { return buf[sidx<W>(pos)]; };
            inv_ntt<W, LG, E>(buf, sload, tws, q, NC);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = threadIdx.x + e * NT;
                st_stream<W>(p + pos, csub(mul_shoup_lazy<W>(buf[sidx<W>(pos)], ni, nip, q), q));
            }
        }
        __syncthreads();   // the next item's first pass rewrites buf
    }
}

// Two warp groups per CTA for the one-CTA integer transforms at 2^12 / 2^13 (the idea
// of the c5 FP64 kernels: with one team every warp reaches the load/store phase of a
// pass together).  Persistent over prime-major items, the prime's twiddle table in
// shared memory; group g takes alternate items of a prime segment into its own buffer
// (forward: pass 1 reads the polynomial straight from HBM, coalesced; inverse: a
// coalesced copy into the buffer first); each thread performs the one-team threads
// vt = t + 256 h, h < H = NT / 256; group-local named barriers between passes.
EPHDC_D void gbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EPHDC_D void gbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int LG, typename W> constexpr size_t ntt2g_smem() {
    return sizeof(TwPair<W>) * ((size_t)1 << LG) + 2 * sizeof(W) * ((size_t)1 << LG);
}

template <int LG, bool INV, typename W>
__global__ void __launch_bounds__(512, 1) k_ntt_batch_2g(W *__restrict__ polys, NttArgsW<W> a, u32 batch) {
    constexpr int E = kE, NC = 1 << LG, NT = NC / E, H = NT / 256;
    static_assert(H >= 1 && NT % 256 == 0, "two groups of 256 threads cover the one-team threads");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TwPair<W> *tws = reinterpret_cast<TwPair<W> *>(smem_raw);
    const int tid = threadIdx.x, g = tid >> 8, gt = tid & 255;
    W *buf = reinterpret_cast<W *>(smem_raw + sizeof(TwPair<W>) * NC) + (size_t)g * NC;
    const u32 items = batch * a.L;
    const u32 w0 = (u32)((u64)items * blockIdx.x / gridDim.x), w1 = (u32)((u64)items * (blockIdx.x + 1) / gridDim.x);
    auto gsync = [&]() { gbar_sync(1 + g, 256); };
    for (u32 i0 = w0; i0 < w1;) {
        const u32 j = i0 / batch, i1 = min(w1, (j + 1) * batch);
        __syncthreads();
        const TwPair<W> *tw = a.tw + (size_t)j * NC;
        for (int i = tid; i < NC; i += 512) tws[i] = tw[i];
        const W q = (W)a.ps.q[j], two_q = (W)(2 * q);
        W ni = 0, nip = 0;
        if constexpr (INV) {
            ni = a.ninv[2 * j];
            nip = a.ninv[2 * j + 1];
        }
        __syncthreads();
        const bool pair = i0 + 1 < i1;
        if (g == 1 && pair) gbar_sync(3, 512);   // group 1 one pass behind
        for (u32 w = i0 + (u32)g; w < i1; w += 2) {
            W *p = polys + ((size_t)(w - j * batch) * a.L + j) * NC;
            if constexpr (!INV) {
                auto load = [&](int pos) -> W { return ld_stream<W>(p + pos); };
                // levels in passes of 4 (T0 = LG-1, LG-5, ...), the last pass the remainder
#pragma unroll 1
                for (int h = 0; h < H; ++h) fwd_pass_vt<W, LG, E, LG - 1, 4, true>(buf, load, tws, NC, q, two_q, gt + 256 * h);
                gsync();
                if (g == 0 && w == i0 && pair) gbar_arrive(3, 512);
#pragma unroll 1
                for (int h = 0; h < H; ++h) fwd_pass_vt<W, LG, E, LG - 5, 4, false>(buf, load, tws, NC, q, two_q, gt + 256 * h);
                gsync();
                if constexpr (LG - 8 > 4) {   // 2^13: 4 + 4 + 4 + 1
#pragma unroll 1
                    for (int h = 0; h < H; ++h) fwd_pass_vt<W, LG, E, LG - 9, 4, false>(buf, load, tws, NC, q, two_q, gt + 256 * h);
                    gsync();
#pragma unroll 1
                    for (int h = 0; h < H; ++h)
                        fwd_pass_vt<W, LG, E, LG - 13, LG - 12, false>(buf, load, tws, NC, q, two_q, gt + 256 * h);
                } else {                        // 2^12: 4 + 4 + 4
#pragma unroll 1
                    for (int h = 0; h < H; ++h)
                        fwd_pass_vt<W, LG, E, LG - 9, LG - 8, false>(buf, load, tws, NC, q, two_q, gt + 256 * h);
                }
                gsync();
#pragma unroll 1
                for (int h = 0; h < H; ++h) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int pos = gt + 256 * h + e * NT;
                        st_stream<W>(p + pos, reduce4<W>(buf[sidx<W>(pos)], q, two_q));
                    }
                }
            } else {
                auto none = [](int) -> W { return 0; };
#pragma unroll 1
                for (int h = 0; h < H; ++h) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int pos = gt + 256 * h + e * NT;
                        buf[sidx<W>(pos)] = ld_stream<W>(p + pos);
                    }
                }
                gsync();
                if (g == 0 && w == i0 && pair) gbar_arrive(3, 512);
                // passes: half-sizes 2^0.., in groups of 4 (DONE = 0, 4, 8, [12])
#pragma unroll 1
                for (int h = 0; h < H; ++h) inv_pass_vt<W, LG, E, 0, 4>(buf, none, tws, NC, q, two_q, gt + 256 * h);
                gsync();
#pragma unroll 1
                for (int h = 0; h < H; ++h) inv_pass_vt<W, LG, E, 4, 4>(buf, none, tws, NC, q, two_q, gt + 256 * h);
                gsync();
                if constexpr (LG - 8 > 4) {
#pragma unroll 1
                    for (int h = 0; h < H; ++h) inv_pass_vt<W, LG, E, 8, 4>(buf, none, tws, NC, q, two_q, gt + 256 * h);
                    gsync();
#pragma unroll 1
                    for (int h = 0; h < H; ++h) inv_pass_vt<W, LG, E, 12, LG - 12>(buf, none, tws, NC, q, two_q, gt + 256 * h);
                } else {
#pragma unroll 1
                    for (int h = 0; h < H; ++h) inv_pass_vt<W, LG, E, 8, LG - 8>(buf, none, tws, NC, q, two_q, gt + 256 * h);
                }
                gsync();
#pragma unroll 1
                for (int h = 0; h < H; ++h) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int pos = gt + 256 * h + e * NT;
                        st_stream<W>(p + pos, csub(mul_shoup_lazy<W>(buf[sidx<W>(pos)], ni, nip, q), q));
                    }
                }
            }
            gsync();   // the next item's first pass rewrites buf
        }
        i0 = i1;
    }
}

// The GS = log2(N) - 14 global stages: forward (CT; first stages, canonical input ->
// lazy [0, 4q)) or inverse (GS; last stages, lazy [0, 2q) input -> times N^-1,
// canonical).  Thread = one radix-2^GS group {i + k * N/2^GS}.
template <int GS, bool INV, typename W = u64>
__global__ void __launch_bounds__(256) k_ntt_global(W *__restrict__ polys, u32 n_polys, NttArgsW<W> a) {
    constexpr int R = 1 << GS;
    const u32 N = 1u << a.log2N, T = N >> GS;
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (size_t)n_polys * T) return;
    const u32 pj = (u32)(gid / T), i = (u32)(gid % T), j = pj % a.L;
    W *p = polys + (size_t)pj * N + i;
    const W q = (W)a.ps.q[j], two_q = (W)(2 * q);
    const TwPair<W> *tw = a.tw + (size_t)j * N;
    W x[R];
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = ld_stream<W>(p + (size_t)k * T);
    if constexpr (!INV) {
#pragma unroll
        for (int sub = 0; sub < GS; ++sub) {
            const int h = R >> (sub + 1);
#pragma unroll
            for (int v = 0; v < (1 << sub); ++v) {
                const TwPair<W> w = tw[(1 << sub) + v];
#pragma unroll
                for (int kk = 0; kk < h; ++kk) ct_bfly<W>(x[v * 2 * h + kk], x[v * 2 * h + kk + h], w, q, two_q);
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) st_stream<W>(p + (size_t)k * T, x[k]);
    } else {
#pragma unroll
        for (int sub = 0; sub < GS; ++sub) {
            const int hs = 1 << sub;
#pragma unroll
            for (int v = 0; v < R / (2 * hs); ++v) {
                const TwPair<W> w = tw[(R >> (sub + 1)) + v];
#pragma unroll
                for (int kk = 0; kk < hs; ++kk) gs_bfly<W>(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], w, q, two_q);
            }
        }
        const W ni = a.ninv[2 * j], nip = a.ninv[2 * j + 1];
#pragma unroll
        for (int k = 0; k < R; ++k) st_stream<W>(p + (size_t)k * T, csub(mul_shoup_lazy<W>(x[k], ni, nip, q), q));
    }
}

// Standalone MAC on u32 words (primes < 2^30): products < 2^60 accumulate exactly in u64
// and are reduced every 15 terms (15 * 2^60 + q < 2^64) by a Barrett step with
// m = floor((2^64 - 1) / q); the per-split partial sums (< q) are folded with 64-bit
// atomics into out64 [L][2][N], reduced by k_mac32_out.  A thread owns 4 consecutive
// coefficients (16-byte streaming loads) and keeps 5 terms' loads in flight.
EPHDC_D u64 barrett64(u64 x, u64 q, u64 m) {
    u64 r = x - mulhi(x, m) * q;   // floor(x m / 2^64) >= floor(x / q) - 2: r < 3q
    r = r >= q ? r - q : r;
    return r >= q ? r - q : r;
}
__global__ void __launch_bounds__(256) k_mac32(const u32 *__restrict__ ct, const u32 *__restrict__ pt, u32 D, u32 L,
                                               u32 N, u32 dsplit, PrimeSet ps, u64 *__restrict__ out) {
    const u32 quads = (L * N) >> 2;
    const u32 g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= quads) return;
    const u32 lin = 4 * g, j = lin / N, i = lin % N;
    const u64 q = ps.q[j], m = ~0ull / q;
    const u32 per = (D + dsplit - 1) / dsplit;
    const u32 d0 = blockIdx.y * per, d1 = min(D, d0 + per);
    u64 a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
    const size_t sp = (size_t)L * N, sc = 2 * sp;   // strides of one term
    const u32 *pp = pt + (size_t)j * N + i, *cp = ct + (size_t)j * 2 * N + i;
    for (u32 d = d0; d < d1; d += 15) {
        const u32 e = min(d1, d + 15);
#pragma unroll 5
        for (u32 dd = d; dd < e; ++dd) {
            const uint4 p = __ldcs(reinterpret_cast<const uint4 *>(pp + dd * sp));
            const uint4 c0 = __ldcs(reinterpret_cast<const uint4 *>(cp + dd * sc));
            const uint4 c1 = __ldcs(reinterpret_cast<const uint4 *>(cp + dd * sc + N));
            a0[0] += (u64)c0.x * p.x;
            a0[1] += (u64)c0.y * p.y;
            a0[2] += (u64)c0.z * p.z;
            a0[3] += (u64)c0.w * p.w;
            a1[0] += (u64)c1.x * p.x;
            a1[1] += (u64)c1.y * p.y;
            a1[2] += (u64)c1.z * p.z;
            a1[3] += (u64)c1.w * p.w;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a0[k] = barrett64(a0[k], q, m);
            a1[k] = barrett64(a1[k], q, m);
        }
    }
    unsigned long long *o = reinterpret_cast<unsigned long long *>(out + (size_t)j * 2 * N + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        atomicAdd(o + k, a0[k]);
        atomicAdd(o + N + k, a1[k]);
    }
}

__global__ void k_mac32_out(const u64 *__restrict__ acc, u32 L, u32 N, PrimeSet ps, u32 *__restrict__ out) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * L * N) return;
    out[i] = (u32)(acc[i] % ps.q[i / (2 * N)]);
}

// Standalone MAC for primes >= 2^50 (u64 words): the exact 128-bit products are summed in
// 128-bit accumulators (32 terms of < 2^122 stay below 2^127) and folded to [0, q) every
// 32 terms with two Montgomery products: hi 2^64 + lo = mont(hi, 2^128 mod q) +
// mont(lo, 2^64 mod q) (mod q) -- one 64x64 -> 128 product per term instead of a
// Montgomery product (4 wide multiplies).  Each thread owns 2 consecutive coefficients of
// one prime and keeps 4 terms' loads in flight; outputs are true residues (k_mod_q).
struct U128 {
    u64 lo, hi;
};
EPHDC_D void mac128(U128 &acc, u64 a, u64 b) {
    const u64 lo = a * b, hi = mulhi(a, b);
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(acc.lo), "+l"(acc.hi) : "l"(lo), "l"(hi));
}
EPHDC_D u64 fold128(const U128 &x, u64 q, u64 qinv, u64 r2, u64 r1) {
    const u64 t = mont_mul(x.hi, r2, q, qinv) + mont_mul(x.lo, r1, q, qinv);   // < 2q
    return t >= q ? t - q : t;
}
// The D range is cut into dsplit pieces (blockIdx.y); piece y folds into row y / per_slot
// of out ([slots][L][2][N]; one row, the caller's output, when dsplit <= per_slot), so
// that a row sums at most per_slot residues < q and cannot wrap 2^64.
__global__ void __launch_bounds__(256) k_mac(const u64 *__restrict__ ct, const u64 *__restrict__ pt, u32 D, u32 L,
                                             u32 N, u32 dsplit, u32 per_slot, PrimeSet ps, u64 *__restrict__ out) {
    const u32 pairs = (L * N) >> 1;
    const u32 g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= pairs) return;
    const u32 lin = 2 * g, j = lin / N, i = lin % N;
    const u64 q = ps.q[j], qinv = ps.qinv[j], r2 = ps.r2[j];
    const u64 r1 = mont_mul(r2, 1, q, qinv);   // 2^64 mod q
    const u32 per = (D + dsplit - 1) / dsplit;
    const u32 d0 = blockIdx.y * per, d1 = min(D, d0 + per);
    U128 a00{0, 0}, a01{0, 0}, a10{0, 0}, a11{0, 0};
    const size_t sp = (size_t)L * N, sc = 2 * sp;
    const u64 *pp = pt + (size_t)j * N + i, *cp = ct + (size_t)j * 2 * N + i;
    for (u32 d = d0; d < d1; d += 32) {
        const u32 e = min(d1, d + 32);
#pragma unroll 4
        for (u32 dd = d; dd < e; ++dd) {
            const ulonglong2 p = __ldcs(reinterpret_cast<const ulonglong2 *>(pp + dd * sp));
            const ulonglong2 c0 = __ldcs(reinterpret_cast<const ulonglong2 *>(cp + dd * sc));
            const ulonglong2 c1 = __ldcs(reinterpret_cast<const ulonglong2 *>(cp + dd * sc + N));
            mac128(a00, c0.x, p.x);
            mac128(a01, c0.y, p.y);
            mac128(a10, c1.x, p.x);
            mac128(a11, c1.y, p.y);
        }
        a00 = U128{fold128(a00, q, qinv, r2, r1), 0};
        a01 = U128{fold128(a01, q, qinv, r2, r1), 0};
        a10 = U128{fold128(a10, q, qinv, r2, r1), 0};
        a11 = U128{fold128(a11, q, qinv, r2, r1), 0};
    }
    unsigned long long *o = reinterpret_cast<unsigned long long *>(
        out + (size_t)(blockIdx.y / per_slot) * 2 * L * N + (size_t)j * 2 * N + i);
    atomicAdd(o, a00.lo);
    atomicAdd(o + 1, a01.lo);
    atomicAdd(o + N, a10.lo);
    atomicAdd(o + N + 1, a11.lo);
}

// The same MAC on the FP64 pipe for primes < 2^50 (modf64.cuh: exact products in
// doubles).  The integer form needs ~12 half/quarter-rate IMAD.WIDE per Montgomery
// product, about the IMAD.WIDE peak at HBM speed; here a product is 6 FP64 operations
// (25% of the FP64 pipe at HBM speed).  Accumulators stay below 2^53 by a reduction
// every red_every terms (red_every (q/2 + 1) < 2^52); sums are true residues (no
// Montgomery factor): k_mod_q finishes.
__global__ void __launch_bounds__(256) k_mac_f64(const u64 *__restrict__ ct, const u64 *__restrict__ pt, u32 D, u32 L,
                                                 u32 N, u32 dsplit, PrimeSet ps, u32 red_every, u64 *__restrict__ out) {
    using namespace ephdc_f64;
    const u32 pairs = (L * N) >> 1;
    const u32 g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= pairs) return;
    const u32 lin = 2 * g, j = lin / N, i = lin % N;
    const double q = (double)ps.q[j], nq = -q, qinv = 1.0 / q;
    const u32 per = (D + dsplit - 1) / dsplit;
    const u32 d0 = blockIdx.y * per, d1 = min(D, d0 + per);
    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
    u32 cnt = 0;
#pragma unroll 4
    for (u32 d = d0; d < d1; ++d) {
        const ulonglong2 p = __ldcs(reinterpret_cast<const ulonglong2 *>(pt + ((size_t)d * L + j) * N + i));
        const ulonglong2 c0 = __ldcs(reinterpret_cast<const ulonglong2 *>(ct + (((size_t)d * L + j) * 2) * N + i));
        const ulonglong2 c1 = __ldcs(reinterpret_cast<const ulonglong2 *>(ct + (((size_t)d * L + j) * 2 + 1) * N + i));
        const double px = from_u64(p.x), py = from_u64(p.y);
        a00 = __dadd_rn(a00, mul_rt(from_u64(c0.x), px, qinv, nq));
        a01 = __dadd_rn(a01, mul_rt(from_u64(c0.y), py, qinv, nq));
        a10 = __dadd_rn(a10, mul_rt(from_u64(c1.x), px, qinv, nq));
        a11 = __dadd_rn(a11, mul_rt(from_u64(c1.y), py, qinv, nq));
        if (++cnt == red_every) {
            cnt = 0;
            a00 = reduce(a00, qinv, nq);
            a01 = reduce(a01, qinv, nq);
            a10 = reduce(a10, qinv, nq);
            a11 = reduce(a11, qinv, nq);
        }
    }
    unsigned long long *o = reinterpret_cast<unsigned long long *>(out + (size_t)j * 2 * N + i);
    atomicAdd(o, (unsigned long long)to_canonical_u64(reduce(a00, qinv, nq), q));
    atomicAdd(o + 1, (unsigned long long)to_canonical_u64(reduce(a01, qinv, nq), q));
    atomicAdd(o + N, (unsigned long long)to_canonical_u64(reduce(a10, qinv, nq), q));
    atomicAdd(o + N + 1, (unsigned long long)to_canonical_u64(reduce(a11, qinv, nq), q));
}

// out[i] <- out[i] mod q_j, prime j = (i / N) % L
__global__ void k_mod_q(u64 *__restrict__ out, u32 L, u32 N, PrimeSet ps, u32 n_total) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_total) return;
    out[i] %= ps.q[(i / N) % L];
}

// out[i] <- sum over the slot rows of (acc[s][i] mod q_j) mod q_j  (k_mac with slots > 1)
__global__ void k_mod_q_slots(const u64 *__restrict__ acc, u32 slots, u64 *__restrict__ out, u32 L, u32 N,
                              PrimeSet ps, u32 n_total) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_total) return;
    const u64 q = ps.q[(i / N) % L];
    u64 sum = 0;
    for (u32 k = 0; k < slots; ++k) {
        sum += acc[(size_t)k * n_total + i] % q;   // < 2q < 2^62
        if (sum >= q) sum -= q;
    }
    out[i] = sum;
}

// =====================================================================================
// launchers
// =====================================================================================
template <class K> static cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static inline cudaError_t counted(cudaError_t e, uint64_t n = 1) {
    if (e == cudaSuccess) g_launches.fetch_add(n, std::memory_order_relaxed);
    return e;
}

cudaError_t launch_encode(const ephdc_ctx *c, const void *d_X, const int8_t *d_P, uint32_t nq, void *d_H, bool raw,
                          cudaStream_t st) {
    // tensor-core path (encode_tc.cu) unless disabled or unsupported (F % 16 != 0,
    // operands not 16-byte aligned for TMA)
    if (c->p.encoder != EPHDC_ENCODER_DP4A && encode_tc_supported(c) && ((uintptr_t)d_X & 15) == 0 &&
        ((uintptr_t)d_P & 15) == 0) {
        cudaError_t e = launch_encode_tc(c, d_X, d_P, nq, d_H, raw, st);
        if (e != cudaErrorInvalidValue) return e;
    }
    dim3 grid((nq + 63) / 64, (c->p.D_live + 63) / 64);
    const int qmax = (1 << (c->p.Qbits - 1)) - 1;
    const uint8_t *X = (const uint8_t *)d_X;
    const u32 F = c->p.F, D = c->p.D_live, s = c->p.qshift;
    if (c->p.feat_unsigned) {
        if (raw) k_encode<true, true><<<grid, 256, 0, st>>>(X, d_P, nq, F, D, s, qmax, d_H);
        else k_encode<true, false><<<grid, 256, 0, st>>>(X, d_P, nq, F, D, s, qmax, d_H);
    } else {
        if (raw) k_encode<false, true><<<grid, 256, 0, st>>>(X, d_P, nq, F, D, s, qmax, d_H);
        else k_encode<false, false><<<grid, 256, 0, st>>>(X, d_P, nq, F, D, s, qmax, d_H);
    }
    return counted(cudaGetLastError());
}

static PackArgs pack_args(const ephdc_ctx *c) {
    PackArgs a;
    a.t = (u32)c->t;
    a.two_t = (u32)(2 * c->t);
    a.ninv = c->ninv_t;
    a.ninv_p = c->ninv_t_p;
    a.k = c->p.k;
    a.B = c->B;
    a.D_live = c->p.D_live;
    a.itw = c->dev.itw_t;
    return a;
}

template <int LG, bool MODEL, bool CENTER>
static cudaError_t pack_launch(const ephdc_ctx *c, const int8_t *src, u32 nq, u32 b, u32 nbat, u32 d0, u32 nd, u32 *M,
                               cudaStream_t st) {
    const size_t smem = sizeof(u32) * padded_len(1 << LG);
    auto kern = k_pack_intt<LG, MODEL, CENTER>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(nd, nbat), (1 << LG) / kE, smem, st>>>(src, nq, b, d0, pack_args(c), M);
    return counted(cudaGetLastError());
}

template <bool MODEL, bool CENTER>
static cudaError_t pack_dispatch(const ephdc_ctx *c, const int8_t *src, u32 nq, u32 b, u32 nbat, u32 d0, u32 nd,
                                 u32 *M, cudaStream_t st) {
    if (nd == 0 || nbat == 0) return cudaSuccess;
    if (nbat > 65535) return cudaErrorInvalidConfiguration;
    switch (c->p.log2N) {
        case 10: return pack_launch<10, MODEL, CENTER>(c, src, nq, b, nbat, d0, nd, M, st);
        case 11: return pack_launch<11, MODEL, CENTER>(c, src, nq, b, nbat, d0, nd, M, st);
        case 12: return pack_launch<12, MODEL, CENTER>(c, src, nq, b, nbat, d0, nd, M, st);
        case 13: return pack_launch<13, MODEL, CENTER>(c, src, nq, b, nbat, d0, nd, M, st);
        case 14: return pack_launch<14, MODEL, CENTER>(c, src, nq, b, nbat, d0, nd, M, st);
    }
    return cudaErrorInvalidValue;
}

template <int LG>
static cudaError_t packq_launch(const ephdc_ctx *c, const int8_t *H, u32 nq, u32 b0, u32 nbat, u32 *M, cudaStream_t st) {
    const size_t smem = sizeof(TwPair<u32>) * (1 << LG) + sizeof(u32) * padded_len(1 << LG);
    auto kern = k_pack_intt_q<LG>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const u32 D = c->p.D_live;
    const int per_sm = LG >= 14 ? 1 : (16384 >> LG);
    const uint64_t rows = (uint64_t)nbat * D;
    const u32 grid = (u32)std::min<uint64_t>(rows, 148ull * per_sm);
    const u32 kmagic = c->p.k > 1 ? (u32)((1ull << 32) / c->p.k + 1) : 0u;   // k = 1: identity
    kern<<<grid, (1 << LG) / kE, smem, st>>>(H, nq, b0, nbat, D, pack_args(c), kmagic, M);
    return counted(cudaGetLastError());
}

cudaError_t launch_pack_intt_queries(const ephdc_ctx *c, const int8_t *d_H, uint32_t nq, uint32_t b, uint32_t nbat,
                                     uint32_t d0, uint32_t nd, uint32_t *d_M, cudaStream_t st, uint32_t plan_flags) {
    const bool alt = (plan_flags & 128u) != 0, no_pf = (plan_flags & 256u) != 0;
    // whole-dimension calls (the hot path) use the persistent kernels -- at N >= 2^12 the
    // ntt32_c5.cu passes (alt: the round-1 kernel, A/B) -- partial ranges (the parity
    // export of single dims) the one-CTA-per-row kernel
    if (d0 == 0 && nd == c->p.D_live && nbat > 0 && nd > 0) {
        if (!alt) {
            const cudaError_t e = launch_pack_intt_q32(c, d_H, nq, b, nbat, d_M, st, no_pf);
            if (e != cudaErrorNotSupported) return e;
        }
        switch (c->p.log2N) {
            case 10: return packq_launch<10>(c, d_H, nq, b, nbat, d_M, st);
            case 11: return packq_launch<11>(c, d_H, nq, b, nbat, d_M, st);
            case 12: return packq_launch<12>(c, d_H, nq, b, nbat, d_M, st);
            case 13: return packq_launch<13>(c, d_H, nq, b, nbat, d_M, st);
            case 14: return packq_launch<14>(c, d_H, nq, b, nbat, d_M, st);
        }
        return cudaErrorInvalidValue;
    }
    return pack_dispatch<false, true>(c, d_H, nq, b, nbat, d0, nd, d_M, st);
}

cudaError_t launch_pack_intt_model(const ephdc_ctx *c, const int8_t *d_C, uint32_t d0, uint32_t nd, uint32_t *d_M,
                                   cudaStream_t st) {
    return pack_dispatch<true, false>(c, d_C, 0, 0, 1, d0, nd, d_M, st);
}

cudaError_t launch_pack_intt_sr(const ephdc_ctx *c, const int8_t *src, bool model, uint32_t nq, uint32_t b,
                                uint32_t d0, uint32_t nd, uint32_t *d_M, cudaStream_t st) {
    // HE-HDC-SR: query plaintexts to encrypt ([0, t)), class tiles to multiply (centered)
    return model ? pack_dispatch<true, true>(c, src, 0, 0, 1, d0, nd, d_M, st)
                 : pack_dispatch<false, false>(c, src, nq, b, 1, d0, nd, d_M, st);
}

static MacArgs mac_args(const ephdc_ctx *c) {
    MacArgs a;
    a.ps = c->ps;
    a.t = (u32)c->t;
    a.half_t = (u32)((c->t - 1) / 2);
    a.L = c->L;
    a.D_live = c->p.D_live;
    a.G = c->fused_G;
    a.tw = c->dev.tw_q;
    return a;
}

size_t ntt_mac_smem_bytes(uint32_t lgc) {
    const size_t nc = (size_t)1 << lgc;
    return sizeof(u64) * (padded_len((int)nc) + 2 * nc);
}

template <int LGC, int S>
static cudaError_t ntt_mac_launch(const ephdc_ctx *c, const u32 *M, const u64 *model, u64 *out, cudaStream_t st,
                                  uint32_t d_lim) {
    const size_t smem = ntt_mac_smem_bytes(LGC);
    auto kern = k_ntt_mac<LGC, S>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const u32 grid = c->L * S * c->fused_chunks;
    MacArgs a = mac_args(c);
    a.D_live = std::min(a.D_live, d_lim);   // ephdc_infer_batch_prefix: the first d_lim dims
    kern<<<grid, (1 << LGC) / kE, smem, st>>>(M, model, out, a);
    return counted(cudaGetLastError());
}

cudaError_t launch_ntt_mac(const ephdc_ctx *c, const uint32_t *d_M, const uint64_t *d_model, uint64_t *d_out,
                           cudaStream_t st, uint32_t d_lim) {
    switch (c->p.log2N) {
        case 10: return ntt_mac_launch<10, 1>(c, d_M, d_model, d_out, st, d_lim);
        case 11: return ntt_mac_launch<11, 1>(c, d_M, d_model, d_out, st, d_lim);
        case 12: return ntt_mac_launch<12, 1>(c, d_M, d_model, d_out, st, d_lim);
        case 13: return ntt_mac_launch<13, 1>(c, d_M, d_model, d_out, st, d_lim);
        case 14: return ntt_mac_launch<13, 2>(c, d_M, d_model, d_out, st, d_lim);
    }
    return cudaErrorInvalidValue;
}

int ntt_mac_occupancy(uint32_t log2N, uint32_t S) {
    const uint32_t lgc = log2N - (S == 2 ? 1 : 0);
    const size_t smem = ntt_mac_smem_bytes(lgc);
    int per_sm = (int)((227 * 1024) / smem);
    return per_sm < 1 ? 1 : per_sm;
}

cudaError_t launch_finalize(const ephdc_ctx *c, uint64_t *d_out, cudaStream_t st) {
    const u32 n = 2 * c->L * c->N;
    k_finalize<<<(n + 255) / 256, 256, 0, st>>>(d_out, c->L, c->N, c->ps, n);
    return counted(cudaGetLastError());
}

template <int LG>
static cudaError_t pt_launch(const ephdc_ctx *c, const u32 *M, u32 nd, u64 *pt, cudaStream_t st) {
    const size_t smem = sizeof(u64) * padded_len(1 << LG);
    auto kern = k_plaintext_ntt<LG>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<nd * c->L, (1 << LG) / batch_E<LG>(), smem, st>>>(M, pt, mac_args(c));
    return counted(cudaGetLastError());
}

cudaError_t launch_plaintext_ntt(const ephdc_ctx *c, const uint32_t *d_M, uint32_t nd, uint64_t *d_pt,
                                 cudaStream_t st) {
    if (nd == 0) return cudaSuccess;
    switch (c->p.log2N) {
        case 10: return pt_launch<10>(c, d_M, nd, d_pt, st);
        case 11: return pt_launch<11>(c, d_M, nd, d_pt, st);
        case 12: return pt_launch<12>(c, d_M, nd, d_pt, st);
        case 13: return pt_launch<13>(c, d_M, nd, d_pt, st);
        case 14: return pt_launch<14>(c, d_M, nd, d_pt, st);
    }
    return cudaErrorInvalidValue;
}

template <int LG>
static cudaError_t enc_launch(const ephdc_ctx *c, const u32 *M, u64 d0, u32 nd, const u64 *shat, const ephdc_seed &key,
                              u64 *model, cudaStream_t st) {
    const size_t smem = sizeof(u64) * padded_len(1 << LG);
    auto kern = k_encrypt<LG>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    EncArgs a;
    a.ps = c->ps;
    a.L = c->L;
    for (int i = 0; i < 8; ++i) a.key.k[i] = key.key[i];
    a.cdt = c->dev.cdt;
    a.shat_mont = shat;
    a.tw = c->dev.tw_q;
    kern<<<nd * c->L, (1 << LG) / batch_E<LG>(), smem, st>>>(M, d0, a, model);
    return counted(cudaGetLastError());
}

cudaError_t launch_encrypt(const ephdc_ctx *c, const uint32_t *d_M, uint64_t d0, uint32_t nd,
                           const uint64_t *d_shat_mont, const ephdc_seed &key, uint64_t *d_model, cudaStream_t st) {
    if (nd == 0) return cudaSuccess;
    switch (c->p.log2N) {
        case 10: return enc_launch<10>(c, d_M, d0, nd, d_shat_mont, key, d_model, st);
        case 11: return enc_launch<11>(c, d_M, d0, nd, d_shat_mont, key, d_model, st);
        case 12: return enc_launch<12>(c, d_M, d0, nd, d_shat_mont, key, d_model, st);
        case 13: return enc_launch<13>(c, d_M, d0, nd, d_shat_mont, key, d_model, st);
        case 14: return enc_launch<14>(c, d_M, d0, nd, d_shat_mont, key, d_model, st);
    }
    return cudaErrorInvalidValue;
}

template <typename W> static NttArgsW<W> ntt_args(const ephdc_ntt_plan *p, bool inv) {
    NttArgsW<W> a;
    a.ps = p->ps;
    a.L = p->L;
    a.log2N = p->log2N;
    if constexpr (sizeof(W) == 8) {
        a.tw = inv ? p->itw : p->tw;
        a.ninv = p->ninv;
    } else {
        a.tw = inv ? p->itw32 : p->tw32;
        a.ninv = p->ninv32;
    }
    return a;
}

template <int LG, bool INV, typename W>
static cudaError_t nttb_launch(const ephdc_ntt_plan *p, W *polys, u32 batch, cudaStream_t st) {
    // one-CTA transforms whose twiddle table fits beside the buffer: the persistent form
    // where it measured faster (r24, fraction of HBM, persistent vs per polynomial):
    // u32 inverse 2^12 0.401 vs 0.357, 2^13 0.300 vs 0.223, 2^14 0.265 vs 0.245; u32
    // forward 2^12 0.445 vs 0.430; u64 (60-bit) forward 2^13 0.203 vs 0.194.  Slower and
    // so not used: u32 forward 2^13 / 2^14 (0.343 / 0.278 vs 0.362 / 0.363 -- one or two
    // CTAs per SM instead of up to four), u64 2^12 (0.216 vs 0.264).
    // u32 words: the two-group persistent kernel where it measured fastest (r28, fraction
    // of HBM, two groups / persistent one team / per polynomial): forward 2^12 0.466 /
    // 0.445 / 0.424, 2^13 0.365 / 0.343 / 0.361; inverse 2^13 0.328 / 0.300 / 0.224
    // (inverse 2^12: 0.354 / 0.401 / 0.356 -- the one-team persistent form below)
    if constexpr (sizeof(W) == 4 && (LG == 13 || (LG == 12 && !INV))) {
        if (p->log2N == LG && !p->int_per_poly) {
            auto k2 = k_ntt_batch_2g<LG, INV, W>;
            constexpr size_t sm2 = ntt2g_smem<LG, W>();
            cudaError_t e = set_smem(k2, sm2);
            if (e != cudaSuccess) return e;
            const uint64_t items = (uint64_t)batch * p->L;
            const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(items, 148u));
            k2<<<grid, 512, sm2, st>>>(polys, ntt_args<W>(p, INV), batch);
            return counted(cudaGetLastError());
        }
    }
    constexpr bool kPersist = sizeof(W) == 4 ? (INV || LG == 12) : (!INV && LG == 13);
    if constexpr (kPersist && LG >= 12 && nttp_smem<LG, INV, W>() <= (200u << 10)) {
        if (p->log2N == LG && !p->int_per_poly) {
            auto kp = k_ntt_batch_p<LG, INV, W>;
            constexpr size_t sm = nttp_smem<LG, INV, W>();
            cudaError_t e = set_smem(kp, sm);
            if (e != cudaSuccess) return e;
            const uint64_t items = (uint64_t)batch * p->L;
            const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(items, 148u * nttp_ctas_per_sm<LG, W>()));
            kp<<<grid, (1 << LG) / batch_E<LG>(), sm, st>>>(polys, ntt_args<W>(p, INV), batch);
            return counted(cudaGetLastError());
        }
    }
    const size_t smem = sizeof(W) * padded_len(1 << LG);
    auto kern = k_ntt_batch<LG, INV, W>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const uint64_t grid = (uint64_t)batch * p->L << (p->log2N - LG);
    if (grid > 0x7fffffffull) return cudaErrorInvalidConfiguration;
    kern<<<(unsigned)grid, (1 << LG) / batch_E<LG>(), smem, st>>>(polys, ntt_args<W>(p, INV));
    return counted(cudaGetLastError());
}

template <int GS, bool INV, typename W>
static cudaError_t nttg_launch(const ephdc_ntt_plan *p, W *polys, u32 batch, cudaStream_t st) {
    const uint64_t n_polys = (uint64_t)batch * p->L;
    const uint64_t threads = n_polys * (p->N >> GS);
    const uint64_t blocks = (threads + 255) / 256;
    if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
    k_ntt_global<GS, INV, W><<<(unsigned)blocks, 256, 0, st>>>(polys, (u32)n_polys, ntt_args<W>(p, INV));
    return counted(cudaGetLastError());
}

// The GS = log2(N) - 14 global stages alone on u32 words (the ntt32_c5.cu slice kernels
// do the 2^14-point rest): forward first, inverse last (with N^-1).
cudaError_t launch_ntt_global32(const ephdc_ntt_plan *p, uint32_t *polys, uint32_t batch, bool inverse,
                                cudaStream_t st) {
    if (p->log2N == 15) return inverse ? nttg_launch<1, true, u32>(p, polys, batch, st) : nttg_launch<1, false, u32>(p, polys, batch, st);
    if (p->log2N == 16) return inverse ? nttg_launch<2, true, u32>(p, polys, batch, st) : nttg_launch<2, false, u32>(p, polys, batch, st);
    return cudaErrorNotSupported;
}

template <bool INV, typename W>
static cudaError_t ntt_large(const ephdc_ntt_plan *p, W *polys, u32 batch, cudaStream_t st) {
    // forward: global stages, then 2^14-point slices; inverse: slices, then global stages
    cudaError_t e = cudaSuccess;
    if (!INV)
        e = p->log2N == 15 ? nttg_launch<1, false, W>(p, polys, batch, st) : nttg_launch<2, false, W>(p, polys, batch, st);
    if (e != cudaSuccess) return e;
    e = nttb_launch<14, INV, W>(p, polys, batch, st);
    if (e != cudaSuccess || !INV) return e;
    return p->log2N == 15 ? nttg_launch<1, true, W>(p, polys, batch, st) : nttg_launch<2, true, W>(p, polys, batch, st);
}

template <typename W>
static cudaError_t ntt_batch_w(const ephdc_ntt_plan *p, W *d_polys, uint32_t batch, bool inverse, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
#define EPHDC_NTTB(LG)                                                             \
    case LG:                                                                       \
        return inverse ? nttb_launch<LG, true, W>(p, d_polys, batch, st)          \
                       : nttb_launch<LG, false, W>(p, d_polys, batch, st);
    switch (p->log2N) {
        EPHDC_NTTB(10)
        EPHDC_NTTB(11)
        EPHDC_NTTB(12)
        EPHDC_NTTB(13)
        EPHDC_NTTB(14)
        case 15:
        case 16: return inverse ? ntt_large<true, W>(p, d_polys, batch, st) : ntt_large<false, W>(p, d_polys, batch, st);
    }
#undef EPHDC_NTTB
    return cudaErrorInvalidValue;
}

cudaError_t launch_ntt_batch(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, bool inverse,
                             cudaStream_t st) {
    return ntt_batch_w<u64>(p, d_polys, batch, inverse, st);
}

cudaError_t launch_ntt_batch32(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, bool inverse,
                               cudaStream_t st) {
    if (!p->tw32) return cudaErrorInvalidValue;
    return ntt_batch_w<u32>(p, d_polys, batch, inverse, st);
}

// CTAs of two full waves of a 256-thread MAC kernel: the u32 MAC's D split is rounded DOWN
// to that count, so no third, nearly empty wave forms (r73: 0.88-0.93 -> 1.00-1.04 of HBM
// at the points whose split had rounded up to 1216 CTAs on 1184 slots).
template <class K> static u32 two_waves(K kernel) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, 0) != cudaSuccess || occ < 1) occ = 4;
    return 2u * 148u * (u32)occ;
}

cudaError_t launch_mac32(const ephdc_ntt_plan *p, const uint32_t *d_ct, const uint32_t *d_pt, uint32_t D,
                         uint32_t *d_out, cudaStream_t st) {
    const u32 L = p->L, N = p->N;
    if (((uintptr_t)d_ct | (uintptr_t)d_pt) & 15) return cudaErrorMisalignedAddress;   // 16-byte loads
    u64 *acc = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&acc), sizeof(u64) * 2 * L * N, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(acc, 0, sizeof(u64) * 2 * L * N, st);
    const u32 quads = (L * N) / 4;
    const u32 bx = (quads + 255) / 256;
    // <= 2^16 partial sums < q < 2^30 per coefficient: the 64-bit fold cannot wrap
    u32 dsplit = std::max<u32>(1, two_waves(k_mac32) / bx);
    dsplit = std::max<u32>(1, std::min(std::min(dsplit, D), 1u << 16));
    if (e == cudaSuccess && D > 0) {
        k_mac32<<<dim3(bx, dsplit), 256, 0, st>>>(d_ct, d_pt, D, L, N, dsplit, p->ps, acc);
        e = counted(cudaGetLastError());
    }
    if (e == cudaSuccess) {
        const u32 n = 2 * L * N;
        k_mac32_out<<<(n + 255) / 256, 256, 0, st>>>(acc, L, N, p->ps, d_out);
        e = counted(cudaGetLastError());
    }
    const cudaError_t e2 = cudaFreeAsync(acc, st);
    return e != cudaSuccess ? e : e2;
}

cudaError_t launch_mac(const ephdc_ntt_plan *p, const uint64_t *d_ct, const uint64_t *d_pt, uint32_t D,
                       uint64_t *d_out, cudaStream_t st) {
    const u32 L = p->L, N = p->N;
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(u64) * 2 * L * N, st);
    if (e != cudaSuccess) return e;
    if (D == 0) return cudaSuccess;
    const u32 pairs = (L * N) / 2;
    const u32 bx = (pairs + 255) / 256;
    u64 qmax = 0;
    for (u32 j = 0; j < L; ++j) qmax = std::max<u64>(qmax, p->q[j]);
    u32 max_split = (u32)std::min<u64>(~0ull / qmax, 1u << 16);
    const bool f64 = qmax < (1ull << 50);
    // ~8 CTAs per SM, rounded up.  Rounding down to two full waves (as launch_mac32 does)
    // was measured on these two kernels too (r74): +4-5 points on average but 1.00 -> 0.86
    // (FP64 form) and 0.95 -> 0.75 (integer form) at L N >= 2^19, where one piece is left --
    // not adopted here.
    const u32 target = std::max<u32>(1, (148u * 8u + bx - 1) / bx);
    u32 dsplit = std::min(std::min(target, D), max_split);
    const u32 n = 2 * L * N;
    if (f64) {   // FP64 pipe: 0.96-1.03 of measured HBM vs 0.74-0.77 (r26, profiles/r02/ab)
        const u32 red_every = (u32)std::max<double>(1.0, std::min<double>(64.0, std::floor(4503599627370496.0 / (double)qmax)));
        k_mac_f64<<<dim3(bx, dsplit), 256, 0, st>>>(d_ct, d_pt, D, L, N, dsplit, p->ps, red_every, d_out);
        e = counted(cudaGetLastError());
        if (e != cudaSuccess) return e;
        k_mod_q<<<(n + 255) / 256, 256, 0, st>>>(d_out, L, 2 * N, p->ps, n);
        return counted(cudaGetLastError());
    }
    // Integer form (primes >= 2^50): a 64-bit row holds at most max_split = floor(2^64 / q)
    // partial sums (15 at 60 bits).  When L N is small that many pieces cannot fill the
    // GPU (L = 1, N = 2^12: 8 x 15 CTAs, 0.48 of HBM, profiles/r02/r67), so the pieces
    // beyond max_split fold into further rows of a scratch [slots][L][2][N] (<= 1.3 MB:
    // it is only needed when bx is small) and k_mod_q_slots sums the rows mod q.
    const u32 want = std::max<u32>(1, std::min(std::min<u32>(target, D), 1u << 16));
    if (want > max_split) {
        const u32 slots = (want + max_split - 1) / max_split;
        u64 *acc = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void **>(&acc), sizeof(u64) * n * slots, st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(acc, 0, sizeof(u64) * n * slots, st);
        if (e == cudaSuccess) {
            k_mac<<<dim3(bx, want), 256, 0, st>>>(d_ct, d_pt, D, L, N, want, max_split, p->ps, acc);
            e = counted(cudaGetLastError());
        }
        if (e == cudaSuccess) {
            k_mod_q_slots<<<(n + 255) / 256, 256, 0, st>>>(acc, slots, d_out, L, 2 * N, p->ps, n);
            e = counted(cudaGetLastError());
        }
        const cudaError_t e2 = cudaFreeAsync(acc, st);
        return e != cudaSuccess ? e : e2;
    }
    k_mac<<<dim3(bx, dsplit), 256, 0, st>>>(d_ct, d_pt, D, L, N, dsplit, max_split, p->ps, d_out);
    e = counted(cudaGetLastError());
    if (e != cudaSuccess) return e;
    // output layout [L][2][N]: prime index = i / (2N); the folded sums are true residues
    k_mod_q<<<(n + 255) / 256, 256, 0, st>>>(d_out, L, 2 * N, p->ps, n);
    return counted(cudaGetLastError());
}

// MAC of D ciphertexts [D][L][2][N] with D plaintexts [D][L][N] under a context's primes,
// output [2][L][N] (the scores-ciphertext layout); d_tmp: [L][2][N] scratch.
cudaError_t launch_mac_ctx(const ephdc_ctx *c, const uint64_t *d_ct, const uint64_t *d_pt, uint32_t D, uint64_t *d_out,
                           cudaStream_t st) {
    ephdc_ntt_plan p;   // only the fields launch_mac reads
    p.q = c->q;
    p.L = c->L;
    p.N = c->N;
    p.log2N = c->p.log2N;
    p.ps = c->ps;
    u64 *tmp = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&tmp), sizeof(u64) * 2 * c->L * c->N, st);
    if (e != cudaSuccess) return e;
    e = launch_mac(&p, d_ct, d_pt, D, tmp, st);
    for (u32 cc = 0; cc < 2 && e == cudaSuccess; ++cc)   // [L][2][N] -> [2][L][N]
        e = cudaMemcpy2DAsync(d_out + (size_t)cc * c->L * c->N, sizeof(u64) * c->N, tmp + (size_t)cc * c->N,
                              sizeof(u64) * 2 * c->N, sizeof(u64) * c->N, c->L, cudaMemcpyDeviceToDevice, st);
    cudaError_t e2 = cudaFreeAsync(tmp, st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace ephdc
