// ntt_dev.cuh -- CTA-resident negacyclic NTT passes in shared memory (sm_100a).
//
// A CTA of NT = NC/E threads transforms NC = 2^LG residues held in shared memory.
// Each pass runs up to 4 butterfly stages (radix 16) in registers: a thread loads
// E = 16 elements (E/R groups of R = 2^r elements at stride tl), applies r stages,
// and writes them back; one __syncthreads() per pass.  Shared memory is padded by
// one word per 16 (pad(i) = i + i/16) for 8-byte words and XOR-swizzled for 4-byte
// words (sidx) so that the pass patterns, including the 16-consecutive-element
// groups of the last forward / first inverse pass, are free of bank conflicts.
//
// Index conventions follow the textbook loops (oracle/oracle_core.c is the
// independent reference):
//   forward (Cooley-Tukey), stage half-size t, block i: W = psi_rev[N/(2t) + i]
//   inverse (Gentleman-Sande), stage half-size t, block i: W = psiinv_rev[N/(2t) + i]
// with psi_rev[k] = psi^brev(k).  A CTA may own one of S = N/NC output slices of a
// forward NTT (the split used by the fused MAC kernel at N = 16384): the caller then
// performs the first global stage while loading and passes tw_num = N + s*NC so the
// block indices are global.
#pragma once
#include "modarith.cuh"

namespace ephdc_ntt {

EPHDC_D int pad(int i) { return i + (i >> 4); }
constexpr int padded_len(int n) { return n + n / 16; }

// Shared-memory slot of element i of a W buffer.  8-byte words: pad(i) (every pass
// pattern conflict-free).  4-byte words: the pad layout puts 32 consecutive words in 33
// banks (a 2-way conflict for the passes whose lanes touch consecutive elements and
// for the row output); the XOR swizzle i ^ ((i >> 4) & 31) keeps all inverse-pass
// patterns and the output conflict-free in the same (unpadded) space.
template <typename W> EPHDC_D int sidx(int i) {
    if constexpr (sizeof(W) == 4) return i ^ ((i >> 4) & 31);
    else return pad(i);
}
// Slot of element base + c where base and the compile-time offset c share no set bits
// (a pass group: base = blk * block + off, c = k * stride).  The u32 swizzle is
// XOR-linear, so sidx(base + c) = sidx(base) ^ sidx(c): one LOP3 with an immediate per
// element.  sb = sidx<W>(base) for 4-byte words, base for 8-byte words.
template <typename W> EPHDC_D int sidx_at(int sb, int c) {
    if constexpr (sizeof(W) == 4) return sb ^ sidx<W>(c);
    else return pad(sb + c);
}
template <typename W> EPHDC_D int sidx_base(int base) {
    if constexpr (sizeof(W) == 4) return sidx<W>(base);
    else return base;
}

// Sub-stages of a forward pass with compile-time trip counts (x[] stays in registers).
template <typename W, int T0_LOG, int R_LOG, int SUB>
EPHDC_D void ct_substages(W (&x)[1 << R_LOG], const TwPair<W> *__restrict__ tw, u32 idx0, W q, W two_q) {
    if constexpr (SUB < R_LOG) {
        constexpr int R = 1 << R_LOG, h = R >> (SUB + 1);
#pragma unroll
        for (int v = 0; v < (1 << SUB); ++v) {
            const TwPair<W> w = tw[(idx0 << SUB) + v];
#pragma unroll
            for (int kk = 0; kk < h; ++kk) ct_bfly<W>(x[v * 2 * h + kk], x[v * 2 * h + kk + h], w, q, two_q);
        }
        ct_substages<W, T0_LOG, R_LOG, SUB + 1>(x, tw, idx0, q, two_q);
    }
}

// One forward pass: local stages with half-sizes 2^T0_LOG ... 2^(T0_LOG-R_LOG+1).
template <typename W, int LG, int E, int T0_LOG, int R_LOG, bool FROM_LOAD, class Load>
EPHDC_D void fwd_pass(W *buf, const Load &load, const TwPair<W> *__restrict__ tw, u32 tw_num, W q, W two_q) {
    constexpr int R = 1 << R_LOG;
    constexpr int TL_LOG = T0_LOG - (R_LOG - 1);
    constexpr int TL = 1 << TL_LOG;
    constexpr int NT = (1 << LG) / E;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> TL_LOG, off = g & (TL - 1);
        const int base = (blk << (T0_LOG + 1)) + off;
        const int sb = sidx_base<W>(base);
        W x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * TL);
            else x[k] = buf[sidx_at<W>(sb, k * TL)];
        }
        const u32 idx0 = (tw_num >> (T0_LOG + 1)) + (u32)blk;
        ct_substages<W, T0_LOG, R_LOG, 0>(x, tw, idx0, q, two_q);
#pragma unroll
        for (int k = 0; k < R; ++k) buf[sidx_at<W>(sb, k * TL)] = x[k];
    }
    __syncthreads();
}

template <typename W, int LG, int E, int REM, bool FIRST, class Load>
EPHDC_D void fwd_passes(W *buf, const Load &load, const TwPair<W> *__restrict__ tw, u32 tw_num, W q, W two_q) {
    if constexpr (REM > 0) {
        constexpr int R_LOG = REM >= 4 ? 4 : REM;
        fwd_pass<W, LG, E, REM - 1, R_LOG, FIRST>(buf, load, tw, tw_num, q, two_q);
        fwd_passes<W, LG, E, REM - R_LOG, false>(buf, load, tw, tw_num, q, two_q);
    }
}

// Forward NTT of NC = 2^LG values produced by load(local_index) (in [0, 4q));
// result (lazy, [0, 4q)) in buf[sidx<W>(i)], bit-reversed evaluation order.
template <typename W, int LG, int E, class Load>
EPHDC_D void fwd_ntt(W *buf, const Load &load, const TwPair<W> *__restrict__ tw, u32 tw_num, W q) {
    fwd_passes<W, LG, E, LG, true>(buf, load, tw, tw_num, q, (W)(2 * q));
}

// Sub-stages of an inverse pass with compile-time trip counts.
template <typename W, int LG, int T0_LOG, int R_LOG, int SUB>
EPHDC_D void gs_substages(W (&x)[1 << R_LOG], const TwPair<W> *__restrict__ itw, u32 tw_num, int blk, W q, W two_q) {
    if constexpr (SUB < R_LOG) {
        constexpr int R = 1 << R_LOG, hs = 1 << SUB;
#pragma unroll
        for (int v = 0; v < R / (2 * hs); ++v) {
            const u32 idx = (tw_num >> (T0_LOG + SUB + 1)) + (u32)((blk * R) >> (SUB + 1)) + v;
            const TwPair<W> w = itw[idx];
#pragma unroll
            for (int kk = 0; kk < hs; ++kk) gs_bfly<W>(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], w, q, two_q);
        }
        gs_substages<W, LG, T0_LOG, R_LOG, SUB + 1>(x, itw, tw_num, blk, q, two_q);
    }
}

// One inverse pass: stages with half-sizes 2^T0_LOG ... 2^(T0_LOG+R_LOG-1).
template <typename W, int LG, int E, int T0_LOG, int R_LOG, bool FROM_LOAD, class Load>
EPHDC_D void inv_pass(W *buf, const Load &load, const TwPair<W> *__restrict__ itw, u32 tw_num, W q, W two_q) {
    constexpr int R = 1 << R_LOG;
    constexpr int T0 = 1 << T0_LOG;
    constexpr int NT = (1 << LG) / E;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> T0_LOG, off = g & (T0 - 1);
        const int base = blk * (T0 * R) + off;
        const int sb = sidx_base<W>(base);
        W x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * T0);
            else x[k] = buf[sidx_at<W>(sb, k * T0)];
        }
        gs_substages<W, LG, T0_LOG, R_LOG, 0>(x, itw, tw_num, blk, q, two_q);
#pragma unroll
        for (int k = 0; k < R; ++k) buf[sidx_at<W>(sb, k * T0)] = x[k];
    }
    __syncthreads();
}

template <typename W, int LG, int E, int DONE, bool FIRST, class Load>
EPHDC_D void inv_passes(W *buf, const Load &load, const TwPair<W> *__restrict__ itw, u32 tw_num, W q, W two_q) {
    if constexpr (DONE < LG) {
        constexpr int R_LOG = (LG - DONE) >= 4 ? 4 : (LG - DONE);
        inv_pass<W, LG, E, DONE, R_LOG, FIRST>(buf, load, itw, tw_num, q, two_q);
        inv_passes<W, LG, E, DONE + R_LOG, false>(buf, load, itw, tw_num, q, two_q);
    }
}

// Inverse NTT (without the final N^-1) of values from load(i) in [0, 2q);
// result (lazy, [0, 2q)) in buf[sidx<W>(i)], natural coefficient order.  As for the
// forward transform, tw_num = N + s*NC makes a CTA that owns slice s of a larger
// transform (the remaining global stages done by the caller) index global blocks.
template <typename W, int LG, int E, class Load>
EPHDC_D void inv_ntt(W *buf, const Load &load, const TwPair<W> *__restrict__ itw, W q, u32 tw_num = 1u << LG) {
    inv_passes<W, LG, E, 0, true>(buf, load, itw, tw_num, q, (W)(2 * q));
}

// ---------------------------------------------------------------------------------
// The same passes for an explicit one-team thread index vt over NT_ONE = 2^LG / E
// threads (the two-group kernels: a thread of an 8-warp group performs vt = t and
// t + 256 in turn); no barrier inside -- the caller synchronises its group.
// ---------------------------------------------------------------------------------
template <typename W, int LG, int E, int T0_LOG, int R_LOG, bool FROM_LOAD, class Load>
EPHDC_D void fwd_pass_vt(W *buf, const Load &load, const TwPair<W> *__restrict__ tw, u32 tw_num, W q, W two_q,
                         int vt) {
    constexpr int R = 1 << R_LOG;
    constexpr int TL_LOG = T0_LOG - (R_LOG - 1);
    constexpr int TL = 1 << TL_LOG;
    constexpr int NT = (1 << LG) / E;
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
        const int g = vt + u * NT;
        const int blk = g >> TL_LOG, off = g & (TL - 1);
        const int base = (blk << (T0_LOG + 1)) + off;
        const int sb = sidx_base<W>(base);
        W x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * TL);
            else x[k] = buf[sidx_at<W>(sb, k * TL)];
        }
        const u32 idx0 = (tw_num >> (T0_LOG + 1)) + (u32)blk;
        ct_substages<W, T0_LOG, R_LOG, 0>(x, tw, idx0, q, two_q);
#pragma unroll
        for (int k = 0; k < R; ++k) buf[sidx_at<W>(sb, k * TL)] = x[k];
    }
}

template <typename W, int LG, int E, int T0_LOG, int R_LOG, class Load>
EPHDC_D void inv_pass_vt(W *buf, const Load &load, const TwPair<W> *__restrict__ itw, u32 tw_num, W q, W two_q,
                         int vt) {
    constexpr int R = 1 << R_LOG;
    constexpr int T0 = 1 << T0_LOG;
    constexpr int NT = (1 << LG) / E;
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
        const int g = vt + u * NT;
        const int blk = g >> T0_LOG, off = g & (T0 - 1);
        const int base = blk * (T0 * R) + off;
        const int sb = sidx_base<W>(base);
        W x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = buf[sidx_at<W>(sb, k * T0)];
        gs_substages<W, LG, T0_LOG, R_LOG, 0>(x, itw, tw_num, blk, q, two_q);
#pragma unroll
        for (int k = 0; k < R; ++k) buf[sidx_at<W>(sb, k * T0)] = x[k];
    }
}

}  // namespace ephdc_ntt
