// ntt_f64.cuh -- CTA-resident negacyclic forward NTT on the FP64 pipe (sm_100a).
//
// A CTA of NT = NC/16 threads transforms NC = 2^LGC residues (signed integers held
// in doubles, modf64.cuh) in padded shared memory.  Passes of up to 4 Cooley-Tukey
// stages run in registers (16 elements per thread, one __syncthreads per pass); the
// LAST stage (half-size 1) is a separate radix-2 pass whose outputs stay in registers
// and are handed to a sink -- the fused MAC, or a store for the parity export -- so
// that a thread owns the coefficient pairs (2g, 2g+1), g = tid + u*NT: consecutive
// threads touch consecutive 16-byte pairs, i.e. the sink's global accesses coalesce.
//
// Twiddles: the CTA's slice of the bit-reversed psi table, (w, fl(w/q)) pairs, in
// shared memory.  In the textbook loop (oracle/oracle_core.c) local stage with m
// blocks uses psi_rev[m + block]; a CTA owning slice s of S = N/NC (first global stage
// done by the caller while loading) needs psi_rev[S*m + s*m + block].  Inside a
// radix-16 pass whose first stage has m0 blocks, sub-stage `sub` of block-group B uses
// entries m0*2^sub + B*2^sub + v (v < 2^sub); the table stores that entry at slot
// m0*2^sub + v*m0 + B so that the lanes of a warp (consecutive B) read consecutive
// 16-byte slots -- free of shared-memory bank conflicts (the natural order has a
// 2^sub * 16-byte lane stride, up to 16-way conflicts).
#pragma once
#include "modf64.cuh"

namespace ephdc_f64 {

EPHDC_D int pad(int i) { return i + (i >> 4); }
constexpr int padded_len(int n) { return n + n / 16; }
constexpr int kE = 16;  // elements per thread

// One pass of R = 2^R_LOG local stages with half-sizes 2^T0_LOG ... 2^(T0_LOG-R_LOG+1).
// (LGC - 1 - T0_LOG is a multiple of 4: pass k starts at local stage level 4k.)
// A radix-16 pass whose blocks span <= 512 elements (T0_LOG <= 8) keeps every warp
// inside the window [512w, 512w + 512) of the buffer: if the next pass (or the tail,
// see fwd_ntt_tail) is warp-local too, the pass needs only __syncwarp().
template <int LGC, int T0_LOG, int R_LOG, int E = kE> constexpr bool warp_local_pass() {
    return R_LOG == 4 && T0_LOG <= 8 && ((1 << LGC) / E) % 32 == 0;
}

template <int LGC, int T0_LOG, int R_LOG, bool FROM_LOAD, bool SYNC_WARP, int E, class Load>
EPHDC_D void fwd_pass(double *buf, const Load &load, const double2 *tw, double nq) {
    constexpr int R = 1 << R_LOG;
    constexpr int TL_LOG = T0_LOG - (R_LOG - 1);
    constexpr int TL = 1 << TL_LOG;
    constexpr int NT = (1 << LGC) / E;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> TL_LOG, off = g & (TL - 1);
        const int base = (blk << (T0_LOG + 1)) + off;
        // pad(base + k*TL) = pad(base) + k*TL + (k*TL >> 4) whenever the block stride
        // 2^(T0+1) is a multiple of 16 (off < TL never carries into the next 16): one
        // address register plus compile-time offsets
        constexpr bool kConstPad = T0_LOG >= 3;
        const int pb = pad(base);
        auto addr = [&](int k) { return kConstPad ? pb + k * TL + ((k * TL) >> 4) : pad(base + k * TL); };
        double x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * TL);
            else x[k] = buf[addr(k)];
        }
        constexpr int m0 = (1 << LGC) >> (T0_LOG + 1);
#pragma unroll
        for (int sub = 0; sub < R_LOG; ++sub) {
            const int h = R >> (sub + 1);
#pragma unroll
            for (int v = 0; v < (1 << sub); ++v) {
                const double2 w = tw[(m0 << sub) + v * m0 + blk];
#pragma unroll
                for (int kk = 0; kk < h; ++kk) ct_bfly(x[v * 2 * h + kk], x[v * 2 * h + kk + h], w.x, w.y, nq);
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) buf[addr(k)] = x[k];
    }
    if constexpr (SYNC_WARP) __syncwarp();
    else __syncthreads();
}

// Stages with half-sizes 2^(REM-1) ... 2^1 in passes of <= 4; the first reads from
// load().  Hooks: before_last() runs before the last of these passes, after_first()
// right after the first (behind its barrier: every thread has consumed load()).
template <int LGC, int REM, bool FIRST, int WL, int E, class Load, class H1, class H2>
EPHDC_D void fwd_passes(double *buf, const Load &load, const double2 *tw, double nq, const H1 &after_first,
                        const H2 &before_last) {
    if constexpr (REM > 1) {
        constexpr int R_LOG = (REM - 1) >= 4 ? 4 : (REM - 1);
        constexpr int NEXT_REM = REM - R_LOG;
        constexpr int NEXT_R = (NEXT_REM - 1) >= 4 ? 4 : (NEXT_REM - 1);
        // the tail (NEXT_REM == 1) is warp-local with the windowed pair mapping (WL == 2)
        constexpr bool next_local = NEXT_REM <= 1 ? WL == 2 : warp_local_pass<LGC, NEXT_REM - 1, NEXT_R, E>();
        constexpr bool sync_warp = WL != 0 && warp_local_pass<LGC, REM - 1, R_LOG, E>() && next_local;
        if constexpr (NEXT_REM <= 1) before_last();
        fwd_pass<LGC, REM - 1, R_LOG, FIRST, sync_warp, E>(buf, load, tw, nq);
        if constexpr (FIRST) after_first();
        fwd_passes<LGC, NEXT_REM, false, WL, E>(buf, load, tw, nq, after_first, before_last);
    }
}

// Fills tw_s[1..n_slots) (n_slots = NC/2: the head stages only, or NC: also the last
// stage) with the slice-s twiddles of a prime (twg = [N] (w, w/q) pairs in psi_rev
// order) in the pass layout described above.  All NT threads call it.
template <int LGC, int S, int E = kE>
EPHDC_D void load_twiddles(double2 *tw_s, const double2 *__restrict__ twg, int s, int n_slots) {
    constexpr int NT = (1 << LGC) / E;
    for (int p = threadIdx.x; p < n_slots; p += NT) {
        if (p == 0) continue;
        const int lm = 31 - __clz(p), m = 1 << lm;
        int i = p;  // last stage (lm = LGC-1): natural order
        if (lm < LGC - 1) {
            const int start = lm & ~3, sub = lm - start, m0 = 1 << start;
            const int r = p - m, v = r / m0, B = r % m0;
            i = m + (B << sub) + v;
        }
        tw_s[p] = twg[S * m + s * m + (i - m)];
    }
}

// Global index (into a prime's psi_rev table) of the last-stage twiddle of pair g.
template <int LGC, int S> EPHDC_D int tail_twiddle_index(int s, int g) {
    constexpr int m = (1 << LGC) >> 1;
    return S * m + s * m + g;
}

// All stages but the last (half-sizes NC/2 ... 2) of the forward NTT of the NC =
// 2^LGC values load(i).  Values stay signed and lazy; DESIGN.md gives their bounds.
// WL: 0 = a CTA barrier after every pass; 1 = __syncwarp between warp-local head
// passes (default: measured fastest, profiles/r01/ab_sync.txt); 2 = also before the
// tail (windowed pair mapping -- fewer barriers, but slower model-load pattern).
template <int LGC, int WL = 1, int E = kE, class Load, class H1, class H2>
EPHDC_D void fwd_ntt_head(double *buf, const Load &load, const double2 *tw, double nq, const H1 &after_first,
                          const H2 &before_last) {
    static_assert(LGC >= 5, "at least one radix-16 pass before the final stage");
    fwd_passes<LGC, LGC, true, WL, E>(buf, load, tw, nq, after_first, before_last);
}

// Pair index of the last stage.  WINDOWED: thread (warp w, lane l) owns, for each of its
// E/16 radix-16 groups v = u/8 (thread group g = tid + v*NT in the head passes), the
// pairs p = v*8*NT + 256w + l + 32(u%8): exactly the 512-element window that warp w
// touched with group v in the warp-local head passes ([512w, 512w+512) shifted by
// v*16*NT), so the last head pass needs no CTA barrier; natural: p = tid + u*NT.
// Either way the lanes of a warp own consecutive 16-byte pairs (coalesced accesses).
template <int LGC, bool WINDOWED, int E = kE> EPHDC_D int tail_pair(int u) {
    constexpr int NT = (1 << LGC) / E;
    if constexpr (WINDOWED)
        return (u >> 3) * (8 * NT) + (threadIdx.x >> 5) * 256 + (threadIdx.x & 31) + 32 * (u & 7);
    else return threadIdx.x + u * NT;
}

// Last stage (half-size 1) for the coefficient pair p = tail_pair(u) with its twiddle
// (w, w/q).  Output order: the CTA's local bit-reversed evaluation order.
template <int LGC, bool WINDOWED, int E = kE>
EPHDC_D void fwd_ntt_tail(const double *buf, int u, double w, double wq, double nq, double &x0, double &x1) {
    const int p = tail_pair<LGC, WINDOWED, E>(u);
    const int a = pad(2 * p);   // 2p is even: 2p + 1 stays in the same 16-word row
    x0 = buf[a];
    x1 = buf[a + 1];
    ct_bfly(x0, x1, w, wq, nq);
}

// ---------------------------------------------------------------------------------
// The same passes for an explicit thread index vt (the two-group fused kernel: each
// thread of an 8-warp group performs the one-team threads vt = t and t + 256 in turn).
// Separate functions on purpose: the one-team kernel's schedule is sensitive to any
// change of its code (kernels_f64.cu, PREFIX).
// ---------------------------------------------------------------------------------
template <int LGC, int T0_LOG, int R_LOG, bool FROM_LOAD, class Load>
EPHDC_D void fwd_pass_vt(double *buf, const Load &load, const double2 *tw, double nq, int vt) {
    constexpr int R = 1 << R_LOG;
    constexpr int TL_LOG = T0_LOG - (R_LOG - 1);
    constexpr int TL = 1 << TL_LOG;
    const int g = vt;
    const int blk = g >> TL_LOG, off = g & (TL - 1);
    const int base = (blk << (T0_LOG + 1)) + off;
    constexpr bool kConstPad = T0_LOG >= 3;
    const int pb = pad(base);
    auto addr = [&](int k) { return kConstPad ? pb + k * TL + ((k * TL) >> 4) : pad(base + k * TL); };
    double x[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        if constexpr (FROM_LOAD) x[k] = load(base + k * TL);
        else x[k] = buf[addr(k)];
    }
    constexpr int m0 = (1 << LGC) >> (T0_LOG + 1);
#pragma unroll
    for (int sub = 0; sub < R_LOG; ++sub) {
        const int h = R >> (sub + 1);
#pragma unroll
        for (int v = 0; v < (1 << sub); ++v) {
            const double2 w = tw[(m0 << sub) + v * m0 + blk];
#pragma unroll
            for (int kk = 0; kk < h; ++kk) ct_bfly(x[v * 2 * h + kk], x[v * 2 * h + kk + h], w.x, w.y, nq);
        }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) buf[addr(k)] = x[k];
}

// windowed last-stage pair (tail_pair<LGC, true>) of one-team thread vt
template <int LGC> EPHDC_D int tail_pair_vt(int u, int vt) {
    constexpr int NT = (1 << LGC) / kE;
    return (u >> 3) * (8 * NT) + (vt >> 5) * 256 + (vt & 31) + 32 * (u & 7);
}

// ---------------------------------------------------------------------------------
// Inverse (Gentleman-Sande) passes on doubles, for the standalone c5 transform.  The
// sums X + Y double their bound every stage, so callers check 2^(LGC-1) * B0 < 2^51
// (ephdc_ntt_plan_create).  Twiddles in shared memory in the pass-major layout: the
// twiddle of (sub-stage sub, block-group blk, v) at slot NC/2^(T0+sub+1) + v*nblk + blk.
// ---------------------------------------------------------------------------------
template <int NC, int T0_LOG, int R_LOG, int SUB>
EPHDC_D void gs_substages_f64(double (&x)[1 << R_LOG], const double2 *tw, int blk, double nq) {
    if constexpr (SUB < R_LOG) {
        constexpr int R = 1 << R_LOG, hs = 1 << SUB, nv = R / (2 * hs), nblk = NC >> (T0_LOG + R_LOG);
#pragma unroll
        for (int v = 0; v < nv; ++v) {
            const double2 w = tw[(NC >> (T0_LOG + SUB + 1)) + v * nblk + blk];
#pragma unroll
            for (int kk = 0; kk < hs; ++kk) gs_bfly(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], w.x, w.y, nq);
        }
        gs_substages_f64<NC, T0_LOG, R_LOG, SUB + 1>(x, tw, blk, nq);
    }
}

// SINK: the last pass hands each output (natural position, value) to sink() -- the
// caller's scaling + global store -- instead of writing shared memory (no barrier).
// Inverse passes run with increasing half-sizes; a radix-16 pass with T0 <= 32 keeps
// each warp in the window [512w, 512w + 512) (one group per thread, blocks of 16 T0
// <= 512 elements), so between two such passes a __syncwarp suffices.
template <int LGC, int T0_LOG, int R_LOG> constexpr bool inv_warp_local() {
    return R_LOG == 4 && T0_LOG <= 5 && ((1 << LGC) / kE) % 32 == 0;
}
template <int LGC, int DONE> constexpr bool inv_next_warp_local() {
    constexpr int NEXT = DONE + ((LGC - DONE) >= 4 ? 4 : (LGC - DONE));
    if constexpr (NEXT >= LGC) return false;
    else return inv_warp_local<LGC, NEXT, ((LGC - NEXT) >= 4 ? 4 : (LGC - NEXT))>();
}
template <int LGC, int T0_LOG, int R_LOG, bool FROM_LOAD, bool SINK, class Load, class Sink>
EPHDC_D void inv_pass_f64(double *buf, const Load &load, const double2 *tw, double nq, const Sink &sink) {
    constexpr int NC = 1 << LGC, NT = NC / kE, R = 1 << R_LOG, T0 = 1 << T0_LOG;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < kE / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> T0_LOG, off = g & (T0 - 1);
        const int base = blk * (T0 * R) + off;
        double x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * T0);
            else x[k] = buf[pad(base + k * T0)];
        }
        gs_substages_f64<NC, T0_LOG, R_LOG, 0>(x, tw, blk, nq);
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (SINK) sink(base + k * T0, x[k]);
            else buf[pad(base + k * T0)] = x[k];
        }
    }
    if constexpr (!SINK) {
        if constexpr (inv_warp_local<LGC, T0_LOG, R_LOG>() && inv_next_warp_local<LGC, T0_LOG>()) __syncwarp();
        else __syncthreads();
    }
}

template <int LGC, int DONE, bool FIRST, class Load, class Sink>
EPHDC_D void inv_ntt_f64(double *buf, const Load &load, const double2 *tw, double nq, const Sink &sink) {
    if constexpr (DONE < LGC) {
        constexpr int R_LOG = (LGC - DONE) >= 4 ? 4 : (LGC - DONE);
        inv_pass_f64<LGC, DONE, R_LOG, FIRST, DONE + R_LOG == LGC>(buf, load, tw, nq, sink);
        inv_ntt_f64<LGC, DONE + R_LOG, false>(buf, load, tw, nq, sink);
    }
}

// Fills tw_s[1..NC) with the inverse twiddles psi^-1_rev of a full NC-point transform
// in the pass-major layout of inv_pass_f64.
template <int LGC>
EPHDC_D void load_inv_twiddles(double2 *tw_s, const double2 *__restrict__ twg) {
    constexpr int NC = 1 << LGC, NT = NC / kE;
    for (int p = threadIdx.x; p < NC; p += NT) {
        if (p == 0) continue;
        const int lsb = 31 - __clz(p), sb = 1 << lsb;
        const int st = LGC - 1 - lsb, done = st & ~3, sub = st - done;
        const int rlog = (LGC - done) < 4 ? (LGC - done) : 4;
        const int nblk = NC >> (done + rlog);
        const int r = p - sb, v = r / nblk, blk = r % nblk;
        tw_s[p] = twg[sb + blk * ((1 << rlog) >> (sub + 1)) + v];
    }
}

// ---------------------------------------------------------------------------------
// Inverse as Cooley-Tukey DIT (standalone c5 transform): the forward output x (bit-
// reversed) is DFT(a psi^j) permuted, so DIT stages with half-sizes 1, 2, ..., NC/2 and
// twiddles omega^-(NC/2h) jj (jj = position in the block of 2h) produce
// IDFT(DFT(a psi^j)) = NC a_j psi^j in natural order; the caller multiplies by
// NC^-1 psi^-j.  CT butterflies grow the bound by <= (1/2 + B 2^-54) q per stage, as in
// the forward transform (the GS form doubles it per stage).  Twiddles: the stage table
// tw[h + jj] (natural order; a warp's lanes read consecutive or identical entries).
// ---------------------------------------------------------------------------------
template <int T0_LOG, int R_LOG, int SUB>
EPHDC_D void dit_substages_f64(double (&x)[1 << R_LOG], const double2 *tw, int off, double nq) {
    if constexpr (SUB < R_LOG) {
        constexpr int R = 1 << R_LOG, hs = 1 << SUB, T0 = 1 << T0_LOG, h = hs * T0;
#pragma unroll
        for (int kk = 0; kk < hs; ++kk) {
            const double2 w = tw[h + off + kk * T0];
#pragma unroll
            for (int v = 0; v < R / (2 * hs); ++v) ct_bfly(x[v * 2 * hs + kk], x[v * 2 * hs + kk + hs], w.x, w.y, nq);
        }
        dit_substages_f64<T0_LOG, R_LOG, SUB + 1>(x, tw, off, nq);
    }
}

template <int LGC, int T0_LOG, int R_LOG, bool FROM_LOAD, bool SINK, class Load, class Sink>
EPHDC_D void dit_pass_f64(double *buf, const Load &load, const double2 *tw, double nq, const Sink &sink) {
    constexpr int NC = 1 << LGC, NT = NC / kE, R = 1 << R_LOG, T0 = 1 << T0_LOG;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < kE / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> T0_LOG, off = g & (T0 - 1);
        const int base = blk * (T0 * R) + off;
        double x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * T0);
            else x[k] = buf[pad(base + k * T0)];
        }
        dit_substages_f64<T0_LOG, R_LOG, 0>(x, tw, off, nq);
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (SINK) sink(base + k * T0, x[k]);
            else buf[pad(base + k * T0)] = x[k];
        }
    }
    if constexpr (!SINK) {
        if constexpr (inv_warp_local<LGC, T0_LOG, R_LOG>() && inv_next_warp_local<LGC, T0_LOG>()) __syncwarp();
        else __syncthreads();
    }
}

template <int LGC, int DONE, bool FIRST, class Load, class Sink>
EPHDC_D void inv_dit_f64(double *buf, const Load &load, const double2 *tw, double nq, const Sink &sink) {
    if constexpr (DONE < LGC) {
        constexpr int R_LOG = (LGC - DONE) >= 4 ? 4 : (LGC - DONE);
        dit_pass_f64<LGC, DONE, R_LOG, FIRST, DONE + R_LOG == LGC>(buf, load, tw, nq, sink);
        inv_dit_f64<LGC, DONE + R_LOG, false>(buf, load, tw, nq, sink);
    }
}

}  // namespace ephdc_f64
