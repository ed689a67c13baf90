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
// shared memory, indexed like the textbook loop (oracle/oracle_core.c): local stage
// with m blocks uses tw[m + block].  A CTA owning slice s of S = N/NC (first global
// stage done by the caller while loading) stores tw_global[S*m + s*m + block] there.
#pragma once
#include "modf64.cuh"

namespace ephdc_f64 {

EPHDC_D int pad(int i) { return i + (i >> 4); }
constexpr int padded_len(int n) { return n + n / 16; }
constexpr int kE = 16;  // elements per thread

// One pass of R = 2^R_LOG local stages with half-sizes 2^T0_LOG ... 2^(T0_LOG-R_LOG+1).
template <int LGC, int T0_LOG, int R_LOG, bool FROM_LOAD, class Load>
EPHDC_D void fwd_pass(double *buf, const Load &load, const double2 *tw, double nq) {
    constexpr int R = 1 << R_LOG;
    constexpr int TL_LOG = T0_LOG - (R_LOG - 1);
    constexpr int TL = 1 << TL_LOG;
    constexpr int NT = (1 << LGC) / kE;
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < kE / R; ++u) {
        const int g = tid + u * NT;
        const int blk = g >> TL_LOG, off = g & (TL - 1);
        const int base = (blk << (T0_LOG + 1)) + off;
        double x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if constexpr (FROM_LOAD) x[k] = load(base + k * TL);
            else x[k] = buf[pad(base + k * TL)];
        }
        const int idx0 = ((1 << LGC) >> (T0_LOG + 1)) + blk;
#pragma unroll
        for (int sub = 0; sub < R_LOG; ++sub) {
            const int h = R >> (sub + 1);
#pragma unroll
            for (int v = 0; v < (1 << sub); ++v) {
                const double2 w = tw[(idx0 << sub) + v];
#pragma unroll
                for (int kk = 0; kk < h; ++kk) ct_bfly(x[v * 2 * h + kk], x[v * 2 * h + kk + h], w.x, w.y, nq);
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) buf[pad(base + k * TL)] = x[k];
    }
    __syncthreads();
}

// Stages with half-sizes 2^(REM-1) ... 2^1 in passes of <= 4; the first reads from load().
template <int LGC, int REM, bool FIRST, class Load>
EPHDC_D void fwd_passes(double *buf, const Load &load, const double2 *tw, double nq) {
    if constexpr (REM > 1) {
        constexpr int R_LOG = (REM - 1) >= 4 ? 4 : (REM - 1);
        fwd_pass<LGC, REM - 1, R_LOG, FIRST>(buf, load, tw, nq);
        fwd_passes<LGC, REM - R_LOG, false>(buf, load, tw, nq);
    }
}

// Forward NTT of the NC = 2^LGC values load(i); the outputs of the last stage are
// passed to sink(u, g, x0, x1) for the coefficient pairs (2g, 2g+1), g = tid + u*NT,
// in the CTA's local bit-reversed evaluation order.  Values stay signed and lazy;
// DESIGN.md gives their bounds.
template <int LGC, class Load, class Sink>
EPHDC_D void fwd_ntt(double *buf, const Load &load, const double2 *tw, double nq, const Sink &sink) {
    static_assert(LGC >= 5, "at least one radix-16 pass before the final stage");
    constexpr int NT = (1 << LGC) / kE;
    fwd_passes<LGC, LGC, true>(buf, load, tw, nq);
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < kE / 2; ++u) {
        const int g = tid + u * NT;
        double x0 = buf[pad(2 * g)], x1 = buf[pad(2 * g + 1)];
        const double2 w = tw[((1 << LGC) >> 1) + g];
        ct_bfly(x0, x1, w.x, w.y, nq);
        sink(u, g, x0, x1);
    }
}

}  // namespace ephdc_f64
