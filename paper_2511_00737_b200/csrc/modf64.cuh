// modf64.cuh -- exact modular arithmetic on the FP64 pipe for primes q < 2^50.
//
// B200 (sm_100a) executes DFMA at 64 lanes/clk/SM (tools/int_peak.cu, profiles/r01/
// int_peak.jsonl), twice the rate of the 32x32-bit IMAD.WIDE / IMAD.HI that a u64
// product decomposes into.  Residues are held as signed integers in IEEE doubles
// (exact below 2^53) and every product is computed EXACTLY:
//
//   h = fl(x*w),  l = x*w - h        (fma; the error of a product is representable)
//   k = round(x*w/q)                 (fma with the 1.5*2^52 rounding constant)
//   r = (h - k*q) + l = x*w - k*q    (fma: h - k*q is an integer < 2^53; then exact add)
//
// so r == x*w (mod q) with no rounding anywhere: results are bit-identical to integer
// arithmetic after the final canonicalisation.  The bounds each function needs are
// stated on it; DESIGN.md "FP64 modular arithmetic" derives them and the host checks
// them per parameter set (ephdc_ctx_create) before selecting this path.
#pragma once
#include <stdint.h>

#ifndef EPHDC_D
#define EPHDC_D __device__ __forceinline__
#endif

namespace ephdc_f64 {

constexpr double kRound = 6755399441055744.0;  // 1.5 * 2^52: x + kRound - kRound = rint(x) for |x| < 2^51
constexpr double kTwo52 = 4503599627370496.0;  // 2^52

struct ModF {
    double q;     // the prime
    double nq;    // -q
    double qinv;  // fl(1/q)
};

// x * w - round(x * w/q) * q with wq = fl(w/q):  exact, |r| <= (1/2 + |x| 2^-54) q.
// Needs |x| < 2^51, 0 <= w < q < 2^50.
EPHDC_D double mul_tw(double x, double w, double wq, double nq) {
    const double h = __dmul_rn(x, w);
    const double l = __fma_rn(x, w, -h);
    const double k = __dadd_rn(__fma_rn(x, wq, kRound), -kRound);
    return __dadd_rn(__fma_rn(k, nq, h), l);
}

// a * b - round(a*b*qinv) * q for runtime operands:  exact, |r| <= (1/2 + 2 |ab/q| 2^-53) q + 1.
// Needs |a b / q| < 2^51.
EPHDC_D double mul_rt(double a, double b, double qinv, double nq) {
    const double h = __dmul_rn(a, b);
    const double l = __fma_rn(a, b, -h);
    const double k = __dadd_rn(__fma_rn(h, qinv, kRound), -kRound);
    return __dadd_rn(__fma_rn(k, nq, h), l);
}

// x - round(x/q) q:  exact, |r| <= q/2 + 1.  Needs |x| < 2^53.
EPHDC_D double reduce(double x, double qinv, double nq) {
    const double k = __dadd_rn(__fma_rn(x, qinv, kRound), -kRound);
    return __fma_rn(k, nq, x);
}

// Cooley-Tukey butterfly (X, Y) -> (X + wY, X - wY), all values signed, exact.
EPHDC_D void ct_bfly(double &X, double &Y, double w, double wq, double nq) {
    const double t = mul_tw(Y, w, wq, nq);
    const double x = X;
    X = __dadd_rn(x, t);
    Y = __dsub_rn(x, t);
}


// Exact conversions without the I2F/F2I conversion unit: an integer v < 2^52 placed in
// the mantissa of 2^52 (bit pattern 0x4330... | v) is the double 2^52 + v.
// Gentleman-Sande butterfly (X, Y) -> (X + Y, (X - Y) w).
EPHDC_D void gs_bfly(double &X, double &Y, double w, double wq, double nq) {
    const double x = X, y = Y;
    X = __dadd_rn(x, y);
    Y = mul_tw(__dsub_rn(x, y), w, wq, nq);
}

EPHDC_D double from_u64(uint64_t v) {  // v < 2^52
    return __dsub_rn(__longlong_as_double((long long)(v | 0x4330000000000000ull)), kTwo52);
}
// signed int32 v -> double, exact: the bit pattern 0x43300000:(v ^ 2^31) is 2^52 + 2^31 + v
EPHDC_D double from_i32(int v) {
    return __dsub_rn(__hiloint2double(0x43300000, v ^ (int)0x80000000), 4503601774854144.0);
}
// canonical residue: r in (-q, q) -> [0, q) as u64
EPHDC_D uint64_t to_canonical_u64(double r, double q) {
    const double c = r < 0.0 ? __dadd_rn(r, q) : r;
    return (uint64_t)__double_as_longlong(__dadd_rn(c, kTwo52)) & 0x000FFFFFFFFFFFFFull;
}

}  // namespace ephdc_f64
