// modarith.cuh -- modular arithmetic for the sm_100a kernels (integer pipe only).
//
// u64 residues (q < 2^61):  Shoup products with precomputed companions w' =
//   floor(w * 2^64 / q) for constant twiddles (Harvey lazy butterflies keep
//   values in [0, 4q)), Montgomery products for runtime x runtime operands
//   (the MAC: model residue times plaintext residue).
// u32 residues (t < 2^30): the same Shoup/Harvey forms on 32-bit words.
#pragma once
#include <stdint.h>

typedef uint64_t u64;
typedef uint32_t u32;

#define EPHDC_HD __host__ __device__ __forceinline__
#define EPHDC_D __device__ __forceinline__

template <typename W> struct TwPair { W w, wp; };
template <> struct __align__(16) TwPair<u64> { u64 w, wp; };
template <> struct __align__(8) TwPair<u32> { u32 w, wp; };

EPHDC_D u64 mulhi(u64 a, u64 b) { return (u64)__umul64hi((unsigned long long)a, (unsigned long long)b); }
EPHDC_D u32 mulhi(u32 a, u32 b) { return __umulhi(a, b); }

// x * w mod q in [0, 2q) for any x < 2^bits (Shoup)
template <typename W> EPHDC_D W mul_shoup_lazy(W x, W w, W wp, W q) { return x * w - mulhi(x, wp) * q; }

template <typename W> EPHDC_D W csub(W x, W m) { return x >= m ? x - m : x; }
// u32, x < 2m: x - m wraps above x exactly when x < m, so min() selects -- IADD + VIMNMX
// instead of ISETP + SEL + IADD
template <> EPHDC_D u32 csub<u32>(u32 x, u32 m) { return min(x, x - m); }

// Cooley-Tukey butterfly, lazy (Harvey): X, Y in [0, 4q) -> X + wY, X - wY in [0, 4q)
template <typename W>
EPHDC_D void ct_bfly(W &X, W &Y, const TwPair<W> tw, W q, W two_q) {
    W x = csub(X, two_q);
    W t = mul_shoup_lazy(Y, tw.w, tw.wp, q);
    X = x + t;
    Y = x - t + two_q;
}

// Gentleman-Sande butterfly, lazy: X, Y in [0, 2q) -> X + Y, (X - Y) w in [0, 2q)
template <typename W>
EPHDC_D void gs_bfly(W &X, W &Y, const TwPair<W> tw, W q, W two_q) {
    W x = X, y = Y;
    X = csub(x + y, two_q);
    Y = mul_shoup_lazy(x - y + two_q, tw.w, tw.wp, q);
}

// [0, 4q) -> [0, q)
template <typename W> EPHDC_D W reduce4(W x, W q, W two_q) { return csub(csub(x, two_q), q); }

// Montgomery: a * b * 2^-64 mod q, a, b < q < 2^63, result in [0, q).
// m = lo(ab) * q^-1 mod 2^64 makes lo(mq) = lo(ab), so (ab - mq) / 2^64 = hi(ab) - hi(mq) in (-q, q).
EPHDC_D u64 mont_mul(u64 a, u64 b, u64 q, u64 qinv) {
    u64 lo = a * b;
    u64 hi = mulhi(a, b);
    u64 m = lo * qinv;
    u64 mh = mulhi(m, q);
    u64 r = hi - mh;
    return hi < mh ? r + q : r;
}
