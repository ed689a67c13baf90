// rng.cuh -- counter-based ChaCha20 streams (reading #7), host and device.
//
// Every random value of the scheme is a 64-bit word of one ChaCha20 block (RFC 8439
// sec. 2.3: 20 rounds, 256-bit key, 32-bit block counter, 96-bit nonce):
//   word64(key, tag, a, ctr, w) = out[2w] | out[2w+1] << 32,
//   out = ChaCha20_block(key, counter = ctr, nonce = (tag, lo32(a), hi32(a))),  w < 8.
// Streams (tags):
//   secret s_i         (2)  ctr = i/8, a = 0, word i%8                       (reading #9)
//   uniform a_{d,j,i}  (3)  first draw: a = d*L + j, ctr = i/8, word i%8     (reading #8)
//                      (5)  retry n >= 1: ctr = i + ((n-1)/8) * 2^16, word (n-1)%8
//   Gaussian e_{d,i}   (4)  a = d, ctr = i/4: magnitude word 2(i%4), sign word 2(i%4)+1
// ChaCha20 is a PRF: the published c1 = a residues reveal nothing about the key (the
// round-1 SplitMix64 output function was invertible).  The key is 256 bits from the OS
// (ephdc_seed_os) unless a caller asks for a deterministic test key (ephdc_seed_u64).
#pragma once
#include <stdint.h>

namespace ephdc_rng {

#define EPHDC_RNG_HD __host__ __device__ __forceinline__

constexpr uint32_t kTagSecret = 2, kTagUniform = 3, kTagError = 4, kTagUniformRetry = 5;
constexpr int kCdtLen = 20;

struct Key {
    uint32_t k[8];
};

EPHDC_RNG_HD uint32_t rotl(uint32_t x, int r) {
#ifdef __CUDA_ARCH__
    return __funnelshift_l(x, x, r);
#else
    return (x << r) | (x >> (32 - r));
#endif
}

#define EPHDC_QR(a, b, c, d)            \
    a += b; d ^= a; d = rotl(d, 16);    \
    c += d; b ^= c; b = rotl(b, 12);    \
    a += b; d ^= a; d = rotl(d, 8);     \
    c += d; b ^= c; b = rotl(b, 7);

// RFC 8439 sec. 2.3 block function: out[16] = state + 20 rounds(state)
EPHDC_RNG_HD void chacha20_block(const Key &key, uint32_t ctr, uint32_t n0, uint32_t n1, uint32_t n2,
                                 uint32_t (&out)[16]) {
    const uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key.k[0], key.k[1], key.k[2],
                             key.k[3],    key.k[4],    key.k[5],    key.k[6],    key.k[7], ctr,      n0,
                             n1,          n2};
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = in[i];
#pragma unroll 2
    for (int r = 0; r < 10; ++r) {
        EPHDC_QR(x[0], x[4], x[8], x[12]);
        EPHDC_QR(x[1], x[5], x[9], x[13]);
        EPHDC_QR(x[2], x[6], x[10], x[14]);
        EPHDC_QR(x[3], x[7], x[11], x[15]);
        EPHDC_QR(x[0], x[5], x[10], x[15]);
        EPHDC_QR(x[1], x[6], x[11], x[12]);
        EPHDC_QR(x[2], x[7], x[8], x[13]);
        EPHDC_QR(x[3], x[4], x[9], x[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = x[i] + in[i];
}
#undef EPHDC_QR

EPHDC_RNG_HD uint64_t word64(const uint32_t (&b)[16], uint32_t w) {
    // w is thread-dependent: select without dynamic register indexing
    uint64_t r = 0;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k)
        if (k == w) r = (uint64_t)b[2 * k] | ((uint64_t)b[2 * k + 1] << 32);
    return r;
}
EPHDC_RNG_HD uint64_t draw(const Key &key, uint32_t tag, uint64_t a, uint32_t ctr, uint32_t w) {
    uint32_t b[16];
    chacha20_block(key, ctr, tag, (uint32_t)a, (uint32_t)(a >> 32), b);
    return word64(b, w);
}

// reading #9
EPHDC_RNG_HD int ternary(const Key &key, uint32_t i) {
    return (int)(draw(key, kTagSecret, 0, i >> 3, i & 7) % 3) - 1;
}
// reading #8: rejection sampling with mask = 2^ceil(log2 q) - 1 (N <= 2^16)
EPHDC_RNG_HD uint64_t uniform_mod(const Key &key, uint64_t d, uint32_t j, uint32_t L, uint32_t i, uint64_t q,
                                  uint64_t mask) {
    const uint64_t a = d * L + j;
    uint64_t u = draw(key, kTagUniform, a, i >> 3, i & 7) & mask;
    for (uint32_t n = 1; u >= q; ++n) u = draw(key, kTagUniformRetry, a, i + (((n - 1) >> 3) << 16), (n - 1) & 7) & mask;
    return u;
}
// reading #10: CDT magnitude, sign from the paired word
EPHDC_RNG_HD int gaussian(const Key &key, uint64_t d, uint32_t i, const uint64_t *cdt) {
    uint32_t b[16];
    chacha20_block(key, i >> 2, kTagError, (uint32_t)d, (uint32_t)(d >> 32), b);
    const uint32_t w = 2 * (i & 3);
    const uint64_t u = word64(b, w) >> 1;
    int k = 0;
    while (k < kCdtLen - 1 && u >= cdt[k]) ++k;
    if (k == 0) return 0;
    return (word64(b, w + 1) >> 63) ? -k : k;
}

}  // namespace ephdc_rng
