// rng.cuh -- counter-based SplitMix64 streams (reading #7), host and device.
//
//   stream(seed, tag, a, b) = mix(mix(mix(seed ^ tag*G) ^ a*C1) ^ b*C2)
//   draw(st, n)             = mix(st + (n+1)*G)      (n-th SplitMix64 output from state st)
// Tags: 2 = secret key, 3 = uniform a, 4 = Gaussian e.
#pragma once
#include <stdint.h>

namespace ephdc_rng {

#define EPHDC_RNG_HD __host__ __device__ __forceinline__

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kStreamA = 0xD1B54A32D192ED03ULL;
constexpr uint64_t kStreamB = 0x8CB92BA72F3D8DD7ULL;
constexpr uint64_t kTagSecret = 2, kTagUniform = 3, kTagError = 4;
constexpr int kCdtLen = 20;

EPHDC_RNG_HD uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
EPHDC_RNG_HD uint64_t stream(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
    return mix(mix(mix(seed ^ (tag * kGold)) ^ (a * kStreamA)) ^ (b * kStreamB));
}
EPHDC_RNG_HD uint64_t draw(uint64_t st, uint64_t n) { return mix(st + (n + 1) * kGold); }

// reading #9
EPHDC_RNG_HD int ternary(uint64_t seed, uint32_t i) {
    return (int)(draw(stream(seed, kTagSecret, 0, i), 0) % 3) - 1;
}
// reading #8: rejection sampling with mask = 2^ceil(log2 q) - 1
EPHDC_RNG_HD uint64_t uniform_mod(uint64_t seed, uint64_t d, uint32_t j, uint32_t L, uint32_t i, uint64_t q,
                                  uint64_t mask) {
    const uint64_t st = stream(seed, kTagUniform, d * L + j, i);
    for (uint64_t n = 0;; ++n) {
        const uint64_t u = draw(st, n) & mask;
        if (u < q) return u;
    }
}
// reading #10: CDT magnitude, sign from the next draw
EPHDC_RNG_HD int gaussian(uint64_t seed, uint64_t d, uint32_t i, const uint64_t *cdt) {
    const uint64_t st = stream(seed, kTagError, d, i);
    const uint64_t u = draw(st, 0) >> 1;
    int k = 0;
    while (k < kCdtLen - 1 && u >= cdt[k]) ++k;
    if (k == 0) return 0;
    return (draw(st, 1) >> 63) ? -k : k;
}

}  // namespace ephdc_rng
