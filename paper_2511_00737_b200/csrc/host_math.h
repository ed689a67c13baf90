// host_math.h -- host-side number theory of libephdc (product side; independent of oracle/).
#pragma once
#include <stdint.h>

#include <vector>

namespace ephdc_host {

typedef unsigned __int128 u128;

inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
uint64_t powmod(uint64_t a, uint64_t e, uint64_t m);
uint64_t invmod(uint64_t a, uint64_t p);  // p prime
bool is_prime_u64(uint64_t n);
uint32_t bit_reverse(uint32_t x, int bits);

// largest primes p < 2^bits[i], p = 1 mod 2N, distinct, not in exclude (reading #18)
bool ntt_prime_chain(uint32_t log2N, const uint32_t *bits, uint32_t count, const uint64_t *exclude,
                     uint32_t n_exclude, uint64_t *out);
// minimal primitive 2N-th root of unity mod p (reading #2); 0 on failure
uint64_t min_primitive_root_2n(uint64_t p, uint32_t log2N);
// Shoup companion floor(w * 2^bits / p)
inline uint64_t shoup64(uint64_t w, uint64_t p) { return (uint64_t)(((u128)w << 64) / p); }
inline uint32_t shoup32(uint32_t w, uint32_t p) { return (uint32_t)(((uint64_t)w << 32) / p); }
// p^-1 mod 2^64 (p odd)
uint64_t inv_mod_2_64(uint64_t p);
// 2^128 mod p
uint64_t two128_mod(uint64_t p);

// x^brev(k) for k < N
void pow_brev(uint64_t x, uint64_t p, uint32_t log2N, uint64_t *out);

// discrete Gaussian CDT (reading #10)
void gaussian_cdt(double sigma, uint64_t out[20]);

// plain host negacyclic NTTs (keygen s_hat; decryption)
struct HostNtt {
    uint32_t log2N = 0;
    uint64_t p = 0;
    std::vector<uint64_t> fw, inv;  // psi^brev(k), psi^-brev(k)
    uint64_t ninv = 0;
    void init(uint64_t p, uint64_t psi, uint32_t log2N);
    void forward(uint64_t *a) const;
    void inverse(uint64_t *a) const;
};

// multi-precision helpers (little-endian u64 limbs)
typedef std::vector<uint64_t> Big;
Big big_from_product(const std::vector<uint64_t> &ps);
Big big_div_small(const Big &a, uint64_t d, uint64_t *rem);
uint64_t big_mod_small(const Big &a, uint64_t m);
int big_cmp(const Big &a, const Big &b);
void big_add_inplace(Big &a, const Big &b);
void big_sub_inplace(Big &a, const Big &b);        // requires a >= b
Big big_mul_small(const Big &a, uint64_t m);
long double big_to_ld(const Big &a);

// CRT decryption context: Q = prod q_j; per coefficient residues -> floor((t*x + floor(Q/2)) / Q) mod t
struct CrtRound {
    std::vector<uint64_t> q;
    uint64_t t = 0;
    Big Q, Qhalf;
    std::vector<Big> Qj;          // Q / q_j
    std::vector<uint64_t> yj;     // (Q/q_j)^-1 mod q_j
    long double Q_ld = 0;
    void init(const std::vector<uint64_t> &q, uint64_t t);
    uint64_t round_coeff(const uint64_t *res, size_t stride) const;  // res[j*stride]
};

}  // namespace ephdc_host
