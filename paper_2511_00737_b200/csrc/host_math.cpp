// host_math.cpp -- host number theory of libephdc (product side).
#include "host_math.h"

#include <math.h>
#include <string.h>

namespace ephdc_host {

uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    a %= m;
    for (; e; e >>= 1) {
        if (e & 1) r = mulmod(r, a, m);
        a = mulmod(a, a, m);
    }
    return r;
}

uint64_t invmod(uint64_t a, uint64_t p) { return powmod(a, p - 2, p); }

// Deterministic Miller-Rabin for all 64-bit n (Sinclair's 7-base set).
bool is_prime_u64(uint64_t n) {
    if (n < 2) return false;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t p : small) {
        if (n == p) return true;
        if (n % p == 0) return false;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    static const uint64_t bases[] = {2, 325, 9375, 28178, 450775, 9780504, 1795265022};
    for (uint64_t a : bases) {
        uint64_t x = a % n;
        if (x == 0) continue;
        x = powmod(x, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; ++r) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

uint32_t bit_reverse(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int b = 0; b < bits; ++b, x >>= 1) r = (r << 1) | (x & 1u);
    return r;
}

bool ntt_prime_chain(uint32_t log2N, const uint32_t *bits, uint32_t count, const uint64_t *exclude,
                     uint32_t n_exclude, uint64_t *out) {
    const uint64_t m = 2ull << log2N;
    std::vector<uint64_t> used(exclude, exclude + n_exclude);
    for (uint32_t i = 0; i < count; ++i) {
        if (bits[i] > 62 || bits[i] < 2) return false;
        const uint64_t bound = 1ull << bits[i];
        if (bound <= m) return false;
        uint64_t c = (bound - 1) / m * m + 1;   // largest x = 1 mod m with x <= bound - 1 ...
        if (c >= bound) c -= m;                  // ... strictly below the bound
        bool found = false;
        for (; c > m; c -= m) {
            bool dup = false;
            for (uint64_t u : used) dup |= (u == c);
            if (!dup && is_prime_u64(c)) { found = true; break; }
        }
        if (!found) return false;
        out[i] = c;
        used.push_back(c);
    }
    return true;
}

// Generator of (Z/p)^*: factor p-1 by trial division, test g^((p-1)/f) != 1.
static uint64_t generator(uint64_t p) {
    std::vector<uint64_t> f;
    uint64_t n = p - 1;
    for (uint64_t d = 2; d * d <= n; d += (d == 2 ? 1 : 2)) {
        if (n % d == 0) {
            f.push_back(d);
            while (n % d == 0) n /= d;
        }
    }
    if (n > 1) f.push_back(n);
    for (uint64_t g = 2; g < p; ++g) {
        bool ok = true;
        for (uint64_t fi : f)
            if (powmod(g, (p - 1) / fi, p) == 1) { ok = false; break; }
        if (ok) return g;
    }
    return 0;
}

uint64_t min_primitive_root_2n(uint64_t p, uint32_t log2N) {
    const uint64_t two_n = 2ull << log2N;
    if ((p - 1) % two_n != 0) return 0;
    uint64_t g = generator(p);
    if (!g) return 0;
    const uint64_t psi0 = powmod(g, (p - 1) / two_n, p);   // order exactly 2N
    const uint64_t sq = mulmod(psi0, psi0, p);
    uint64_t best = psi0, x = psi0;
    for (uint64_t k = 1; k < (two_n >> 1); ++k) {            // odd powers 3, 5, ..., 2N-1
        x = mulmod(x, sq, p);
        if (x < best) best = x;
    }
    return best;
}

uint64_t inv_mod_2_64(uint64_t p) {
    uint64_t x = p;                 // Newton: x <- x (2 - p x), 5 doublings from 3 bits
    for (int i = 0; i < 6; ++i) x *= 2 - p * x;
    return x;
}

uint64_t two128_mod(uint64_t p) {
    uint64_t r = (uint64_t)(((u128)1 << 64) % p);
    return mulmod(r, r, p);
}

void pow_brev(uint64_t x, uint64_t p, uint32_t log2N, uint64_t *out) {
    const uint32_t N = 1u << log2N;
    std::vector<uint64_t> pw(N);
    pw[0] = 1;
    for (uint32_t i = 1; i < N; ++i) pw[i] = mulmod(pw[i - 1], x, p);
    for (uint32_t k = 0; k < N; ++k) out[k] = pw[bit_reverse(k, log2N)];
}

void gaussian_cdt(double sigma, uint64_t out[20]) {
    long double rho[20], Z = 0;
    for (int k = 0; k < 20; ++k) {
        rho[k] = expl(-(long double)k * k / (2.0L * sigma * sigma));
        Z += (k == 0 ? 1.0L : 2.0L) * rho[k];
    }
    long double acc = 0;
    for (int k = 0; k < 20; ++k) {
        acc += (k == 0 ? 1.0L : 2.0L) * rho[k];
        const long double v = acc / Z * 1099511627776.0L;   // 2^40
        out[k] = (uint64_t)llroundl(v) << 23;
    }
    out[19] = 1ull << 63;
}

void HostNtt::init(uint64_t p_, uint64_t psi, uint32_t lg) {
    p = p_;
    log2N = lg;
    const uint32_t N = 1u << lg;
    fw.resize(N);
    inv.resize(N);
    pow_brev(psi, p, lg, fw.data());
    pow_brev(invmod(psi, p), p, lg, inv.data());
    ninv = invmod(N % p, p);
}

void HostNtt::forward(uint64_t *a) const {
    const uint32_t N = 1u << log2N;
    for (uint32_t m = 1, t = N >> 1; m < N; m <<= 1, t >>= 1)
        for (uint32_t i = 0; i < m; ++i) {
            const uint64_t w = fw[m + i];
            uint64_t *x = a + 2 * i * t;
            for (uint32_t j = 0; j < t; ++j) {
                const uint64_t u = x[j], v = mulmod(x[j + t], w, p);
                x[j] = u + v >= p ? u + v - p : u + v;
                x[j + t] = u >= v ? u - v : u + p - v;
            }
        }
}

void HostNtt::inverse(uint64_t *a) const {
    const uint32_t N = 1u << log2N;
    for (uint32_t t = 1, h = N >> 1; t < N; t <<= 1, h >>= 1)
        for (uint32_t i = 0; i < h; ++i) {
            const uint64_t w = inv[h + i];
            uint64_t *x = a + 2 * i * t;
            for (uint32_t j = 0; j < t; ++j) {
                const uint64_t u = x[j], v = x[j + t];
                x[j] = u + v >= p ? u + v - p : u + v;
                x[j + t] = mulmod(u >= v ? u - v : u + p - v, w, p);
            }
        }
    for (uint32_t j = 0; j < N; ++j) a[j] = mulmod(a[j], ninv, p);
}

// ---------------- multi-precision ----------------
static void trim(Big &a) {
    while (a.size() > 1 && a.back() == 0) a.pop_back();
}

Big big_from_product(const std::vector<uint64_t> &ps) {
    Big r{1};
    for (uint64_t p : ps) r = big_mul_small(r, p);
    return r;
}

Big big_mul_small(const Big &a, uint64_t m) {
    Big r(a.size() + 1, 0);
    u128 carry = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        u128 v = (u128)a[i] * m + carry;
        r[i] = (uint64_t)v;
        carry = v >> 64;
    }
    r[a.size()] = (uint64_t)carry;
    trim(r);
    return r;
}

Big big_div_small(const Big &a, uint64_t d, uint64_t *rem) {
    Big r(a.size(), 0);
    u128 cur = 0;
    for (size_t i = a.size(); i-- > 0;) {
        cur = (cur << 64) | a[i];
        r[i] = (uint64_t)(cur / d);
        cur %= d;
    }
    if (rem) *rem = (uint64_t)cur;
    trim(r);
    return r;
}

uint64_t big_mod_small(const Big &a, uint64_t m) {
    u128 r = 0;
    for (size_t i = a.size(); i-- > 0;) r = ((r << 64) | a[i]) % m;
    return (uint64_t)r;
}

int big_cmp(const Big &a, const Big &b) {
    size_t n = a.size() > b.size() ? a.size() : b.size();
    for (size_t i = n; i-- > 0;) {
        uint64_t x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

void big_add_inplace(Big &a, const Big &b) {
    if (a.size() < b.size()) a.resize(b.size(), 0);
    u128 carry = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        u128 v = (u128)a[i] + (i < b.size() ? b[i] : 0) + carry;
        a[i] = (uint64_t)v;
        carry = v >> 64;
    }
    if (carry) a.push_back((uint64_t)carry);
}

void big_sub_inplace(Big &a, const Big &b) {
    uint64_t borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        uint64_t y = i < b.size() ? b[i] : 0;
        u128 sub = (u128)y + borrow;
        borrow = (u128)a[i] < sub;
        a[i] = (uint64_t)((u128)a[i] - sub);
    }
    trim(a);
}

long double big_to_ld(const Big &a) {
    long double r = 0;
    for (size_t i = a.size(); i-- > 0;) r = r * 18446744073709551616.0L + (long double)a[i];
    return r;
}

void CrtRound::init(const std::vector<uint64_t> &q_, uint64_t t_) {
    q = q_;
    t = t_;
    Q = big_from_product(q);
    Qhalf = big_div_small(Q, 2, nullptr);
    Qj.clear();
    yj.clear();
    for (uint64_t p : q) {
        uint64_t rem;
        Big qj = big_div_small(Q, p, &rem);
        Qj.push_back(qj);
        yj.push_back(invmod(big_mod_small(qj, p), p));
    }
    Q_ld = big_to_ld(Q);
}

// x = sum_j [res_j * y_j]_{q_j} * Q_j  (< L*Q), reduced mod Q, then the BFV rounding.
uint64_t CrtRound::round_coeff(const uint64_t *res, size_t stride) const {
    Big x{0};
    for (size_t j = 0; j < q.size(); ++j) {
        const uint64_t v = mulmod(res[j * stride], yj[j], q[j]);
        big_add_inplace(x, big_mul_small(Qj[j], v));
    }
    while (big_cmp(x, Q) >= 0) big_sub_inplace(x, Q);
    Big num = big_mul_small(x, t);
    big_add_inplace(num, Qhalf);
    // quotient estimate, then exact correction
    long double est = floorl(big_to_ld(num) / Q_ld);
    uint64_t qt = est < 0 ? 0 : (uint64_t)est;
    for (int it = 0; it < 4; ++it) {
        Big prod = big_mul_small(Q, qt);
        if (big_cmp(prod, num) > 0) { --qt; continue; }
        Big next = prod;
        big_add_inplace(next, Q);
        if (big_cmp(next, num) <= 0) { ++qt; continue; }
        break;
    }
    return qt % t;
}

}  // namespace ephdc_host
