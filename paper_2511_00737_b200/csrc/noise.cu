// noise.cu -- GPU noise probe of scores ciphertexts: the measurement behind findDmax
// (Algorithm 1 lines 17-24: "evalHEcomputation(N, T, D) is
// correct"; batch the trials on the GPU).
//
// For each ciphertext (c0, c1) in NTT form mod q_j:
//   x = INTT(c0 + c1 * s_hat) mod Q            (phase, coefficient form, RNS)
//   m = round(t x / Q) mod t                   (the decryption of ephdc_decrypt_*)
//   e = x - Delta m  (mod Q, centered), Delta = floor(Q/t)
//   bits = bit length of max_i |e_i|           (exact)
// When the decryption is correct, e is the ciphertext noise of the oracle's
// noise_bits (x - Delta m_expected); decryption stays correct while |e| < Delta/2.
// Exactness: the centered |e_i| is compared and sized in mixed-radix form (Garner:
// x = v_0 + v_1 q_0 + v_2 q_0 q_1 + ..., digits v_i < q_i exact) -- e or Q - e,
// whichever has the lexicographically smaller digits from the top, is expanded to a
// multi-limb integer by Horner's rule.  Only m uses floating point: t x / Q from the
// digits in doubles (error < 2^-20 for t < 2^31); a coefficient whose t x / Q lies
// within 2^-16 of a rounding boundary (|e| within ~2^-16 Delta of Delta/2: the
// decryption itself is ambiguous there) sets the ciphertext's flag.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "internal.h"
#include "modarith.cuh"

namespace {

constexpr int kMaxL = EPHDC_MAX_PRIMES;
constexpr int kLimbs = (kMaxL * 61 + 63) / 64 + 1;

struct NoiseTab {
    u32 L;
    u64 t;
    u64 q[kMaxL];
    u64 dl[kMaxL], dl_p[kMaxL];            // Delta mod q_j and its Shoup companion
    u64 inv[kMaxL][kMaxL], inv_p[kMaxL][kMaxL];  // q_k^-1 mod q_i (k < i)
    double inv_tail[kMaxL];                // 1 / prod_{k >= i} q_k
};

__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ u64 mul_c(u64 x, u64 w, u64 wp, u64 q) { return csub(mul_shoup_lazy<u64>(x, w, wp, q), q); }

// Garner: residues r (canonical) -> mixed-radix digits v.
__device__ void garner(const NoiseTab &T, const u64 *r, u64 *v) {
    for (u32 i = 0; i < T.L; ++i) {
        u64 a = r[i];
        for (u32 k = 0; k < i; ++k) a = mul_c(sub_mod(a, v[k] % T.q[i], T.q[i]), T.inv[i][k], T.inv_p[i][k], T.q[i]);
        v[i] = a;
    }
}

// -1 if digits a < b, 0 if equal, 1 if a > b (most significant digit first)
__device__ int cmp_digits(const NoiseTab &T, const u64 *a, const u64 *b) {
    for (int i = (int)T.L - 1; i >= 0; --i)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

// bit length of sum_i v_i prod_{k<i} q_k, and (via *lg) its log2 from the top limbs
__device__ u32 bit_length(const NoiseTab &T, const u64 *v, double *lg) {
    u64 limb[kLimbs];
    for (int w = 0; w < kLimbs; ++w) limb[w] = 0;
    for (int i = (int)T.L - 1; i >= 0; --i) {
        // limb = limb * q_i + v_i   (q_{L-1} multiplies nothing: start from the top digit)
        u64 carry = v[i];
        if (i < (int)T.L - 1) {
            for (int w = 0; w < kLimbs; ++w) {
                const u64 lo = limb[w] * T.q[i], hi = __umul64hi(limb[w], T.q[i]);
                const u64 s = lo + carry;
                carry = hi + (s < lo ? 1u : 0u);
                limb[w] = s;
            }
        } else {
            limb[0] = carry;
        }
    }
    for (int w = kLimbs - 1; w >= 0; --w)
        if (limb[w]) {
            const double top = (double)limb[w] + (w > 0 ? (double)limb[w - 1] * 5.421010862427522e-20 : 0.0);
            *lg = log2(top) + 64.0 * w;
            return (u32)(64 * w + 64 - __clzll((long long)limb[w]));
        }
    *lg = 0.0;
    return 0;
}

__global__ void k_phase(const u64 *__restrict__ ct, const TwPair<u64> *__restrict__ sh, const u64 *__restrict__ q,
                        u32 L, u32 N, u64 nct, u64 *__restrict__ x) {
    const u64 n = nct * L * N;
    for (u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (u64)gridDim.x * blockDim.x) {
        const u64 b = idx / ((u64)L * N), r = idx % ((u64)L * N);
        const u32 j = (u32)(r / N);
        const u64 qj = q[j];
        const u64 c0 = ct[(b * 2 + 0) * L * N + r] % qj, c1 = ct[(b * 2 + 1) * L * N + r] % qj;
        const u64 v = mul_c(c1, sh[r].w, sh[r].wp, qj);
        x[idx] = c0 + v >= qj ? c0 + v - qj : c0 + v;
    }
}

__global__ void k_noise(const u64 *__restrict__ x, const NoiseTab *__restrict__ tab, u32 N, u64 nct,
                        u32 *__restrict__ bits, u32 *__restrict__ flags, unsigned long long *__restrict__ lg2) {
    const NoiseTab &T = *tab;
    const u64 n = nct * N;
    for (u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (u64)gridDim.x * blockDim.x) {
        const u64 b = idx / N, i = idx % N;
        u64 r[kMaxL], v[kMaxL], e[kMaxL], ve[kMaxL];
        for (u32 j = 0; j < T.L; ++j) r[j] = x[(b * T.L + j) * N + i];
        garner(T, r, v);
        double f = 0.0;                                  // x / Q in [0, 1)
        for (u32 k = 0; k < T.L; ++k) f += (double)v[k] * T.inv_tail[k];
        const double tf = (double)T.t * f;
        const double mf = rint(tf);
        if (fabs(fabs(tf - mf) - 0.5) < 1.0 / 65536.0) atomicOr(&flags[b], 1u);
        u64 m = (u64)mf;
        if (m >= T.t) m -= T.t;
        for (u32 j = 0; j < T.L; ++j) e[j] = sub_mod(r[j], mul_c(m % T.q[j], T.dl[j], T.dl_p[j], T.q[j]), T.q[j]);
        garner(T, e, ve);
        for (u32 j = 0; j < T.L; ++j) e[j] = e[j] ? T.q[j] - e[j] : 0;   // -e
        garner(T, e, v);
        double lg;
        const u32 bl = bit_length(T, cmp_digits(T, v, ve) < 0 ? v : ve, &lg);
        atomicMax(&bits[b], bl);
        // max of non-negative doubles = max of their bit patterns
        atomicMax(&lg2[b], (unsigned long long)__double_as_longlong(lg));
    }
}

u64 mod_inv(u64 a, u64 q) {  // q prime
    unsigned __int128 r = 1, base = a % q;
    u64 e = q - 2;
    while (e) {
        if (e & 1) r = r * base % q;
        base = base * base % q;
        e >>= 1;
    }
    return (u64)r;
}

u64 shoup(u64 w, u64 q) { return (u64)(((unsigned __int128)w << 64) / q); }

cudaError_t counted(cudaError_t e) {
    if (e == cudaSuccess) ephdc::g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

}  // namespace

extern "C" ephdc_status ephdc_noise_probe(const ephdc_ctx *c, const ephdc_sk *sk, const uint64_t *d_ct,
                                          uint32_t nct, uint32_t *h_bits, uint32_t *h_flags, double *h_log2,
                                          void *stream) {
    if (!c || !sk || ((!d_ct || !h_bits) && nct)) return EPHDC_ENULL;
    if (sk->ctx != c) return EPHDC_ECONTEXT;
    if (c->device < 0) return EPHDC_ECONTEXT;
    if (nct == 0) return EPHDC_OK;
    const u32 L = c->L, N = c->N;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaSetDevice(c->device) != cudaSuccess) return EPHDC_ECUDA;

    NoiseTab T{};
    T.L = L;
    T.t = c->t;
    for (u32 j = 0; j < L; ++j) {
        T.q[j] = c->q[j];
        T.dl[j] = c->delta[j] % c->q[j];
        T.dl_p[j] = shoup(T.dl[j], c->q[j]);
    }
    for (u32 i = 0; i < L; ++i)
        for (u32 k = 0; k < i; ++k) {
            T.inv[i][k] = mod_inv(c->q[k] % c->q[i], c->q[i]);
            T.inv_p[i][k] = shoup(T.inv[i][k], c->q[i]);
        }
    for (u32 i = 0; i < L; ++i) {
        double p = 1.0;
        for (u32 k = i; k < L; ++k) p *= (double)c->q[k];
        T.inv_tail[i] = 1.0 / p;
    }
    std::vector<TwPair<u64>> sh((size_t)L * N);
    for (u32 j = 0; j < L; ++j)
        for (u32 i = 0; i < N; ++i) {
            const u64 w = sk->s_hat[(size_t)j * N + i] % c->q[j];
            sh[(size_t)j * N + i] = TwPair<u64>{w, shoup(w, c->q[j])};
        }

    ephdc_ntt_plan *plan = nullptr;
    ephdc_status s = ephdc_ntt_plan_create(c->q.data(), L, c->p.log2N, c->device, 0u, &plan);
    if (s != EPHDC_OK) return s;
    std::unique_ptr<ephdc_ntt_plan, void (*)(ephdc_ntt_plan *)> plan_guard(plan, ephdc_ntt_plan_free);

    void *mem = nullptr;
    const size_t x_bytes = sizeof(u64) * (size_t)nct * L * N, sh_bytes = sizeof(TwPair<u64>) * sh.size();
    const size_t q_bytes = sizeof(u64) * L, out_bytes = sizeof(u64) * 2 * (size_t)nct;
    const size_t total = x_bytes + sh_bytes + sizeof(NoiseTab) + q_bytes + out_bytes + 64;
    if (cudaMalloc(&mem, total) != cudaSuccess) return EPHDC_ERESOURCE;
    std::unique_ptr<void, cudaError_t (*)(void *)> mem_guard(mem, cudaFree);
    char *base = static_cast<char *>(mem);
    u64 *d_x = reinterpret_cast<u64 *>(base);
    TwPair<u64> *d_sh = reinterpret_cast<TwPair<u64> *>(base + x_bytes);
    NoiseTab *d_tab = reinterpret_cast<NoiseTab *>(base + x_bytes + sh_bytes);
    u64 *d_q = reinterpret_cast<u64 *>(base + x_bytes + sh_bytes + sizeof(NoiseTab));
    // outputs: [nct] u64 log2 bit patterns, then [nct] u32 bits, [nct] u32 flags
    unsigned long long *d_lg = reinterpret_cast<unsigned long long *>(base + x_bytes + sh_bytes + sizeof(NoiseTab) +
                                                                      q_bytes);
    u32 *d_out = reinterpret_cast<u32 *>(d_lg + nct);
    if (cudaMemcpyAsync(d_sh, sh.data(), sh_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(d_tab, &T, sizeof(T), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(d_q, c->q.data(), q_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemsetAsync(d_lg, 0, out_bytes, st) != cudaSuccess)
        return EPHDC_ECUDA;
    const u64 n1 = (u64)nct * L * N;
    k_phase<<<(unsigned)std::min<u64>((n1 + 255) / 256, 148ull * 16), 256, 0, st>>>(d_ct, d_sh, d_q, L, N, nct, d_x);
    if (counted(cudaGetLastError()) != cudaSuccess) return EPHDC_ECUDA;
    s = ephdc_ntt_inv(plan, d_x, nct, st);
    if (s != EPHDC_OK) return s;
    const u64 n2 = (u64)nct * N;
    k_noise<<<(unsigned)std::min<u64>((n2 + 127) / 128, 148ull * 8), 128, 0, st>>>(d_x, d_tab, N, nct, d_out,
                                                                                 d_out + nct, d_lg);
    if (counted(cudaGetLastError()) != cudaSuccess) return EPHDC_ECUDA;
    std::vector<unsigned long long> hl(nct);
    std::vector<u32> h(2 * (size_t)nct);
    if (cudaMemcpyAsync(hl.data(), d_lg, sizeof(u64) * nct, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(h.data(), d_out, sizeof(u32) * 2 * nct, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return EPHDC_ECUDA;
    std::copy(h.begin(), h.begin() + nct, h_bits);
    if (h_flags) std::copy(h.begin() + nct, h.end(), h_flags);
    if (h_log2)
        for (uint32_t b = 0; b < nct; ++b) {
            double v;
            std::memcpy(&v, &hl[b], sizeof v);
            h_log2[b] = v;
        }
    return EPHDC_OK;
}
