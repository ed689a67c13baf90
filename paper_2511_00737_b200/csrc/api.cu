// api.cu -- implementation of the C ABI declared in include/ephdc.h.
#include <cuda_runtime.h>
#include <string.h>
#include <sys/random.h>
#include <cstdlib>

#include <algorithm>
#include <memory>
#include <new>
#include <thread>
#include <vector>

#include "internal.h"
#include "rng.cuh"

using namespace ephdc;
using namespace ephdc_host;

namespace {

#define EPHDC_CUDA_TRY(expr)                     \
    do {                                         \
        cudaError_t _e = (expr);                 \
        if (_e != cudaSuccess) return EPHDC_ECUDA; \
    } while (0)

const char *kClassNames[ephdc_workspace::kClasses] = {"encode", "pack_intt", "ntt_mac", "finalize"};
enum { kClsEncode = 0, kClsPack = 1, kClsMac = 2, kClsFinal = 3 };

template <class T> cudaError_t dev_alloc(T **p, size_t n) {
    return cudaMalloc(reinterpret_cast<void **>(p), sizeof(T) * (n ? n : 1));
}

// RAII device buffer for temporaries
struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
};

// Timed launch helper for the workspace instrumentation.
struct Timer {
    ephdc_workspace *ws;
    cudaStream_t st;
    int cls;
    int idx = -1;
    Timer(ephdc_workspace *w, cudaStream_t s, int c) : ws(w), st(s), cls(c) {
        if (ws && ws->timing) {
            size_t need = ws->ev_marks.size() * 2 + 2;
            while (ws->ev_pool.size() < need) {
                cudaEvent_t e;
                if (cudaEventCreate(&e) != cudaSuccess) return;
                ws->ev_pool.push_back(e);
            }
            idx = (int)ws->ev_marks.size() * 2;
            cudaEventRecord(ws->ev_pool[idx], st);
        }
    }
    void done() {
        if (idx >= 0) {
            cudaEventRecord(ws->ev_pool[idx + 1], st);
            ws->ev_marks.push_back({cls, idx});
            ws->launches[cls] += 1;
            idx = -1;
        }
    }
};

bool is_ntt_prime(uint64_t p, uint32_t log2N) { return p > 2 && (p - 1) % (2ull << log2N) == 0 && is_prime_u64(p); }

uint64_t mask_for(uint64_t q) {
    uint64_t m = 1;
    while (m < q) m = (m << 1) | 1;
    return m;
}

void fill_prime_set(PrimeSet &ps, const std::vector<uint64_t> &q, uint64_t t) {
    memset(&ps, 0, sizeof(ps));
    for (size_t j = 0; j < q.size(); ++j) {
        ps.q[j] = q[j];
        ps.qinv[j] = inv_mod_2_64(q[j]);
        ps.r2[j] = two128_mod(q[j]);
        ps.qmt[j] = t ? q[j] - t : 0;
        ps.mask[j] = mask_for(q[j]);
    }
}

std::vector<TwPair<u64>> make_tw64(uint64_t psi, uint64_t p, uint32_t log2N) {
    const uint32_t N = 1u << log2N;
    std::vector<uint64_t> pw(N);
    pow_brev(psi, p, log2N, pw.data());
    std::vector<TwPair<u64>> out(N);
    for (uint32_t i = 0; i < N; ++i) out[i] = TwPair<u64>{pw[i], shoup64(pw[i], p)};
    return out;
}

}  // namespace

extern "C" {

const char *ephdc_status_string(ephdc_status s) {
    switch (s) {
        case EPHDC_OK: return "ok";
        case EPHDC_EPARAM: return "invalid parameter";
        case EPHDC_ECONTEXT: return "context mismatch or host-only context";
        case EPHDC_EOVERFLOW: return "output capacity too small";
        case EPHDC_ERESOURCE: return "allocation failed";
        case EPHDC_ECUDA: return "CUDA error";
        case EPHDC_EDOMAIN: return "value outside its modular domain";
        case EPHDC_ENULL: return "null pointer";
    }
    return "unknown status";
}

int ephdc_abi_version(void) { return EPHDC_ABI_VERSION; }

// ------------------------------------------------------------------------------------
// random-stream keys (reading #7)
// ------------------------------------------------------------------------------------
ephdc_status ephdc_seed_os(ephdc_seed *out) {
    if (!out) return EPHDC_ENULL;
    unsigned char *p = reinterpret_cast<unsigned char *>(out->key);
    size_t got = 0;
    while (got < sizeof out->key) {
        const ssize_t r = getrandom(p + got, sizeof out->key - got, 0);
        if (r < 0) return EPHDC_ERESOURCE;
        got += (size_t)r;
    }
    return EPHDC_OK;
}

ephdc_status ephdc_seed_u64(uint64_t v, ephdc_seed *out) {
    if (!out) return EPHDC_ENULL;
    memset(out, 0, sizeof *out);
    out->key[0] = (uint32_t)v;
    out->key[1] = (uint32_t)(v >> 32);
    return EPHDC_OK;
}

ephdc_status ephdc_chacha20_block(const ephdc_seed *key, uint32_t counter, const uint32_t nonce[3], uint32_t out[16]) {
    if (!key || !nonce || !out) return EPHDC_ENULL;
    ephdc_rng::Key k;
    memcpy(k.k, key->key, sizeof k.k);
    uint32_t b[16];
    ephdc_rng::chacha20_block(k, counter, nonce[0], nonce[1], nonce[2], b);
    memcpy(out, b, sizeof b);
    return EPHDC_OK;
}

namespace {
// NULL -> a fresh OS key (the default: streams the client cannot reproduce)
ephdc_status resolve_seed(const ephdc_seed *in, ephdc_seed *key) {
    if (in) {
        *key = *in;
        return EPHDC_OK;
    }
    return ephdc_seed_os(key);
}
}  // namespace

ephdc_status ephdc_query_bits(uint32_t D_live, uint32_t Cbits, uint64_t t, uint32_t *Qbits) {
    if (!Qbits) return EPHDC_ENULL;
    if (Cbits < 2 || Cbits > 8 || t < 3) return EPHDC_EPARAM;
    const uint64_t cmax = (1u << (Cbits - 1)) - 1, limit = (t - 1) / 2;
    for (uint32_t Q = 8; Q >= 2; --Q)
        if ((uint64_t)D_live * ((1u << (Q - 1)) - 1) * cmax <= limit) {
            *Qbits = Q;
            return EPHDC_OK;
        }
    return EPHDC_EPARAM;
}

ephdc_status ephdc_train_model(uint32_t D_live, uint32_t n, uint32_t k, uint32_t Cbits, uint32_t Qbits,
                               const int32_t *h_acc, const int64_t *h_labels, int8_t *h_class_hv,
                               uint32_t *qshift) {
    if (!h_class_hv || !qshift || ((!h_acc || !h_labels) && n && D_live)) return EPHDC_ENULL;
    if (k == 0 || Cbits < 2 || Cbits > 8 || Qbits < 2 || Qbits > 8) return EPHDC_EPARAM;
    for (uint32_t i = 0; i < n; ++i)
        if (h_labels[i] < 0 || (uint64_t)h_labels[i] >= k) return EPHDC_EPARAM;
    const int64_t cmax = (1 << (Cbits - 1)) - 1, qmax = (1 << (Qbits - 1)) - 1;
    std::vector<int64_t> v((size_t)k * D_live, 0);
    int64_t peak = 0;
    for (uint32_t d = 0; d < D_live; ++d) {
        const int32_t *row = h_acc + (size_t)d * n;
        for (uint32_t i = 0; i < n; ++i) {
            v[(size_t)h_labels[i] * D_live + d] += row[i];
            peak = std::max<int64_t>(peak, row[i] < 0 ? -(int64_t)row[i] : row[i]);
        }
    }
    for (uint32_t c = 0; c < k; ++c) {
        const int64_t *vc = v.data() + (size_t)c * D_live;
        int64_t M = 0;
        for (uint32_t d = 0; d < D_live; ++d) M = std::max<int64_t>(M, vc[d] < 0 ? -vc[d] : vc[d]);
        for (uint32_t d = 0; d < D_live; ++d) {
            const int64_t a = vc[d] < 0 ? -vc[d] : vc[d];
            const int64_t r = M == 0 ? 0 : (2 * a * cmax + M) / (2 * M);
            h_class_hv[(size_t)c * D_live + d] = (int8_t)(vc[d] < 0 ? -r : r);
        }
    }
    uint32_t s = 0;
    while ((qmax << s) < peak) ++s;
    *qshift = s;
    return EPHDC_OK;
}

uint64_t ephdc_launch_count(void) { return g_launches.load(); }

ephdc_status ephdc_find_ntt_primes(uint32_t log2N, const uint32_t *bits, uint32_t count, const uint64_t *exclude,
                                   uint32_t n_exclude, uint64_t *out) {
    if (!bits || !out || (n_exclude && !exclude)) return EPHDC_ENULL;
    if (log2N < 1 || log2N > 20) return EPHDC_EPARAM;
    return ntt_prime_chain(log2N, bits, count, exclude, n_exclude, out) ? EPHDC_OK : EPHDC_EPARAM;
}

ephdc_status ephdc_min_psi(uint64_t p, uint32_t log2N, uint64_t *psi) {
    if (!psi) return EPHDC_ENULL;
    if (log2N > 20 || !is_ntt_prime(p, log2N)) return EPHDC_EPARAM;
    *psi = min_primitive_root_2n(p, log2N);
    return *psi ? EPHDC_OK : EPHDC_EPARAM;
}

ephdc_status ephdc_gaussian_cdt(double sigma, uint64_t *out20) {
    if (!out20) return EPHDC_ENULL;
    if (!(sigma > 0.0) || sigma > 100.0) return EPHDC_EPARAM;
    gaussian_cdt(sigma, out20);
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// context
// ------------------------------------------------------------------------------------
void ephdc_ctx_free(ephdc_ctx *c) {
    if (!c) return;
    if (c->device >= 0) {
        cudaSetDevice(c->device);
        cudaFree(c->dev.tw_q);
        cudaFree(c->dev.tw_f64);
        cudaFree(c->dev.itw_t);
        cudaFree(c->dev.cdt);
    }
    delete c;
}

ephdc_status ephdc_ctx_create(const ephdc_params *p, int device, ephdc_ctx **out) {
    if (!p || !out || !p->q) return EPHDC_ENULL;
    *out = nullptr;
    if (p->log2N < 10 || p->log2N > 14 || p->L < 1 || p->L > EPHDC_MAX_PRIMES) return EPHDC_EPARAM;
    const uint32_t N = 1u << p->log2N;
    if (p->k < 1 || p->k > N || p->D_live < 1 || p->D_stored < p->D_live || p->F < 4 || p->F % 4) return EPHDC_EPARAM;
    if (p->Qbits < 2 || p->Qbits > 8 || p->Cbits < 2 || p->Cbits > 8 || p->qshift > 30) return EPHDC_EPARAM;
    if (!(p->sigma_e > 0.0) || p->sigma_e > 100.0) return EPHDC_EPARAM;
    if (p->t >= (1ull << 30) || !is_ntt_prime(p->t, p->log2N)) return EPHDC_EPARAM;
    for (uint32_t j = 0; j < p->L; ++j) {
        if (p->q[j] >= (1ull << 60) || p->q[j] <= p->t || !is_ntt_prime(p->q[j], p->log2N)) return EPHDC_EPARAM;
        for (uint32_t i = 0; i < j; ++i)
            if (p->q[i] == p->q[j]) return EPHDC_EPARAM;
    }
    std::unique_ptr<ephdc_ctx> c(new (std::nothrow) ephdc_ctx());
    if (!c) return EPHDC_ERESOURCE;
    c->p = *p;
    c->q.assign(p->q, p->q + p->L);
    c->p.q = c->q.data();
    c->N = N;
    c->L = p->L;
    c->t = p->t;
    c->B = N / p->k;
    c->psi_t = min_primitive_root_2n(p->t, p->log2N);
    if (!c->psi_t) return EPHDC_EPARAM;
    for (uint64_t qj : c->q) {
        uint64_t ps = min_primitive_root_2n(qj, p->log2N);
        if (!ps) return EPHDC_EPARAM;
        c->psi.push_back(ps);
    }
    // Delta = floor(Q / t) (reading #4), reduced per prime
    Big Q = big_from_product(c->q);
    Big delta = big_div_small(Q, p->t, nullptr);
    fill_prime_set(c->ps, c->q, p->t);
    for (uint32_t j = 0; j < c->L; ++j) {
        c->delta.push_back(big_mod_small(delta, c->q[j]));
        c->ps.delta[j] = c->delta[j];
        c->ps.delta_p[j] = shoup64(c->delta[j], c->q[j]);
    }
    const uint32_t ninv = (uint32_t)invmod(N % p->t, p->t);
    c->ninv_t = ninv;
    c->ninv_t_p = shoup32(ninv, (uint32_t)p->t);
    gaussian_cdt(p->sigma_e, c->cdt);
    c->host_q.resize(c->L);
    for (uint32_t j = 0; j < c->L; ++j) c->host_q[j].init(c->q[j], c->psi[j], p->log2N);
    c->host_t.init(p->t, c->psi_t, p->log2N);
    c->crt.init(c->q, p->t);
    for (uint64_t qj : c->q) {
        uint32_t b = 0;
        while (b < 64 && (qj >> b)) ++b;
        c->qbits.push_back(b);
    }
    // fused MAC kernel geometry: S CTAs per polynomial (N = 16384 -> 2 halves of 8192),
    // dims split in chunks so the grid holds ~8 waves; all partial sums < 2^64.
    c->fused_S = p->log2N >= 14 ? (1u << (p->log2N - 13)) : 1u;
    {
        const uint32_t occ = (uint32_t)ntt_mac_occupancy(p->log2N, c->fused_S);
        const uint64_t target = 8ull * 148 * occ;
        uint64_t chunks = (target + c->L * c->fused_S - 1) / (c->L * c->fused_S);
        chunks = std::max<uint64_t>(1, std::min<uint64_t>(chunks, p->D_live));
        uint64_t qmax = *std::max_element(c->q.begin(), c->q.end());
        chunks = std::min<uint64_t>(chunks, ~0ull / qmax);
        c->fused_G = (uint32_t)((p->D_live + chunks - 1) / chunks);
        c->fused_chunks = (p->D_live + c->fused_G - 1) / c->fused_G;
    }
    if (p->arith > EPHDC_ARITH_F64 || p->encoder > EPHDC_ENCODER_DP4A) return EPHDC_EPARAM;
    if (p->arith != EPHDC_ARITH_INT) {
        const bool ok = plan_f64(c->q, p->t, p->log2N, &c->f64);
        if (!ok && p->arith == EPHDC_ARITH_F64) return EPHDC_EPARAM;
    }
    c->device = device;
    if (device >= 0) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) return EPHDC_ECUDA;
        EPHDC_CUDA_TRY(cudaSetDevice(device));
        std::vector<TwPair<u64>> twq((size_t)c->L * N);
        for (uint32_t j = 0; j < c->L; ++j) {
            auto tj = make_tw64(c->psi[j], c->q[j], p->log2N);
            std::copy(tj.begin(), tj.end(), twq.begin() + (size_t)j * N);
        }
        if (c->f64.enabled) {
            // (psi_rev[i], fl(psi_rev[i] / q_j)): exact integers < 2^50 and correctly rounded quotients
            std::vector<double> twd((size_t)c->L * N * 2);
            for (size_t i = 0; i < (size_t)c->L * N; ++i) {
                const double qd = (double)c->q[i / N];
                twd[2 * i] = (double)twq[i].w;
                twd[2 * i + 1] = (double)twq[i].w / qd;
                if (i % N == 0) {  // index 0 is never a twiddle: it carries (q_j, fl(1/q_j))
                    twd[2 * i] = qd;
                    twd[2 * i + 1] = 1.0 / qd;
                }
            }
            if (cudaMalloc(&c->dev.tw_f64, sizeof(double) * twd.size()) != cudaSuccess) {
                ephdc_ctx_free(c.release());
                return EPHDC_ERESOURCE;
            }
            if (cudaMemcpy(c->dev.tw_f64, twd.data(), sizeof(double) * twd.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
                ephdc_ctx_free(c.release());
                return EPHDC_ECUDA;
            }
        }
        std::vector<uint64_t> ipw(N);
        pow_brev(invmod(c->psi_t, p->t), p->t, p->log2N, ipw.data());
        std::vector<TwPair<u32>> itw(N);
        for (uint32_t i = 0; i < N; ++i) itw[i] = TwPair<u32>{(u32)ipw[i], shoup32((u32)ipw[i], (u32)p->t)};
        if (dev_alloc(&c->dev.tw_q, twq.size()) != cudaSuccess || dev_alloc(&c->dev.itw_t, itw.size()) != cudaSuccess ||
            dev_alloc(&c->dev.cdt, 20) != cudaSuccess) {
            ephdc_ctx_free(c.release());
            return EPHDC_ERESOURCE;
        }
        if (cudaMemcpy(c->dev.tw_q, twq.data(), sizeof(twq[0]) * twq.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c->dev.itw_t, itw.data(), sizeof(itw[0]) * itw.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c->dev.cdt, c->cdt, sizeof(c->cdt), cudaMemcpyHostToDevice) != cudaSuccess) {
            ephdc_ctx_free(c.release());
            return EPHDC_ECUDA;
        }
    }
    *out = c.release();
    return EPHDC_OK;
}

ephdc_status ephdc_ctx_query(const ephdc_ctx *c, ephdc_ctx_info *info) {
    if (!c || !info) return EPHDC_ENULL;
    memset(info, 0, sizeof(*info));
    info->N = c->N;
    info->L = c->L;
    info->B = c->B;
    info->k = c->p.k;
    info->t = c->t;
    info->psi_t = c->psi_t;
    for (uint32_t j = 0; j < c->L; ++j) {
        info->q[j] = c->q[j];
        info->psi[j] = c->psi[j];
        info->delta[j] = c->delta[j];
    }
    info->fused_split = c->fused_S;
    info->fused_chunks = c->fused_chunks;
    info->device = c->device;
    info->arith = c->f64.enabled ? EPHDC_ARITH_F64 : EPHDC_ARITH_INT;
    info->f64_red_every = c->f64.enabled ? c->f64.red_every : 0u;
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// keys and model
// ------------------------------------------------------------------------------------
ephdc_status ephdc_keygen(const ephdc_ctx *c, const ephdc_seed *seed, ephdc_sk **out) {
    if (!c || !out) return EPHDC_ENULL;
    ephdc_seed key;
    if (ephdc_status e = resolve_seed(seed, &key)) return e;
    ephdc_rng::Key rk;
    memcpy(rk.k, key.key, sizeof rk.k);
    std::unique_ptr<ephdc_sk> sk(new (std::nothrow) ephdc_sk());
    if (!sk) return EPHDC_ERESOURCE;
    sk->ctx = c;
    const uint32_t N = c->N;
    sk->s.resize(N);
    for (uint32_t i = 0; i < N; ++i) sk->s[i] = (int8_t)ephdc_rng::ternary(rk, i);
    sk->s_hat.resize((size_t)c->L * N);
    for (uint32_t j = 0; j < c->L; ++j) {
        uint64_t *sh = sk->s_hat.data() + (size_t)j * N;
        for (uint32_t i = 0; i < N; ++i) sh[i] = sk->s[i] < 0 ? c->q[j] - 1 : (uint64_t)sk->s[i];
        c->host_q[j].forward(sh);
    }
    *out = sk.release();
    return EPHDC_OK;
}

void ephdc_sk_free(ephdc_sk *sk) {
    if (!sk) return;
    if (sk->d_shat_mont) {
        cudaSetDevice(sk->ctx->device);
        cudaFree(sk->d_shat_mont);
    }
    delete sk;
}

// s_hat * 2^64 mod q_j on the host ([L][N]): mont_mul(a, this) = a * s_hat
static std::vector<uint64_t> shat_mont_host(const ephdc_ctx *c, const ephdc_sk *sk) {
    const uint32_t N = c->N, L = c->L;
    std::vector<uint64_t> shm((size_t)L * N);
    for (uint32_t j = 0; j < L; ++j) {
        const uint64_t r = (uint64_t)(((u128)1 << 64) % c->q[j]);
        for (uint32_t i = 0; i < N; ++i) shm[(size_t)j * N + i] = mulmod(sk->s_hat[(size_t)j * N + i], r, c->q[j]);
    }
    return shm;
}

ephdc_status ephdc_sk_export(const ephdc_sk *sk, int8_t *s_out, uint64_t *s_hat_out) {
    if (!sk || !s_out) return EPHDC_ENULL;
    memcpy(s_out, sk->s.data(), sk->s.size());
    if (s_hat_out) memcpy(s_hat_out, sk->s_hat.data(), sizeof(uint64_t) * sk->s_hat.size());
    return EPHDC_OK;
}

void ephdc_model_free(ephdc_model *m) { delete m; }   // ~ephdc_model frees d_ct

ephdc_status ephdc_encrypt_model(const ephdc_ctx *c, const ephdc_sk *sk, const int8_t *class_hv,
                                 const ephdc_seed *seed, ephdc_model **out) {
    if (!c || !sk || !class_hv || !out) return EPHDC_ENULL;
    *out = nullptr;
    ephdc_seed key;
    if (ephdc_status e = resolve_seed(seed, &key)) return e;
    if (sk->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    const uint32_t N = c->N, L = c->L, D = c->p.D_live, k = c->p.k;
    for (size_t i = 0; i < (size_t)k * D; ++i)
        if (2 * (int64_t)(class_hv[i] < 0 ? -class_hv[i] : class_hv[i]) >= (int64_t)c->t) return EPHDC_EDOMAIN;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    std::unique_ptr<ephdc_model> m(new (std::nothrow) ephdc_model());
    if (!m) return EPHDC_ERESOURCE;
    m->ctx = c;
    m->D = D;
    if (dev_alloc(&m->d_ct, (size_t)D * L * 2 * N) != cudaSuccess) return EPHDC_ERESOURCE;
    // s_hat in Montgomery form (s_hat * 2^64 mod q): mont_mul(a, s_hat*2^64) = a * s_hat
    const std::vector<uint64_t> shm = shat_mont_host(c, sk);
    const uint32_t chunk = std::min<uint32_t>(D, 2048);
    DevBuf bC, bS, bM;
    if (cudaMalloc(&bC.p, (size_t)k * D) != cudaSuccess || cudaMalloc(&bS.p, sizeof(uint64_t) * shm.size()) != cudaSuccess ||
        cudaMalloc(&bM.p, sizeof(uint32_t) * (size_t)chunk * N) != cudaSuccess)
        return EPHDC_ERESOURCE;
    EPHDC_CUDA_TRY(cudaMemcpy(bC.p, class_hv, (size_t)k * D, cudaMemcpyHostToDevice));
    EPHDC_CUDA_TRY(cudaMemcpy(bS.p, shm.data(), sizeof(uint64_t) * shm.size(), cudaMemcpyHostToDevice));
    cudaStream_t st = 0;
    for (uint32_t d0 = 0; d0 < D; d0 += chunk) {
        const uint32_t nd = std::min(chunk, D - d0);
        EPHDC_CUDA_TRY(launch_pack_intt_model(c, (const int8_t *)bC.p, d0, nd, (uint32_t *)bM.p, st));
        EPHDC_CUDA_TRY(launch_encrypt(c, (const uint32_t *)bM.p, d0, nd, (const uint64_t *)bS.p, key,
                                      m->d_ct + (size_t)d0 * L * 2 * N, st));
    }
    // FP64 path: keep the residues as exact doubles (the fused kernel's operand format)
    if (c->f64.enabled) EPHDC_CUDA_TRY(launch_u64_to_f64(m->d_ct, (size_t)D * L * 2 * N, st));
    EPHDC_CUDA_TRY(cudaDeviceSynchronize());
    *out = m.release();
    return EPHDC_OK;
}

ephdc_status ephdc_model_export(const ephdc_model *m, uint32_t d0, uint32_t nd, uint64_t *host_out) {
    if (!m || !host_out) return EPHDC_ENULL;
    if ((uint64_t)d0 + nd > m->D) return EPHDC_EPARAM;
    const ephdc_ctx *c = m->ctx;
    const size_t per = (size_t)c->L * 2 * c->N;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    EPHDC_CUDA_TRY(cudaMemcpy(host_out, m->d_ct + per * d0, sizeof(uint64_t) * per * nd, cudaMemcpyDeviceToHost));
    if (c->f64.enabled) {  // stored as exact doubles < 2^50: back to canonical u64
        for (size_t i = 0; i < per * nd; ++i) {
            double v;
            memcpy(&v, &host_out[i], sizeof v);
            host_out[i] = (uint64_t)v;
        }
    }
    return EPHDC_OK;
}

ephdc_status ephdc_model_scale(const ephdc_ctx *c, ephdc_model *m, uint32_t g, const uint64_t *h_scales,
                               uint32_t n_scales) {
    if (!c || !m || (!h_scales && n_scales)) return EPHDC_ENULL;
    if (m->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    const uint32_t D = m->D, L = c->L;
    if (g == 0 || n_scales != (D + g - 1) / g) return EPHDC_EPARAM;
    for (uint32_t J = 0; J < n_scales; ++J)
        if (h_scales[J] % c->t == 0) return EPHDC_EPARAM;
    // cumulative factor of group J per prime: prod_{J' >= J} lift(s_J'^-1 mod t) mod q_j
    std::vector<uint64_t> fac((size_t)n_scales * L);
    std::vector<uint64_t> run(L, 1);
    for (uint32_t J = n_scales; J-- > 0;) {
        const uint64_t inv = invmod(h_scales[J] % c->t, c->t);
        const bool neg = inv > (c->t - 1) / 2;
        for (uint32_t j = 0; j < L; ++j) {
            const uint64_t q = c->q[j];
            const uint64_t lift = neg ? q - (c->t - inv) : inv;   // centered lift into [0, q)
            run[j] = mulmod(run[j], lift, q);
            // integer path: Montgomery form (x 2^64) for mont_mul; FP64 path: plain factor
            fac[(size_t)J * L + j] = c->f64.enabled ? run[j] : (uint64_t)(((u128)run[j] << 64) % q);
        }
    }
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    DevBuf bf;
    if (cudaMalloc(&bf.p, sizeof(uint64_t) * fac.size()) != cudaSuccess) return EPHDC_ERESOURCE;
    EPHDC_CUDA_TRY(cudaMemcpy(bf.p, fac.data(), sizeof(uint64_t) * fac.size(), cudaMemcpyHostToDevice));
    EPHDC_CUDA_TRY(launch_model_scale(c, m->d_ct, D, g, (const uint64_t *)bf.p, 0));
    EPHDC_CUDA_TRY(cudaDeviceSynchronize());
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// workspace
// ------------------------------------------------------------------------------------
void ephdc_workspace_free(ephdc_workspace *ws) {
    if (!ws) return;
    cudaSetDevice(ws->ctx->device);
    cudaFree(ws->d_M);
    cudaFree(ws->d_X);
    cudaFree(ws->d_H);
    cudaFree(ws->d_out);
    cudaFree(ws->d_msg);
    cudaFree(ws->d_dlim);
    for (cudaEvent_t e : ws->ev_pool) cudaEventDestroy(e);
    delete ws;
}

ephdc_status ephdc_workspace_create(const ephdc_ctx *c, uint32_t max_nq, const ephdc_plan *plan,
                                    ephdc_workspace **out) {
    if (!c || !out) return EPHDC_ENULL;
    *out = nullptr;
    if (c->device < 0) return EPHDC_ECONTEXT;
    if (max_nq == 0) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    std::unique_ptr<ephdc_workspace> ws(new (std::nothrow) ephdc_workspace());
    if (!ws) return EPHDC_ERESOURCE;
    ws->ctx = c;
    ws->max_nq = max_nq;
    if (plan) ws->plan = *plan;
    ws->nb_max = (max_nq + c->B - 1) / c->B;
    const size_t D = c->p.D_live;
    // FP64 path: the encoded plaintexts of all batches are kept (one fused launch over
    // every batch), up to a 32 GB cap; the integer path keeps one batch.
    ws->m_batches = 1;
    if (c->f64.enabled) {
        const size_t per = D * c->N * sizeof(uint32_t);
        const size_t cap = std::max<size_t>(1, (32ull << 30) / per);
        ws->m_batches = (uint32_t)std::min<size_t>(std::min<size_t>(ws->nb_max, cap), 65535);
        // plan override (tests): smaller batch groups exercise the grouped path (taken above 32 GB)
        if (ws->plan.m_batches) ws->m_batches = std::min<uint32_t>(ws->m_batches, ws->plan.m_batches);
    }
    if (dev_alloc(&ws->d_M, D * c->N * ws->m_batches) != cudaSuccess || cudaMalloc(&ws->d_X, (size_t)max_nq * c->p.F) != cudaSuccess ||
        dev_alloc(&ws->d_H, D * max_nq) != cudaSuccess ||
        dev_alloc(&ws->d_out, (size_t)ws->nb_max * 2 * c->L * c->N) != cudaSuccess ||
        dev_alloc(&ws->d_msg, ephdc_scores_message_bytes(c, ws->nb_max)) != cudaSuccess ||
        dev_alloc(&ws->d_dlim, ws->nb_max) != cudaSuccess) {
        ephdc_workspace_free(ws.release());
        return EPHDC_ERESOURCE;
    }
    *out = ws.release();
    return EPHDC_OK;
}

ephdc_status ephdc_workspace_set_timing(ephdc_workspace *ws, int enable) {
    if (!ws) return EPHDC_ENULL;
    ws->timing = enable != 0;
    return EPHDC_OK;
}

ephdc_status ephdc_workspace_timing(ephdc_workspace *ws, const char **names, double *ms, uint64_t *launches,
                                    uint32_t *n) {
    if (!ws || !n) return EPHDC_ENULL;
    EPHDC_CUDA_TRY(cudaSetDevice(ws->ctx->device));
    if (!ws->ev_marks.empty()) {
        EPHDC_CUDA_TRY(cudaEventSynchronize(ws->ev_pool[ws->ev_marks.back().second + 1]));
        for (auto &mk : ws->ev_marks) {
            float e = 0;
            EPHDC_CUDA_TRY(cudaEventElapsedTime(&e, ws->ev_pool[mk.second], ws->ev_pool[mk.second + 1]));
            ws->ms[mk.first] += e;
        }
        ws->ev_marks.clear();
    }
    const uint32_t cnt = std::min<uint32_t>(*n, ephdc_workspace::kClasses);
    for (uint32_t i = 0; i < cnt; ++i) {
        if (names) names[i] = kClassNames[i];
        if (ms) ms[i] = ws->ms[i];
        if (launches) launches[i] = ws->launches[i];
        ws->ms[i] = 0;
        ws->launches[i] = 0;
    }
    *n = cnt;
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// client hot path
// ------------------------------------------------------------------------------------
static ephdc_status encode_impl(const ephdc_ctx *c, ephdc_workspace *ws, const void *d_X, const int8_t *d_P,
                                uint32_t nq, int8_t *d_H, cudaStream_t st) {
    if (nq == 0) return EPHDC_OK;
    Timer tm(ws, st, kClsEncode);
    EPHDC_CUDA_TRY(launch_encode(c, d_X, d_P, nq, d_H, false, st));
    tm.done();
    return EPHDC_OK;
}

ephdc_status ephdc_encode_queries(const ephdc_ctx *c, const void *d_X, const int8_t *d_P, uint32_t nq, int8_t *d_H,
                                  void *stream) {
    if (!c || ((!d_X || !d_P || !d_H) && nq)) return EPHDC_ENULL;
    if (c->device < 0) return EPHDC_ECONTEXT;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    return encode_impl(c, nullptr, d_X, d_P, nq, d_H, (cudaStream_t)stream);
}

ephdc_status ephdc_encode_raw(const ephdc_ctx *c, const void *d_X, const int8_t *d_P, uint32_t n, int32_t *d_acc,
                              void *stream) {
    if (!c || ((!d_X || !d_P || !d_acc) && n)) return EPHDC_ENULL;
    if (c->device < 0) return EPHDC_ECONTEXT;
    if (n == 0) return EPHDC_OK;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    EPHDC_CUDA_TRY(launch_encode(c, d_X, d_P, n, d_acc, true, (cudaStream_t)stream));
    return EPHDC_OK;
}

static ephdc_status infer_impl(const ephdc_ctx *c, const ephdc_model *m, ephdc_workspace *ws, const int8_t *d_H,
                               uint32_t nq, uint64_t *d_out, cudaStream_t st, const uint32_t *h_dims = nullptr) {
    const uint32_t nb = (nq + c->B - 1) / c->B;
    const size_t per = (size_t)2 * c->L * c->N;
    if (nb == 0) return EPHDC_OK;
    EPHDC_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(uint64_t) * per * nb, st));
    if (h_dims && c->f64.enabled)   // per-batch dim counts for the fused kernel (pageable copy: synchronous)
        EPHDC_CUDA_TRY(cudaMemcpyAsync(ws->d_dlim, h_dims, sizeof(uint32_t) * nb, cudaMemcpyHostToDevice, st));
    if (c->f64.enabled) {
        // FP64 path: pack + INTT_t of a group of batches, then ONE fused launch over the group
        for (uint32_t b0 = 0; b0 < nb; b0 += ws->m_batches) {
            const uint32_t g = std::min(ws->m_batches, nb - b0);
            {
                Timer tm(ws, st, kClsPack);
                EPHDC_CUDA_TRY(launch_pack_intt_queries(c, d_H, nq, b0, g, 0, c->p.D_live, ws->d_M, st, ws->plan.flags));
                tm.done();
            }
            {
                Timer tm(ws, st, kClsMac);
                EPHDC_CUDA_TRY(launch_ntt_mac_f64(c, ws->plan, ws->d_M, g, reinterpret_cast<const double *>(m->d_ct),
                                                  d_out + per * b0, st, h_dims ? ws->d_dlim + b0 : nullptr));
                tm.done();
            }
        }
        Timer tm(ws, st, kClsFinal);
        EPHDC_CUDA_TRY(launch_reduce_out(c, d_out, nb, st));
        tm.done();
        ws->last_stream = st;
        return EPHDC_OK;
    }
    for (uint32_t b = 0; b < nb; ++b) {
        {
            Timer tm(ws, st, kClsPack);
            EPHDC_CUDA_TRY(launch_pack_intt_queries(c, d_H, nq, b, 1, 0, c->p.D_live, ws->d_M, st, ws->plan.flags));
            tm.done();
        }
        {
            Timer tm(ws, st, kClsMac);
            EPHDC_CUDA_TRY(launch_ntt_mac(c, ws->d_M, m->d_ct, d_out + per * b, st, h_dims ? h_dims[b] : 0xffffffffu));
            tm.done();
        }
        {
            Timer tm(ws, st, kClsFinal);
            EPHDC_CUDA_TRY(launch_finalize(c, d_out + per * b, st));
            tm.done();
        }
    }
    ws->last_stream = st;
    return EPHDC_OK;
}

ephdc_status ephdc_infer_batch(const ephdc_ctx *c, const ephdc_model *m, ephdc_workspace *ws, const int8_t *d_H,
                               uint32_t nq, uint64_t *d_out, uint32_t cap_ct, void *stream) {
    if (!c || !m || !ws || ((!d_H || !d_out) && nq)) return EPHDC_ENULL;
    if (m->ctx != c || ws->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    const uint32_t nb = (nq + c->B - 1) / c->B;
    if (cap_ct < nb) return EPHDC_EOVERFLOW;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    return infer_impl(c, m, ws, d_H, nq, d_out, (cudaStream_t)stream);
}

ephdc_status ephdc_infer_batch_prefix(const ephdc_ctx *c, const ephdc_model *m, ephdc_workspace *ws,
                                      const int8_t *d_H, uint32_t nq, const uint32_t *h_dims, uint64_t *d_out,
                                      uint32_t cap_ct, void *stream) {
    if (!c || !m || !ws || ((!d_H || !d_out || !h_dims) && nq)) return EPHDC_ENULL;
    if (m->ctx != c || ws->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    const uint32_t nb = (nq + c->B - 1) / c->B;
    if (cap_ct < nb) return EPHDC_EOVERFLOW;
    if (nq > ws->max_nq) return EPHDC_EPARAM;
    for (uint32_t b = 0; b < nb; ++b)
        if (h_dims[b] > c->p.D_live) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    return infer_impl(c, m, ws, d_H, nq, d_out, (cudaStream_t)stream, h_dims);
}

ephdc_status ephdc_encode_plaintexts(const ephdc_ctx *c, ephdc_workspace *ws, const int8_t *d_H, uint32_t nq,
                                     uint32_t b, uint32_t d0, uint32_t nd, uint64_t *d_pt, void *stream) {
    if (!c || !ws || !d_H || !d_pt) return EPHDC_ENULL;
    if (ws->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    if ((uint64_t)b * c->B >= nq || (uint64_t)d0 + nd > c->p.D_live) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (nd > c->p.D_live * ws->m_batches) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(launch_pack_intt_queries(c, d_H, nq, b, 1, d0, nd, ws->d_M, st));
    if (c->f64.enabled) EPHDC_CUDA_TRY(launch_plaintext_ntt_f64(c, ws->d_M, nd, d_pt, st));
    else EPHDC_CUDA_TRY(launch_plaintext_ntt(c, ws->d_M, nd, d_pt, st));
    return EPHDC_OK;
}

ephdc_status ephdc_classify_host(const ephdc_ctx *c, const ephdc_model *m, ephdc_workspace *ws, const void *h_X,
                                 const int8_t *d_P, uint32_t nq, uint64_t *h_out, uint32_t cap_ct, void *stream) {
    if (!c || !m || !ws || ((!h_X || !d_P || !h_out) && nq)) return EPHDC_ENULL;
    if (m->ctx != c || ws->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    if (nq > ws->max_nq) return EPHDC_EPARAM;
    const uint32_t nb = (nq + c->B - 1) / c->B;
    if (cap_ct < nb) return EPHDC_EOVERFLOW;
    if (nq == 0) return EPHDC_OK;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    EPHDC_CUDA_TRY(cudaMemcpyAsync(ws->d_X, h_X, (size_t)nq * c->p.F, cudaMemcpyHostToDevice, st));
    ephdc_status s = encode_impl(c, ws, ws->d_X, d_P, nq, ws->d_H, st);
    if (s != EPHDC_OK) return s;
    s = infer_impl(c, m, ws, ws->d_H, nq, ws->d_out, st);
    if (s != EPHDC_OK) return s;
    EPHDC_CUDA_TRY(cudaMemcpyAsync(h_out, ws->d_out, sizeof(uint64_t) * 2 * c->L * c->N * nb, cudaMemcpyDeviceToHost, st));
    EPHDC_CUDA_TRY(cudaStreamSynchronize(st));
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// HE-HDC-SR, the server-side SIMD baseline
// ------------------------------------------------------------------------------------
ephdc_status ephdc_sr_encrypt_queries(const ephdc_ctx *c, ephdc_sk *sk, ephdc_workspace *ws, const int8_t *d_H,
                                      uint32_t nq, uint32_t b, const ephdc_seed *seed, uint64_t *d_qct,
                                      void *stream) {
    if (!c || !sk || !ws || !d_H || !d_qct) return EPHDC_ENULL;
    ephdc_seed key;
    if (ephdc_status e = resolve_seed(seed, &key)) return e;
    if (sk->ctx != c || ws->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    if ((uint64_t)b * c->B >= nq) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (!sk->d_shat_mont) {
        const std::vector<uint64_t> shm = shat_mont_host(c, sk);
        if (dev_alloc(&sk->d_shat_mont, shm.size()) != cudaSuccess) return EPHDC_ERESOURCE;
        EPHDC_CUDA_TRY(cudaMemcpy(sk->d_shat_mont, shm.data(), sizeof(uint64_t) * shm.size(), cudaMemcpyHostToDevice));
    }
    const uint32_t D = c->p.D_live;
    EPHDC_CUDA_TRY(launch_pack_intt_sr(c, d_H, false, nq, b, 0, D, ws->d_M, st));
    // stream indices 2^32 + b*D + d: disjoint from the model's d < D_live (reading #25)
    EPHDC_CUDA_TRY(launch_encrypt(c, ws->d_M, (1ull << 32) + (uint64_t)b * D, D, sk->d_shat_mont, key, d_qct, st));
    return EPHDC_OK;
}

ephdc_status ephdc_sr_model_plaintexts(const ephdc_ctx *c, const int8_t *h_class_hv, uint64_t *d_pt) {
    if (!c || !h_class_hv || !d_pt) return EPHDC_ENULL;
    if (c->device < 0) return EPHDC_ECONTEXT;
    const uint32_t N = c->N, D = c->p.D_live, k = c->p.k;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    const uint32_t chunk = std::min<uint32_t>(D, 2048);
    DevBuf bC, bM;
    if (cudaMalloc(&bC.p, (size_t)k * D) != cudaSuccess || cudaMalloc(&bM.p, sizeof(uint32_t) * (size_t)chunk * N) != cudaSuccess)
        return EPHDC_ERESOURCE;
    EPHDC_CUDA_TRY(cudaMemcpy(bC.p, h_class_hv, (size_t)k * D, cudaMemcpyHostToDevice));
    for (uint32_t d0 = 0; d0 < D; d0 += chunk) {
        const uint32_t nd = std::min(chunk, D - d0);
        EPHDC_CUDA_TRY(launch_pack_intt_sr(c, (const int8_t *)bC.p, true, 0, 0, d0, nd, (uint32_t *)bM.p, 0));
        uint64_t *out = d_pt + (size_t)d0 * c->L * N;
        if (c->f64.enabled) EPHDC_CUDA_TRY(launch_plaintext_ntt_f64(c, (const uint32_t *)bM.p, nd, out, 0));
        else EPHDC_CUDA_TRY(launch_plaintext_ntt(c, (const uint32_t *)bM.p, nd, out, 0));
    }
    EPHDC_CUDA_TRY(cudaDeviceSynchronize());
    return EPHDC_OK;
}

ephdc_status ephdc_sr_evaluate(const ephdc_ctx *c, const uint64_t *d_pt, const uint64_t *d_qct, uint64_t *d_out,
                               void *stream) {
    if (!c || !d_pt || !d_qct || !d_out) return EPHDC_ENULL;
    if (c->device < 0) return EPHDC_ECONTEXT;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    EPHDC_CUDA_TRY(launch_mac_ctx(c, d_qct, d_pt, c->p.D_live, d_out, (cudaStream_t)stream));
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// scores message (bit-packed residues)
// ------------------------------------------------------------------------------------
size_t ephdc_scores_message_bytes(const ephdc_ctx *c, uint32_t nb) {
    if (!c) return 0;
    size_t bits = 0;
    for (uint32_t b : c->qbits) bits += b;
    return (size_t)nb * 2 * c->N * bits / 8;
}

ephdc_status ephdc_pack_scores(const ephdc_ctx *c, const uint64_t *d_ct, uint32_t nb, uint8_t *d_msg, void *stream) {
    if (!c || ((!d_ct || !d_msg) && nb)) return EPHDC_ENULL;
    if (c->device < 0) return EPHDC_ECONTEXT;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    EPHDC_CUDA_TRY(launch_pack_bits(c, d_ct, nb, d_msg, (cudaStream_t)stream));
    return EPHDC_OK;
}

ephdc_status ephdc_unpack_scores(const ephdc_ctx *c, const uint8_t *h_msg, uint32_t nb, uint64_t *h_ct) {
    if (!c || ((!h_msg || !h_ct) && nb)) return EPHDC_ENULL;
    const uint32_t N = c->N, L = c->L;
    size_t bitpos = 0;
    for (uint32_t bc = 0; bc < 2 * nb; ++bc)
        for (uint32_t j = 0; j < L; ++j) {
            const uint32_t bj = c->qbits[j];
            uint64_t *o = h_ct + ((size_t)bc * L + j) * N;
            for (uint32_t i = 0; i < N; ++i) {
                uint64_t v = 0;
                for (uint32_t k = 0; k < bj; ++k, ++bitpos)
                    v |= (uint64_t)((h_msg[bitpos >> 3] >> (bitpos & 7)) & 1u) << k;
                if (v >= c->q[j]) return EPHDC_EDOMAIN;
                o[i] = v;
            }
        }
    return EPHDC_OK;
}

ephdc_status ephdc_classify_host_packed(const ephdc_ctx *c, const ephdc_model *m, ephdc_workspace *ws,
                                        const void *h_X, const int8_t *d_P, uint32_t nq, uint8_t *h_msg,
                                        size_t cap_bytes, void *stream) {
    if (!c || !m || !ws || ((!h_X || !d_P || !h_msg) && nq)) return EPHDC_ENULL;
    if (m->ctx != c || ws->ctx != c || c->device < 0) return EPHDC_ECONTEXT;
    if (nq > ws->max_nq) return EPHDC_EPARAM;
    if (nq == 0) return EPHDC_OK;
    const uint32_t nb = (nq + c->B - 1) / c->B;
    if (cap_bytes < ephdc_scores_message_bytes(c, nb)) return EPHDC_EOVERFLOW;
    EPHDC_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t st = (cudaStream_t)stream;
    EPHDC_CUDA_TRY(cudaMemcpyAsync(ws->d_X, h_X, (size_t)nq * c->p.F, cudaMemcpyHostToDevice, st));
    ephdc_status s = encode_impl(c, ws, ws->d_X, d_P, nq, ws->d_H, st);
    if (s != EPHDC_OK) return s;
    s = infer_impl(c, m, ws, ws->d_H, nq, ws->d_out, st);
    if (s != EPHDC_OK) return s;
    EPHDC_CUDA_TRY(launch_pack_bits(c, ws->d_out, nb, ws->d_msg, st));
    EPHDC_CUDA_TRY(cudaMemcpyAsync(h_msg, ws->d_msg, ephdc_scores_message_bytes(c, nb), cudaMemcpyDeviceToHost, st));
    EPHDC_CUDA_TRY(cudaStreamSynchronize(st));
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// server decide (host)
// ------------------------------------------------------------------------------------
static void decrypt_one(const ephdc_ctx *c, const ephdc_sk *sk, const uint64_t *ct, uint64_t *slots) {
    const uint32_t N = c->N, L = c->L;
    std::vector<uint64_t> x((size_t)L * N);
    for (uint32_t j = 0; j < L; ++j) {
        const uint64_t q = c->q[j];
        const uint64_t *c0 = ct + (size_t)j * N;
        const uint64_t *c1 = ct + ((size_t)L + j) * N;
        const uint64_t *sh = sk->s_hat.data() + (size_t)j * N;
        uint64_t *xj = x.data() + (size_t)j * N;
        for (uint32_t i = 0; i < N; ++i) {
            const uint64_t v = mulmod(c1[i] % q, sh[i], q);
            const uint64_t u = c0[i] % q;
            xj[i] = u + v >= q ? u + v - q : u + v;
        }
        c->host_q[j].inverse(xj);
    }
    const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nth; ++w)
        pool.emplace_back([&, w] {
            for (uint32_t i = w; i < N; i += nth) slots[i] = c->crt.round_coeff(x.data() + i, N);
        });
    for (auto &th : pool) th.join();
    c->host_t.forward(slots);
}

ephdc_status ephdc_decrypt_slots(const ephdc_ctx *c, const ephdc_sk *sk, const uint64_t *h_ct, uint64_t *h_slots) {
    if (!c || !sk || !h_ct || !h_slots) return EPHDC_ENULL;
    if (sk->ctx != c) return EPHDC_ECONTEXT;
    decrypt_one(c, sk, h_ct, h_slots);
    return EPHDC_OK;
}

ephdc_status ephdc_decrypt_scores(const ephdc_ctx *c, const ephdc_sk *sk, const uint64_t *h_ct, uint32_t nq,
                                  int64_t *h_scores, uint32_t *h_labels) {
    if (!c || !sk || ((!h_ct || !h_scores) && nq)) return EPHDC_ENULL;
    if (sk->ctx != c) return EPHDC_ECONTEXT;
    const uint32_t N = c->N, k = c->p.k, B = c->B;
    const uint32_t nb = (nq + B - 1) / B;
    const int64_t t = (int64_t)c->t;
    // batches are independent ciphertexts: host threads over them (the NTT tables and the
    // CRT context are read-only)
    auto work = [&](uint32_t b0, uint32_t b1) {
        std::vector<uint64_t> slots(N);
        for (uint32_t b = b0; b < b1; ++b) {
            decrypt_one(c, sk, h_ct + (size_t)b * 2 * c->L * N, slots.data());
            const uint32_t n_b = std::min(B, nq - b * B);
            for (uint32_t qi = 0; qi < n_b; ++qi) {
                const uint32_t qg = b * B + qi;
                int64_t best = 0;
                uint32_t arg = 0;
                for (uint32_t cl = 0; cl < k; ++cl) {
                    int64_t v = (int64_t)slots[(size_t)qi * k + cl];
                    if (v > (t - 1) / 2) v -= t;
                    h_scores[(size_t)qg * k + cl] = v;
                    if (cl == 0 || v > best) { best = v; arg = cl; }
                }
                if (h_labels) h_labels[qg] = arg;
            }
        }
    };
    const uint32_t nt = std::max<uint32_t>(1, std::min<uint32_t>(nb, std::thread::hardware_concurrency()));
    if (nt <= 1) {
        work(0, nb);
        return EPHDC_OK;
    }
    std::vector<std::thread> pool;
    for (uint32_t i = 0; i < nt; ++i) pool.emplace_back(work, (uint32_t)((uint64_t)nb * i / nt), (uint32_t)((uint64_t)nb * (i + 1) / nt));
    for (auto &th : pool) th.join();
    return EPHDC_OK;
}

// ------------------------------------------------------------------------------------
// standalone kernels (c5)
// ------------------------------------------------------------------------------------
void ephdc_ntt_plan_free(ephdc_ntt_plan *p) {
    if (!p) return;
    if (p->device >= 0) {
        cudaSetDevice(p->device);
        cudaFree(p->tw);
        cudaFree(p->itw);
        cudaFree(p->ninv);
        cudaFree(p->tw_f64);
        cudaFree(p->itw_f64);
        cudaFree(p->post_f64);
        cudaFree(p->tw32);
        cudaFree(p->itw32);
        cudaFree(p->ninv32);
        ephdc_ntt_plan_c5_free(p);
    }
    delete p;
}

ephdc_status ephdc_ntt_plan_create(const uint64_t *q, uint32_t L, uint32_t log2N, int device, uint32_t flags,
                                   ephdc_ntt_plan **out) {
    if (!q || !out) return EPHDC_ENULL;
    *out = nullptr;
    if (L < 1 || L > EPHDC_MAX_PRIMES || log2N < 10 || log2N > 16 || (flags & ~(EPHDC_NTT_FORCE_INT | EPHDC_NTT_ALT_TEAMS | EPHDC_NTT_U32_GENERIC)))
        return EPHDC_EPARAM;
    for (uint32_t j = 0; j < L; ++j)
        if (q[j] >= (1ull << 61) || !is_ntt_prime(q[j], log2N)) return EPHDC_EPARAM;
    if (device < 0) return EPHDC_ECONTEXT;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) return EPHDC_ECUDA;
    EPHDC_CUDA_TRY(cudaSetDevice(device));
    std::unique_ptr<ephdc_ntt_plan> p(new (std::nothrow) ephdc_ntt_plan());
    if (!p) return EPHDC_ERESOURCE;
    p->q.assign(q, q + L);
    p->L = L;
    p->log2N = log2N;
    p->N = 1u << log2N;
    p->device = device;
    fill_prime_set(p->ps, p->q, 0);
    const uint32_t N = p->N;
    std::vector<TwPair<u64>> tw((size_t)L * N), itw((size_t)L * N);
    std::vector<uint64_t> ninv(2 * L);
    for (uint32_t j = 0; j < L; ++j) {
        const uint64_t psi = min_primitive_root_2n(q[j], log2N);
        auto f = make_tw64(psi, q[j], log2N);
        auto g = make_tw64(invmod(psi, q[j]), q[j], log2N);
        std::copy(f.begin(), f.end(), tw.begin() + (size_t)j * N);
        std::copy(g.begin(), g.end(), itw.begin() + (size_t)j * N);
        ninv[2 * j] = invmod(N % q[j], q[j]);
        ninv[2 * j + 1] = shoup64(ninv[2 * j], q[j]);
    }
    plan_ntt_f64(p->q, log2N, &p->fwd_f64, &p->inv_f64, &p->inv_dit);
    if (flags & EPHDC_NTT_FORCE_INT) p->fwd_f64 = p->inv_f64 = false;
    p->c5_alt_teams = (flags & EPHDC_NTT_ALT_TEAMS) != 0;
    p->int_per_poly = p->c5_alt_teams;
    p->u32_generic = (flags & EPHDC_NTT_U32_GENERIC) != 0;
    // the c5 kernels (ntt_c5.cu) use the FP64 forward table at every N >= 2^12 whose
    // primes are all < 2^50; their own bounds are decided in plan_ntt_c5
    const bool c5_candidate = !(flags & EPHDC_NTT_FORCE_INT) && log2N >= 12 &&
                              *std::max_element(p->q.begin(), p->q.end()) < (1ull << 50);

    if (p->fwd_f64 || p->inv_f64 || c5_candidate) {
        // FP64 tables: forward psi_rev; inverse = Cooley-Tukey DIT on the bit-reversed
        // input (x[r] = DFT(a psi^j)[brev r]): stage of half-size h uses omega^-(N/2h) jj
        // for the block position jj < h (entry h + jj), then a_j = N^-1 psi^-j x_j
        std::vector<double> f((size_t)L * N * 2), g((size_t)L * N * 2), po((size_t)L * N * 2);
        for (uint32_t j = 0; j < L; ++j) {
            const double qd = (double)q[j];
            const uint64_t psi_inv = invmod(min_primitive_root_2n(q[j], log2N), q[j]);
            for (uint32_t i = 0; i < N; ++i) {
                const size_t k = (size_t)j * N + i;
                f[2 * k] = i ? (double)tw[k].w : qd;
                f[2 * k + 1] = i ? (double)tw[k].w / qd : 1.0 / qd;
            }
            g[2 * (size_t)j * N] = qd;
            g[2 * (size_t)j * N + 1] = 1.0 / qd;
            if (p->inv_dit) {
                for (uint32_t h = 1; h < N; h *= 2) {
                    const uint64_t wh = powmod(psi_inv, N / h, q[j]);   // omega^-(N/2h), omega = psi^2
                    uint64_t w = 1;
                    for (uint32_t jj = 0; jj < h; ++jj, w = mulmod(w, wh, q[j])) {
                        const size_t k = (size_t)j * N + h + jj;
                        g[2 * k] = (double)w;
                        g[2 * k + 1] = (double)w / qd;
                    }
                }
                uint64_t c = ninv[2 * j];                                  // N^-1 psi^-i
                for (uint32_t i = 0; i < N; ++i, c = mulmod(c, psi_inv, q[j])) {
                    const size_t k = (size_t)j * N + i;
                    po[2 * k] = (double)c;
                    po[2 * k + 1] = (double)c / qd;
                }
            } else {
                for (uint32_t i = 1; i < N; ++i) {                       // psi^-1_rev (GS)
                    const size_t k = (size_t)j * N + i;
                    g[2 * k] = (double)itw[k].w;
                    g[2 * k + 1] = (double)itw[k].w / qd;
                }
                po[2 * (size_t)j * N] = (double)ninv[2 * j];           // [j][0] = N^-1
                po[2 * (size_t)j * N + 1] = (double)ninv[2 * j] / qd;
            }
        }
        if (cudaMalloc(&p->tw_f64, sizeof(double) * f.size()) != cudaSuccess ||
            cudaMalloc(&p->itw_f64, sizeof(double) * g.size()) != cudaSuccess ||
            cudaMalloc(&p->post_f64, sizeof(double) * po.size()) != cudaSuccess) {
            ephdc_ntt_plan_free(p.release());
            return EPHDC_ERESOURCE;
        }
        if (cudaMemcpy(p->tw_f64, f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(p->itw_f64, g.data(), sizeof(double) * g.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(p->post_f64, po.data(), sizeof(double) * po.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            ephdc_ntt_plan_free(p.release());
            return EPHDC_ECUDA;
        }
    }
    if (dev_alloc(&p->tw, tw.size()) != cudaSuccess || dev_alloc(&p->itw, itw.size()) != cudaSuccess ||
        dev_alloc(&p->ninv, ninv.size()) != cudaSuccess) {
        ephdc_ntt_plan_free(p.release());
        return EPHDC_ERESOURCE;
    }
    if (cudaMemcpy(p->tw, tw.data(), sizeof(tw[0]) * tw.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->itw, itw.data(), sizeof(itw[0]) * itw.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->ninv, ninv.data(), sizeof(uint64_t) * ninv.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        ephdc_ntt_plan_free(p.release());
        return EPHDC_ECUDA;
    }
    // u32 words when every prime < 2^30 (lazy [0, 4q) fits 32 bits)
    if (*std::max_element(p->q.begin(), p->q.end()) < (1ull << 30)) {
        std::vector<TwPair<u32>> t32((size_t)L * N), it32((size_t)L * N);
        std::vector<uint32_t> n32(2 * L);
        for (size_t i = 0; i < t32.size(); ++i) {
            const uint32_t qj = (uint32_t)q[i / N];
            t32[i] = TwPair<u32>{(u32)tw[i].w, shoup32((u32)tw[i].w, qj)};
            it32[i] = TwPair<u32>{(u32)itw[i].w, shoup32((u32)itw[i].w, qj)};
        }
        for (uint32_t j = 0; j < L; ++j) {
            n32[2 * j] = (uint32_t)ninv[2 * j];
            n32[2 * j + 1] = shoup32(n32[2 * j], (uint32_t)q[j]);
        }
        if (dev_alloc(&p->tw32, t32.size()) != cudaSuccess || dev_alloc(&p->itw32, it32.size()) != cudaSuccess ||
            dev_alloc(&p->ninv32, n32.size()) != cudaSuccess) {
            ephdc_ntt_plan_free(p.release());
            return EPHDC_ERESOURCE;
        }
        if (cudaMemcpy(p->tw32, t32.data(), sizeof(t32[0]) * t32.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(p->itw32, it32.data(), sizeof(it32[0]) * it32.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(p->ninv32, n32.data(), sizeof(uint32_t) * n32.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            ephdc_ntt_plan_free(p.release());
            return EPHDC_ECUDA;
        }
    }
    p->u32_for_u64 = p->tw32 && !p->u32_generic && !(flags & EPHDC_NTT_FORCE_INT) && log2N >= 12 && log2N <= 14;
    if (c5_candidate && plan_ntt_c5(p.get()) != cudaSuccess) {
        ephdc_ntt_plan_free(p.release());
        return EPHDC_ECUDA;
    }
    *out = p.release();
    return EPHDC_OK;
}

ephdc_status ephdc_ntt_fwd(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, void *stream) {
    if (!p || (!d_polys && batch)) return EPHDC_ENULL;
    EPHDC_CUDA_TRY(cudaSetDevice(p->device));
    cudaError_t e = launch_ntt32_c5_u64(p, d_polys, batch, false, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) e = launch_ntt_c5(p, d_polys, batch, false, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) e = launch_ntt_batch_f64(p, d_polys, batch, false, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) EPHDC_CUDA_TRY(launch_ntt_batch(p, d_polys, batch, false, (cudaStream_t)stream));
    else EPHDC_CUDA_TRY(e);
    return EPHDC_OK;
}

ephdc_status ephdc_ntt_inv(const ephdc_ntt_plan *p, uint64_t *d_polys, uint32_t batch, void *stream) {
    if (!p || (!d_polys && batch)) return EPHDC_ENULL;
    EPHDC_CUDA_TRY(cudaSetDevice(p->device));
    cudaError_t e = launch_ntt32_c5_u64(p, d_polys, batch, true, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) e = launch_ntt_c5(p, d_polys, batch, true, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) e = launch_ntt_batch_f64(p, d_polys, batch, true, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) EPHDC_CUDA_TRY(launch_ntt_batch(p, d_polys, batch, true, (cudaStream_t)stream));
    else EPHDC_CUDA_TRY(e);
    return EPHDC_OK;
}

ephdc_status ephdc_ntt_fwd32(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, void *stream) {
    if (!p || (!d_polys && batch)) return EPHDC_ENULL;
    if (!p->tw32) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(p->device));
    const cudaError_t e = launch_ntt32_c5(p, d_polys, batch, false, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) EPHDC_CUDA_TRY(launch_ntt_batch32(p, d_polys, batch, false, (cudaStream_t)stream));
    else EPHDC_CUDA_TRY(e);
    return EPHDC_OK;
}

ephdc_status ephdc_ntt_inv32(const ephdc_ntt_plan *p, uint32_t *d_polys, uint32_t batch, void *stream) {
    if (!p || (!d_polys && batch)) return EPHDC_ENULL;
    if (!p->tw32) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(p->device));
    const cudaError_t e = launch_ntt32_c5(p, d_polys, batch, true, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) EPHDC_CUDA_TRY(launch_ntt_batch32(p, d_polys, batch, true, (cudaStream_t)stream));
    else EPHDC_CUDA_TRY(e);
    return EPHDC_OK;
}

ephdc_status ephdc_mac32(const ephdc_ntt_plan *p, const uint32_t *d_ct, const uint32_t *d_pt, uint32_t D,
                         uint32_t *d_out, void *stream) {
    if (!p || !d_out || ((!d_ct || !d_pt) && D)) return EPHDC_ENULL;
    if (!p->tw32) return EPHDC_EPARAM;
    EPHDC_CUDA_TRY(cudaSetDevice(p->device));
    EPHDC_CUDA_TRY(launch_mac32(p, d_ct, d_pt, D, d_out, (cudaStream_t)stream));
    return EPHDC_OK;
}

ephdc_status ephdc_ntt_plan_query(const ephdc_ntt_plan *p, ephdc_ntt_plan_info *info) {
    if (!p || !info) return EPHDC_ENULL;
    info->fwd_kernel = p->u32_for_u64 ? EPHDC_NTT_KERNEL_C5_U32
                       : p->c5_fwd    ? EPHDC_NTT_KERNEL_C5_F64
                       : p->fwd_f64   ? EPHDC_NTT_KERNEL_F64
                                      : EPHDC_NTT_KERNEL_INT;
    info->inv_kernel = p->u32_for_u64 ? EPHDC_NTT_KERNEL_C5_U32
                       : p->c5_inv    ? EPHDC_NTT_KERNEL_C5_F64
                       : p->inv_f64   ? EPHDC_NTT_KERNEL_F64
                                      : EPHDC_NTT_KERNEL_INT;
    info->u32_words = p->tw32 != nullptr;
    info->u32_kernel = !p->tw32 ? EPHDC_NTT_KERNEL_INT
                       : (!p->u32_generic && p->log2N >= 12) ? EPHDC_NTT_KERNEL_C5_U32
                                                                               : EPHDC_NTT_KERNEL_INT;
    return EPHDC_OK;
}

ephdc_status ephdc_mac(const ephdc_ntt_plan *p, const uint64_t *d_ct, const uint64_t *d_pt, uint32_t D, uint64_t *d_out,
                       void *stream) {
    if (!p || !d_out || ((!d_ct || !d_pt) && D)) return EPHDC_ENULL;
    EPHDC_CUDA_TRY(cudaSetDevice(p->device));
    EPHDC_CUDA_TRY(launch_mac(p, d_ct, d_pt, D, d_out, (cudaStream_t)stream));
    return EPHDC_OK;
}

}  // extern "C"
