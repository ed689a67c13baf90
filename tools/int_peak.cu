// int_peak.cu -- measured integer-pipe throughput on the B200 (denominator of the "alu" roofline).
// Each kernel runs 8 independent dependency chains per thread of one PTX op; the SASS op
// it lowers to is checked with cuobjdump. Reports ops/clk/SM using clock64/globaltimer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;

#define KERNEL(NAME, T, INIT, BODY)                                                        \
    __global__ void NAME(T *out, unsigned long long *clk) {                               \
        T r[CH];                                                                           \
        for (int c = 0; c < CH; ++c) r[c] = (T)(threadIdx.x * 7 + c * 13 + INIT);          \
        const T m = (T)(blockIdx.x | 0x9e3779b9u);                                         \
        unsigned long long c0 = clock64(), g0;                                             \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));                             \
        for (int i = 0; i < ITERS; ++i) {                                                  \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }                       \
        }                                                                                  \
        unsigned long long c1 = clock64(), g1;                                             \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));                             \
        T s = 0;                                                                           \
        for (int c = 0; c < CH; ++c) s += r[c];                                            \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                    \
        if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }   \
    }

// IMAD (32-bit multiply-add, lo)
KERNEL(k_imad, uint32_t, 1, asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(r[c]) : "r"(m)))
// IMAD.HI (32x32 -> high 32)
KERNEL(k_imadhi, uint32_t, 1, asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(r[c]) : "r"(m)))
// IMAD.WIDE (32x32 -> 64 + 64)
KERNEL(k_imadwide, uint64_t, 1,
       asm volatile("{ .reg .u32 lo; cvt.u32.u64 lo, %0; mad.wide.u32 %0, lo, %1, %0; }" : "+l"(r[c]) : "r"((uint32_t)m)))
// IADD3 (alu pipe)
KERNEL(k_iadd3, uint32_t, 1, asm volatile("add.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(m)))
// u64 multiply high (emulated: several IMAD-class ops)
KERNEL(k_mul64hi, uint64_t, 3, asm volatile("mul.hi.u64 %0, %0, %1;" : "+l"(r[c]) : "l"((uint64_t)m * 0x9E3779B97F4A7C15ull)))
// u64 multiply low
KERNEL(k_mul64lo, uint64_t, 3, asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(r[c]) : "l"((uint64_t)m * 0x9E3779B97F4A7C15ull | 1)))
// FP64 FMA (for reference: the DFMA pipe)
KERNEL(k_dfma, double, 1, asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(r[c]) : "d"(1.0000001)))
KERNEL(k_dadd, double, 1, asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(r[c]) : "d"(1.0000001)))
KERNEL(k_dmul, double, 1, asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(r[c]) : "d"(1.0000001)))
// int32 -> double conversion (I2F.F64): which pipe, what rate
KERNEL(k_cvt, double, 1, {
    const int v = __double2loint(r[c]);
    asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(r[c]) : "r"(v));
})
// DFMA chains plus as many independent cvt chains: if the conversion has its own pipe
// this runs at the DFMA-only rate (ops counted = DFMAs only)
__global__ void k_dfma_cvt(double *out, unsigned long long *clk) {
    double r[CH], z[CH];
    for (int c = 0; c < CH; ++c) { r[c] = threadIdx.x * 7 + c; z[c] = c; }
    unsigned long long c0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(r[c]) : "d"(1.0000001));
            const int v = __double2loint(z[c]);
            asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(z[c]) : "r"(v));
        }
    }
    unsigned long long c1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    double s = 0;
    for (int c = 0; c < CH; ++c) s += r[c] + z[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
}

// The exact FP64 Cooley-Tukey butterfly of csrc/modf64.cuh (8 FP64 instructions:
// DMUL, 3 DFMA, 4 DADD) on CH independent (X, Y) pairs: the achievable FP64 rate of
// the NTT's instruction mix.  Counted as 8 ops per butterfly.
__global__ void k_bfly(double *out, unsigned long long *clk) {
    const double q = 281474976546817.0, nq = -q, w = 23720796222.0, wq = w / q, R = 6755399441055744.0;
    double X[CH], Y[CH];
    for (int c = 0; c < CH; ++c) { X[c] = threadIdx.x * 7 + c; Y[c] = threadIdx.x * 3 + c * 11; }
    unsigned long long c0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const double y = Y[c], x = X[c];
            const double h = __dmul_rn(y, w);
            const double l = __fma_rn(y, w, -h);
            const double k = __dadd_rn(__fma_rn(y, wq, R), -R);
            const double t = __dadd_rn(__fma_rn(k, nq, h), l);
            X[c] = __dadd_rn(x, t);
            Y[c] = __dsub_rn(x, t);
        }
    }
    unsigned long long c1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    double s = 0;
    for (int c = 0; c < CH; ++c) s += X[c] + Y[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
}

template <class K, class T>
static void run(const char *name, K kern, int blocks, int threads) {
    T *out;
    unsigned long long *clk, h[2];
    cudaMalloc(&out, sizeof(T) * blocks * threads);
    cudaMalloc(&clk, 16);
    kern<<<blocks, threads>>>(out, clk);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    const double ops = (double)blocks * threads * ITERS * CH;
    const double mhz = (double)h[0] / (double)h[1] * 1e3;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double per_sm_clk = ops / (ms * 1e-3) / sms / (mhz * 1e6);
    printf("{\"op\": \"%s\", \"Gops\": %.1f, \"per_sm_per_clk\": %.2f, \"sm_mhz\": %.0f, \"ms\": %.3f}\n", name,
           ops / (ms * 1e-3) / 1e9, per_sm_clk, mhz, ms);
    cudaFree(out);
    cudaFree(clk);
}

// Sustained: the butterfly mix at the c5 kernels' occupancy (one 512-thread CTA per SM)
// launched back to back for `seconds`, so the clock and power state are those of a long
// run (an external nvidia-smi sampler records them): the measured FP64 ceiling of the
// NTT's instruction mix.
static void sustained(double seconds) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    unsigned long long *clk;
    cudaMalloc(&out, sizeof(double) * sms * 512);
    cudaMalloc(&clk, 16);
    k_bfly<<<sms, 512>>>(out, clk);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int launches = 0;
    float ms = 0.f;
    cudaEventRecord(a);
    while (ms < seconds * 1e3) {
        for (int i = 0; i < 64; ++i) k_bfly<<<sms, 512>>>(out, clk);
        launches += 64;
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    const double ops = (double)launches * sms * 512 * ITERS * CH;
    printf("{\"op\": \"FP64 butterfly mix sustained (1x512 thr/SM)\", \"Gops\": %.1f, \"seconds\": %.2f, "
           "\"launches\": %d}\n",
           ops / (ms * 1e-3) / 1e9, ms * 1e-3, launches);
}

int main(int argc, char **argv) {
    if (argc > 2 && argv[1][0] == 's') {   // int_peak sustained <seconds>
        sustained(atof(argv[2]));
        return 0;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    run<decltype(k_imad), uint32_t>("IMAD(mad.lo.u32)", k_imad, blocks, threads);
    run<decltype(k_imadhi), uint32_t>("IMAD.HI(mad.hi.u32)", k_imadhi, blocks, threads);
    run<decltype(k_imadwide), uint64_t>("IMAD.WIDE(mad.wide.u32)", k_imadwide, blocks, threads);
    run<decltype(k_iadd3), uint32_t>("IADD3(add.u32)", k_iadd3, blocks, threads);
    run<decltype(k_mul64hi), uint64_t>("mul.hi.u64", k_mul64hi, blocks, threads);
    run<decltype(k_mul64lo), uint64_t>("mul.lo.u64", k_mul64lo, blocks, threads);
    run<decltype(k_dfma), double>("DFMA(fma.rn.f64)", k_dfma, blocks, threads);
    run<decltype(k_dadd), double>("DADD(add.rn.f64)", k_dadd, blocks, threads);
    run<decltype(k_dmul), double>("DMUL(mul.rn.f64)", k_dmul, blocks, threads);
    run<decltype(k_cvt), double>("I2F.F64(cvt.rn.f64.s32)", k_cvt, blocks, threads);
    run<decltype(k_dfma_cvt), double>("DFMA + independent cvt.f64.s32 (DFMA counted)", k_dfma_cvt, blocks, threads);
    // butterfly mix: ITERS/8 iterations x CH butterflies x 8 FP64 instructions = ITERS*CH ops
    run<decltype(k_bfly), double>("FP64 butterfly mix (8 ops/bfly), 8x256 thr/SM", k_bfly, blocks, threads);
    run<decltype(k_bfly), double>("FP64 butterfly mix (8 ops/bfly), 1x512 thr/SM", k_bfly, sms, 512);
    return 0;
}
