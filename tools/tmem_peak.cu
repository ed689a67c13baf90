// tmem_peak.cu -- measured TMEM <-> register throughput on the B200 with the access
// pattern of the fused kernel's tail (tcgen05.ld/st .32x32b, 16 warps x 32 lanes, each
// warp its own 128 columns of its lane quarter).  Reports bytes/clk/SM for
//   ld1: one x16 load then wait::ld, repeated;  ld4: four x16 loads, one wait;
//   st4: four x16 stores, one wait::st;  ldst: x16 load, wait, x16 store (the tail's
//   read-modify-write of one accumulator block).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2511_00737_b200/csrc -o tmem_peak tmem_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tmem.cuh"

constexpr int ITERS = 2048;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_tmem(uint32_t *out, unsigned long long *clk) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ephdc_tmem::alloc(&slot, 512);
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    const uint32_t base = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 128u;
    uint32_t r[4][16];
    for (int b = 0; b < 4; ++b)
        for (int i = 0; i < 16; ++i) r[b][i] = threadIdx.x * 16 + i + b;
    for (int b = 0; b < 4; ++b) ephdc_tmem::st16(base + 16 * b, r[b]);
    ephdc_tmem::wait_st();
    __syncthreads();
    unsigned long long c0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < ITERS; ++it) {
        if constexpr (MODE == 0) {
            ephdc_tmem::ld16(base + 16 * (it & 3), r[0]);
            ephdc_tmem::wait_ld(r[0]);
            acc += r[0][it & 15];
        } else if constexpr (MODE == 1) {
#pragma unroll
            for (int b = 0; b < 4; ++b) ephdc_tmem::ld16(base + 16 * b, r[b]);
            ephdc_tmem::wait_ld(r[0]);
#pragma unroll
            for (int b = 1; b < 4; ++b) ephdc_tmem::after_wait(r[b]);
            acc += r[0][it & 15] + r[1][3] + r[2][5] + r[3][7];
        } else if constexpr (MODE == 2) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                r[b][0] += it;
                ephdc_tmem::st16(base + 16 * b, r[b]);
            }
            ephdc_tmem::wait_st();
        } else {
            ephdc_tmem::ld16(base + 16 * (it & 3), r[0]);
            ephdc_tmem::wait_ld(r[0]);
            r[0][0] += 1u;
            ephdc_tmem::st16(base + 16 * (it & 3), r[0]);
        }
    }
    ephdc_tmem::wait_st();
    unsigned long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + r[0][0] + r[3][1];
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = c1 - c0;
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(slot, 512);
}

template <int MODE> static void run(const char *name, double bytes_per_iter_thread) {
    uint32_t *out;
    unsigned long long *clk, h = 0;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 16);
    k_tmem<MODE><<<148, 512>>>(out, clk);
    cudaDeviceSynchronize();
    k_tmem<MODE><<<148, 512>>>(out, clk);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    const double bytes = bytes_per_iter_thread * 512.0 * ITERS;
    printf("{\"op\": \"%s\", \"bytes_per_clk_sm\": %.2f, \"clk\": %llu, \"err\": \"%s\"}\n", name, bytes / (double)h, h,
           cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    run<0>("tmem_ld_x16_wait", 64.0);
    run<1>("tmem_ld_4x16_wait", 256.0);
    run<2>("tmem_st_4x16_wait", 256.0);
    run<3>("tmem_ld_wait_st_x16", 128.0);
    return 0;
}
