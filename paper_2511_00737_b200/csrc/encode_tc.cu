// encode_tc.cu -- HDC encoding GEMM on the 5th-generation tensor cores (sm_100a).
//
//   acc[d][q] = sum_f P[d][f] * X[q][f]           (BASELINE.json subsystem (a))
//   h[d][q]   = clamp(floor((acc + 2^(s-1)) / 2^s), +-(2^(Q-1)-1))   (readings #12, #13)
//
// A = P [D_stored][F] int8 (K-major), B = X [nq][F] int8 or uint8 (K-major): a dense
// int8 contraction, exact in int32 (|acc| <= F * 255 < 2^18).  One CTA (4 warps)
// computes a 128 (dims) x 128 (queries) tile:
//   * warp 0 / lane 0: TMA producer -- cp.async.bulk.tensor.2d of 128 x 128-byte boxes
//     (SWIZZLE_128B) of P and X into a 3-stage shared-memory ring (full/empty mbarriers);
//     the tensor maps zero-fill beyond F, D_stored and nq, so ragged tiles need no code;
//   * warp 1 / lane 0: MMA issuer -- tcgen05.mma.cta_group::1.kind::i8, M = N = 128,
//     K = 32 per instruction, accumulator (int32) in 128 TMEM columns;
//     tcgen05.commit releases each stage and finally signals the epilogue;
//   * all 4 warps: epilogue -- tcgen05.ld.32x32b (thread = TMEM lane = dim row),
//     quantise, write 16-byte runs of H[d][q0..] (dim-major, row d feeds plaintext d).
// DESIGN.md "Kernels".
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "internal.h"
#include "tma_host.h"
#include "tmem.cuh"

namespace ephdc {

namespace {

constexpr int kTileM = 128, kTileN = 128, kTileK = 128;  // K tile in bytes (= int8 elements)
constexpr int kStages = 3;
constexpr int kThreads = 128;
constexpr uint32_t kStageBytes = (kTileM + kTileN) * kTileK;  // 32 KB
constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024;  // + alignment slack

EPHDC_D uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

EPHDC_D void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
EPHDC_D void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
EPHDC_D void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

EPHDC_D void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_addr(bar))
        : "memory");
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, rows 128 bytes apart, 8-row
// atoms 1024 bytes apart (SBO), version 1 (sm_100).  addr must be 1024-byte aligned
// up to the K offset inside the atom (added in 16-byte units).
EPHDC_D uint64_t smem_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor of kind::i8: D = S32, A = S8, B = S8 or U8, both K-major, M = N = 128.
template <bool B_UNSIGNED> constexpr uint32_t idesc_i8() {
    return (2u << 4) | (1u << 7) | ((B_UNSIGNED ? 0u : 1u) << 10) | ((uint32_t)(kTileN >> 3) << 17) |
           ((uint32_t)(kTileM >> 4) << 24);
}

EPHDC_D void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}

EPHDC_D void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

EPHDC_D void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory");
}

struct EncTcArgs {
    u32 nq, F, D_live, shift;
    int qmax;
};

template <bool B_UNSIGNED, bool RAW>
__global__ void __launch_bounds__(kThreads, 1)
    k_encode_tc(const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapX, EncTcArgs a,
                void *__restrict__ Hout) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
    __shared__ uint32_t tmem_slot;
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q0 = blockIdx.x * kTileN, d0 = blockIdx.y * kTileM;
    const int nk = (int)((a.F + kTileK - 1) / kTileK);

    if (warp == 0) ephdc_tmem::alloc(&tmem_slot, (uint32_t)kTileN);
    if (tid == 32) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(&done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    const uint32_t tmem_d = tmem_slot;

    if (tid == 0) {
        // TMA producer
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapP) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % kStages;
            if (kb >= kStages) mbar_wait(&empty_bar[s], (uint32_t)((kb / kStages - 1) & 1));
            unsigned char *sa = smem + (size_t)s * kStageBytes;
            unsigned char *sb = sa + kTileM * kTileK;
            mbar_expect_tx(&full_bar[s], kStageBytes);
            tma_load_2d(sa, &mapP, kb * kTileK, d0, &full_bar[s]);
            tma_load_2d(sb, &mapX, kb * kTileK, q0, &full_bar[s]);
        }
    } else if (tid == 32) {
        // MMA issuer
        constexpr uint32_t idesc = idesc_i8<B_UNSIGNED>();
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % kStages;
            mbar_wait(&full_bar[s], (uint32_t)((kb / kStages) & 1));
            ephdc_tmem::fence_after_sync();
            const uint32_t sa = smem_addr(smem + (size_t)s * kStageBytes);
            const uint32_t sb = sa + kTileM * kTileK;
#pragma unroll
            for (int k = 0; k < kTileK / 32; ++k)
                mma_i8(tmem_d, smem_desc(sa + 32 * k), smem_desc(sb + 32 * k), idesc, (kb | k) != 0);
            mma_commit(&empty_bar[s]);  // stage s free once these MMAs have read it
        }
        mma_commit(&done_bar);          // accumulator complete
    }
    __syncwarp();
    // epilogue: thread (warp w, lane l) owns dim row d0 + 32w + l, TMEM lane 32w + l
    mbar_wait(&done_bar, 0);
    ephdc_tmem::fence_after_sync();
    const int d = d0 + 32 * warp + lane;
    const bool row_ok = d < (int)a.D_live;
    const int rnd = a.shift ? (1 << (a.shift - 1)) : 0;
#pragma unroll 1
    for (int c = 0; c < kTileN / 32; ++c) {
        uint32_t r[32];
        ld32(tmem_d + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * c), r);
        const int qc = q0 + 32 * c;
        if (!row_ok) continue;
        if constexpr (RAW) {
            int *o = reinterpret_cast<int *>(Hout) + (size_t)d * a.nq + qc;
            if (qc + 32 <= (int)a.nq && ((a.nq & 3) == 0)) {
#pragma unroll
                for (int v = 0; v < 8; ++v)
                    reinterpret_cast<int4 *>(o)[v] = make_int4((int)r[4 * v], (int)r[4 * v + 1], (int)r[4 * v + 2], (int)r[4 * v + 3]);
            } else {
                for (int e = 0; e < 32 && qc + e < (int)a.nq; ++e) o[e] = (int)r[e];
            }
        } else {
            uint32_t packed[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                uint32_t w = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    int h = ((int)r[4 * v + b] + rnd) >> a.shift;  // arithmetic shift = floor division
                    h = max(-a.qmax, min(a.qmax, h));
                    w |= ((uint32_t)(h & 0xFF)) << (8 * b);
                }
                packed[v] = w;
            }
            int8_t *o = reinterpret_cast<int8_t *>(Hout) + (size_t)d * a.nq + qc;
            if (qc + 32 <= (int)a.nq && ((a.nq & 15) == 0)) {
                reinterpret_cast<uint4 *>(o)[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
                reinterpret_cast<uint4 *>(o)[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
            } else {
                for (int e = 0; e < 32 && qc + e < (int)a.nq; ++e) o[e] = (int8_t)((packed[e >> 2] >> (8 * (e & 3))) & 0xFF);
            }
        }
    }
    ephdc_tmem::fence_before_sync();
    __syncthreads();
    ephdc_tmem::fence_after_sync();
    if (warp == 0) ephdc_tmem::dealloc(tmem_d, (uint32_t)kTileN);
}

}  // namespace

// ---- host: tensor maps through the driver entry point (no -lcuda link; tma_host.h) ----
EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

namespace {

// rows x F bytes, row-major; box 128 rows x 128 bytes, 128-byte swizzle, zero fill
bool make_map(CUtensorMap *m, const void *base, uint64_t rows, uint64_t F) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {F, rows};
    const cuuint64_t strides[1] = {F};
    const cuuint32_t box[2] = {(cuuint32_t)kTileK, 128u};
    const cuuint32_t estr[2] = {1u, 1u};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool U, bool RAW> cudaError_t launch_tc(const CUtensorMap &mp, const CUtensorMap &mx, EncTcArgs a, void *H,
                                                 dim3 grid, cudaStream_t st) {
    auto kern = k_encode_tc<U, RAW>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, kSmemBytes, st>>>(mp, mx, a, H);
    e = cudaGetLastError();
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

}  // namespace

bool encode_tc_supported(const ephdc_ctx *c) { return c->p.F % 16 == 0 && encode_tiled_fn() != nullptr; }

cudaError_t launch_encode_tc(const ephdc_ctx *c, const void *d_X, const int8_t *d_P, uint32_t nq, void *d_H, bool raw,
                             cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    CUtensorMap mp, mx;
    if (!make_map(&mp, d_P, c->p.D_stored, c->p.F) || !make_map(&mx, d_X, nq, c->p.F)) return cudaErrorInvalidValue;
    EncTcArgs a;
    a.nq = nq;
    a.F = c->p.F;
    a.D_live = c->p.D_live;
    a.shift = c->p.qshift;
    a.qmax = (1 << (c->p.Qbits - 1)) - 1;
    const dim3 grid((nq + kTileN - 1) / kTileN, (c->p.D_live + kTileM - 1) / kTileM);
    if (c->p.feat_unsigned)
        return raw ? launch_tc<true, true>(mp, mx, a, d_H, grid, st) : launch_tc<true, false>(mp, mx, a, d_H, grid, st);
    return raw ? launch_tc<false, true>(mp, mx, a, d_H, grid, st) : launch_tc<false, false>(mp, mx, a, d_H, grid, st);
}

}  // namespace ephdc
