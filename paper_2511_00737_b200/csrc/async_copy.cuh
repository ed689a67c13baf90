// async_copy.cuh -- one-thread bulk (TMA 1-D) copies global -> shared with an mbarrier.
#pragma once
#include <stdint.h>

#ifndef EPHDC_D
#define EPHDC_D __device__ __forceinline__
#endif

namespace ephdc_async {

EPHDC_D uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

EPHDC_D void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// The calling thread arrives and announces `bytes` of transactions for this phase.
EPHDC_D void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

EPHDC_D void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Orders this thread's earlier generic-proxy shared-memory accesses (made visible to it
// by a preceding barrier) before subsequent async-proxy (bulk copy) writes.
EPHDC_D void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// bytes: multiple of 16, src/dst 16-byte aligned; completion counted on *bar.
EPHDC_D void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace ephdc_async
