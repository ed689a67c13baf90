// tmem_x.cuh -- per-thread TMEM loads/stores of 4 / 8 / 16 / 32 columns (tcgen05 .32x32b).
//
// Thread l of warp w addresses lane 32*(w%4)+l of the allocation: TMEM is thread-private
// storage for values a thread reuses across many iterations (the c5 NTT keeps its
// pass-3 and last-stage twiddles there, one (w, w/q) pair = 4 columns).
#pragma once
#include <stdint.h>

#include "tmem.cuh"

namespace ephdc_tmem {

template <int X> EPHDC_D void ldx(uint32_t taddr, uint32_t (&r)[X]);
template <int X> EPHDC_D void stx(uint32_t taddr, const uint32_t (&r)[X]);
// wait for this thread's outstanding tcgen05.ld; r is valid afterwards
template <int X> EPHDC_D void waitx(uint32_t (&r)[X]);

#define EPHDC_R4(o) "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3])
#define EPHDC_W4(o) "r"(r[o + 0]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3])
#define EPHDC_P4(o) "+r"(r[o + 0]), "+r"(r[o + 1]), "+r"(r[o + 2]), "+r"(r[o + 3])

template <> EPHDC_D void ldx<4>(uint32_t t, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : EPHDC_R4(0) : "r"(t) : "memory");
}
template <> EPHDC_D void ldx<8>(uint32_t t, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : EPHDC_R4(0), EPHDC_R4(4)
                 : "r"(t)
                 : "memory");
}
template <> EPHDC_D void ldx<16>(uint32_t t, uint32_t (&r)[16]) { ld16(t, r); }
template <> EPHDC_D void ldx<32>(uint32_t t, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : EPHDC_R4(0), EPHDC_R4(4), EPHDC_R4(8), EPHDC_R4(12), EPHDC_R4(16), EPHDC_R4(20), EPHDC_R4(24), EPHDC_R4(28)
        : "r"(t)
        : "memory");
}
template <> EPHDC_D void stx<4>(uint32_t t, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(t), EPHDC_W4(0) : "memory");
}
template <> EPHDC_D void stx<16>(uint32_t t, const uint32_t (&r)[16]) { st16(t, r); }

template <> EPHDC_D void waitx<4>(uint32_t (&r)[4]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : EPHDC_P4(0)::"memory");
}
template <> EPHDC_D void waitx<8>(uint32_t (&r)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : EPHDC_P4(0), EPHDC_P4(4)::"memory");
}
template <> EPHDC_D void waitx<16>(uint32_t (&r)[16]) { wait_ld(r); }
template <> EPHDC_D void waitx<32>(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : EPHDC_P4(0), EPHDC_P4(4), EPHDC_P4(8), EPHDC_P4(12), EPHDC_P4(16), EPHDC_P4(20), EPHDC_P4(24),
                   EPHDC_P4(28)::"memory");
}

#undef EPHDC_R4
#undef EPHDC_W4
#undef EPHDC_P4

// (w, w/q) pair k of a register block loaded from TMEM (4 columns per pair)
template <int X> EPHDC_D double2 pair_at(const uint32_t (&r)[X], int k) {
    return make_double2(__hiloint2double(r[4 * k + 1], r[4 * k]), __hiloint2double(r[4 * k + 3], r[4 * k + 2]));
}
EPHDC_D void put_pair(uint32_t *r, double2 w) {
    r[0] = (uint32_t)__double2loint(w.x);
    r[1] = (uint32_t)__double2hiint(w.x);
    r[2] = (uint32_t)__double2loint(w.y);
    r[3] = (uint32_t)__double2hiint(w.y);
}

}  // namespace ephdc_tmem
