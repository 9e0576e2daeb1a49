// topk_row.cuh -- Top-k selection of ONE bf16 row held by one thread (steps 1-2), shared by
// the stand-alone top-k kernel (topk.cu) and the fused-Q attention prologue (attn_sm100_ot.cu), so
// both produce the same support bit for bit.
//
// Input: the row as NW = d/2 words of two |x| bit patterns (sign cleared; for finite non-negative bf16
// the numeric order IS the order of the 15-bit keys).  Output: gm[d/32] selection masks, bit f =
// feature f selected: every key > T and the lowest-index keys == T (A2), where T is the largest
// threshold with #{key >= T} >= k, found by a 15-step bitwise binary search counting on the FP16
// pipe (set.ge.bf16x2 gives 1.0 per key >= T; four bf16x2 accumulators count exactly).
#pragma once
#include <cstdint>

namespace sfa {
namespace tk {

template <int NW>
__device__ __forceinline__ int count_ge(const uint32_t (&ab)[NW], uint32_t T) {
    const uint32_t t2 = T * 0x10001u;
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        uint32_t m;
        asm("set.ge.bf16x2.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(ab[i]), "r"(t2));
        asm("add.rn.bf16x2 %0, %0, %1;" : "+r"(acc[i & 3]) : "r"(m));
    }
    uint32_t s01, s23, s;
    asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(s01) : "r"(acc[0]), "r"(acc[1]));
    asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(s23) : "r"(acc[2]), "r"(acc[3]));
    asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(s) : "r"(s01), "r"(s23));  // <= 64 per half: exact
    return (int)(__uint_as_float(s << 16) + __uint_as_float(s & 0xFFFF0000u));
}

// max key of the row (>= 0x7F80: a non-finite entry, A14)
template <int NW>
__device__ __forceinline__ uint32_t row_max_key(const uint32_t (&ab)[NW]) {
    uint32_t mx2 = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        uint32_t m;
        asm("max.u16x2 %0, %1, %2;" : "=r"(m) : "r"(mx2), "r"(ab[i]));
        mx2 = m;
    }
    return max(mx2 & 0xFFFFu, mx2 >> 16);
}

// mx: the row's max key (row_max_key).  T is found exponent first: walking down from the max key's
// exponent, the first exponent e with #{key >= e.2^7} >= k is T's (the count is monotone in the
// threshold), typically one or two passes since the top k of a row sit within a binade or two of its
// max; then the 7 mantissa bits by bisection -- ~9 counting passes instead of 15.
template <int NW>
__device__ __forceinline__ void select_masks(const uint32_t (&ab)[NW], int k, uint32_t (&gm)[NW / 16], uint32_t mx) {
    constexpr int NM = NW / 16;
    // largest T with #{key >= T} >= k
    int e = (int)((mx > 0x7FFFu ? 0x7FFFu : mx) >> 7);
#pragma unroll 1
    while (e > 0 && count_ge(ab, (uint32_t)e << 7) < k) --e;
    uint32_t T = (uint32_t)e << 7;
#pragma unroll 1
    for (int bit = 6; bit >= 0; --bit) {
        const uint32_t cand = T | (1u << bit);
        if (count_ge(ab, cand) >= k) T = cand;
    }
    // key > T always, key == T for the lowest-index ties
    uint32_t em[NM];
#pragma unroll
    for (int w = 0; w < NM; ++w) gm[w] = em[w] = 0u;
    const uint32_t tg = (T + 1u) * 0x10001u, te = T * 0x10001u;  // T + 1 <= 0x7F80 (+inf) on finite rows
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        uint32_t g, e;  // bf16 1.0 (0x3F80, bit 7 set) per true half
        asm("set.ge.bf16x2.bf16x2 %0, %1, %2;" : "=r"(g) : "r"(ab[i]), "r"(tg));
        asm("set.eq.bf16x2.bf16x2 %0, %1, %2;" : "=r"(e) : "r"(ab[i]), "r"(te));
        gm[i >> 4] |= (((g >> 7) & 1u) | ((g >> 22) & 2u)) << (2 * (i & 15));
        em[i >> 4] |= (((e >> 7) & 1u) | ((e >> 22) & 2u)) << (2 * (i & 15));
    }
    int need = k;
#pragma unroll
    for (int w = 0; w < NM; ++w) need -= __popc(gm[w]);
#ifndef SFA_FAULT_TOPK_TIE_HIGH
#pragma unroll
    for (int w = 0; w < NM; ++w)
        while (need > 0 && em[w] != 0u) {  // lowest-index ties first (A2)
            gm[w] |= em[w] & (0u - em[w]);
            em[w] &= em[w] - 1u;
            --need;
        }
#else  // negative control (tools/gpu_mutants.sh): ties taken from the highest index
#pragma unroll
    for (int w = NM - 1; w >= 0; --w)
        while (need > 0 && em[w] != 0u) {
            const uint32_t hb = 0x80000000u >> __clz(em[w]);
            gm[w] |= hb;
            em[w] &= ~hb;
            --need;
        }
#endif
}

}  // namespace tk
}  // namespace sfa
