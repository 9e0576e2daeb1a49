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
    // the two exact integer halves summed, then converted on the FMA pipe (1.5 * 2^23 shifter) rather
    // than by an F2I on the XU pipe
    return __float_as_int(__uint_as_float(s << 16) + __uint_as_float(s & 0xFFFF0000u) + 12582912.f) - 0x4B400000;
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

// ---------------------------------------------------------------------------------------------
// Split row layout (the stand-alone kernel, topk.cu): word i = |x_i| | |x_{i+D/2}| << 16, i < D/2 = NW.
// The selection is the same function of the row as select_masks (the same T, the same lowest-index
// tie rule); only the register layout differs, so that the selection masks can be built with one
// compare and one LOP3 per word (a 0xFFFF-per-half compare result ANDed into bit j of both halves)
// and land in feature order with four byte permutes, no bit interleaving.

// gm[w] bit b = feature 32w + b has key >= T
template <int NW>
__device__ __forceinline__ void ge_masks_split(const uint32_t (&ab)[NW], uint32_t T, uint32_t (&gm)[NW / 16]) {
    constexpr int NG = NW / 16;  // groups of 16 words: lo halves = features [16g, 16g+16), hi = + NW
    const uint32_t t2 = T * 0x10001u;
    uint32_t W[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        W[g] = 0u;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t m;  // 0xFFFF per half with key >= T
            asm("set.ge.u32.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(ab[16 * g + j]), "r"(t2));
            W[g] |= m & (0x10001u << j);
        }
    }
#pragma unroll
    for (int w = 0; w < NG / 2; ++w) {
        gm[w] = __byte_perm(W[2 * w], W[2 * w + 1], 0x5410);           // features [32w, 32w+32)
        gm[w + NG / 2] = __byte_perm(W[2 * w], W[2 * w + 1], 0x7632);  // features NW + [32w, 32w+32)
    }
}

// T = the largest threshold with #{key >= T} >= k, cnt = #{key >= T}: the exponent first, walking down
// from the row max's, then the 7 mantissa bits by bisection, stopping once every lane of the warp has
// cnt == k (the set {key >= T} is then final: raising T further cannot change it).  (A byte-domain
// bisection counting with vabsdiff4, two instructions per four keys, measured slower: the count is
// bound by the ALU pipe, which vabsdiff4 shares with the compare it replaces; so did moving 3/8 of the
// compares to the FMA pipe as fma.sat.f16x2 on the keys read as f16 -- profiles/r02_topk.md.)
// Call with the whole warp converged.
template <int NW>
__device__ __forceinline__ uint32_t threshold_split(const uint32_t (&ab)[NW], int k, uint32_t mx, int &cnt) {
    int e = (int)((mx > 0x7FFFu ? 0x7FFFu : mx) >> 7);
#pragma unroll 1
    for (;;) {  // count_ge(0) = 2 NW >= k ends the walk at e = 0 at the latest
        cnt = count_ge(ab, (uint32_t)e << 7);
        if (cnt >= k || e == 0) break;
        --e;
    }
    uint32_t T = (uint32_t)e << 7;
#pragma unroll 1
    for (int bit = 6; bit >= 0; --bit) {
        if (__all_sync(0xffffffffu, cnt == k)) break;
        const uint32_t cand = T | (1u << bit);
        const int c = count_ge(ab, cand);
        if (c >= k) {
            T = cand;
            cnt = c;
        }
    }
    return T;
}

// Exact selection masks (every key > T, then the lowest-index keys == T, A2).
template <int NW>
__device__ __forceinline__ void select_masks_split(const uint32_t (&ab)[NW], int k, uint32_t (&gm)[NW / 16], uint32_t mx) {
    constexpr int NM = NW / 16;
    int cnt;
    const uint32_t T = threshold_split(ab, k, mx, cnt);
    ge_masks_split(ab, T, gm);
    if (cnt != k) {  // ties at T: keep key > T, add the lowest-index keys == T
        uint32_t em[NM];
        ge_masks_split(ab, T + 1u, em);  // T + 1 <= 0x7F80 (+inf) on finite rows
        int need = k;
#pragma unroll
        for (int w = 0; w < NM; ++w) {
            const uint32_t gt = em[w];
            em[w] = gm[w] & ~gt;  // key == T
            gm[w] = gt;
            need -= __popc(gt);
        }
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
}

}  // namespace tk
}  // namespace sfa
