// densify.cuh -- decompression of k-sparse codes into 128B-swizzled K-major UMMA operand
// tiles in shared memory (steps 4 of DESIGN.md): the on-chip half of "a key arrives as its code".
#pragma once
#include <cstdint>

namespace sfa {
namespace dz {

// byte offset of feature f of row r inside a 128B-swizzled K-major tile with `rows` rows
__device__ __forceinline__ uint32_t swz_off(int r, int f, int rows) {
    return (uint32_t)((f >> 6) * rows * 128 + r * 128 + ((((f >> 3) & 7) ^ (r & 7)) << 4) + (f & 7) * 2);
}

__device__ __forceinline__ void sts_zero16(uint32_t addr) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0u) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((uint16_t)v) : "memory");
}

// the code row (idx, val) a later densify_row will read: into L1 ahead of time (issued one tile early,
// so the decompression after the ring slot frees does not wait on L2)
__device__ __forceinline__ void prefetch_code_row(const uint8_t *idx, const uint16_t *val) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(idx));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(val));
}

// zero row r of a swizzled tile (D features) then write its k code values
template <int D>
__device__ __forceinline__ void densify_row(uint32_t tile, int rows, int r, bool valid, const uint8_t *__restrict__ idx,
                                            const uint16_t *__restrict__ val, int k) {
    if (k == D && valid) {
        // k = d: every feature is selected and the indices are ascending (A4), so idx[t] = t and the
        // row IS the value vector -- 16-byte copies into the swizzled row, no zeroing, no scatter
        const uint4 *src = reinterpret_cast<const uint4 *>(val);
#pragma unroll
        for (int kb = 0; kb < D / 64; ++kb)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint4 w = __ldg(src + kb * 8 + c);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(tile + kb * rows * 128 + r * 128 +
                                                                                ((c ^ (r & 7)) << 4)),
                             "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                             : "memory");
            }
        return;
    }
#pragma unroll
    for (int kb = 0; kb < D / 64; ++kb)
#pragma unroll
        for (int c = 0; c < 8; ++c) sts_zero16(tile + kb * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4));
    if (!valid) return;
    if ((k & 7) == 0) {
        for (int c0 = 0; c0 < k; c0 += 8) {
            const uint2 ii = __ldg(reinterpret_cast<const uint2 *>(idx + c0));
            const uint4 vv = __ldg(reinterpret_cast<const uint4 *>(val + c0));
            const uint32_t iw[2] = {ii.x, ii.y};
            const uint32_t vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int f = (iw[e >> 2] >> (8 * (e & 3))) & 0xFF;
                sts_u16(tile + swz_off(r, f, rows), (vw[e >> 1] >> (16 * (e & 1))) & 0xFFFF);
            }
        }
    } else if ((k & 3) == 0) {
        for (int c0 = 0; c0 < k; c0 += 4) {
            const uint32_t ii = __ldg(reinterpret_cast<const uint32_t *>(idx + c0));
            const uint2 vv = __ldg(reinterpret_cast<const uint2 *>(val + c0));
            const uint32_t vw[2] = {vv.x, vv.y};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int f = (ii >> (8 * e)) & 0xFF;
                sts_u16(tile + swz_off(r, f, rows), (vw[e >> 1] >> (16 * (e & 1))) & 0xFFFF);
            }
        }
    } else {
        for (int c = 0; c < k; ++c) sts_u16(tile + swz_off(r, __ldg(idx + c), rows), __ldg(val + c));
    }
}

}  // namespace dz
}  // namespace sfa
