// common.cuh -- shared device helpers and the key-tile bucket layout of the CUDA path.
//
// Key-tile bucketing (our form of the paper's CSC_feat,
// P:L786-795, which replaces the per-tile BinarySearchRange of Alg. 1 L723 / P:L757-758):
// for every (batch b, kv head g, key tile t of BK keys) the workspace holds
//     off[d+1]  uint16   bucket f spans entries [off[f], off[f+1]) ; every bucket is padded
//                        to a multiple of 4 entries so it can be read with 16-byte loads
//     ent[cap]  entries  bf16 path: uint32 = (bf16 bits of k~_jf) << 16 | j_local * SLAB_ROW_BYTES
//                        f32 path : uint2  = { j_local * SLAB_ROW_BYTES, fp32 bits of k~_jf }
// The pad entries point at the trash row j_local = BK with value +0.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sfa {

// bytes between consecutive key rows of a per-warp score slab S_w[j][lane] (fp32, bank = lane)
constexpr int SLAB_ROW_BYTES = 32 * 4;

struct BucketLayout {
    int32_t bk;          // keys per tile
    int32_t ntiles;      // ceil(n_kv / bk)
    int32_t off_bytes;   // align16((d+1)*2)
    int32_t cap;         // max entries per tile, multiple of 4: bk*k + 3*d rounded up
    int32_t ent_bytes;   // 4 (bf16) or 8 (f32)
    int64_t tile_bytes;  // align16(off_bytes + cap*ent_bytes)
};

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

inline BucketLayout make_layout(int d, int k, int64_t n_kv, int bk, bool bf16) {
    BucketLayout L;
    L.bk = bk;
    L.ntiles = (int32_t)((n_kv + bk - 1) / bk);
    L.off_bytes = (int32_t)align_up((d + 1) * 2, 16);
    L.cap = (int32_t)align_up((int64_t)bk * k + 3 * d, 4);
    L.ent_bytes = bf16 ? 4 : 8;
    L.tile_bytes = align_up(L.off_bytes + (int64_t)L.cap * L.ent_bytes, 16);
    return L;
}

// ---- scalar helpers -------------------------------------------------------------------------
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t b16) { return __uint_as_float(b16 << 16); }

__device__ __forceinline__ uint16_t f32_to_bf16_bits_rn(float x) {
    __nv_bfloat16 h = __float2bfloat16_rn(x);
    return *reinterpret_cast<uint16_t *>(&h);
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
struct DT;
template <>
struct DT<float> {
    static constexpr bool is_bf16 = false;
    __device__ static float to_f(float x) { return x; }
};
template <>
struct DT<__nv_bfloat16> {
    static constexpr bool is_bf16 = true;
    __device__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
};

}  // namespace sfa
