// gen.cu -- device side of the seeded input generator (include/sfa_gen.h); no method arithmetic.
#include "../../include/sfa_gen.h"
#include "common.cuh"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t hash3(uint64_t seed, int tid, uint64_t i) {
    return splitmix64((seed * 0x100000001B3ull) ^ ((uint64_t)(tid & 0xFF) << 56) ^ i);
}

__device__ __forceinline__ float irwin_hall(uint64_t h) {
    const int64_t z = (int64_t)((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + (h >> 48)) - 131070;
    return (float)z * 3.0517578125e-05f;  // 2^-15, exact
}

__global__ void gen_kernel(void *out, int bf16, int64_t count, int64_t offset, uint64_t seed, int tid, int variant,
                           int64_t n, int d, int span) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)(offset + t);
        const uint64_t h = hash3(seed, tid, i);
        float x;
        if (variant == 1) {
            x = (float)((int)(h % 9ull) - 4);
        } else {
            x = irwin_hall(h);
            if (variant == 2) {
                const uint64_t feat = i % (uint64_t)d, head = i / ((uint64_t)d * (uint64_t)n);
                const uint64_t g = hash3(seed, 8 + tid, head * (uint64_t)d + feat);
                const int e = (int)(g % (uint64_t)(2 * span + 1)) - span;
                x = ldexpf(x, e);  // exact power-of-two gain
            }
        }
        if (bf16)
            reinterpret_cast<uint16_t *>(out)[t] = sfa::f32_to_bf16_bits_rn(x);
        else
            reinterpret_cast<float *>(out)[t] = x;
    }
}

}  // namespace

extern "C" sfa_status sfa_gen_fill(void *out, sfa_dtype dtype, int64_t count, int64_t offset, uint64_t seed,
                                   int32_t tensor_id, int32_t variant, int64_t n, int32_t d, int32_t skew_span,
                                   sfa_stream_t stream) {
    if (count < 0 || offset < 0 || (dtype != SFA_F32 && dtype != SFA_BF16) || variant < 0 || variant > 2)
        return SFA_ERR_INVALID_ARGUMENT;
    if (variant == 2 && (n < 1 || d < 1 || skew_span < 0)) return SFA_ERR_INVALID_ARGUMENT;
    if (count == 0) return SFA_OK;
    if (!out) return SFA_ERR_INVALID_ARGUMENT;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, dtype == SFA_BF16, count, offset, seed,
                                                                   tensor_id, variant, n, d, skew_span);
    return cudaGetLastError() == cudaSuccess ? SFA_OK : SFA_ERR_CUDA;
}
