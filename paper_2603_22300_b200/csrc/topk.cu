// topk.cu -- stage 1: row-wise Top-k coding (Sec. 3.1 Eq. topk_QK).
//
// One warp per row of d values (d = 32*E, E = 2 or 4 values per lane, one 4..16-byte load
// per lane, the warp reading the row as one contiguous coalesced segment).  Selection is a
// bitwise binary search for the k-th largest magnitude key (the IEEE bits with the sign
// cleared: monotone in |x| for finite x, exact for denormals and +-0, A21), counting with
// redux.sync; entries strictly above the threshold are taken, and entries equal to it are
// taken lowest index first (A2) using a ballot-sliced exclusive prefix over lanes.  Output
// is in ascending feature order (A4), values are bit copies (A7).  HBM-bound.
#include "launch.cuh"

namespace sfa {

template <typename Bits, int E>
struct RowVec;
template <>
struct RowVec<uint16_t, 2> {
    using V = uint32_t;
    __device__ static void split(V v, uint32_t (&b)[2]) { b[0] = v & 0xFFFFu; b[1] = v >> 16; }
};
template <>
struct RowVec<uint16_t, 4> {
    using V = uint2;
    __device__ static void split(V v, uint32_t (&b)[4]) {
        b[0] = v.x & 0xFFFFu; b[1] = v.x >> 16; b[2] = v.y & 0xFFFFu; b[3] = v.y >> 16;
    }
};
template <>
struct RowVec<uint32_t, 2> {
    using V = uint2;
    __device__ static void split(V v, uint32_t (&b)[2]) { b[0] = v.x; b[1] = v.y; }
};
template <>
struct RowVec<uint32_t, 4> {
    using V = uint4;
    __device__ static void split(V v, uint32_t (&b)[4]) { b[0] = v.x; b[1] = v.y; b[2] = v.z; b[3] = v.w; }
};

// exclusive prefix over lanes of a small per-lane count c < 8
__device__ __forceinline__ int lane_exclusive_prefix(int c) {
    const uint32_t lt = lanemask_lt();
    return __popc(__ballot_sync(0xffffffffu, c & 1) & lt) + 2 * __popc(__ballot_sync(0xffffffffu, c & 2) & lt) +
           4 * __popc(__ballot_sync(0xffffffffu, c & 4) & lt);
}

template <typename Bits, int D>
__global__ void __launch_bounds__(256) topk_codes_kernel(const Bits *__restrict__ x, int64_t rows, int64_t ld, int k,
                                                         uint8_t *__restrict__ idx, Bits *__restrict__ val,
                                                         uint32_t *status_word) {
    constexpr int E = D / 32;
    constexpr bool kBF16 = sizeof(Bits) == 2;
    constexpr int NBITS = kBF16 ? 15 : 31;
    constexpr uint32_t ABS = kBF16 ? 0x7FFFu : 0x7FFFFFFFu;
    constexpr uint32_t EXP = kBF16 ? 0x7F80u : 0x7F800000u;
    using RV = RowVec<Bits, E>;
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    bool bad = false;
    for (int64_t r = warp0; r < rows; r += nwarps) {
        const typename RV::V raw = __ldcs(reinterpret_cast<const typename RV::V *>(x + r * ld) + lane);
        uint32_t b[E], key[E];
        RV::split(raw, b);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            key[e] = b[e] & ABS;
            bad |= (b[e] & EXP) == EXP;
        }
        // largest T with #{key >= T} >= k: the k-th largest magnitude
        uint32_t T = 0;
#pragma unroll 4
        for (int bit = NBITS - 1; bit >= 0; --bit) {
            const uint32_t cand = T | (1u << bit);
            int c = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) c += key[e] >= cand;
            if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) >= k) T = cand;
        }
        int gt = 0, eq = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            gt += key[e] > T;
            eq += key[e] == T;
        }
        const int need = k - (int)__reduce_add_sync(0xffffffffu, (unsigned)gt);  // >= 1 ties to take
        int eq_seen = lane_exclusive_prefix(eq);
        bool sel[E];
        int nsel = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const bool tie = key[e] == T;
            sel[e] = key[e] > T || (tie && eq_seen < need);
            eq_seen += tie;
            nsel += sel[e];
        }
        int pos = lane_exclusive_prefix(nsel);
        uint8_t *ir = idx + r * k;
        Bits *vr = val + r * k;
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (sel[e]) {
                ir[pos] = (uint8_t)(lane * E + e);
                vr[pos] = (Bits)b[e];
                ++pos;
            }
    }
    if (status_word != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status_word, 1u);
}

// host launcher (called from api.cu after validation)
cudaError_t launch_topk(const void *x, bool bf16, int64_t rows, int d, int64_t ld, int k, uint8_t *idx, void *val,
                        uint32_t *status_word, cudaStream_t stream) {
    if (rows == 0) return cudaSuccess;
    int sms = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (rows + 7) / 8;
    const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
    if (bf16) {
        if (d == 64)
            topk_codes_kernel<uint16_t, 64><<<grid, 256, 0, stream>>>((const uint16_t *)x, rows, ld, k, idx,
                                                                     (uint16_t *)val, status_word);
        else
            topk_codes_kernel<uint16_t, 128><<<grid, 256, 0, stream>>>((const uint16_t *)x, rows, ld, k, idx,
                                                                      (uint16_t *)val, status_word);
    } else {
        if (d == 64)
            topk_codes_kernel<uint32_t, 64><<<grid, 256, 0, stream>>>((const uint32_t *)x, rows, ld, k, idx,
                                                                     (uint32_t *)val, status_word);
        else
            topk_codes_kernel<uint32_t, 128><<<grid, 256, 0, stream>>>((const uint32_t *)x, rows, ld, k, idx,
                                                                      (uint32_t *)val, status_word);
    }
    return cudaGetLastError();
}

}  // namespace sfa
