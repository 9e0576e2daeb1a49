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
#include "topk_row.cuh"

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

// ---------------------------------------------------------------------------------------------
// bf16 rows: one THREAD per row (the warp-per-row kernel above issues ~500 warp instructions per
// row and is ALU-bound at ~9% of HBM bandwidth).  A CTA of 128 threads owns 128 consecutive rows:
//   1. coalesced 16-byte loads of the rows into shared memory, 16-byte chunks XOR-swizzled by
//      (row & 15) so each thread then reads its own row with conflict-free LDS.128;
//   2. the row as 64 (d=128) or 32 (d=64) registers of two |bf16| bit patterns each (sign cleared:
//      for finite non-negative bf16 the numeric order IS the order of the 15-bit keys);
//   3. the same bitwise binary search for the k-th largest key T (15 steps), counting on the FP16
//      pipe: set.ge.bf16x2 (1.0 per key >= T) + add.bf16x2 into four exact accumulators, 2
//      instructions per 2 keys (the integer subtract/popc version kept the ALU pipe at 82 %);
//   4. selection bit masks (set.ge against T + 1, set.eq against T), ties == T taken lowest index
//      first (A2), then the set bits walked in ascending feature order (A4) with the values
//      re-read from the row in shared memory; staged and written out with coalesced stores.
// Non-finite inputs: max key (max.u16x2) >= 0x7F80.
constexpr int TK_ROWS = 128;

// One tensor's rows for the row-per-thread kernel.  A launch covers one or two of them (Q and K of
// the same step in ONE grid: blocks [0, nb0) take segment 0, the rest segment 1), which saves a
// launch and its tail on small problems (GPT-2 shape: ~16 us per top-k launch).
struct TkSeg {
    const uint16_t *x;
    int64_t rows, ld;
    uint8_t *idx;
    uint16_t *val;
};
struct TkSegs {
    TkSeg s[2];
    int64_t nb0;  // blocks of segment 0
};

template <int D>
__global__ void __launch_bounds__(TK_ROWS) topk_rows_bf16_kernel(const __grid_constant__ TkSegs segs, int k,
                                                                 uint32_t *status_word) {
    constexpr int NW = D / 2;     // u32 words per row
    constexpr int NC = D / 8;     // 16-byte chunks per row
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t *rowbuf = sm;                                   // [TK_ROWS][D*2] swizzled
    uint8_t *oidx = sm + TK_ROWS * D * 2;                   // [TK_ROWS][k]
    uint16_t *oval = reinterpret_cast<uint16_t *>(oidx + ((TK_ROWS * k + 15) & ~15));  // [TK_ROWS][k]
    const int t = threadIdx.x;
    const bool second = (int64_t)blockIdx.x >= segs.nb0;
    const TkSeg &sg = second ? segs.s[1] : segs.s[0];
    const uint16_t *__restrict__ x = sg.x;
    const int64_t rows = sg.rows, ld = sg.ld;
    uint8_t *__restrict__ idx = sg.idx;
    uint16_t *__restrict__ val = sg.val;
    const int64_t row0 = ((int64_t)blockIdx.x - (second ? segs.nb0 : 0)) * TK_ROWS;
    const int nrows = (int)((rows - row0) < TK_ROWS ? (rows - row0) : TK_ROWS);

    // 1. coalesced loads (16 B per thread per step), swizzled stores
    for (int v = t; v < nrows * NC; v += TK_ROWS) {
        const int r = v / NC, c = v % NC;
        const uint4 w = __ldcs(reinterpret_cast<const uint4 *>(x + (row0 + r) * ld) + c);
        *reinterpret_cast<uint4 *>(rowbuf + r * D * 2 + ((c ^ (r & 15) & (NC - 1)) << 4)) = w;
    }
    __syncthreads();

    const bool active = t < nrows;
    uint32_t ab[NW];  // |x| bit patterns, two keys per word
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const uint4 w = *reinterpret_cast<const uint4 *>(rowbuf + t * D * 2 + ((c ^ (t & 15) & (NC - 1)) << 4));
        ab[4 * c + 0] = w.x & 0x7FFF7FFFu;
        ab[4 * c + 1] = w.y & 0x7FFF7FFFu;
        ab[4 * c + 2] = w.z & 0x7FFF7FFFu;
        ab[4 * c + 3] = w.w & 0x7FFF7FFFu;
    }
    const uint32_t mx = tk::row_max_key(ab);
    if (active && mx >= 0x7F80u && status_word != nullptr) atomicOr(status_word, 1u);
    // 3-4. threshold search and selection masks (topk_row.cuh)
    constexpr int NM = D / 32;
    uint32_t gm[NM];
    tk::select_masks(ab, k, gm, mx);
    // 5. ascending compaction into the staging area (values re-read from the row in shared memory)
    uint8_t *my_i = oidx + t * k;
    uint16_t *my_v = oval + t * k;
    int pos = 0;
#pragma unroll
    for (int w = 0; w < NM; ++w) {
        uint32_t m = active ? gm[w] : 0u;
        while (m != 0u) {
            const int f = 32 * w + (__ffs(m) - 1);
            m &= m - 1u;
            const int c = f >> 3;
            my_i[pos] = (uint8_t)f;
            my_v[pos] = *reinterpret_cast<const uint16_t *>(rowbuf + t * D * 2 + ((c ^ (t & 15) & (NC - 1)) << 4) + (f & 7) * 2);
            ++pos;
        }
    }
    __syncthreads();
    // coalesced copy-out of the CTA's contiguous [nrows][k] index and value blocks
    const int nib = nrows * k;
    uint8_t *gi = idx + row0 * k;
    uint16_t *gv = val + row0 * k;
    if ((k & 15) == 0) {
        for (int v = t; v < nib / 16; v += TK_ROWS)
            reinterpret_cast<uint4 *>(gi)[v] = reinterpret_cast<const uint4 *>(oidx)[v];
    } else {
        for (int v = t; v < nib; v += TK_ROWS) gi[v] = oidx[v];
    }
    if ((k & 7) == 0) {
        for (int v = t; v < nib / 8; v += TK_ROWS)
            reinterpret_cast<uint4 *>(gv)[v] = reinterpret_cast<const uint4 *>(oval)[v];
    } else {
        for (int v = t; v < nib; v += TK_ROWS) gv[v] = oval[v];
    }
}

// 16-byte row loads and stores of the row-per-thread kernel: aligned rows and outputs
bool rows_kernel_ok(const void *x, int64_t ld, const void *idx, const void *val) {
    return (ld * 2) % 16 == 0 && ((uintptr_t)x & 15u) == 0 && ((uintptr_t)idx & 15u) == 0 && ((uintptr_t)val & 15u) == 0;
}

cudaError_t launch_rows(const TkSegs &sg, int64_t blocks, int d, int k, uint32_t *status_word, cudaStream_t stream) {
    if (blocks > 0x7FFFFFFF) return cudaErrorInvalidValue;
    const size_t smem = (size_t)TK_ROWS * d * 2 + ((TK_ROWS * k + 15) & ~15) + (size_t)TK_ROWS * k * 2;
    auto kern = d == 64 ? topk_rows_bf16_kernel<64> : topk_rows_bf16_kernel<128>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)blocks, TK_ROWS, smem, stream>>>(sg, k, status_word);
    return cudaGetLastError();
}

// host launcher (called from api.cu after validation)
// k = d: Topk_k is the identity (every entry selected, indices ascending): idx[r][t] = t, val = x bit
// copy, non-finite entries still flagged (A14).  One thread per element, HBM-bound.
template <typename T>
__global__ void __launch_bounds__(256) topk_identity_kernel(const T *__restrict__ x, int64_t rows, int d, int64_t ld,
                                                            uint8_t *__restrict__ idx, T *__restrict__ val,
                                                            uint32_t *status_word) {
    const int64_t n = rows * d;
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / d;
        const int c = (int)(e % d);
        const T v = x[r * ld + c];
        val[e] = v;
        idx[e] = (uint8_t)c;
        const uint32_t mag = sizeof(T) == 2 ? ((uint32_t)v & 0x7FFFu) : ((uint32_t)v & 0x7FFFFFFFu);
        bad |= sizeof(T) == 2 ? (mag >= 0x7F80u) : (mag >= 0x7F800000u);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && status_word != nullptr) atomicOr(status_word, 1u);
}

cudaError_t launch_topk(const void *x, bool bf16, int64_t rows, int d, int64_t ld, int k, uint8_t *idx, void *val,
                        uint32_t *status_word, cudaStream_t stream) {
    if (rows == 0) return cudaSuccess;
    if (k == d) {
        const int64_t n = rows * d;
        const unsigned g = (unsigned)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
        if (bf16)
            topk_identity_kernel<uint16_t><<<g, 256, 0, stream>>>((const uint16_t *)x, rows, d, ld, idx, (uint16_t *)val,
                                                                  status_word);
        else
            topk_identity_kernel<uint32_t><<<g, 256, 0, stream>>>((const uint32_t *)x, rows, d, ld, idx, (uint32_t *)val,
                                                                  status_word);
        return cudaGetLastError();
    }
    int sms = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (rows + 7) / 8;
    const int grid = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
    if (bf16) {
        // row-per-thread kernel; 16-byte row loads need ld*2 % 16 == 0 (else the warp-per-row kernel)
        if (rows_kernel_ok(x, ld, idx, val)) {
            TkSegs sg;
            sg.s[0] = {(const uint16_t *)x, rows, ld, idx, (uint16_t *)val};
            sg.s[1] = sg.s[0];
            sg.nb0 = (rows + TK_ROWS - 1) / TK_ROWS;
            return launch_rows(sg, sg.nb0, d, k, status_word, stream);
        } else if (d == 64)
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

// Q and K codes of one step in one launch (bf16, d in {64, 128}, 1 <= k < d, both row-kernel aligned);
// otherwise two launch_topk calls
cudaError_t launch_topk_pair(const void *x0, int64_t rows0, int64_t ld0, uint8_t *idx0, void *val0, const void *x1,
                             int64_t rows1, int64_t ld1, uint8_t *idx1, void *val1, int d, int k,
                             uint32_t *status_word, cudaStream_t stream) {
    if (k < d && rows0 > 0 && rows1 > 0 && rows_kernel_ok(x0, ld0, idx0, val0) && rows_kernel_ok(x1, ld1, idx1, val1)) {
        TkSegs sg;
        sg.s[0] = {(const uint16_t *)x0, rows0, ld0, idx0, (uint16_t *)val0};
        sg.s[1] = {(const uint16_t *)x1, rows1, ld1, idx1, (uint16_t *)val1};
        sg.nb0 = (rows0 + TK_ROWS - 1) / TK_ROWS;
        return launch_rows(sg, sg.nb0 + (rows1 + TK_ROWS - 1) / TK_ROWS, d, k, status_word, stream);
    }
    cudaError_t e = launch_topk(x0, true, rows0, d, ld0, k, idx0, val0, status_word, stream);
    if (e != cudaSuccess) return e;
    return launch_topk(x1, true, rows1, d, ld1, k, idx1, val1, status_word, stream);
}

}  // namespace sfa
