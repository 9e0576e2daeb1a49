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
// row and is ALU-bound at ~9% of HBM bandwidth).  A CTA of 128 threads owns blocks of 128
// consecutive rows; the grid is persistent (a few CTAs per SM, each walking blocks with a stride of
// the grid) and double-buffered:
//   1. the NEXT block's rows stream into the second shared-memory buffer with cp.async (16 bytes per
//      thread per step, coalesced), 16-byte chunks XOR-swizzled by (row & 15) so each thread then
//      reads its own row with conflict-free LDS.128, while the current block is selected;
//   2. the row as D/2 registers in the split layout of topk_row.cuh (word i = |x_i|, |x_{i+D/2}|,
//      sign cleared: for finite non-negative bf16 the numeric order IS the order of the 15-bit keys);
//   3. the k-th largest key T: exponent first from the row max, then the mantissa bits, counting on
//      the FP16 pipe (set.ge.bf16x2 + add.bf16x2, 2 instructions per 2 keys), stopping once every
//      row of the warp counts exactly k keys >= T;
//   4. selection bit masks (one set.ge.u32.bf16x2 + one LOP3 per 2 keys), ties == T taken lowest
//      index first (A2) on the rare rows that have them, then the set bits walked in ascending
//      feature order (A4) with the values re-read from the row in shared memory; staged and written
//      out with coalesced stores.
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
    int64_t nb;   // blocks of both segments
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

// KC = k when k is 8 or 16 (compile time: the row's code is assembled in registers and stored with
// 16-byte stores straight to global, coalesced across the warp's consecutive rows), else 0 (runtime k:
// staged in shared memory and copied out per block)
template <int D, int KC>
__global__ void __launch_bounds__(TK_ROWS, 3) topk_rows_bf16_kernel(const __grid_constant__ TkSegs segs, int k,
                                                                    uint32_t *status_word) {
    constexpr int NW = D / 2;            // u32 words per row
    constexpr int NC = D / 8;            // 16-byte chunks per row
    constexpr int NM = D / 32;           // selection mask words
    constexpr int RB = TK_ROWS * D * 2;  // bytes of one row buffer
    constexpr int RPI = TK_ROWS / NC;    // rows per cp.async step of the CTA
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t *oidx = sm + 2 * RB;                                                       // KC = 0: [TK_ROWS][k]
    uint16_t *oval = reinterpret_cast<uint16_t *>(oidx + ((TK_ROWS * k + 15) & ~15));  // KC = 0: [TK_ROWS][k]
    const int t = threadIdx.x;
    const int cc = t % NC, r0 = t / NC;  // this thread's 16-byte chunk column and first row of every copy

    // block b -> (segment, first row, rows in it)
    auto locate = [&](int64_t b, int64_t &row0, int &nrows) -> const TkSeg & {
        const bool second = b >= segs.nb0;
        const TkSeg &sg = second ? segs.s[1] : segs.s[0];
        row0 = (b - (second ? segs.nb0 : 0)) * TK_ROWS;
        nrows = (int)((sg.rows - row0) < TK_ROWS ? (sg.rows - row0) : TK_ROWS);
        return sg;
    };
    auto issue = [&](int64_t b, int buf) {
        int64_t row0;
        int nrows;
        const TkSeg &sg = locate(b, row0, nrows);
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm + buf * RB) + (uint32_t)r0 * (D * 2);
        const char *src = reinterpret_cast<const char *>(sg.x + (row0 + r0) * sg.ld + cc * 8);
        const int64_t step = (int64_t)RPI * sg.ld * 2;  // bytes between this thread's consecutive rows
#pragma unroll
        for (int i = 0; i < NC; ++i, src += step) {
            const int r = r0 + i * RPI;
            if (r < nrows)
                cp_async16(base + (uint32_t)(i * RPI * D * 2) + ((uint32_t)(cc ^ (r & 15) & (NC - 1)) << 4), src);
        }
    };

    int64_t b = blockIdx.x;
    if (b < segs.nb) issue(b, 0);
    cp_async_commit();
    for (int buf = 0; b < segs.nb; b += gridDim.x, buf ^= 1) {
        if (b + gridDim.x < segs.nb) issue(b + gridDim.x, buf ^ 1);
        cp_async_commit();
        cp_async_wait1();  // this block's group has landed (the next one may still be in flight)
        __syncthreads();
        const uint8_t *rowbuf = sm + buf * RB;
        const uint32_t myrow = (uint32_t)__cvta_generic_to_shared(rowbuf) + (uint32_t)t * (D * 2);
        int64_t row0;
        int nrows;
        const TkSeg &sg = locate(b, row0, nrows);
        const bool active = t < nrows;

        uint32_t ab[NW];  // split layout: word i = |x_i| | |x_{i+NW}| << 16
#pragma unroll
        for (int c = 0; c < NC / 2; ++c) {
            const uint4 X = *reinterpret_cast<const uint4 *>(rowbuf + t * D * 2 + ((c ^ (t & 15) & (NC - 1)) << 4));
            const uint4 Y =
                *reinterpret_cast<const uint4 *>(rowbuf + t * D * 2 + (((c + NC / 2) ^ (t & 15) & (NC - 1)) << 4));
            const uint32_t xs[4] = {X.x, X.y, X.z, X.w}, ys[4] = {Y.x, Y.y, Y.z, Y.w};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                ab[8 * c + 2 * m] = __byte_perm(xs[m], ys[m], 0x5410) & 0x7FFF7FFFu;
                ab[8 * c + 2 * m + 1] = __byte_perm(xs[m], ys[m], 0x7632) & 0x7FFF7FFFu;
            }
        }
        uint32_t mx = tk::row_max_key(ab);
        if (mx >= 0x7F80u) {  // non-finite row (A14): flagged; NaN keys clamped to +inf so that every count
            // below (bf16 compares and byte arithmetic alike) sees the same numbers and the walk terminates
            if (active && status_word != nullptr) atomicOr(status_word, 1u);
#pragma unroll
            for (int i = 0; i < NW; ++i) asm("min.u16x2 %0, %0, %1;" : "+r"(ab[i]) : "r"(0x7F807F80u));
            mx = 0x7F80u;
        }
        auto val_addr = [&](int f) { return myrow + ((uint32_t)((f >> 3) ^ (t & 15) & (NC - 1)) << 4) + (uint32_t)(f & 7) * 2; };
        if constexpr (KC > 0) {
            // exactly KC bits are set over q[]: walk them in ascending order through a queue of the mask
            // words (an empty word is shifted out, at most NM - 1 times per row)
            uint32_t q[NM];
            tk::select_masks_split(ab, KC, q, mx);
            if (!active) {  // a ragged block's idle rows: any KC bits, nothing stored
                q[0] = (KC >= 32) ? 0xFFFFFFFFu : ((1u << KC) - 1u);
#pragma unroll
                for (int w = 1; w < NM; ++w) q[w] = 0u;
            }
            int base = 0;
            uint32_t iw[KC / 4], vw[KC / 2];  // the row's code: KC index bytes, KC bf16 values
#pragma unroll
            for (int i = 0; i < KC / 4; ++i) iw[i] = 0u;
#pragma unroll
            for (int i = 0; i < KC / 2; ++i) vw[i] = 0u;
#pragma unroll
            for (int pos = 0; pos < KC; ++pos) {
                while (q[0] == 0u && base < D) {
#pragma unroll
                    for (int w = 0; w + 1 < NM; ++w) q[w] = q[w + 1];
                    q[NM - 1] = 0u;
                    base += 32;
                }
                const int f = q[0] != 0u ? base + __ffs(q[0]) - 1 : 0;  // (never 0 bits: never spin)
                q[0] &= q[0] - 1u;
                iw[pos >> 2] |= (uint32_t)f << (8 * (pos & 3));
                vw[pos >> 1] |= lds_u16(val_addr(f)) << (16 * (pos & 1));
            }
            if (active) {
                const int64_t row = row0 + t;
                if constexpr (KC == 16) {
                    reinterpret_cast<uint4 *>(sg.idx)[row] = make_uint4(iw[0], iw[1], iw[2], iw[3]);
                    uint4 *vr = reinterpret_cast<uint4 *>(sg.val) + 2 * row;
                    vr[0] = make_uint4(vw[0], vw[1], vw[2], vw[3]);
                    vr[1] = make_uint4(vw[4], vw[5], vw[6], vw[7]);
                } else {  // KC == 8
                    reinterpret_cast<uint2 *>(sg.idx)[row] = make_uint2(iw[0], iw[1]);
                    reinterpret_cast<uint4 *>(sg.val)[row] = make_uint4(vw[0], vw[1], vw[2], vw[3]);
                }
            }
            // every thread's reads of this row buffer precede the next iteration's cp.async into it
            __syncthreads();
        } else {
            uint32_t gm[NM];
            tk::select_masks_split(ab, k, gm, mx);
            // ascending compaction into the staging area (values re-read from the row in shared memory)
            uint8_t *my_i = oidx + t * k;
            uint16_t *my_v = oval + t * k;
            int pos = 0;
#pragma unroll
            for (int w = 0; w < NM; ++w) {
                uint32_t m = active ? gm[w] : 0u;
                while (m != 0u) {
                    const int f = 32 * w + (__ffs(m) - 1);
                    m &= m - 1u;
                    my_i[pos] = (uint8_t)f;
                    my_v[pos] = (uint16_t)lds_u16(val_addr(f));
                    ++pos;
                }
            }
            __syncthreads();  // staging complete
            // coalesced copy-out of the block's contiguous [nrows][k] index and value blocks
            const int nib = nrows * k;
            uint8_t *gi = sg.idx + row0 * k;
            uint16_t *gv = sg.val + row0 * k;
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
            // the next iteration's __syncthreads orders these staging reads before the next writes
        }
    }
}

// 16-byte row loads and stores of the row-per-thread kernel: aligned rows and outputs
bool rows_kernel_ok(const void *x, int64_t ld, const void *idx, const void *val) {
    return (ld * 2) % 16 == 0 && ((uintptr_t)x & 15u) == 0 && ((uintptr_t)idx & 15u) == 0 && ((uintptr_t)val & 15u) == 0;
}

template <int D, int KC>
cudaError_t launch_rows_t(const TkSegs &sg, int k, uint32_t *status_word, cudaStream_t stream) {
    const size_t smem = (size_t)2 * TK_ROWS * D * 2 + (KC > 0 ? 0 : ((TK_ROWS * k + 15) & ~15) + (size_t)TK_ROWS * k * 2);
    auto kern = topk_rows_bf16_kernel<D, KC>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TK_ROWS, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int64_t grid = sg.nb < (int64_t)sms * per_sm ? sg.nb : (int64_t)sms * per_sm;
    kern<<<(unsigned)grid, TK_ROWS, smem, stream>>>(sg, k, status_word);
    return cudaGetLastError();
}

cudaError_t launch_rows(TkSegs sg, int64_t blocks, int d, int k, uint32_t *status_word, cudaStream_t stream) {
    if (blocks > 0x7FFFFFFF) return cudaErrorInvalidValue;
    sg.nb = blocks;
    if (d == 64)
        return k == 8 ? launch_rows_t<64, 8>(sg, k, status_word, stream)
             : k == 16 ? launch_rows_t<64, 16>(sg, k, status_word, stream)
                       : launch_rows_t<64, 0>(sg, k, status_word, stream);
    return k == 8 ? launch_rows_t<128, 8>(sg, k, status_word, stream)
         : k == 16 ? launch_rows_t<128, 16>(sg, k, status_word, stream)
                   : launch_rows_t<128, 0>(sg, k, status_word, stream);
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
