// vprep.cu -- P.V operand preparation for the sm_100a kernel (reading A12).
//
// The tensor-core P.V takes A = P and B = V in the same 16-bit format.  Rounding P to bf16 costs
// 2^-9 relative per weight, which alone can exceed the 2e-3 bar on |O| ~ 1 rows; fp16 P costs
// 2^-12.  V therefore goes to fp16 too, EXACTLY: V' = V * 2^-e with one power of two per
// (batch, kv head) chosen so max|V'| lies in [2^14, 2^15) -- scaled down for large heads and UP for
// small ones (bf16's 8-bit significand fits fp16's 11 bits; only |V'| < 2^-14, i.e. below about
// 2^-28 max|V| of the head, loses bits to fp16 subnormals).  The attention epilogue
// multiplies O by 2^e.  Two HBM-bound passes: absmax per head, then convert.
#include <cuda_fp16.h>

#include "launch.cuh"

namespace sfa {

namespace {

// absmax of |V| per (b, kv head): float bits of a non-negative value order like unsigned ints
__global__ void __launch_bounds__(256) v_absmax_kernel(const uint4 *__restrict__ v, int64_t vec_per_head,
                                                        int64_t n_bh, uint32_t *__restrict__ amax) {
    for (int64_t bh = blockIdx.y; bh < n_bh; bh += gridDim.y) {  // grid.y <= 65535: heads strided
    const uint4 *src = v + (int64_t)bh * vec_per_head;
    uint32_t m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < vec_per_head;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = __ldg(src + i);
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            m = max(m, (w[e] << 16) & 0x7FFFFFFFu);
            m = max(m, w[e] & 0x7FFF0000u);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(amax + bh, m);
    }
}

// out rows are dvp >= d_v features wide: features [d_v, dvp) are written as zeros (SM100_OT with
// d_v = 64 runs its d_v = 128 P.V over the padded copy)
__global__ void __launch_bounds__(256) v_to_f16_kernel(const uint4 *__restrict__ v, int64_t vec_per_head,
                                                        int64_t n_bh, const uint32_t *__restrict__ amax,
                                                        uint2 *__restrict__ out, int cin, int cout) {
    // cin / cout: 16-byte vectors per row of V (d_v / 8) and of the copy (dvp / 8)
    const int64_t out_per_head = vec_per_head / cin * cout;
    for (int64_t bh = blockIdx.y; bh < n_bh; bh += gridDim.y) {
    const int e = vprep_head_exp(__ldg(amax + bh));
#ifndef SFA_FAULT_VSCALE
    const float sc = __uint_as_float((uint32_t)(127 - e) << 23);  // 2^-e, exact
#else  // negative control: V' = V 2^(1-e) while the epilogue multiplies by 2^e
    const float sc = __uint_as_float((uint32_t)(128 - e) << 23);
#endif
    const uint4 *src = v + (int64_t)bh * vec_per_head;
    uint4 *dst = reinterpret_cast<uint4 *>(out) + (int64_t)bh * out_per_head;
    const auto cvt = [sc](const uint4 x) {
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const __half2 h = __floats2half2_rn(__uint_as_float(w[q] << 16) * sc, __uint_as_float(w[q] & 0xFFFF0000u) * sc);
            o[q] = *reinterpret_cast<const uint32_t *>(&h);
        }
        return make_uint4(o[0], o[1], o[2], o[3]);
    };
    if (cin == cout) {  // unpadded copy: a plain streaming loop
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < out_per_head;
             i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = cvt(__ldcs(src + i));
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < out_per_head;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t row = i / cout;
            const int c = (int)(i - row * cout);
            dst[i] = c < cin ? cvt(__ldcs(src + row * cin + c)) : make_uint4(0u, 0u, 0u, 0u);
        }
    }
    }
}

// K~ for the SM100_OT kernel's TMA: the decompressed key rows, bf16 [rows][D], written once per key
// (the attention kernel would otherwise rebuild every key tile in shared memory once per work item,
// ~630 shared-memory wavefronts per key tile, profiles/r02_ot_ab.txt).  Bit copies of the code values
// at their indices, zeros elsewhere.  A CTA stages 128 rows in shared memory (zero fill,
// thread per row scatters its k values), then writes them out with coalesced 16-byte stores.
constexpr int KD_ROWS = 128;
template <int D>
__global__ void __launch_bounds__(KD_ROWS) k_dense_kernel(const uint8_t *__restrict__ idx,
                                                           const uint16_t *__restrict__ val, int64_t rows, int k,
                                                           uint4 *__restrict__ out) {
    constexpr int NC = D / 8;  // 16-byte chunks per row
    extern __shared__ uint4 kd_sm[];  // [KD_ROWS][NC]
    const int t = threadIdx.x;
    const int64_t row0 = (int64_t)blockIdx.x * KD_ROWS;
    const int nrows = (int)((rows - row0) < KD_ROWS ? (rows - row0) : KD_ROWS);
    for (int v = t; v < KD_ROWS * NC; v += KD_ROWS) kd_sm[v] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (t < nrows) {
        uint16_t *row = reinterpret_cast<uint16_t *>(kd_sm + t * NC);
        const uint8_t *ir = idx + (row0 + t) * k;
        const uint16_t *vr = val + (row0 + t) * k;
        if ((k & 7) == 0) {
            for (int e0 = 0; e0 < k; e0 += 8) {
                const uint2 ii = __ldg(reinterpret_cast<const uint2 *>(ir + e0));
                const uint4 vv = __ldg(reinterpret_cast<const uint4 *>(vr + e0));
                const uint32_t iw[2] = {ii.x, ii.y}, vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
#ifdef SFA_FAULT_KDENSE_DROP_LAST  // negative control: the row's last selected feature left at 0
                    if (e0 + e == k - 1) continue;
#endif
                    row[(iw[e >> 2] >> (8 * (e & 3))) & 0xFFu] = (uint16_t)(vw[e >> 1] >> (16 * (e & 1)));
                }
            }
        } else {
            for (int e = 0; e < k; ++e) row[__ldg(ir + e)] = __ldg(vr + e);
        }
    }
    __syncthreads();
    uint4 *dst = out + row0 * NC;
    for (int v = t; v < nrows * NC; v += KD_ROWS) dst[v] = kd_sm[v];
}

// Small heads (n_kv * d_v * 2 <= 128 KB, e.g. GPT-2's): the whole key preparation in ONE launch with no
// memset.  Blocks [0, bh_kv) own one (batch, kv head) each: 1024 threads load the head's V into registers
// at once (<= 8 16-byte vectors per thread: the whole head in flight), max|V| by a block reduction,
// then the exact fp16 copy from the same registers, and the max's bits into amax[bh].  Blocks
// [bh_kv, ...) build K~ rows like k_dense_kernel (SM100_OT only).
constexpr int VS_THREADS = 1024;
constexpr int VS_VPT = 8;  // vectors per thread: heads up to VS_THREADS * VS_VPT * 16 B = 128 KB
template <int D>
__global__ void __launch_bounds__(VS_THREADS) prep_small_kernel(const uint4 *__restrict__ v, int64_t vec_per_head,
                                                                 int64_t n_bh, uint32_t *__restrict__ amax,
                                                                 uint4 *__restrict__ out, int cin, int cout,
                                                                 const uint8_t *__restrict__ kidx,
                                                                 const uint16_t *__restrict__ kval, int64_t krows, int k,
                                                                 uint4 *__restrict__ kout) {
    __shared__ uint32_t red[VS_THREADS / 32];
    const int t = threadIdx.x;
    if ((int64_t)blockIdx.x < n_bh) {
        const int64_t bh = blockIdx.x;
        const int nvec = (int)vec_per_head;  // <= VS_THREADS * VS_VPT
        const uint4 *src = v + bh * vec_per_head;
        uint4 x[VS_VPT];
#pragma unroll
        for (int i = 0; i < VS_VPT; ++i) {
            const int iv = t + i * VS_THREADS;
            x[i] = iv < nvec ? __ldcs(src + iv) : make_uint4(0u, 0u, 0u, 0u);
        }
        uint32_t m = 0;
#pragma unroll
        for (int i = 0; i < VS_VPT; ++i) {
            const uint32_t w[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                m = max(m, (w[e] << 16) & 0x7FFFFFFFu);
                m = max(m, w[e] & 0x7FFF0000u);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((t & 31) == 0) red[t >> 5] = m;
        __syncthreads();
        m = red[t & 31];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (t == 0) amax[bh] = m;
        const int e = vprep_head_exp(m);
#ifndef SFA_FAULT_VSCALE
        const float sc = __uint_as_float((uint32_t)(127 - e) << 23);  // 2^-e, exact
#else  // negative control: V' = V 2^(1-e) while the epilogue multiplies by 2^e
        const float sc = __uint_as_float((uint32_t)(128 - e) << 23);
#endif
        uint4 *dst = out + bh * (vec_per_head / cin * cout);
#pragma unroll
        for (int i = 0; i < VS_VPT; ++i) {
            const int iv = t + i * VS_THREADS;
            if (iv < nvec) {
                const uint32_t w[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
                uint32_t o[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const __half2 h =
                        __floats2half2_rn(__uint_as_float(w[q] << 16) * sc, __uint_as_float(w[q] & 0xFFFF0000u) * sc);
                    o[q] = *reinterpret_cast<const uint32_t *>(&h);
                }
                const int row = cin == cout ? 0 : iv / cin;
                dst[cin == cout ? iv : row * cout + (iv - row * cin)] = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
        if (cout > cin) {  // the zero padding of the copy's rows (SM100_OT with d_v = 64)
            const int pad = cout - cin, nz = nvec / cin * pad;
            for (int z = t; z < nz; z += VS_THREADS) dst[(z / pad) * cout + cin + z % pad] = make_uint4(0u, 0u, 0u, 0u);
        }
        return;
    }
    // ---- K~ rows: KD_ROWS rows per block, thread t < KD_ROWS scatters row t
    constexpr int NC = D / 8;
    __shared__ uint4 kd[KD_ROWS * NC];
    const int64_t row0 = ((int64_t)blockIdx.x - n_bh) * KD_ROWS;
    const int nrows = (int)((krows - row0) < KD_ROWS ? (krows - row0) : KD_ROWS);
    for (int i = t; i < KD_ROWS * NC; i += VS_THREADS) kd[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (t < nrows) {
        uint16_t *row = reinterpret_cast<uint16_t *>(kd + t * NC);
        const uint8_t *ir = kidx + (row0 + t) * k;
        const uint16_t *vr = kval + (row0 + t) * k;
        for (int e = 0; e < k; ++e) {
#ifdef SFA_FAULT_KDENSE_DROP_LAST  // negative control: the row's last selected feature left at 0
            if (e == k - 1) continue;
#endif
            row[__ldg(ir + e)] = __ldg(vr + e);
        }
    }
    __syncthreads();
    uint4 *dst = kout + row0 * NC;
    for (int i = t; i < nrows * NC; i += VS_THREADS) dst[i] = kd[i];
}

}  // namespace

cudaError_t launch_kdense(const uint8_t *k_idx, const void *k_val, int64_t rows, int d, int k, void *out,
                          cudaStream_t stream) {
    if (rows == 0) return cudaSuccess;
    const int64_t blocks = (rows + KD_ROWS - 1) / KD_ROWS;
    if (blocks > 0x7FFFFFFF) return cudaErrorInvalidValue;
    const size_t smem = (size_t)KD_ROWS * d * 2;
    if (d == 64)
        k_dense_kernel<64><<<(unsigned)blocks, KD_ROWS, smem, stream>>>(k_idx, (const uint16_t *)k_val, rows, k, (uint4 *)out);
    else
        k_dense_kernel<128><<<(unsigned)blocks, KD_ROWS, smem, stream>>>(k_idx, (const uint16_t *)k_val, rows, k, (uint4 *)out);
    return cudaGetLastError();
}

bool prep_small_ok(int64_t bh_kv, int64_t n_kv, int d_v, int64_t krows) {
    return n_kv * d_v / 8 <= (int64_t)VS_THREADS * VS_VPT && bh_kv + (krows + KD_ROWS - 1) / KD_ROWS <= 0x7FFFFFFF;
}

cudaError_t launch_prep_small(const void *v, int64_t bh_kv, int64_t n_kv, int d_v, int dvp, uint32_t *amax, void *v16,
                              const uint8_t *k_idx, const void *k_val, int d, int k, void *k_dense, cudaStream_t stream) {
    if (bh_kv == 0) return cudaSuccess;
    const int64_t krows = k_dense != nullptr ? bh_kv * n_kv : 0;
    const int64_t blocks = bh_kv + (krows + KD_ROWS - 1) / KD_ROWS;
    const int64_t vec = n_kv * d_v / 8;
    if (d == 64)
        prep_small_kernel<64><<<(unsigned)blocks, VS_THREADS, 0, stream>>>(
            (const uint4 *)v, vec, bh_kv, amax, (uint4 *)v16, d_v / 8, dvp / 8, k_idx, (const uint16_t *)k_val, krows,
            k, (uint4 *)k_dense);
    else
        prep_small_kernel<128><<<(unsigned)blocks, VS_THREADS, 0, stream>>>(
            (const uint4 *)v, vec, bh_kv, amax, (uint4 *)v16, d_v / 8, dvp / 8, k_idx, (const uint16_t *)k_val, krows,
            k, (uint4 *)k_dense);
    return cudaGetLastError();
}

cudaError_t launch_vprep(const void *v, int64_t bh_kv, int64_t n_kv, int d_v, int dvp, uint32_t *amax, void *v16,
                         cudaStream_t stream) {
    if (bh_kv == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(amax, 0, (size_t)bh_kv * 4, stream);
    if (e != cudaSuccess) return e;
    const int64_t vec = n_kv * d_v / 8;  // 16-byte vectors per head (d_v is a multiple of 8)
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t gx = (vec + 255) / 256;
    const int64_t cap = ((int64_t)sms * 8 + bh_kv - 1) / bh_kv;  // about 8 CTAs per SM in total
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    dim3 grid((unsigned)gx, (unsigned)(bh_kv < 65535 ? bh_kv : 65535));
    v_absmax_kernel<<<grid, 256, 0, stream>>>((const uint4 *)v, vec, bh_kv, amax);
    v_to_f16_kernel<<<grid, 256, 0, stream>>>((const uint4 *)v, vec, bh_kv, amax, (uint2 *)v16, d_v / 8, dvp / 8);
    return cudaGetLastError();
}

}  // namespace sfa
