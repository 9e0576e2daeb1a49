// attn_simt.cu -- FlashSFA forward on CUDA cores (steps 4-8; Alg. 1, Sec. 3.2).
//
// The reference kernel of the path and the only one for fp32 (P.V by FFMA: TF32 would miss
// the 1e-5 bar, reading A12).  One CTA = 128 query rows of one (b, h); thread = query row
// (the "exclusive ownership, no atomics" contract of App. C, re-mapped: a row
// owner instead of a 2x2 patch).  Per key tile of BK keys (tiles above the causal diagonal
// are skipped):
//   step 4  scatter: for each of the row's k features f, for each (j, k~_jf) in bucket f of
//           the tile, S_w[j][lane] += q~_if * k~_jf  -- the per-warp fp32 slab in shared memory,
//           bank = lane, so the read-modify-writes are conflict-free; about BK*k^2/d products
//           per row instead of BK*d.  scale*log2(e) is pre-folded into q~ (A5/A17).
//   step 5  causal mask: keys beyond q_pos0 + i (A9) and beyond n_kv are never absorbed.
//   step 6  online softmax in the log2 domain (m, l in registers); the slab is read and
//           re-zeroed in the same pass.
//   step 7  O += p * V_j with V_j broadcast from shared memory (fp32 accumulate in registers).
//   step 8  O /= l, round to the output dtype (RNE); LSE = (m + log2 l) ln 2.
// EDGE (reading A1/R2): the scatter itself finds the edges -- P:L101 "Traversing
// active coordinates yields only the nonzero attention edges".  Slab entries start as the
// sentinel UNTOUCHED (a NaN bit pattern no fmaf produces from finite inputs); the first product
// that lands on (j, lane) replaces it, so after the scatter an entry still UNTOUCHED is a pair with
// disjoint supports and is left out of the softmax (zero-valued support entries still touch: A8).
#include "launch.cuh"

namespace sfa {

constexpr uint32_t UNTOUCHED = 0xFFFFFFFFu;

template <typename T, int D, int DV, int BK, bool EDGE>
__global__ void __launch_bounds__(128) attn_simt_kernel(const AttnParams p) {
    constexpr bool kBF16 = DT<T>::is_bf16;
    constexpr int EB = kBF16 ? 4 : 8;
    extern __shared__ __align__(16) uint8_t smem[];
    float *slab_all = reinterpret_cast<float *>(smem);                       // [4][BK+1][32]
    uint8_t *btile = smem + 4 * (BK + 1) * 32 * 4;                            // off + entries
    T *Vs = reinterpret_cast<T *>(btile + p.L.tile_bytes);                    // [BK][DV]

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nqb = (int)((p.n_q + 127) / 128);
    const int qb = nqb - 1 - (int)blockIdx.x;  // heaviest causal blocks first
    const int bh = blockIdx.y;
    const int b = bh / p.H, h = bh % p.H;
    const int g = h / (p.H / p.H_kv);
    const int64_t r = (int64_t)qb * 128 + tid;
    const bool valid = r < p.n_q;
    const int64_t qrow = ((int64_t)bh) * p.n_q + r;
    const uint8_t *qi = p.q_idx + qrow * p.k;
    const T *qv = reinterpret_cast<const T *>(p.q_val) + qrow * p.k;
    float *slab = slab_all + w * (BK + 1) * 32 + lane;
    const uint16_t *off = reinterpret_cast<const uint16_t *>(btile);

    const float slab_init = EDGE ? __uint_as_float(UNTOUCHED) : 0.f;
    for (int i = tid; i < 4 * (BK + 1) * 32; i += 128) slab_all[i] = slab_init;

    const int64_t last_row = ((int64_t)qb * 128 + 127 < p.n_q - 1) ? (int64_t)qb * 128 + 127 : p.n_q - 1;
    int ntiles = p.L.ntiles;
    if (p.causal) {
        const int64_t lim = (p.q_pos0 + last_row) / BK + 1;
        if (lim < ntiles) ntiles = (int)lim;
    }
    const int64_t kvb = (int64_t)b * p.H_kv + g;
    const uint8_t *tiles = p.ws + kvb * p.L.ntiles * p.L.tile_bytes;
    const T *vbase = reinterpret_cast<const T *>(p.v) + kvb * p.n_kv * DV;

    float m = -INFINITY, l = 0.f;
    float O[DV];
#pragma unroll
    for (int c = 0; c < DV; ++c) O[c] = 0.f;

    int t0 = 0;  // N4 sliding window: key tiles before the window of the block's first row are skipped
    if (p.window > 0) {
        const int64_t kb = p.q_pos0 + (int64_t)qb * 128 - p.window + 1;
        if (kb > 0) t0 = (int)(kb / BK);
        if (t0 > ntiles - 1) t0 = ntiles - 1 < 0 ? 0 : ntiles - 1;
    }
    for (int t = t0; t < ntiles; ++t) {
        __syncthreads();
        {  // stage bucket tile and V tile
            const uint8_t *tb = tiles + (int64_t)t * p.L.tile_bytes;
            const int used = reinterpret_cast<const uint16_t *>(tb)[D];
            const int nvec = (p.L.off_bytes + used * EB) / 16;
            for (int i = tid; i < nvec; i += 128)
                reinterpret_cast<uint4 *>(btile)[i] = reinterpret_cast<const uint4 *>(tb)[i];
            constexpr int VPR = DV * sizeof(T) / 16;  // 16-byte vectors per V row
            const int64_t key0 = (int64_t)t * BK;
            for (int i = tid; i < BK * VPR; i += 128) {
                const int j = i / VPR, c = i % VPR;
                uint4 x = make_uint4(0, 0, 0, 0);
                if (key0 + j < p.n_kv) x = reinterpret_cast<const uint4 *>(vbase + (key0 + j) * DV)[c];
                reinterpret_cast<uint4 *>(Vs + j * DV)[c] = x;
            }
        }
        __syncthreads();
        if (valid) {
            // step 4: scatter-accumulate the support overlaps into this row's slab column
            for (int tt = 0; tt < p.k; ++tt) {
                const int f = qi[tt];
                const float q = DT<T>::to_f(qv[tt]) * p.scale_log2;
                const int e0 = off[f], e1 = off[f + 1];
                if (kBF16) {
                    const uint32_t *ent = reinterpret_cast<const uint32_t *>(btile + p.L.off_bytes);
                    for (int e = e0; e < e1; ++e) {
                        const uint32_t x = ent[e];
                        float *s = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(slab) + (x & 0xFFFFu));
                        const float cur = *s;
                        *s = fmaf(q, __uint_as_float(x & 0xFFFF0000u), (EDGE && __float_as_uint(cur) == UNTOUCHED) ? 0.f : cur);
                    }
                } else {
                    const uint2 *ent = reinterpret_cast<const uint2 *>(btile + p.L.off_bytes);
                    for (int e = e0; e < e1; ++e) {
                        const uint2 x = ent[e];
                        float *s = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(slab) + x.x);
                        const float cur = *s;
                        *s = fmaf(q, __uint_as_float(x.y), (EDGE && __float_as_uint(cur) == UNTOUCHED) ? 0.f : cur);
                    }
                }
            }
            // step 5: allowed keys of this row inside the tile
            const int64_t key0 = (int64_t)t * BK;
            int64_t jv = p.n_kv - key0;
            if (p.causal && p.q_pos0 + r - key0 + 1 < jv) jv = p.q_pos0 + r - key0 + 1;
            if (jv > BK) jv = BK;
            int jl = 0;  // first key of the window in this tile
            if (p.window > 0) {
                const int64_t lo = p.q_pos0 + r - p.window + 1 - key0;
                jl = lo < 0 ? 0 : (lo > BK ? BK : (int)lo);
            }
            // step 6: online softmax (log2 domain)
            float mx = -INFINITY;
            for (int j = jl; j < jv; ++j) {
                const float sj = slab[j * 32];
                if (!EDGE || __float_as_uint(sj) != UNTOUCHED) mx = fmaxf(mx, sj);
            }
            if (mx > m) {
                const float alpha = fast_exp2(m - mx);  // m = -inf -> 0
                l *= alpha;
#pragma unroll
                for (int c = 0; c < DV; ++c) O[c] *= alpha;
                m = mx;
            }
            // steps 6-7: p = 2^(s - m), l += p, O += p V_j ; re-zero the slab
            for (int j = 0; j < BK; ++j) {
                const float s = slab[j * 32];
                slab[j * 32] = slab_init;
                if (j >= jl && j < jv && (!EDGE || __float_as_uint(s) != UNTOUCHED)) {
                    const float pj = fast_exp2(s - m);
                    l += pj;
                    const T *vr = Vs + j * DV;
                    if (kBF16) {
#pragma unroll
                        for (int c = 0; c < DV; c += 8) {
                            const uint4 x = *reinterpret_cast<const uint4 *>(vr + c);
                            O[c + 0] = fmaf(pj, __uint_as_float(x.x << 16), O[c + 0]);
                            O[c + 1] = fmaf(pj, __uint_as_float(x.x & 0xFFFF0000u), O[c + 1]);
                            O[c + 2] = fmaf(pj, __uint_as_float(x.y << 16), O[c + 2]);
                            O[c + 3] = fmaf(pj, __uint_as_float(x.y & 0xFFFF0000u), O[c + 3]);
                            O[c + 4] = fmaf(pj, __uint_as_float(x.z << 16), O[c + 4]);
                            O[c + 5] = fmaf(pj, __uint_as_float(x.z & 0xFFFF0000u), O[c + 5]);
                            O[c + 6] = fmaf(pj, __uint_as_float(x.w << 16), O[c + 6]);
                            O[c + 7] = fmaf(pj, __uint_as_float(x.w & 0xFFFF0000u), O[c + 7]);
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < DV; c += 4) {
                            const float4 x = *reinterpret_cast<const float4 *>(vr + c);
                            O[c + 0] = fmaf(pj, x.x, O[c + 0]);
                            O[c + 1] = fmaf(pj, x.y, O[c + 1]);
                            O[c + 2] = fmaf(pj, x.z, O[c + 2]);
                            O[c + 3] = fmaf(pj, x.w, O[c + 3]);
                        }
                    }
                }
            }
        }
    }
    if (!valid) return;
    // step 8: epilogue
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (kBF16) {
        uint16_t *orow = reinterpret_cast<uint16_t *>(p.o) + qrow * DV;
#pragma unroll
        for (int c = 0; c < DV; c += 8) {
            uint4 x;
            x.x = (uint32_t)f32_to_bf16_bits_rn(O[c + 0] * inv) | ((uint32_t)f32_to_bf16_bits_rn(O[c + 1] * inv) << 16);
            x.y = (uint32_t)f32_to_bf16_bits_rn(O[c + 2] * inv) | ((uint32_t)f32_to_bf16_bits_rn(O[c + 3] * inv) << 16);
            x.z = (uint32_t)f32_to_bf16_bits_rn(O[c + 4] * inv) | ((uint32_t)f32_to_bf16_bits_rn(O[c + 5] * inv) << 16);
            x.w = (uint32_t)f32_to_bf16_bits_rn(O[c + 6] * inv) | ((uint32_t)f32_to_bf16_bits_rn(O[c + 7] * inv) << 16);
            reinterpret_cast<uint4 *>(orow + c)[0] = x;
        }
    } else {
        float *orow = reinterpret_cast<float *>(p.o) + qrow * DV;
#pragma unroll
        for (int c = 0; c < DV; c += 4)
            reinterpret_cast<float4 *>(orow + c)[0] = make_float4(O[c] * inv, O[c + 1] * inv, O[c + 2] * inv, O[c + 3] * inv);
    }
    p.lse[qrow] = l > 0.f ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
}

template <typename T, int D, int DV, int BK>
static cudaError_t launch_simt_t(const AttnParams &p, cudaStream_t stream) {
    const size_t smem = 4 * (BK + 1) * 32 * 4 + p.L.tile_bytes + (size_t)BK * DV * sizeof(T);
    auto kern = p.edges_only ? attn_simt_kernel<T, D, DV, BK, true> : attn_simt_kernel<T, D, DV, BK, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((p.n_q + 127) / 128), (unsigned)(p.B * p.H));
    kern<<<grid, 128, smem, stream>>>(p);
    return cudaGetLastError();
}

template <typename T, int D, int DV>
static cudaError_t launch_simt_bk(const AttnParams &p, cudaStream_t stream) {
    return p.L.bk == 128 ? launch_simt_t<T, D, DV, 128>(p, stream) : launch_simt_t<T, D, DV, 64>(p, stream);
}

template <typename T>
static cudaError_t launch_simt_dt(const AttnParams &p, int d, int d_v, cudaStream_t stream) {
    if (d == 64) return d_v == 64 ? launch_simt_bk<T, 64, 64>(p, stream) : launch_simt_bk<T, 64, 128>(p, stream);
    return d_v == 64 ? launch_simt_bk<T, 128, 64>(p, stream) : launch_simt_bk<T, 128, 128>(p, stream);
}

cudaError_t launch_attn_simt(const AttnParams &p, bool bf16, int d, int d_v, cudaStream_t stream) {
    return bf16 ? launch_simt_dt<__nv_bfloat16>(p, d, d_v, stream) : launch_simt_dt<float>(p, d, d_v, stream);
}

}  // namespace sfa
