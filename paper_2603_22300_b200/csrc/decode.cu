// decode.cu -- SURVEY 8(f) N2: FlashSFA forward for few query rows over a long key/value cache
// (decode / speculative-decode shape: n_q * H/H_kv <= 16 rows per kv head).  Same definition as
// sfa_attn_fwd (Eq. s_ij P:L97-101 on the codes, reading A1/R1; softmax and P V, Alg. 1
// L739-751; causal alignment q_pos0, reading A9) -- only the work shape differs: the tensor-core
// kernel needs 128-row query tiles, while here a kv head has a handful of query rows and n_kv keys,
// so the forward is bound by reading the cache: per key its code (3k bytes) and its V row (2 d_v
// bytes).  This is where feature sparsity pays on B200: the code is 6x smaller than a dense
// 128-dim bf16 key (the paper's KV-cache claim).
//
// Split-KV: CTA (b, kv head g, split s) owns keys [s*chunk, (s+1)*chunk).  The group's query rows
// (R = H/H_kv heads x n_q rows) are decompressed into shared memory as fp32 (q~ scaled by
// scale*log2 e).  Each warp walks 32-key blocks: lane l scores key l of the block against every row
// with k FMAs (its code read with 16-byte loads), the warp reduces the block max per row, updates
// the running max (online softmax, fp32), then accumulates O[row][:] += p V[key] with lanes over
// d_v (V rows read coalesced, 8 bytes per lane) and p broadcast by shuffles.  Each warp keeps its
// own (m, l, O) in registers; the CTA merges its warps in shared memory and writes one partial per
// split; `decode_combine_kernel` merges the splits with their log-sum-exps.  fp32 throughout, bf16
// V read as is; O rounded to bf16 once.
#include "launch.cuh"

namespace sfa {

namespace {

constexpr int DEC_THREADS = 256;
constexpr int DEC_WARPS = DEC_THREADS / 32;
constexpr int MAXROWS = 16;

// partial layout per (b, g, split): m[rows], l[rows], O[rows][d_v] fp32
struct DecArgs {
    const uint8_t *q_idx;
    const uint16_t *q_val;
    const uint8_t *k_idx;
    const uint16_t *k_val;
    const uint16_t *v;
    uint16_t *o;
    float *lse;
    float *part;
    int B, H, H_kv, R, k, d;
    int64_t n_q, n_kv, q_pos0;
    int causal;
    float c_scale;
    int nsplit;
    int64_t chunk;
};

template <int DV, int ROWS>
__global__ void __launch_bounds__(DEC_THREADS) decode_partial_kernel(const DecArgs a) {
    constexpr int DPL = DV / 32;  // value dims per lane (2 or 4)
    extern __shared__ __align__(16) float dsm[];
    float *qs = dsm;                                         // [ROWS][d] fp32 decompressed, pre-scaled queries
    float(*red_m)[ROWS] = reinterpret_cast<float(*)[ROWS]>(dsm + ROWS * a.d);  // [warps][ROWS]
    float(*red_l)[ROWS] = red_m + DEC_WARPS;
    float(*red_o)[ROWS][DV] = reinterpret_cast<float(*)[ROWS][DV]>(dsm + ROWS * a.d + 2 * DEC_WARPS * ROWS);
    const int bg = blockIdx.x, split = blockIdx.y;
    const int b = bg / a.H_kv, g = bg % a.H_kv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = a.R * (int)a.n_q;
    // decompress the group's query rows: row = hr * n_q + i (hr = head within the group)
    for (int x = threadIdx.x; x < ROWS * a.d; x += DEC_THREADS) qs[x] = 0.f;
    __syncthreads();
    for (int row = threadIdx.x; row < rows; row += DEC_THREADS) {
        const int hr = row / (int)a.n_q, i = row % (int)a.n_q;
        const int64_t qrow = ((int64_t)b * a.H + g * a.R + hr) * a.n_q + i;
        for (int t = 0; t < a.k; ++t)
            qs[row * a.d + a.q_idx[qrow * a.k + t]] = __uint_as_float((uint32_t)a.q_val[qrow * a.k + t] << 16) * a.c_scale;
    }
    __syncthreads();

    const int64_t k0 = (int64_t)split * a.chunk;
    int64_t k1 = k0 + a.chunk;
    if (k1 > a.n_kv) k1 = a.n_kv;
    const int64_t kvbase = ((int64_t)b * a.H_kv + g) * a.n_kv;
    float m[ROWS], l[ROWS], acc[ROWS][DPL];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[r][e] = 0.f;
    }
    // warps take interleaved 32-key blocks of the split
    for (int64_t kb = k0 + (int64_t)warp * 32; kb < k1; kb += (int64_t)DEC_WARPS * 32) {
        const int64_t key = kb + lane;
        const bool kval = key < k1;
        // ---- step 4: scores of key `key` against every row from its code
        float s[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) s[r] = 0.f;
        if (kval) {
            const uint8_t *ci = a.k_idx + (kvbase + key) * a.k;
            const uint16_t *cv = a.k_val + (kvbase + key) * a.k;
            if ((a.k & 7) == 0) {  // 8 codes per step: 8-byte index + 16-byte value loads
                for (int t0 = 0; t0 < a.k; t0 += 8) {
                    const uint2 ii = __ldg(reinterpret_cast<const uint2 *>(ci + t0));
                    const uint4 vv = __ldg(reinterpret_cast<const uint4 *>(cv + t0));
                    const uint32_t iw[2] = {ii.x, ii.y}, vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int f = (iw[e >> 2] >> (8 * (e & 3))) & 0xFF;
                        const float kvf = __uint_as_float((e & 1) ? (vw[e >> 1] & 0xFFFF0000u) : (vw[e >> 1] << 16));
#pragma unroll
                        for (int r = 0; r < ROWS; ++r) s[r] = fmaf(qs[r * a.d + f], kvf, s[r]);
                    }
                }
            } else {
                for (int t = 0; t < a.k; ++t) {
                    const int f = __ldg(ci + t);
                    const float kvf = __uint_as_float((uint32_t)__ldg(cv + t) << 16);
#pragma unroll
                    for (int r = 0; r < ROWS; ++r) s[r] = fmaf(qs[r * a.d + f], kvf, s[r]);
                }
            }
        }
        // ---- step 5: causal / ragged mask; step 6: online softmax per row (warp-wide block max)
        float p[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            bool ok = kval && r < rows;
            if (ok && a.causal) ok = key <= a.q_pos0 + (r % (int)a.n_q);
            float x = ok ? s[r] : -INFINITY;
            float bm = x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
            const float mn = fmaxf(m[r], bm);
            const float ms = mn == -INFINITY ? 0.f : mn;
            const float alpha = fast_exp2(m[r] - ms);  // m = -inf -> 0
            p[r] = ok ? fast_exp2(x - ms) : 0.f;
            float ps = p[r];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            l[r] = l[r] * alpha + ps;
#pragma unroll
            for (int e = 0; e < DPL; ++e) acc[r][e] *= alpha;
            m[r] = mn;
        }
        // ---- step 7: O[r][lane dims] += sum over the block's keys of p * V[key][lane dims]
        const int nk = (int)((k1 - kb) < 32 ? (k1 - kb) : 32);
        const uint16_t *vb = a.v + (kvbase + kb) * DV + lane * DPL;
#pragma unroll 4
        for (int kk = 0; kk < nk; ++kk) {
            float vv[DPL];
            if (DPL == 4) {
                const uint2 w = __ldg(reinterpret_cast<const uint2 *>(vb + (int64_t)kk * DV));
                vv[0] = __uint_as_float(w.x << 16);
                vv[1] = __uint_as_float(w.x & 0xFFFF0000u);
                vv[2 % DPL] = __uint_as_float(w.y << 16);
                vv[3 % DPL] = __uint_as_float(w.y & 0xFFFF0000u);
            } else {
                const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(vb + (int64_t)kk * DV));
                vv[0] = __uint_as_float(w << 16);
                vv[1 % DPL] = __uint_as_float(w & 0xFFFF0000u);
            }
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                const float pr = __shfl_sync(0xffffffffu, p[r], kk);
#pragma unroll
                for (int e = 0; e < DPL; ++e) acc[r][e] = fmaf(pr, vv[e], acc[r][e]);
            }
        }
    }
    // ---- merge the CTA's warps (shared memory), write this split's partial
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        if (lane == 0) {
            red_m[warp][r] = m[r];
            red_l[warp][r] = l[r];
        }
#pragma unroll
        for (int e = 0; e < DPL; ++e) red_o[warp][r][lane * DPL + e] = acc[r][e];
    }
    __syncthreads();
    float *part = a.part + ((int64_t)bg * a.nsplit + split) * ROWS * (2 + DV);
    for (int x = threadIdx.x; x < ROWS * DV; x += DEC_THREADS) {
        const int r = x / DV, c = x % DV;
        float M = -INFINITY;
        for (int w = 0; w < DEC_WARPS; ++w) M = fmaxf(M, red_m[w][r]);
        const float Ms = M == -INFINITY ? 0.f : M;
        float L = 0.f, O = 0.f;
        for (int w = 0; w < DEC_WARPS; ++w) {
            const float f = fast_exp2(red_m[w][r] - Ms);
            L += red_l[w][r] * f;
            O += red_o[w][r][c] * f;
        }
        part[2 * ROWS + x] = O;
        if (c == 0) {
            part[r] = M;
            part[ROWS + r] = L;
        }
    }
}

// merge the splits of every row: O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s (step 8)
template <int DV, int ROWS>
__global__ void __launch_bounds__(DV) decode_combine_kernel(const DecArgs a) {
    const int bg = blockIdx.x, r = blockIdx.y, c = threadIdx.x;
    const int rows = a.R * (int)a.n_q;
    if (r >= rows) return;
    const int b = bg / a.H_kv, g = bg % a.H_kv;
    const float *base = a.part + (int64_t)bg * a.nsplit * ROWS * (2 + DV);
    float M = -INFINITY;
    for (int s = 0; s < a.nsplit; ++s) M = fmaxf(M, base[(int64_t)s * ROWS * (2 + DV) + r]);
    const float Ms = M == -INFINITY ? 0.f : M;
    float L = 0.f, O = 0.f;
    for (int s = 0; s < a.nsplit; ++s) {
        const float *ps = base + (int64_t)s * ROWS * (2 + DV);
        const float f = fast_exp2(ps[r] - Ms);
        L += ps[ROWS + r] * f;
        O += ps[2 * ROWS + r * DV + c] * f;
    }
    const int hr = r / (int)a.n_q, i = r % (int)a.n_q;
    const int64_t orow = ((int64_t)b * a.H + g * a.R + hr) * a.n_q + i;
    a.o[orow * DV + c] = f32_to_bf16_bits_rn(L > 0.f ? O / L : 0.f);
    if (c == 0) a.lse[orow] = L > 0.f ? (M + __log2f(L)) * 0.69314718055994530942f : -INFINITY;
}

template <int DV, int ROWS>
cudaError_t launch_decode_t(const DecArgs &a, cudaStream_t st) {
    const size_t smem = ((size_t)ROWS * a.d + 2 * DEC_WARPS * ROWS + (size_t)DEC_WARPS * ROWS * DV) * 4;
    auto kern = decode_partial_kernel<DV, ROWS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 g1(a.B * a.H_kv, a.nsplit);
    kern<<<g1, DEC_THREADS, smem, st>>>(a);
    dim3 g2(a.B * a.H_kv, ROWS);
    decode_combine_kernel<DV, ROWS><<<g2, DV, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

int decode_nsplit(int64_t bh_kv, int64_t n_kv) {
    // enough CTAs for ~4 waves over 148 SMs, each split at least 256 keys
    int64_t want = (148 * 8 + bh_kv - 1) / bh_kv;
    const int64_t maxs = (n_kv + 255) / 256;
    if (want > maxs) want = maxs;
    if (want < 1) want = 1;
    if (want > 4096) want = 4096;
    return (int)want;
}

size_t decode_workspace_bytes(int64_t bh_kv, int64_t n_kv, int d_v) {
    return (size_t)bh_kv * decode_nsplit(bh_kv, n_kv) * MAXROWS * (2 + d_v) * 4;
}

cudaError_t launch_decode(const AttnParams &p, int d, int d_v, cudaStream_t st, void *ws) {
    const int R = p.H / p.H_kv;
    const int rows = R * (int)p.n_q;
    if (rows > MAXROWS || (d_v != 64 && d_v != 128)) return cudaErrorNotSupported;
    DecArgs a;
    a.q_idx = p.q_idx;
    a.q_val = (const uint16_t *)p.q_val;
    a.k_idx = p.k_idx;
    a.k_val = (const uint16_t *)p.k_val;
    a.v = (const uint16_t *)p.v;
    a.o = (uint16_t *)p.o;
    a.lse = p.lse;
    a.part = (float *)ws;
    a.B = p.B;
    a.H = p.H;
    a.H_kv = p.H_kv;
    a.R = R;
    a.k = p.k;
    a.d = d;
    a.n_q = p.n_q;
    a.n_kv = p.n_kv;
    a.q_pos0 = p.q_pos0;
    a.causal = p.causal;
    a.c_scale = p.scale_log2;
    a.nsplit = decode_nsplit((int64_t)p.B * p.H_kv, p.n_kv);
    a.chunk = (p.n_kv + a.nsplit - 1) / a.nsplit;
    if (rows <= 4) return d_v == 64 ? launch_decode_t<64, 4>(a, st) : launch_decode_t<128, 4>(a, st);
    if (rows <= 8) return d_v == 64 ? launch_decode_t<64, 8>(a, st) : launch_decode_t<128, 8>(a, st);
    return d_v == 64 ? launch_decode_t<64, 16>(a, st) : launch_decode_t<128, 16>(a, st);
}

}  // namespace sfa
