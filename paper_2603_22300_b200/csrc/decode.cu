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
// scale*log2 e).  A producer warp streams the split's V rows through a shared-memory ring of 128-key
// blocks (2 stages, 3 CTAs per SM; 256-key blocks, 3 stages, 1 CTA per SM for more than 4 rows) with
// cp.async.bulk (mbarrier transaction counts); the consumer warps (one per 32 keys of a block, every
// block read by all of them) take 32 keys of every block each: lane l scores its key against every
// row with k FMAs from the key's code (16-byte loads prefetched one block ahead), the warp reduces
// the block max per row and updates the running max (online softmax, fp32), then accumulates
// O[row][:] += p V[key] from the ring with lanes over d_v and p broadcast by shuffles.  Each warp
// keeps its own (m, l, O) in registers; the CTA merges its warps (in the drained ring) and writes
// one partial per split; `decode_combine_kernel` merges the splits with their log-sum-exps.  fp32
// throughout, bf16 V read as is; O rounded to bf16 once.
#include <algorithm>
#include <cstdlib>

#include "launch.cuh"
#include "sm100.cuh"

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

#ifndef SFA_DEC_WAVES
#define SFA_DEC_WAVES 4
#endif
// keys per V block streamed by the producer = 32 x the consumer warps: 128 (several CTAs per SM, 4
// consumer warps each: one CTA's prologue and merge overlap the others' streaming) or 256 (one CTA per
// SM, 8 consumer warps; more than 4 rows per kv head need its registers).
// Configurations (A/B through SFA_DEC_DB, read once; 8 sequences x Qwen3 heads x 32K cache, one B200):
// 1282 = 128-key blocks, 2 ring stages, 3 CTAs per SM (default, 0.133 ms = 0.73 of HBM); 128 = 128-key
// blocks, 3 stages, 2 CTAs per SM (0.138 ms); 256 = 256-key blocks, 3 stages, 1 CTA per SM (0.146 ms).
// Measured and dropped: 64-key blocks with 3 / 2 stages at 4 / 6 CTAs per SM (0.138 / 0.150 ms).
int dec_cfg() {
    static const int c = [] {
        const char *e = getenv("SFA_DEC_DB");
        const int v = e != nullptr ? atoi(e) : 1282;
        return (v == 256 || v == 128) ? v : 1282;
    }();
    return c;
}
int dec_db() { return dec_cfg() == 256 ? 256 : 128; }
constexpr int dec_minb(int db, int nst) { return db == 256 ? 1 : (nst == 2 ? 3 : 2); }
int dec_minb_rt() { return dec_cfg() == 256 ? 1 : dec_cfg() == 128 ? 2 : 3; }

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// one key's code in registers (k % 8 == 0, k <= 32), loaded a block ahead of its use
struct Code32 {
    uint2 idx[4];
    uint4 val[4];
};

// CW consumer warps (8 or 16): warps 8g..8g+7 take the blocks blk = g (mod CW / 8), 32 keys each
template <int DV, int ROWS, int CW, int DB, int NST>
__global__ void __launch_bounds__(CW * 32 + 32, dec_minb(DB, NST)) decode_partial_kernel(const DecArgs a) {
    constexpr int WPB = DB / 32;      // consumer warps per V block (32 keys each)
    static_assert(CW == WPB, "one consumer group: every V block is read by all consumer warps");
    constexpr int DPL = DV / 32;      // value dims per lane (2 or 4)
    constexpr int VT = DB * DV * 2;   // bytes of one V block
    extern __shared__ __align__(1024) uint8_t dsm_raw[];
    float *qs = reinterpret_cast<float *>(dsm_raw);                        // [d][ROWS] pre-scaled queries
    float *pbuf = reinterpret_cast<float *>(dsm_raw + ROWS * a.d * 4);     // [CW][32][ROWS] weights
    uint8_t *vring = dsm_raw + ((ROWS * a.d * 4 + CW * 32 * ROWS * 4 + 1023) & ~1023);  // [NST][DB][DV] bf16
    uint64_t *bars = reinterpret_cast<uint64_t *>(vring + NST * VT);        // full[NST], empty[NST]
    const uint32_t vring_s = (uint32_t)__cvta_generic_to_shared(vring);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
    const int bg = blockIdx.x, split = blockIdx.y;
    const int b = bg / a.H_kv, g = bg % a.H_kv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = a.R * (int)a.n_q;
    const int64_t k0 = (int64_t)split * a.chunk;
    int64_t k1 = k0 + a.chunk;
    if (k1 > a.n_kv) k1 = a.n_kv;
    const int nblk = k1 > k0 ? (int)((k1 - k0 + DB - 1) / DB) : 0;
    const int64_t kvbase = ((int64_t)b * a.H_kv + g) * a.n_kv;

    for (int x = threadIdx.x; x < ROWS * a.d; x += blockDim.x) qs[x] = 0.f;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s + 8 * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_s + 8 * (NST + i)), "r"(WPB));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (int row = threadIdx.x; row < rows; row += blockDim.x) {
        const int hr = row / (int)a.n_q, i = row % (int)a.n_q;
        const int64_t qrow = ((int64_t)b * a.H + g * a.R + hr) * a.n_q + i;
        for (int t = 0; t < a.k; ++t)
            qs[a.q_idx[qrow * a.k + t] * ROWS + row] = __uint_as_float((uint32_t)a.q_val[qrow * a.k + t] << 16) * a.c_scale;
    }
    __syncthreads();

    auto wait = [](uint32_t bar, uint32_t parity) {
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                bar),
            "r"(parity)
            : "memory");
    };

    float m[ROWS], l[ROWS], acc[ROWS][DPL];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[r][e] = 0.f;
    }
    constexpr int GROUPS = CW / WPB;
    if (warp == CW) {
        // ============ producer: V blocks of the split into the ring (cp.async.bulk, mbarrier tx) ============
        if (lane == 0) {
            for (int blk = 0; blk < nblk; ++blk) {
                const int st = blk % NST, u = blk / NST;
                wait(bar_s + 8 * (NST + st), (u & 1) ^ 1);
                const int64_t ks = k0 + (int64_t)blk * DB;
                const int nk = (int)((k1 - ks) < DB ? (k1 - ks) : DB);
                const uint32_t bytes = (uint32_t)nk * DV * 2;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s + 8 * st), "r"(bytes)
                             : "memory");
                bulk_g2s(vring_s + st * VT, a.v + (kvbase + ks) * DV, bytes, bar_s + 8 * st);
            }
        }
    } else {
        // ============ consumers: warp w takes keys [32 (w % 8), +32) of blocks w / 8, w / 8 + GROUPS, ... ============
        const int sub = warp % WPB, grp0 = warp / WPB;
        const bool pre = (a.k & 7) == 0 && a.k <= 32;
        Code32 nxt;
        auto load_code = [&](Code32 &c, int64_t key) {
            const uint2 *ci = reinterpret_cast<const uint2 *>(a.k_idx + (kvbase + key) * a.k);
            const uint4 *cv = reinterpret_cast<const uint4 *>(a.k_val + (kvbase + key) * a.k);
#pragma unroll
            for (int gg = 0; gg < 4; ++gg)
                if (8 * gg < a.k) {
                    c.idx[gg] = __ldg(ci + gg);
                    c.val[gg] = __ldg(cv + gg);
                }
        };
        {
            const int64_t key = k0 + (int64_t)grp0 * DB + sub * 32 + lane;
            if (pre && grp0 < nblk && key < k1) load_code(nxt, key);
        }
        for (int blk = grp0; blk < nblk; blk += GROUPS) {
            const int st = blk % NST, u = blk / NST;
            const int64_t kb = k0 + (int64_t)blk * DB + sub * 32;
            const int64_t key = kb + lane;
            const bool kval = key < k1;
            // ---- step 4: scores from the key's code (prefetched one block ahead)
            float sc[ROWS];
#pragma unroll
            for (int r = 0; r < ROWS; ++r) sc[r] = 0.f;
            if (pre) {
                const Code32 cur = nxt;
                const int64_t nkey = key + (int64_t)GROUPS * DB;
                if (blk + GROUPS < nblk && nkey < k1) load_code(nxt, nkey);
                if (kval) {
#pragma unroll
                    for (int gg = 0; gg < 4; ++gg)
                        if (8 * gg < a.k) {
                            const uint32_t iw[2] = {cur.idx[gg].x, cur.idx[gg].y};
                            const uint32_t vw[4] = {cur.val[gg].x, cur.val[gg].y, cur.val[gg].z, cur.val[gg].w};
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                const int f = (iw[e >> 2] >> (8 * (e & 3))) & 0xFF;
                                const float kvf =
                                    __uint_as_float((e & 1) ? (vw[e >> 1] & 0xFFFF0000u) : (vw[e >> 1] << 16));
                                const float4 *qf = reinterpret_cast<const float4 *>(qs + f * ROWS);
#pragma unroll
                                for (int r4 = 0; r4 < ROWS / 4; ++r4) {
                                    const float4 qq = qf[r4];
                                    sm100::ffma2v(sc[4 * r4], sc[4 * r4 + 1], qq.x, qq.y, kvf, kvf, sc[4 * r4], sc[4 * r4 + 1]);
                                    sm100::ffma2v(sc[4 * r4 + 2], sc[4 * r4 + 3], qq.z, qq.w, kvf, kvf, sc[4 * r4 + 2],
                                                  sc[4 * r4 + 3]);
                                }
                            }
                        }
                }
            } else if (kval) {
                const uint8_t *ci = a.k_idx + (kvbase + key) * a.k;
                const uint16_t *cv = a.k_val + (kvbase + key) * a.k;
                for (int t = 0; t < a.k; ++t) {
                    const int f = __ldg(ci + t);
                    const float kvf = __uint_as_float((uint32_t)__ldg(cv + t) << 16);
#pragma unroll
                    for (int r = 0; r < ROWS; ++r) sc[r] = fmaf(qs[f * ROWS + r], kvf, sc[r]);
                }
            }
            // ---- steps 5-6: mask + online softmax per row.  The block max is one redux.sync.max.f32
            // (warp-uniform, so the rescale branch is uniform and taken only when the max grows); the
            // row sum l stays a per-lane partial (same reference max in every lane), summed once at the end.
            float p[ROWS];
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                bool ok = kval && r < rows;
                if (ok && a.causal) ok = key <= a.q_pos0 + (r % (int)a.n_q);
                const float x = ok ? sc[r] : -INFINITY;
                float bm;
                asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(bm) : "f"(x));
                if (bm > m[r]) {
                    const float alpha = fast_exp2(m[r] - bm);  // m = -inf -> 0
                    l[r] *= alpha;
#pragma unroll
                    for (int e = 0; e < DPL; ++e) acc[r][e] *= alpha;
                    m[r] = bm;
                }
                const float ms = m[r] == -INFINITY ? 0.f : m[r];
                p[r] = ok ? fast_exp2(x - ms) : 0.f;
                l[r] += p[r];
            }
            // ---- step 7: O += p V over this warp's 32 keys, V from the ring, p from shared memory
            float *pw = pbuf + warp * 32 * ROWS;
#pragma unroll
            for (int r4 = 0; r4 < ROWS / 4; ++r4)
                reinterpret_cast<float4 *>(pw + lane * ROWS)[r4] = make_float4(p[4 * r4], p[4 * r4 + 1], p[4 * r4 + 2], p[4 * r4 + 3]);
            __syncwarp();
            wait(bar_s + 8 * st, u & 1);
            int nk = (int)(k1 - kb);
            nk = nk < 0 ? 0 : (nk > 32 ? 32 : nk);
            const uint8_t *vrow = vring + st * VT + (size_t)(sub * 32) * DV * 2 + lane * DPL * 2;
#pragma unroll 8
            for (int kk = 0; kk < nk; ++kk) {
                float vv[4];
                if (DPL == 4) {
                    const uint2 w = *reinterpret_cast<const uint2 *>(vrow + (size_t)kk * DV * 2);
                    vv[0] = __uint_as_float(w.x << 16);
                    vv[1] = __uint_as_float(w.x & 0xFFFF0000u);
                    vv[2] = __uint_as_float(w.y << 16);
                    vv[3] = __uint_as_float(w.y & 0xFFFF0000u);
                } else {
                    const uint32_t w = *reinterpret_cast<const uint32_t *>(vrow + (size_t)kk * DV * 2);
                    vv[0] = __uint_as_float(w << 16);
                    vv[1] = __uint_as_float(w & 0xFFFF0000u);
                }
                const float4 *pk4 = reinterpret_cast<const float4 *>(pw + kk * ROWS);
#pragma unroll
                for (int r4 = 0; r4 < ROWS / 4; ++r4) {
                    const float4 pp = pk4[r4];  // broadcast read
                    const float pr[4] = {pp.x, pp.y, pp.z, pp.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = 4 * r4 + q;
#pragma unroll
                        for (int e = 0; e < DPL; e += 2)
                            sm100::ffma2v(acc[r][e], acc[r][e + 1], vv[e], vv[e + 1], pr[q], pr[q], acc[r][e], acc[r][e + 1]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_s + 8 * (NST + st)) : "memory");
        }
    }
    __syncthreads();  // every V block consumed: the ring is reused for the warps' partials
    float *red_m = reinterpret_cast<float *>(vring);           // [CW][ROWS]
    float *red_l = red_m + CW * ROWS;                          // [CW][ROWS]
    float *red_o = red_l + CW * ROWS;                          // [CW][ROWS][DV]
    if (warp < CW) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            float ls = l[r];  // per-lane partial sums -> the warp's l
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
            if (lane == 0) {
                red_m[warp * ROWS + r] = m[r];
                red_l[warp * ROWS + r] = ls;
            }
#pragma unroll
            for (int e = 0; e < DPL; ++e) red_o[(warp * ROWS + r) * DV + lane * DPL + e] = acc[r][e];
        }
    }
    __syncthreads();
    float *part = a.part + ((int64_t)bg * a.nsplit + split) * ROWS * (2 + DV);
    for (int x = threadIdx.x; x < ROWS * DV; x += blockDim.x) {
        const int r = x / DV, c = x % DV;
        float M = -INFINITY;
        for (int w = 0; w < CW; ++w) M = fmaxf(M, red_m[w * ROWS + r]);
        const float Ms = M == -INFINITY ? 0.f : M;
        float L = 0.f, O = 0.f;
        for (int w = 0; w < CW; ++w) {
            const float f = fast_exp2(red_m[w * ROWS + r] - Ms);
            L += red_l[w * ROWS + r] * f;
            O += red_o[(w * ROWS + r) * DV + c] * f;
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

template <int DV, int ROWS, int DB, int NST>
cudaError_t launch_decode_t(const DecArgs &a, cudaStream_t st) {
    // consumer warps = DB / 32: every V block is consumed by ALL consumer warps (one group).  With two
    // groups taking alternate blocks of one shared stage ring (the round-1 shape for <= 4 rows: 16 warps,
    // 256-key blocks), a group can wait on a stage's full barrier two phases ahead of the other group's
    // use of that stage, and the parity test then passes on the wrong phase.
    constexpr int CW = DB / 32;
    const size_t smem = ((size_t)ROWS * a.d * 4 + (size_t)CW * 32 * ROWS * 4 + 1023) / 1024 * 1024 +
                        (size_t)NST * DB * DV * 2 + 2 * NST * 8 + 1024;
    static_assert((size_t)CW * ROWS * (2 + DV) * 4 <= (size_t)NST * DB * DV * 2, "merge area fits the V ring");
    auto kern = decode_partial_kernel<DV, ROWS, CW, DB, NST>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 g1(a.B * a.H_kv, a.nsplit);
    kern<<<g1, CW * 32 + 32, smem, st>>>(a);
    dim3 g2(a.B * a.H_kv, ROWS);
    decode_combine_kernel<DV, ROWS><<<g2, DV, 0, st>>>(a);
    return cudaGetLastError();
}

// the V block size of a launch: 128 keys (two CTAs per SM) for up to 4 rows per kv head -- more rows
// need more registers than two CTAs of 288 threads leave (spills) -- else 256
int dec_db_for(int rows) { return rows <= 4 ? dec_db() : 256; }

template <int DV, int ROWS>
cudaError_t launch_decode_r(const DecArgs &a, cudaStream_t st) {
    if constexpr (ROWS <= 4) {
        if (dec_db_for(ROWS) != 256) {
            return dec_cfg() == 128 ? launch_decode_t<DV, ROWS, 128, 3>(a, st) : launch_decode_t<DV, ROWS, 128, 2>(a, st);
        }
    }
    return launch_decode_t<DV, ROWS, 256, 3>(a, st);
}

}  // namespace

// keys per split: a multiple of 32 (one consumer warp's slice); splits need not be whole V blocks
int64_t decode_chunk(int64_t n_kv, int nsplit) { return ((n_kv + nsplit - 1) / nsplit + 31) / 32 * 32; }

int decode_nsplit(int64_t bh_kv, int64_t n_kv, int DB) {
    // 148 x (1 or 2) resident CTAs (the V ring is ~200 KB or ~100 KB).  Pick the split count that minimises the streaming time
    // waves x keys-per-CTA plus a per-wave ramp (first V block latency + merge, ~512 keys' worth),
    // among splits of >= 2 V blocks and at most SFA_DEC_WAVES * 2 waves: a last wave that is mostly
    // empty costs as much as a full one.
    const int64_t per_wave = 148 * (DB == 256 ? 1 : dec_minb_rt());
    const int64_t maxs = (n_kv + 2 * DB - 1) / (2 * DB);
    int best = 1;
    double best_cost = 1e300;
    for (int64_t s = 1; s <= maxs && s <= 4096; ++s) {
        const int64_t ctas = bh_kv * s;
        const int64_t waves = (ctas + per_wave - 1) / per_wave;
        if (waves > 2 * SFA_DEC_WAVES && s > 1) break;
        const double cost = (double)waves * ((double)decode_chunk(n_kv, (int)s) + 2.0 * DB);
        if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = (int)s;
        }
    }
    return best;
}

size_t decode_workspace_bytes(int64_t bh_kv, int64_t n_kv, int d_v) {
    const int s = std::max(decode_nsplit(bh_kv, n_kv, dec_db()), decode_nsplit(bh_kv, n_kv, 256));
    return (size_t)bh_kv * s * MAXROWS * (2 + d_v) * 4;
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
    a.nsplit = decode_nsplit((int64_t)p.B * p.H_kv, p.n_kv, dec_db_for(rows));
    a.chunk = decode_chunk(p.n_kv, a.nsplit);
    if (rows <= 4) return d_v == 64 ? launch_decode_r<64, 4>(a, st) : launch_decode_r<128, 4>(a, st);
    if (rows <= 8) return d_v == 64 ? launch_decode_r<64, 8>(a, st) : launch_decode_r<128, 8>(a, st);
    return d_v == 64 ? launch_decode_r<64, 16>(a, st) : launch_decode_r<128, 16>(a, st);
}

}  // namespace sfa
