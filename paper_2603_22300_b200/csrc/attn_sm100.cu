// attn_sm100.cu -- FlashSFA forward on sm_100a tensor cores (steps 4-8 of DESIGN.md; Alg. 1
// P:L701-755, Sec. 3.2).
//
// The logits s_ij = scale * sum_{u in S_i and S_j} q~_iu k~_ju are exactly the dot
// products of the DECOMPRESSED k-sparse rows (zeros off the support, reading A1/R1), so a key
// tile's scores are one dense contraction S = Q~ . K~^T.  On B200 that contraction is cheapest
// on the 5th-generation tensor cores even though 1 - k/d of the operands are zero: a 128x128x128
// bf16 tcgen05 MMA costs 512 tensor-pipe clocks, the shared-memory scatter over feature buckets
// (kernel attn_simt.cu) about 4000 LSU clocks at k=16, d=128 (DESIGN.md "Why the scores run on
// tensor cores").  What sparsity still buys on B200 is traffic: a key arrives as its k-sparse
// code (3k bytes) instead of a dense d-vector (2d bytes) and is decompressed into shared memory
// on chip.  Products of bf16 values are exact in fp32, so the MMA computes the same sums as the
// scatter up to fp32 summation order.
//
// One CTA per work item = two 128-row query tiles that read the same key/value sequence (two
// query heads of one GQA group at the same query block, or two consecutive query blocks of one
// head).  Warp roles (512 threads):
//   warps 0-3   softmax for query tile 0  (thread = query row = TMEM lane)
//   warps 4-7   softmax for query tile 1
//   warps 8-11  decompression: Q~ tiles once, then K~ tile j from the key codes (thread = key),
//               into a 2-stage ring of 128B-swizzled K-major UMMA operand tiles
//   warp 12     tcgen05.mma issuer (one thread) + TMEM owner
//   warp 13     TMA producer for the V tiles (3-D tensor map, 128B swizzle, 2-stage ring)
// TMEM (512 columns): S_t / P_t at columns [128t, 128t+128), O_t at [256 + t*d_v, ...).
// Per key tile j the MMA warp issues  O_0 += P_0(j) V(j),  S_0(j+1) = Q~_0 K~(j+1)^T,
//                                     O_1 += P_1(j) V(j),  S_1(j+1) = Q~_1 K~(j+1)^T
// so each softmax group computes exp2 while the tensor pipe works for the other group.
// Softmax: scores are scaled by scale*log2(e) in fp32 (FFMA), row max, ex2.approx per allowed
// pair (causal / ragged keys excluded, step 5), P packed to bf16 (RNE, reading A12) into the
// TMEM columns of S, the lazy O rescale (only when the running max grows by more than 2^8)
// done on TMEM rows; epilogue O/l -> bf16 (RNE), LSE = (m + log2 l) ln 2 (step 8).
#include <cudaTypedefs.h>
#include <mutex>

#include "launch.cuh"
#include "sm100.cuh"

namespace sfa {
using namespace sm100;

namespace {

constexpr int BM = 128;  // query rows per tile (UMMA M)
constexpr int BN = 128;  // keys per tile (UMMA N of S, UMMA K of P.V)
constexpr int NTHREADS = 512;

template <int D, int DV>
struct Cfg {
    static constexpr int QT = BM * D * 2;  // bytes of one decompressed Q~ tile
    static constexpr int KT = BN * D * 2;  // one K~ stage
    static constexpr int VT = BN * DV * 2; // one V stage
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + 2 * QT;
    static constexpr int OFF_V = OFF_K + 2 * KT;
    static constexpr int OFF_BAR = OFF_V + 2 * VT;
    static constexpr int SMEM = OFF_BAR + 256 + 1024;  // + slack to align the base to 1024 B
    static constexpr int O_COL = 256;
};

// mbarrier slots
enum { KFULL = 0, KEMPTY = 2, VFULL = 4, VEMPTY = 6, SFULL = 8, PFULL = 10, OFULL = 12, QFULL = 13, NBAR = 14 };

struct Sm100Args {
    AttnParams p;
    int32_t nqb;         // ceil(n_q / BM)
    int32_t pair_heads;  // 1: tiles (2hp, 2hp+1) at one q block; 0: (h, 2p), (h, 2p+1)
    int32_t per_rank;    // work items per q-block rank
    int32_t nkt;         // ceil(n_kv / BN)
    float c_scale;       // scale * log2(e)
    float *dbg;          // optional: raw S of the first key tile of work item 0, tile 0 (tests)
};

// P is stored as fp16 * 2^P_SHIFT: with the lazy-rescale threshold 2^8 every weight is <= 2^15
// (fp16 max 65504) and weights down to 2^-31 of the running max stay normal/subnormal-exact enough
// (flush bias <= 2^-32 per key; reading A12).
constexpr float P_SHIFT = 7.f;

struct Tile {
    int h, qb;
    bool valid;
};

__device__ __forceinline__ void decode_item(const Sm100Args &a, int item, int &b, Tile (&t)[2]) {
    const AttnParams &p = a.p;
    const int rank = item / a.per_rank, rest = item % a.per_rank;
    if (a.pair_heads) {
        const int qb = a.nqb - 1 - rank;  // heaviest causal blocks first (LPT)
        const int hp2 = p.H / 2;
        b = rest / hp2;
        const int hp = rest % hp2;
        t[0] = {2 * hp, qb, true};
        t[1] = {2 * hp + 1, qb, true};
    } else {
        const int npairs = (a.nqb + 1) / 2;
        const int pr = npairs - 1 - rank;
        b = rest / p.H;
        const int h = rest % p.H;
        t[0] = {h, 2 * pr, 2 * pr < a.nqb};
        t[1] = {h, 2 * pr + 1, 2 * pr + 1 < a.nqb};
    }
}

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

// zero row r of a swizzled tile (D features) then write its k code values
template <int D>
__device__ __forceinline__ void densify_row(uint32_t tile, int rows, int r, bool valid, const uint8_t *__restrict__ idx,
                                            const uint16_t *__restrict__ val, int k) {
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

// Debug timeline (build with SFA_NVCC_FLAGS=-DSFA_TIMELINE): CTA 0 appends (tag, clock64) records
// after the score tile in the diagnostic buffer of sfa_debug_sm100_scores.
#ifdef SFA_TIMELINE
// slot = (kind-1) * 2048 + group * 1024 + j: a plain store, no atomic on the critical path
#define TLREC(tag)                                                                                   \
    do {                                                                                             \
        if (a.dbg != nullptr && blockIdx.x == 0) {                                                   \
            unsigned long long *tb_ = reinterpret_cast<unsigned long long *>(a.dbg + BM * BN);       \
            const unsigned slot_ = ((((tag) >> 12) - 1) << 11) | ((tag) & 2047);                    \
            if (slot_ < 8191) tb_[1 + slot_] = ((unsigned long long)(tag) << 48) | (clock64() & 0xFFFFFFFFFFFFull); \
        }                                                                                            \
    } while (0)
#else
#define TLREC(tag) do {} while (0)
#endif

template <int D, int DV>
__global__ void __launch_bounds__(NTHREADS, 1) attn_sm100_kernel(const __grid_constant__ CUtensorMap tmap_v,
                                                                   const Sm100Args a) {
    using C = Cfg<D, DV>;
    const AttnParams &p = a.p;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t sbase = (raw_s + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (sbase - raw_s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = sbase + C::OFF_BAR;
#define BAR(i) (bar0 + 8u * (uint32_t)(i))
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + C::OFF_BAR + 128);

    int b;
    Tile tl[2];
    decode_item(a, blockIdx.x, b, tl);
    const int g = tl[0].h / (p.H / p.H_kv);
    // key tiles this item needs: causal -> up to the diagonal of its last valid row
    int nt = a.nkt;
    if (p.causal) {
        const int qbl = tl[1].valid ? tl[1].qb : tl[0].qb;
        int64_t last = (int64_t)qbl * BM + BM - 1;
        if (last > p.n_q - 1) last = p.n_q - 1;
        const int64_t lim = (p.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i) {
            const uint32_t cnt = (i == KFULL || i == KFULL + 1 || i == PFULL || i == PFULL + 1 || i == QFULL) ? 4u : 1u;
            mbar_init(BAR(i), cnt);
        }
        fence_mbar_init();
    }
    if (warp == 12) tmem_alloc<512>(smem_u32(tmem_slot));
    if (warp == 13 && lane == 0) tma_prefetch_desc(&tmap_v);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // register budget per warpgroup (setmaxnreg): 2 x 184 (softmax) + 64 (decompress) + 80 = 512 x 128
    const int wg = warp >> 2;
    if (wg < 2) {
        reg_alloc<184>();
        // ============================ softmax (steps 5, 6, 8) ============================
        const int t = wg, wq = warp & 3, r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_off + (uint32_t)(t * 128);
        const uint32_t tO = tmem + lane_off + (uint32_t)(C::O_COL + t * DV);
        const int64_t i = (int64_t)tl[t].qb * BM + r;
        const bool row_ok = tl[t].valid && i < p.n_q;
        int64_t kend = p.n_kv;
        if (p.causal && p.q_pos0 + i + 1 < kend) kend = p.q_pos0 + i + 1;
        const float cs = a.c_scale;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            mbar_wait(BAR(SFULL + t), j & 1);
            if (lane == 0 && wq == 0) TLREC(0x1000 | (t << 10) | (j & 1023));
            tc_fence_after();
            uint32_t s[4][32];
#pragma unroll
            for (int q = 0; q < 4; ++q) tmem_ld32(tS + 32 * q, s[q]);
            tmem_ld_wait();
            if (a.dbg != nullptr && blockIdx.x == 0 && t == 0 && j == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c) a.dbg[r * BN + 32 * q + c] = __uint_as_float(s[q][c]);
            }
            int64_t lim64 = kend - (int64_t)j * BN;
            const int lim = lim64 < 0 ? 0 : (lim64 > BN ? BN : (int)lim64);
            if (lim < BN) {  // step 5 on diagonal / ragged tiles: excluded keys -> -inf -> p = 0
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (32 * q + c >= lim) s[q][c] = 0xFF800000u;
            }
#ifdef SFA_MAXTREE
            float mq[4];  // four independent FMNMX3 chains instead of one 64-deep chain
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                mq[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < 32; ++c) mq[q] = fmaxf(mq[q], __uint_as_float(s[q][c]));
            }
            float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
#else
            float mx = -INFINITY;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 32; ++c) mx = fmaxf(mx, __uint_as_float(s[q][c]));
#endif
            mx *= cs;
            if (lane == 0 && wq == 0) TLREC(0x4000 | (t << 10) | (j & 1023));
            const float m_new = fmaxf(m, mx);
            const bool need = m_new > m + 8.f;
            const bool rescale = __any_sync(0xffffffffu, need);  // warp-uniform (tcgen05.ld/st are warp-wide)
            float alpha = 1.f;
            if (rescale) {
                alpha = (m_new == -INFINITY) ? 1.f : fast_exp2(m - m_new);
                l *= alpha;
                m = m_new;
            }
            const float ms = ((m == -INFINITY) ? 0.f : m) - P_SHIFT;  // p = 2^(s - m + P_SHIFT)
            float rs = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // 32 keys -> 16 packed columns; s[q] dies here
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float x0 = fmaf(__uint_as_float(s[q][2 * c]), cs, -ms);
                    const float x1 = fmaf(__uint_as_float(s[q][2 * c + 1]), cs, -ms);
                    float p0, p1;
#if defined(SFA_V1_POLY)
                    if ((c & 3) < SFA_V1_POLY) {
                        exp2_poly2(x0, x1, p0, p1);
                    } else
#endif
                    {
                        p0 = fast_exp2(x0);
                        p1 = fast_exp2(x1);
                    }
                    rs += p0 + p1;
                    pk[c] = pack_f16x2(p0, p1);
                }
                tmem_st16(tS + 16 * q, pk);  // P (bf16 pairs) over the first 64 columns of S
            }
            l += rs;
            if (rescale && j > 0) {  // O holds sum_{j' < j} P V: those MMAs completed before S(j)'s commit
#pragma unroll 1
                for (int q = 0; q < DV / 32; ++q) {
                    uint32_t o[32];
                    tmem_ld32(tO + 32 * q, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
                    tmem_st32(tO + 32 * q, o);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(PFULL + t));
            if (lane == 0 && wq == 0) TLREC(0x2000 | (t << 10) | (j & 1023));
        }
        // ---- epilogue (step 8)
        mbar_wait(BAR(OFULL), 0);
        tc_fence_after();
        // O = 2^e (sum_j P'_j V'_j) / l with V' = V 2^-e (vprep.cu); l carries the same 2^P_SHIFT as P'
        const float inv = l > 0.f ? __uint_as_float((uint32_t)(127 + vprep_head_exp(__ldg(p.v_amax + b * p.H_kv + g))) << 23) / l : 0.f;
        const int64_t orow = ((int64_t)b * p.H + tl[t].h) * p.n_q + i;
#pragma unroll
        for (int q = 0; q < DV / 32; ++q) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * q, o);
            tmem_ld_wait();
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.o) + orow * DV + 32 * q);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    uint4 w;
                    w.x = pack_bf16x2(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
                    w.y = pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
                    w.z = pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
                    w.w = pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
                    dst[v] = w;
                }
            }
        }
        if (row_ok) p.lse[orow] = l > 0.f ? (m + __log2f(l) - P_SHIFT) * 0.69314718055994530942f : -INFINITY;
    } else if (wg == 2) {
        reg_dealloc<64>();
        // ============================ decompression of Q~ and K~ ============================
        const int r = threadIdx.x - 256;
        const int k = p.k;
        const uint16_t *qv = reinterpret_cast<const uint16_t *>(p.q_val);
        const uint16_t *kv = reinterpret_cast<const uint16_t *>(p.k_val);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int64_t i = (int64_t)tl[t].qb * BM + r;
            const bool ok = tl[t].valid && i < p.n_q;
            const int64_t row = ((int64_t)b * p.H + tl[t].h) * p.n_q + i;
            densify_row<D>(sbase + C::OFF_Q + t * C::QT, BM, r, ok, p.q_idx + row * k, qv + row * k, k);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(QFULL));
        const int64_t kv0 = ((int64_t)b * p.H_kv + g) * p.n_kv;
        for (int j = 0; j < nt; ++j) {
            const int s = j & 1, u = j >> 1;
            const int64_t key = (int64_t)j * BN + r;
            const bool ok = key < p.n_kv;
            mbar_wait(BAR(KEMPTY + s), (u & 1) ^ 1);
            densify_row<D>(sbase + C::OFF_K + s * C::KT, BN, r, ok, p.k_idx + (kv0 + key) * k, kv + (kv0 + key) * k, k);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(KFULL + s));
        }
    } else {
        reg_dealloc<80>();
        if (warp == 12) {
            // ============================ tcgen05.mma issuer ============================
            if (lane == 0) {
                constexpr uint32_t idS = umma_idesc_f16kind(BM, BN, 0, 0, 1);  // bf16 Q~ x bf16 K~
                constexpr uint32_t idO = umma_idesc_f16kind(BM, DV, 0, 1, 0);  // fp16 P (TMEM) x fp16 V (smem)
                auto mma_S = [&](int t, int s) {
                    const uint32_t qa = sbase + C::OFF_Q + t * C::QT, ka = sbase + C::OFF_K + s * C::KT;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off_q = (kk >> 2) * BM * 128 + (kk & 3) * 32;
                        const uint32_t off_k = (kk >> 2) * BN * 128 + (kk & 3) * 32;
                        umma_ss(tmem + t * 128, umma_desc_sw128(qa + off_q, 16, 1024),
                                umma_desc_sw128(ka + off_k, 16, 1024), idS, kk > 0);
                    }
                };
                auto mma_O = [&](int t, int s, bool acc) {
                    const uint32_t va = sbase + C::OFF_V + s * C::VT;
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk)
                        umma_ts(tmem + C::O_COL + t * DV, tmem + t * 128 + kk * 8,
                                umma_desc_sw128(va + kk * 2048, BN * 128, 1024), idO, (acc || kk > 0) ? 1u : 0u);
                };
                mbar_wait(BAR(QFULL), 0);
                mbar_wait(BAR(KFULL + 0), 0);
                tc_fence_after();
                mma_S(0, 0);
                umma_commit(BAR(SFULL + 0));
                mma_S(1, 0);
                umma_commit(BAR(SFULL + 1));
                umma_commit(BAR(KEMPTY + 0));
                for (int j = 0; j < nt; ++j) {
                    const int s = j & 1, u = j >> 1;
                    const bool nxt = j + 1 < nt;
                    const int s1 = (j + 1) & 1, u1 = (j + 1) >> 1;
                    mbar_wait(BAR(VFULL + s), u & 1);
                    mbar_wait(BAR(PFULL + 0), j & 1);
                    TLREC(0x3000 | (j & 1023));
                    tc_fence_after();
                    mma_O(0, s, j > 0);
                    if (nxt) {
                        mbar_wait(BAR(KFULL + s1), u1 & 1);
                        tc_fence_after();
                        mma_S(0, s1);
                        umma_commit(BAR(SFULL + 0));
                    }
                    mbar_wait(BAR(PFULL + 1), j & 1);
                    TLREC(0x3400 | (j & 1023));
                    tc_fence_after();
                    mma_O(1, s, j > 0);
                    umma_commit(BAR(VEMPTY + s));
                    if (nxt) {
                        mma_S(1, s1);
                        umma_commit(BAR(SFULL + 1));
                        umma_commit(BAR(KEMPTY + s1));
                    }
                }
                umma_commit(BAR(OFULL));
            }
            __syncwarp();
        } else if (warp == 13) {
            // ============================ TMA producer for V ============================
            if (lane == 0) {
                const int bhkv = b * p.H_kv + g;
                for (int j = 0; j < nt; ++j) {
                    const int s = j & 1, u = j >> 1;
                    mbar_wait(BAR(VEMPTY + s), (u & 1) ^ 1);
                    mbar_arrive_expect_tx(BAR(VFULL + s), C::VT);
                    const uint32_t dst = sbase + C::OFF_V + s * C::VT;
#pragma unroll
                    for (int cb = 0; cb < DV / 64; ++cb)
                        tma_load_3d(dst + cb * BN * 128, &tmap_v, BAR(VFULL + s), cb * 64, j * BN, bhkv);
                }
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 12) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
#undef BAR
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

template <int D, int DV>
cudaError_t launch_t(const Sm100Args &a, cudaStream_t stream, int items) {
    using C = Cfg<D, DV>;
    const AttnParams &p = a.p;
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)DV, (cuuint64_t)p.n_kv, (cuuint64_t)p.B * p.H_kv};
    cuuint64_t strides[2] = {(cuuint64_t)DV * 2, (cuuint64_t)p.n_kv * DV * 2};
    cuuint32_t box[3] = {64, BN, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void *>(p.v16), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    auto kern = attn_sm100_kernel<D, DV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<items, NTHREADS, C::SMEM, stream>>>(tm, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg) {
    if ((d != 64 && d != 128) || (d_v != 64 && d_v != 128)) return cudaErrorNotSupported;
    Sm100Args a;
    a.p = p;
    a.nqb = (int)((p.n_q + BM - 1) / BM);
    a.nkt = (int)((p.n_kv + BN - 1) / BN);
    a.c_scale = p.scale_log2;
    a.dbg = dbg;
    const int R = p.H / p.H_kv;
    a.pair_heads = (R % 2 == 0) ? 1 : 0;
    int64_t items;
    if (a.pair_heads) {
        a.per_rank = p.B * (p.H / 2);
        items = (int64_t)a.per_rank * a.nqb;
    } else {
        a.per_rank = p.B * p.H;
        items = (int64_t)a.per_rank * ((a.nqb + 1) / 2);
    }
    if (items == 0) return cudaSuccess;
    if (items > INT32_MAX) return cudaErrorNotSupported;
    if (d == 64) return d_v == 64 ? launch_t<64, 64>(a, stream, (int)items) : launch_t<64, 128>(a, stream, (int)items);
    return d_v == 64 ? launch_t<128, 64>(a, stream, (int)items) : launch_t<128, 128>(a, stream, (int)items);
}

}  // namespace sfa
