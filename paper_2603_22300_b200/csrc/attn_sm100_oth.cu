// attn_sm100_oth.cu -- FlashSFA forward on sm_100a: the transposed-output kernel with Q~ held in TMEM and
// 64-key score halves (steps 4-8 of DESIGN.md; Alg. 1, Sec. 3.2).
// SFA_KERNEL_SM100_OTH.
//
// Same arithmetic as attn_sm100_ot.cu (scores = dense contraction of the decompressed k-sparse rows,
// readings A1/R1 and A22; fp16 P x 2^7 against the per-head exactly scaled fp16 V copy, A12; lazy O
// rescale at 2^8; 1/4 of the exponentials on the FMA pipe, A23; the persistent tile scheduler), laid out
// for the resource that binds the OT kernel, the shared-memory data path (profiles/r02_ot_ab.txt):
//
//   * Q~ of the item's two query tiles lives in TMEM (the A operand of S, TS-MMA), so the score MMAs
//     read only K~ from shared memory: 2 KB per M128 N64 K16 instruction instead of Q~ + K~ = 8 KB per
//     M128 N128 K16 -- the S reads of a 128-key step drop from 1,024 to 512 wavefronts;
//   * TMEM then holds Q~ (128 columns) + O^T (256), so each tile's scores come in 64-key halves
//     S_t(j, h) (64 columns per tile); the softmax treats a half like a key tile (max, lazy rescale,
//     exponentials) and hands P over per half, and O^T += V(j, h)^T P(j, h)^T runs per half (K = 64,
//     N = 256 queries of both tiles);
//   * the MMA warp issues warp-converged with elect.sync: an N = 64 instruction from a one-lane branch
//     costs 56 clk instead of its 32-clock floor (profiles/r02_umma_issue_bench.txt).
// Per 128-key step of both tiles: S 512 + P.V 768 + P stores 512 + K~ / V TMA 512 = 2,304 shared-memory
// wavefronts, against ~2,816 for attn_sm100_ot.cu.
//
// Warp roles (512 threads):
//   warps 0-3 / 4-7  softmax of query tile 0 / 1 (thread = query row = TMEM lane); O^T rescale, epilogue
//   warps 8-11       Q~ of both tiles straight into TMEM (rows built in registers), once per item
//   warp 12          tcgen05.mma issuer (warp-converged, one elected lane) + TMEM owner
//   warp 13          TMA producer for V;  warp 14  TMA producer for K~ + the item claims (scheduler)
// TMEM: Q~_t [t * D/2, ...) (bf16 pairs), S_t [128 + 64 t, +64), O^T [256, 512) (lane = feature).
#include <cudaTypedefs.h>
#include <cstring>
#include <mutex>

#include "densify.cuh"
#include "launch.cuh"
#include "sm100.cuh"

namespace sfa {
using namespace sm100;
using namespace dz;

namespace {

#ifndef SFA_OTH_POLY  // exponentials per group of 8 pairs on the FMA pipe (exp2_poly2, reading A23)
#define SFA_OTH_POLY 2
#endif

constexpr int BM = 128;   // query rows per tile
constexpr int BN = 128;   // keys per K~ / V tile (TMA box)
constexpr int HK = 64;    // keys per score half (UMMA N of S, UMMA K of a P.V half)
constexpr int DV = 128;   // output features (UMMA M of O^T)
constexpr int NTHREADS = 512;
constexpr int NRING = 4;  // work-item ring slots
constexpr float P_SHIFT = 7.f;

template <int D>
struct Cfg {
    static constexpr int KT = BN * D * 2;        // one K~ stage
    static constexpr int VT = BN * DV * 2;       // one V stage
    static constexpr int PT = 2 * BM * BN * 2;   // P of both tiles: [half h][256 rows][64 keys fp16]
    static constexpr int NK = 2, NV = 2;
    static constexpr int OFF_K = 0;
    static constexpr int OFF_V = OFF_K + NK * KT;
    static constexpr int OFF_P = OFF_V + NV * VT;
    static constexpr int OFF_BAR = OFF_P + PT;
    static constexpr int OFF_F = OFF_BAR + 256;  // 2 x 128 fp32 per-query factors (alpha, then 1/l)
    static constexpr int SMEM = OFF_F + 1024 + 1024;
    static constexpr int Q_COL = 0, S_COL = 128, O_COL = 256;
};
static_assert(Cfg<128>::SMEM <= 232448, "shared memory budget");

enum {
    KFULL = 0, KEMPTY = 2, VFULL = 4, VEMPTY = 6, SFULL = 8, SEMPTY = 10, PFULL = 12, PEMPTY = 14, OFULL = 16,
    QFULL = 17, QEMPTY = 18, OEMPTY = 19, IFULL = 20, IEMPTY = 24, NBAR = 28
};

struct OthArgs {
    AttnParams p;
    int32_t nqb, pair_heads, nkt, items;
    float c_scale;
    float *dbg;  // optional: raw S of the first key tile of work item 0, tile 0 (tests)
};

struct Tile {
    int h, qb;
    bool valid;
};
struct ItemGeo {
    int b, g, nt;
    Tile tl[2];
};
// kv-group-major, heaviest causal query blocks first (as attn_sm100_ot.cu)
__device__ __forceinline__ ItemGeo item_geo(const OthArgs &a, int item) {
    const AttnParams &p = a.p;
    ItemGeo G;
    if (a.pair_heads) {
        const int PG = p.H / p.H_kv / 2;
        const int per_g = PG * a.nqb;
        const int gi = item / per_g, rem = item % per_g;
        const int qb = a.nqb - 1 - rem / PG, pl = rem % PG;
        G.b = gi / p.H_kv;
        const int h0 = 2 * ((gi % p.H_kv) * PG + pl);
        G.tl[0] = {h0, qb, true};
        G.tl[1] = {h0 + 1, qb, true};
    } else {
        const int npairs = (a.nqb + 1) / 2;
        const int bh = item / npairs, pr = npairs - 1 - item % npairs;
        G.b = bh / p.H;
        const int h = bh % p.H;
        G.tl[0] = {h, 2 * pr, 2 * pr < a.nqb};
        G.tl[1] = {h, 2 * pr + 1, 2 * pr + 1 < a.nqb};
    }
    G.g = G.tl[0].h / (p.H / p.H_kv);
    int nt = a.nkt;
    if (p.causal) {
        const int qbl = G.tl[1].valid ? G.tl[1].qb : G.tl[0].qb;
        int64_t last = (int64_t)qbl * BM + BM - 1;
        if (last > p.n_q - 1) last = p.n_q - 1;
        const int64_t lim = (p.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }
    G.nt = nt;
    return G;
}
__device__ __forceinline__ int ring_get(volatile int *ring, uint32_t ifull, uint32_t iempty, int m, bool whole_warp) {
    const int slot = m & (NRING - 1);
    mbar_wait(ifull + 8u * slot, (m / NRING) & 1);
    const int item = ring[slot];
    if (whole_warp) __syncwarp();
    if (!whole_warp || (threadIdx.x & 31) == 0) mbar_arrive(iempty + 8u * slot);
    return item;
}

// Debug timeline (SFA_NVCC_FLAGS=-DSFA_TIMELINE, tools/timeline.py ... oth): CTA 0 stores (tag, clock64)
// records after the score tile in the diagnostic buffer; tag = kind << 12 | tile << 10 | half index
#ifdef SFA_TIMELINE
#define TLREC(tag)                                                                                   \
    do {                                                                                             \
        if (a.dbg != nullptr && blockIdx.x == 0) {                                                   \
            unsigned long long *tb_ = reinterpret_cast<unsigned long long *>(a.dbg + BM * BN);       \
            const unsigned slot_ = ((((tag) >> 12) - 1) << 10) | ((((tag) >> 10) & 1) << 9) | ((tag) & 511); \
            if (slot_ < 8191) tb_[1 + slot_] = ((unsigned long long)(tag) << 48) | (clock64() & 0xFFFFFFFFFFFFull); \
        }                                                                                            \
    } while (0)
#else
#define TLREC(tag) do {} while (0)
#endif

// tcgen05 issue from a converged warp: one lane elected inside the asm (no per-instruction waterfall)
__device__ __forceinline__ void umma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_ts_e(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_e(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

// 32 words (features [64c, 64c + 64)) of a Q~ row as bf16 pairs (feature 2w in the low half), from the
// row's ascending code (A4): each word ORs in the entries whose index falls in it -- a merge over the
// sorted code whose cursor (e, f) carries from block c to block c + 1; once per item
__device__ __forceinline__ void q_row_block(const uint8_t *__restrict__ idx, const uint16_t *__restrict__ val, int k,
                                            int c, int &e, int &f, uint32_t (&w)[32]) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        uint32_t word = 0u;
        while ((f >> 1) == 32 * c + q) {
            word |= (uint32_t)__ldg(val + e) << (16 * (f & 1));
            ++e;
            f = e < k ? __ldg(idx + e) : 1 << 20;
        }
        w[q] = word;
    }
}

template <int D, bool DBG>
__global__ void __launch_bounds__(NTHREADS, 1) attn_sm100_oth_kernel(const __grid_constant__ CUtensorMap tmap_v,
                                                                       const __grid_constant__ CUtensorMap tmap_k,
                                                                       const OthArgs a) {
    using C = Cfg<D>;
    const AttnParams &p = a.p;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t sbase = (raw_s + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (sbase - raw_s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = sbase + C::OFF_BAR;
#define BAR(i) (bar0 + 8u * (uint32_t)(i))
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + C::OFF_BAR + 232);
    volatile int *ring = reinterpret_cast<volatile int *>(gbase + C::OFF_BAR + 240);
    float *fac = reinterpret_cast<float *>(gbase + C::OFF_F);

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i) {
            uint32_t cnt = 1;
            if (i == SEMPTY || i == SEMPTY + 1 || i == QFULL) cnt = 4;
            if (i == PFULL || i == PFULL + 1 || i == OEMPTY) cnt = 8;
            if (i >= IEMPTY && i < IEMPTY + NRING) cnt = 14;  // V, MMA, 8 softmax, 4 Q~ warps
            mbar_init(BAR(i), cnt);
        }
        fence_mbar_init();
    }
    if (warp == 12) tmem_alloc<512>(smem_u32(tmem_slot));
    if (warp == 13 && lane == 0) {
        tma_prefetch_desc(&tmap_v);
        tma_prefetch_desc(&tmap_k);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int wg = warp >> 2;
    if (wg < 2) {
        reg_alloc<184>();
        // ============================ softmax (steps 5, 6, 8) ============================
        const int t = wg, wq = warp & 3, r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_off + (uint32_t)(C::S_COL + t * HK);
        const uint32_t tO = tmem + lane_off + (uint32_t)(C::O_COL + t * BM);  // O^T lane = feature r
        const uint32_t prow = sbase + C::OFF_P + (uint32_t)(t * BM + r) * 128u;  // P row (t*128 + r), half 0
        const int bar_id = 1 + t;
        float *f_t = fac + t * BM;
        const float cs = a.c_scale;
        uint32_t sh = 0;  // score halves of this tile consumed so far, over all items
        uint32_t jg = 0;  // key tiles consumed so far, over all items
        for (int m_ = 0;; ++m_) {
            const int item = ring_get(ring, BAR(IFULL), BAR(IEMPTY), m_, true);
            if (item < 0) break;
            const ItemGeo G = item_geo(a, item);
            const Tile my = t ? G.tl[1] : G.tl[0];
            const int64_t i = (int64_t)my.qb * BM + r;
            const bool row_ok = my.valid && i < p.n_q;
            int64_t kend = p.n_kv;
            if (p.causal && p.q_pos0 + i + 1 < kend) kend = p.q_pos0 + i + 1;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < G.nt; ++j, ++jg) {
#pragma unroll 1
                for (int h = 0; h < 2; ++h, ++sh) {
                    mbar_wait(BAR(SFULL + t), sh & 1);
                    const int hx = (2 * j + h) & 511;
                    if (lane == 0 && wq == 0 && m_ == 0) TLREC(0x1000 | (t << 10) | hx);
                    tc_fence_after();
                    uint32_t s[2][32];
                    tmem_ld32(tS, s[0]);
                    tmem_ld32(tS + 32, s[1]);
                    tmem_ld_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(BAR(SEMPTY + t));  // S_t may take the next half
                    if (DBG && blockIdx.x == 0 && m_ == 0 && t == 0 && j == 0) {
#pragma unroll
                        for (int q = 0; q < 2; ++q)
#pragma unroll
                            for (int c = 0; c < 32; ++c) a.dbg[r * BN + HK * h + 32 * q + c] = __uint_as_float(s[q][c]);
                    }
                    const int64_t lim64 = kend - ((int64_t)j * BN + HK * h);
                    const int lim = lim64 < 0 ? 0 : (lim64 > HK ? HK : (int)lim64);
                    float mq0 = -INFINITY, mq1 = -INFINITY;
                    if (lim < HK) {  // step 5 on the diagonal / ragged half: excluded keys -> -inf
#pragma unroll
                        for (int q = 0; q < 2; ++q)
#pragma unroll
                            for (int c = 0; c < 32; ++c)
                                if (32 * q + c >= lim) s[q][c] = 0xFF800000u;
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        mq0 = fmaxf(mq0, __uint_as_float(s[0][c]));
                        mq1 = fmaxf(mq1, __uint_as_float(s[1][c]));
                    }
                    const float m_new = fmaxf(m, fmaxf(mq0, mq1) * cs);
                    // O^T columns are shared by the warpgroup: rescale all of tile t or none of it
                    const bool rescale = named_bar_or(bar_id, 128, m_new > m + 8.f);
                    if (lane == 0 && wq == 0 && m_ == 0) TLREC(0x5000 | (t << 10) | hx);
                    const bool prior = j > 0 || h == 1;  // O^T already holds P.V of this item
                    if (rescale) {
                        const float alpha = (m_new == -INFINITY) ? 1.f : fast_exp2(m - m_new);
                        l *= alpha;
                        m = m_new;
                        if (prior) f_t[r] = alpha;
                    }
                    const float ms = ((m == -INFINITY) ? 0.f : m) - P_SHIFT;  // p = 2^(s - m + P_SHIFT)
                    float rs0 = 0.f, rs1 = 0.f;
                    uint32_t pk[32];
#pragma unroll
                    for (int q = 0; q < 2; ++q)
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            float x0, x1, p0, p1;
                            ffma2(x0, x1, __uint_as_float(s[q][2 * c]), __uint_as_float(s[q][2 * c + 1]), cs, -ms);
                            if ((c & 7) < SFA_OTH_POLY) {
                                exp2_poly2(x0, x1, p0, p1);
                            } else {
                                p0 = fast_exp2(x0);
                                p1 = fast_exp2(x1);
                            }
                            fadd2(rs0, rs1, p0, p1);
                            pk[16 * q + c] = pack_f16x2(p0, p1);
                        }
                    l += rs0 + rs1;
                    // P half h is free once P.V(previous key tile, h) has read it
                    if (lane == 0 && wq == 0 && m_ == 0) TLREC(0x4000 | (t << 10) | hx);
                    mbar_wait(BAR(PEMPTY + h), (jg & 1) ^ 1);
                    if (lane == 0 && wq == 0 && m_ == 0) TLREC(0x7000 | (t << 10) | hx);
                    if (rescale && prior) {
                        // every P.V issued so far must be complete: the last one is P.V(j, 0) (h = 1)
                        // or P.V(j - 1, 1) (h = 0)
                        if (h == 1) mbar_wait(BAR(PEMPTY + 0), jg & 1);
                        else mbar_wait(BAR(PEMPTY + 1), (jg & 1) ^ 1);
                        named_bar_sync(bar_id, 128);  // every row's alpha is in f_t
                        tc_fence_after();
#pragma unroll 1
                        for (int q = 0; q < BM / 32; ++q) {
                            uint32_t o[32];
                            tmem_ld32(tO + 32 * q, o);
                            tmem_ld_wait();
#pragma unroll
                            for (int c = 0; c < 32; c += 4) {
                                const float4 al = *reinterpret_cast<const float4 *>(f_t + 32 * q + c);
                                o[c + 0] = __float_as_uint(__uint_as_float(o[c + 0]) * al.x);
                                o[c + 1] = __float_as_uint(__uint_as_float(o[c + 1]) * al.y);
                                o[c + 2] = __float_as_uint(__uint_as_float(o[c + 2]) * al.z);
                                o[c + 3] = __float_as_uint(__uint_as_float(o[c + 3]) * al.w);
                            }
                            tmem_st32(tO + 32 * q, o);
                        }
                        tmem_st_wait();
                    }
                    // P row (t*128 + r), half h: 16-byte chunk c8 swizzled by row
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8)
                        sts_v4(prow + (uint32_t)h * (2 * BM * 128) + ((uint32_t)(c8 ^ (r & 7)) << 4), pk[4 * c8],
                               pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
                    fence_proxy_async_smem();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(BAR(PFULL + h));
                    if (lane == 0 && wq == 0 && m_ == 0) TLREC(0x2000 | (t << 10) | hx);
                }
            }
            // ---- epilogue (step 8): O = 2^e (sum_j P'_j V'_j) / l, V' = V 2^-e (vprep.cu)
            mbar_wait(BAR(OFULL), m_ & 1);
            tc_fence_after();
            const float inv = l > 0.f ? __uint_as_float((uint32_t)(127 + vprep_head_exp(__ldg(p.v_amax + G.b * p.H_kv + G.g))) << 23) / l : 0.f;
            f_t[r] = inv;
            named_bar_sync(bar_id, 128);
            const uint32_t so = sbase + C::OFF_P + (uint32_t)t * (BM * DV * 2);
#pragma unroll 1
            for (int q = 0; q < BM / 32; ++q) {
                uint32_t o[32];
                tmem_ld32(tO + 32 * q, o);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int qq = 32 * q + c;
                    const float v = __uint_as_float(o[c]) * f_t[qq];
                    const uint32_t addr = so + (uint32_t)qq * (DV * 2) + ((uint32_t)((r >> 3) ^ (qq & 15)) << 4) + (uint32_t)(r & 7) * 2;
                    sts_u16(addr, __bfloat16_as_ushort(__float2bfloat16_rn(v)));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(OEMPTY));  // O^T read out: the next item's first P.V may overwrite it
            named_bar_sync(bar_id, 128);
            const int64_t orow = ((int64_t)G.b * p.H + my.h) * p.n_q + i;
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.o) + orow * DV);
#pragma unroll
                for (int c = 0; c < DV / 8; ++c) dst[c] = lds_v4(so + (uint32_t)r * (DV * 2) + ((uint32_t)(c ^ (r & 15)) << 4));
                p.lse[orow] = l > 0.f ? (m + __log2f(l) - P_SHIFT) * 0.69314718055994530942f : -INFINITY;
            }
            named_bar_sync(5, 2 * BM);  // both tiles' staging read before either stores the next item's P
        }
    } else if (wg == 2) {
        reg_dealloc<64>();
        // ============================ Q~ of both tiles into TMEM (per item) ============================
        const int r = (warp - 8) * 32 + lane;  // warp 8 + w accesses TMEM lanes [32w, 32w + 32)
        const uint32_t lane_off = (uint32_t)((warp - 8) * 32) << 16;
        const uint16_t *qv = reinterpret_cast<const uint16_t *>(p.q_val);
        for (int m_ = 0;; ++m_) {
            const int item = ring_get(ring, BAR(IFULL), BAR(IEMPTY), m_, true);
            if (item < 0) break;
            const ItemGeo G = item_geo(a, item);
            if (m_ > 0) mbar_wait(BAR(QEMPTY), (m_ - 1) & 1);  // the previous item's S MMAs are complete
            tc_fence_after();
#pragma unroll 1
            for (int t = 0; t < 2; ++t) {
                const int64_t i = (int64_t)G.tl[t].qb * BM + r;
                const bool ok = G.tl[t].valid && i < p.n_q;
                const int64_t row = ((int64_t)G.b * p.H + G.tl[t].h) * p.n_q + (ok ? i : 0);
                const uint8_t *ir = p.q_idx + row * p.k;
                const uint16_t *vr = qv + row * p.k;
                int e = 0, f = ok ? __ldg(ir) : 1 << 20;  // an invalid row stays zero
#pragma unroll 1
                for (int c = 0; c < D / 64; ++c) {
                    uint32_t w[32];
                    if (ok && p.k == D) {  // identity code (A4): the row is the value vector
                        const uint4 *src = reinterpret_cast<const uint4 *>(vr) + 8 * c;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const uint4 x = __ldg(src + u);
                            w[4 * u] = x.x; w[4 * u + 1] = x.y; w[4 * u + 2] = x.z; w[4 * u + 3] = x.w;
                        }
                    } else {
                        q_row_block(ir, vr, p.k, c, e, f, w);
                    }
                    tmem_st32(tmem + lane_off + (uint32_t)(C::Q_COL + t * (D / 2) + 32 * c), w);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(QFULL));
        }
    } else {
        reg_dealloc<80>();
        if (warp == 12) {
            // ============================ tcgen05.mma issuer (warp-converged) ============================
            constexpr uint32_t idS = umma_idesc_f16kind(BM, HK, 0, 0, 1);      // bf16 Q~ (TMEM) x bf16 K~ half
            constexpr uint32_t idO = umma_idesc_f16kind(DV, 2 * BM, 1, 0, 0);  // fp16 V^T (MN-major) x fp16 P
            uint32_t kc = 0, sh = 0, vc = 0, jg = 0;  // K~ tiles, S halves issued (per tile), V tiles, key tiles
            // S_t(j, h) for both tiles into the 64-column S buffers, each after its tile read the last half
            auto issue_S = [&](int s, int h) {
                const uint32_t ka = sbase + C::OFF_K + s * C::KT + (uint32_t)h * (HK * 128);
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (sh > 0) mbar_wait(BAR(SEMPTY + t), (sh - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        umma_ts_e(tmem + C::S_COL + t * HK, tmem + C::Q_COL + t * (D / 2) + kk * 8,
                                  umma_desc_sw128(ka + (kk >> 2) * (BN * 128) + (kk & 3) * 32, 16, 1024), idS, kk > 0);
                    umma_commit_e(BAR(SFULL + t));
                }
                ++sh;
            };
            // O^T += V(j, h)^T P(j, h)^T: 64 keys, N = 256 queries of both tiles
            auto issue_PV = [&](int vs, int h, bool acc) {
                const uint32_t va = sbase + C::OFF_V + vs * C::VT, pa = sbase + C::OFF_P + h * (2 * BM * 128);
#pragma unroll
                for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
                    umma_ss_e(tmem + C::O_COL, umma_desc_sw128(va + kk * 2048, BN * 128, 1024),
                              umma_desc_sw128(pa + (kk & 3) * 32, 16, 1024), idO, (acc || kk > 4 * h) ? 1u : 0u);
            };
            int m = 0, item = ring_get(ring, BAR(IFULL), BAR(IEMPTY), 0, true);
            if (item >= 0) {
                ItemGeo G = item_geo(a, item);
                mbar_wait(BAR(QFULL), 0);
                mbar_wait(BAR(KFULL + 0), 0);
                issue_S((int)(kc % C::NK), 0);
                for (;;) {
                    int item_n = -1;
                    ItemGeo Gn = G;
                    for (int j = 0; j < G.nt; ++j, ++jg) {
                        const int s = (int)(kc % C::NK), vs = (int)(vc % C::NV);
                        issue_S(s, 1);  // S(j, 1)
                        umma_commit_e(BAR(KEMPTY + s));
                        ++kc;
                        if (j + 1 == G.nt) umma_commit_e(BAR(QEMPTY));  // Q~ may be rebuilt for the next item
                        // P.V(j, 0)
                        mbar_wait(BAR(VFULL + vs), (vc / C::NV) & 1);
                        mbar_wait(BAR(PFULL + 0), jg & 1);
                        if (m == 0) TLREC(0x3000 | ((2 * j) & 511));
                        if (j == 0 && m > 0) mbar_wait(BAR(OEMPTY), (m - 1) & 1);  // O^T read out
                        tc_fence_after();
                        issue_PV(vs, 0, j > 0);
                        umma_commit_e(BAR(PEMPTY + 0));
                        // the next S half: S(j + 1, 0), or the next item's first (read only now: the K~
                        // producer publishes the next item after this item's last K~ load)
                        if (j + 1 < G.nt) {
                            mbar_wait(BAR(KFULL + (int)(kc % C::NK)), (kc / C::NK) & 1);
                            issue_S((int)(kc % C::NK), 0);
                        } else {
                            item_n = ring_get(ring, BAR(IFULL), BAR(IEMPTY), m + 1, true);
                            if (item_n >= 0) {
                                Gn = item_geo(a, item_n);
                                mbar_wait(BAR(QFULL), (m + 1) & 1);
                                mbar_wait(BAR(KFULL + (int)(kc % C::NK)), (kc / C::NK) & 1);
                                issue_S((int)(kc % C::NK), 0);
                            }
                        }
                        // P.V(j, 1)
                        mbar_wait(BAR(PFULL + 1), jg & 1);
                        if (m == 0) TLREC(0x3000 | ((2 * j + 1) & 511));
                        tc_fence_after();
                        issue_PV(vs, 1, true);
                        umma_commit_e(BAR(PEMPTY + 1));
                        umma_commit_e(BAR(VEMPTY + vs));
                        ++vc;
                    }
                    umma_commit_e(BAR(OFULL));
                    if (item_n < 0) break;
                    G = Gn;
                    ++m;
                }
            }
            __syncwarp();
        } else if (warp == 13) {
            // ============================ TMA producer for V ============================
            if (lane == 0) {
                uint32_t vc = 0;
                for (int m_ = 0;; ++m_) {
                    const int item = ring_get(ring, BAR(IFULL), BAR(IEMPTY), m_, false);
                    if (item < 0) break;
                    const ItemGeo G = item_geo(a, item);
                    const int bhkv = G.b * p.H_kv + G.g;
                    for (int j = 0; j < G.nt; ++j, ++vc) {
                        const int vs = (int)(vc % C::NV);
                        mbar_wait(BAR(VEMPTY + vs), ((vc / C::NV) & 1) ^ 1);
                        mbar_arrive_expect_tx(BAR(VFULL + vs), C::VT);
                        const uint32_t dst = sbase + C::OFF_V + vs * C::VT;
#pragma unroll
                        for (int cb = 0; cb < DV / 64; ++cb)
                            tma_load_3d(dst + cb * BN * 128, &tmap_v, BAR(VFULL + vs), cb * 64, j * BN, bhkv);
                    }
                }
            }
            __syncwarp();
        } else if (warp == 14) {
            // ============================ item claims + TMA producer for K~ ============================
            if (lane == 0) {
                uint32_t kc = 0;
                for (int m_ = 0;; ++m_) {
                    const int slot = m_ & (NRING - 1);
                    mbar_wait(BAR(IEMPTY + slot), ((m_ / NRING) & 1) ^ 1);
                    int item = m_ == 0 ? (int)blockIdx.x : (int)atomicAdd(p.sched, 1u) + (int)gridDim.x;
                    if (item >= a.items) item = -1;
                    ring[slot] = item;
                    mbar_arrive(BAR(IFULL + slot));
                    if (item < 0) break;
                    const ItemGeo G = item_geo(a, item);
                    const int bhkv = G.b * p.H_kv + G.g;
                    for (int j = 0; j < G.nt; ++j, ++kc) {
                        const int s = (int)(kc % C::NK);
                        mbar_wait(BAR(KEMPTY + s), ((kc / C::NK) & 1) ^ 1);
                        mbar_arrive_expect_tx(BAR(KFULL + s), C::KT);
                        const uint32_t dst = sbase + C::OFF_K + s * C::KT;
#pragma unroll
                        for (int cb = 0; cb < D / 64; ++cb)
                            tma_load_3d(dst + cb * BN * 128, &tmap_k, BAR(KFULL + s), cb * 64, j * BN, bhkv);
                    }
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

template <int D>
cudaError_t launch_t(const OthArgs &a, cudaStream_t stream) {
    using C = Cfg<D>;
    const AttnParams &p = a.p;
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap tv, tk;
    memset(&tv, 0, sizeof(tv));
    memset(&tk, 0, sizeof(tk));
    {
        cuuint64_t dims[3] = {(cuuint64_t)DV, (cuuint64_t)p.n_kv, (cuuint64_t)p.B * p.H_kv};
        cuuint64_t strides[2] = {(cuuint64_t)DV * 2, (cuuint64_t)p.n_kv * DV * 2};
        cuuint32_t box[3] = {64, BN, 1};
        if (encode(&tv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void *>(p.v16), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)p.n_kv, (cuuint64_t)p.B * p.H_kv};
        cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)p.n_kv * D * 2};
        cuuint32_t box[3] = {64, BN, 1};
        if (encode(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(p.k_dense), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    auto kern = a.dbg != nullptr ? attn_sm100_oth_kernel<D, true> : attn_sm100_oth_kernel<D, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.sched, 0, sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = a.items < sms ? a.items : sms;
    kern<<<grid, NTHREADS, C::SMEM, stream>>>(tv, tk, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100_oth(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg) {
    if ((d != 64 && d != 128) || d_v != DV) return cudaErrorNotSupported;
    if (p.k_dense == nullptr || p.sched == nullptr || p.edges_only || p.window > 0 || p.q_dense != nullptr)
        return cudaErrorNotSupported;
    OthArgs a;
    a.p = p;
    a.nqb = (int)((p.n_q + BM - 1) / BM);
    a.nkt = (int)((p.n_kv + BN - 1) / BN);
    a.c_scale = p.scale_log2;
    a.dbg = dbg;
    const int R = p.H / p.H_kv;
    a.pair_heads = (R % 2 == 0) ? 1 : 0;
    const int64_t items = a.pair_heads ? (int64_t)p.B * (p.H / 2) * a.nqb : (int64_t)p.B * p.H * ((a.nqb + 1) / 2);
    if (items == 0) return cudaSuccess;
    if (items > INT32_MAX) return cudaErrorNotSupported;
    a.items = (int)items;
    return d == 64 ? launch_t<64>(a, stream) : launch_t<128>(a, stream);
}

}  // namespace sfa
