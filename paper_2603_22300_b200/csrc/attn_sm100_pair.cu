// attn_sm100_pair.cu -- FlashSFA forward with M = 256 tensor-core MMAs over a CTA pair
// (tcgen05 cta_group::2; steps 4-8 of DESIGN.md, Alg. 1, Sec. 3.2).
//
// Same method and per-row arithmetic as attn_sm100.cu (scores S = Q~ K~^T of the decompressed codes,
// reading A22; fp16 P x exactly scaled fp16 V, reading A12), laid out for the tensor pipe's rate:
// an M = 128 tcgen05.mma with N <= 128 costs ~100 clocks when its operands stream from shared memory
// (tools/umma_bench.cu), so a single CTA tops out near 16 such MMAs per 16K pairs.  Here two CTAs on
// neighbouring SMs form a cluster; each owns 128 query rows (two heads of one GQA group at the same
// query block, or two consecutive query blocks of one head), and one thread of the leader CTA issues
// M = 256 MMAs that read A (Q~ or P) from each CTA's own shared / tensor memory and B split by N:
// each CTA decompresses only HALF of every key tile (64 keys) and TMA-loads only HALF of V's columns
// (64 of d_v = 128).  Per SM that halves the MMA instructions and the operand traffic per pair.
//
// Per CTA (512 threads):
//   warps 0-7   two softmax groups (keys 0-63 / 64-127 of every tile) for the CTA's 128 rows
//   warps 8-11  decompression: Q~ (128 rows), then 64 keys of every K~ tile (2-stage ring)
//   warp 12     TMEM owner (both CTAs); in the leader, the single-thread MMA issuer
//   warp 13     TMA producer of the CTA's half of every V tile (completion counted on the leader)
// TMEM per CTA: three score buffers [128b, 128b+128) and O at [384, 512): S(j) in buffer j % 3,
// P(j) in place, S(j+3) issued right after O += P(j) V(j) -- the v5 pipeline of attn_sm100.cu's
// history (profiles/r01_timeline_v1.txt).  Hand-offs: producers in both CTAs arrive on the
// leader's full barriers (mapa + release.cluster); the leader's tcgen05.commit multicasts to both.
#include <cudaTypedefs.h>
#include <mutex>

#include "launch.cuh"
#include "sm100.cuh"

namespace sfa {
using namespace sm100;

namespace {

constexpr int BM = 128;         // query rows per CTA (M = 256 per pair)
constexpr int BN = 128;         // keys per tile
constexpr int HALF = BN / 2;    // keys per softmax group; keys decompressed per CTA
constexpr int DV = 128;         // value width (the pair kernel splits it 64 / 64)
constexpr int NTHREADS = 512;
constexpr int NSB = 3;          // score buffers
constexpr float P_SHIFT = 7.f;  // P = fp16 * 2^7 (reading A12)

template <int D>
struct Cfg {
    static constexpr int QT = BM * D * 2;            // this CTA's Q~ tile
    static constexpr int KT = HALF * D * 2;          // this CTA's half of a K~ tile (64 keys)
    static constexpr int VT = BN * (DV / 2) * 2;     // this CTA's half of a V tile (64 columns)
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + QT;
    static constexpr int OFF_V = OFF_K + 2 * KT;
    static constexpr int OFF_RED = OFF_V + 2 * VT;
    static constexpr int OFF_BAR = OFF_RED + 4 * BM * 4;
    static constexpr int SMEM = OFF_BAR + 256 + 1024;
    static constexpr int O_COL = 384;
};

enum {
    KFULL = 0,   // + stage (leader): both CTAs' K~ halves decompressed (4 warps x 2 CTAs)
    KEMPTY = 2,  // + stage (both, multicast commit): S MMA that read it completed
    VFULL = 4,   // + stage (leader): both V halves landed (TMA tx, 2 x VT bytes)
    VEMPTY = 6,  // + stage (both, multicast): P.V MMA that read it completed
    SFULL = 8,   // + buffer (both, multicast): S computed
    PFULL = 11,  // + buffer (leader): P written by both CTAs' softmax groups (8 warps x 2 CTAs)
    OPV = 14,    // + (j & 1) (both, multicast): O += P(j) V(j) completed
    OFULL = 16,  // (both, multicast): all MMAs completed
    QFULL = 17,  // (leader): both Q~ tiles decompressed (4 warps x 2 CTAs)
    NBAR = 18
};

struct PairArgs {
    AttnParams p;
    int32_t nqb;         // ceil(n_q / BM)
    int32_t pair_heads;  // 1: the pair is heads (2hp, 2hp+1) at one q block; 0: q blocks (2p, 2p+1) of one head
    int32_t per_rank;    // pairs per q-block rank
    int32_t nkt;         // ceil(n_kv / BN)
    float c_scale;       // scale * log2(e)
    float *dbg;          // optional: raw S of the first key tile of pair 0, CTA 0 (tests)
};

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

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    attn_sm100_pair_kernel(const __grid_constant__ CUtensorMap tmap_v, const PairArgs a) {
    using C = Cfg<D>;
    const AttnParams &p = a.p;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t sbase = (raw_s + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (sbase - raw_s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = sbase + C::OFF_BAR;
#define BAR(i) (bar0 + 8u * (uint32_t)(i))
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + C::OFF_BAR + 192);
    float *red = reinterpret_cast<float *>(gbase + C::OFF_RED);
    const int rank = (int)cluster_ctarank();
    const bool leader = rank == 0;

    // ---- the pair's work item (heaviest causal blocks first) and this CTA's rows
    const int item = blockIdx.x >> 1;
    const int qrank = item / a.per_rank, rest = item % a.per_rank;
    int b, h, qb, nqb_pair;
    bool valid = true;
    if (a.pair_heads) {
        qb = a.nqb - 1 - qrank;
        b = rest / (p.H / 2);
        h = 2 * (rest % (p.H / 2)) + rank;
        nqb_pair = qb;
    } else {
        const int pr = (a.nqb + 1) / 2 - 1 - qrank;
        b = rest / p.H;
        h = rest % p.H;
        qb = 2 * pr + rank;
        valid = qb < a.nqb;
        nqb_pair = (2 * pr + 1 < a.nqb) ? 2 * pr + 1 : 2 * pr;
    }
    const int g = h / (p.H / p.H_kv);
    int nt = a.nkt;  // identical in both CTAs: the diagonal of the pair's last query block
    if (p.causal) {
        int64_t last = (int64_t)nqb_pair * BM + BM - 1;
        if (last > p.n_q - 1) last = p.n_q - 1;
        const int64_t lim = (p.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i) {
            uint32_t cnt = 1;
            if (i == KFULL || i == KFULL + 1 || i == QFULL) cnt = 8;
            if (i >= PFULL && i < PFULL + NSB) cnt = 16;
            mbar_init(BAR(i), cnt);
        }
        fence_mbar_init();
    }
    if (warp == 12) tmem_alloc_pair<512>(smem_u32(tmem_slot));
    if (warp == 13 && lane == 0) tma_prefetch_desc(&tmap_v);
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // register budget per warpgroup (setmaxnreg): 2 x 152 (softmax) + 96 (decompress) + 112 = 4 x 128
    const int wg = warp >> 2;
    if (wg < 2) {
        reg_alloc<152>();
        // ============================ softmax (steps 5, 6, 8) ============================
        const int grp = wg, wq = warp & 3, r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_off + (uint32_t)(grp * HALF);     // + 128 * buffer
        const uint32_t tP = tmem + lane_off + (uint32_t)(grp * HALF / 2); // P of this group's keys
        const uint32_t tO = tmem + lane_off + (uint32_t)(C::O_COL + grp * (DV / 2));
        const int64_t i = (int64_t)qb * BM + r;
        const bool row_ok = valid && i < p.n_q;
        int64_t kend = p.n_kv;
        if (p.causal && p.q_pos0 + i + 1 < kend) kend = p.q_pos0 + i + 1;
        const float cs = a.c_scale;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            const int bsel = j % NSB;
            mbar_wait_cluster(BAR(SFULL + bsel), (j / NSB) & 1);
            if (lane == 0 && wq == 0) TLREC(0x1000 | (grp << 10) | (j & 1023));
            tc_fence_after();
            uint32_t s[2][32];
            tmem_ld32(tS + 128 * bsel, s[0]);
            tmem_ld32(tS + 128 * bsel + 32, s[1]);
            tmem_ld_wait();
            if (a.dbg != nullptr && blockIdx.x == 0 && j == 0) {
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c) a.dbg[r * BN + grp * HALF + 32 * q + c] = __uint_as_float(s[q][c]);
            }
            const int64_t lim64 = kend - (int64_t)j * BN - grp * HALF;
            const int lim = lim64 < 0 ? 0 : (lim64 > HALF ? HALF : (int)lim64);
            if (lim < HALF) {  // step 5 on diagonal / ragged tiles: excluded keys -> -inf -> p = 0
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (32 * q + c >= lim) s[q][c] = 0xFF800000u;
            }
            float pm0 = __uint_as_float(s[0][0]), pm1 = __uint_as_float(s[0][1]), pm2 = __uint_as_float(s[0][2]),
                  pm3 = __uint_as_float(s[0][3]);
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    pm0 = fmaxf(pm0, __uint_as_float(s[q][c]));
                    pm1 = fmaxf(pm1, __uint_as_float(s[q][c + 1]));
                    pm2 = fmaxf(pm2, __uint_as_float(s[q][c + 2]));
                    pm3 = fmaxf(pm3, __uint_as_float(s[q][c + 3]));
                }
            // exchange partial maxima with the other group (also: both groups now hold S(j)).  The
            // buffer alternates with the tile parity: a group can run at most one tile ahead.
            float *rj = red + (j & 1) * 2 * BM;
            rj[grp * BM + r] = fmaxf(fmaxf(pm0, pm1), fmaxf(pm2, pm3));
            named_bar_sync(1, 256);
            const float mx = fmaxf(rj[r], rj[BM + r]) * cs;
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
            float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
            for (int q = 0; q < 2; ++q) {  // 32 keys -> 16 packed fp16 columns, in place over S
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float p0 = fast_exp2(fmaf(__uint_as_float(s[q][2 * c]), cs, -ms));
                    const float p1 = fast_exp2(fmaf(__uint_as_float(s[q][2 * c + 1]), cs, -ms));
                    ps0 += p0;
                    ps1 += p1;
                    pk[c] = pack_f16x2(p0, p1);
                }
                tmem_st16(tP + 128 * bsel + 16 * q, pk);
            }
            l += ps0 + ps1;
            if (rescale && j > 0) {
                // O holds sum_{j' < j} P V.  S(j) was issued after P V of tile j-3, so the P V MMAs
                // of tiles j-2 and j-1 may still run: wait for P V(j-1) (in-order completion covers
                // j-2).  One barrier per tile parity keeps the wait unambiguous.
                mbar_wait_cluster(BAR(OPV + ((j - 1) & 1)), ((j - 1) >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int q = 0; q < DV / 64; ++q) {
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
            if (lane == 0) mbar_arrive_cluster(BAR(PFULL + bsel), 0);  // on the leader's barrier
            if (lane == 0 && wq == 0) TLREC(0x2000 | (grp << 10) | (j & 1023));
        }
        // ---- epilogue (step 8): combine the two groups' row sums, each group stores half of O
        named_bar_sync(1, 256);
        red[grp * BM + r] = l;
        named_bar_sync(1, 256);
        const float lt = red[r] + red[BM + r];
        mbar_wait_cluster(BAR(OFULL), 0);
        tc_fence_after();
        // O = 2^e (sum_j P'_j V'_j) / l with V' = V 2^-e (vprep.cu); l carries the same 2^P_SHIFT as P'
        const float inv =
            lt > 0.f ? __uint_as_float((uint32_t)(127 + vprep_head_exp(__ldg(p.v_amax + b * p.H_kv + g))) << 23) / lt
                     : 0.f;
        const int64_t orow = ((int64_t)b * p.H + h) * p.n_q + i;
#pragma unroll
        for (int q = 0; q < DV / 64; ++q) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * q, o);
            tmem_ld_wait();
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.o) + orow * DV +
                                                       grp * (DV / 2) + 32 * q);
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
        if (row_ok && grp == 0)
            p.lse[orow] = lt > 0.f ? (m + __log2f(lt) - P_SHIFT) * 0.69314718055994530942f : -INFINITY;
    } else if (wg == 2) {
        reg_dealloc<96>();
        // ============================ decompression of Q~ and this CTA's half of K~ ============================
        const int r = threadIdx.x - 256;
        const int k = p.k;
        const uint16_t *qv = reinterpret_cast<const uint16_t *>(p.q_val);
        const uint16_t *kv = reinterpret_cast<const uint16_t *>(p.k_val);
        {
            const int64_t i = (int64_t)qb * BM + r;
            const bool ok = valid && i < p.n_q;
            const int64_t row = ((int64_t)b * p.H + h) * p.n_q + (ok ? i : 0);
            densify_row<D>(sbase + C::OFF_Q, BM, r, ok, p.q_idx + row * k, qv + row * k, k);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(BAR(QFULL), 0);
        const int64_t kv0 = ((int64_t)b * p.H_kv + g) * p.n_kv;
        for (int j = 0; j < nt; ++j) {
            const int s = j & 1, u = j >> 1;
            mbar_wait_cluster(BAR(KEMPTY + s), (u & 1) ^ 1);
            if (r < HALF) {  // key rows rank*64 + r of tile j
                const int64_t key = (int64_t)j * BN + rank * HALF + r;
                const bool ok = key < p.n_kv;
                densify_row<D>(sbase + C::OFF_K + s * C::KT, HALF, r, ok, p.k_idx + (kv0 + (ok ? key : 0)) * k,
                               kv + (kv0 + (ok ? key : 0)) * k, k);
                fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(BAR(KFULL + s), 0);
        }
    } else {
        reg_dealloc<112>();
        if (warp == 12 && leader) {
            // ============================ tcgen05.mma issuer (leader CTA) ============================
            if (lane == 0) {
                constexpr uint32_t idS = umma_idesc_f16kind(2 * BM, BN, 0, 0, 1);  // bf16 Q~ x bf16 K~
                constexpr uint32_t idO = umma_idesc_f16kind(2 * BM, DV, 0, 1, 0);  // fp16 P x fp16 V
                const uint32_t qa = sbase + C::OFF_Q;
                auto mma_S = [&](int j) {
                    const uint32_t ka = sbase + C::OFF_K + (j & 1) * C::KT;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off_q = (kk >> 2) * BM * 128 + (kk & 3) * 32;
                        const uint32_t off_k = (kk >> 2) * HALF * 128 + (kk & 3) * 32;
                        umma_ss_pair(tmem + (j % NSB) * 128, umma_desc_sw128(qa + off_q, 16, 1024),
                                     umma_desc_sw128(ka + off_k, 16, 1024), idS, kk > 0);
                    }
                };
                auto mma_O = [&](int j) {
                    const uint32_t va = sbase + C::OFF_V + (j & 1) * C::VT;
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk)
                        umma_ts_pair(tmem + C::O_COL, tmem + (j % NSB) * 128 + kk * 8,
                                     umma_desc_sw128(va + kk * 2048, BN * 128, 1024), idO, (j > 0 || kk > 0) ? 1u : 0u);
                };
                mbar_wait_cluster(BAR(QFULL), 0);
                for (int j = 0; j < NSB && j < nt; ++j) {
                    mbar_wait_cluster(BAR(KFULL + (j & 1)), (j >> 1) & 1);
                    tc_fence_after();
                    mma_S(j);
                    umma_commit_pair(BAR(SFULL + j), 3);
                    umma_commit_pair(BAR(KEMPTY + (j & 1)), 3);
                }
                for (int j = 0; j < nt; ++j) {
                    const int s = j & 1, u = j >> 1, bsel = j % NSB;
                    mbar_wait_cluster(BAR(VFULL + s), u & 1);
                    mbar_wait_cluster(BAR(PFULL + bsel), (j / NSB) & 1);
                    if (threadIdx.x == 384) TLREC(0x3000 | (j & 1023));
                    tc_fence_after();
                    mma_O(j);
                    umma_commit_pair(BAR(OPV + (j & 1)), 3);
                    umma_commit_pair(BAR(VEMPTY + s), 3);
                    const int j3 = j + NSB;
                    if (j3 < nt) {
                        mbar_wait_cluster(BAR(KFULL + (j3 & 1)), (j3 >> 1) & 1);
                        tc_fence_after();
                        mma_S(j3);
                        umma_commit_pair(BAR(SFULL + bsel), 3);
                        umma_commit_pair(BAR(KEMPTY + (j3 & 1)), 3);
                    }
                    if (threadIdx.x == 384) TLREC(0x3400 | (j & 1023));
                }
                umma_commit_pair(BAR(OFULL), 3);
            }
            __syncwarp();
        } else if (warp == 13) {
            // ============================ TMA: this CTA's half of every V tile ============================
            if (lane == 0) {
                const int bhkv = b * p.H_kv + g;
                for (int j = 0; j < nt; ++j) {
                    const int s = j & 1, u = j >> 1;
                    mbar_wait_cluster(BAR(VEMPTY + s), (u & 1) ^ 1);
                    if (leader) mbar_arrive_expect_tx(BAR(VFULL + s), 2 * C::VT);
                    tma_load_3d_pair(sbase + C::OFF_V + s * C::VT, &tmap_v, BAR(VFULL + s), rank * (DV / 2), j * BN,
                                     bhkv);
                }
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    cluster_sync();  // the leader's MMAs are complete (OFULL) and both CTAs are done with TMEM
    if (warp == 12) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
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
cudaError_t launch_pair_t(const PairArgs &a, cudaStream_t stream, int pairs) {
    using C = Cfg<D>;
    const AttnParams &p = a.p;
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)DV, (cuuint64_t)p.n_kv, (cuuint64_t)p.B * p.H_kv};
    cuuint64_t strides[2] = {(cuuint64_t)DV * 2, (cuuint64_t)p.n_kv * DV * 2};
    cuuint32_t box[3] = {DV / 2, BN, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void *>(p.v16), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    auto kern = attn_sm100_pair_kernel<D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<2 * pairs, NTHREADS, C::SMEM, stream>>>(tm, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100_pair(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg) {
    if ((d != 64 && d != 128) || d_v != DV) return cudaErrorNotSupported;
    PairArgs a;
    a.p = p;
    a.nqb = (int)((p.n_q + BM - 1) / BM);
    a.nkt = (int)((p.n_kv + BN - 1) / BN);
    a.c_scale = p.scale_log2;
    a.dbg = dbg;
    const int R = p.H / p.H_kv;
    a.pair_heads = (R % 2 == 0) ? 1 : 0;
    int64_t pairs;
    if (a.pair_heads) {
        a.per_rank = p.B * (p.H / 2);
        pairs = (int64_t)a.per_rank * a.nqb;
    } else {
        a.per_rank = p.B * p.H;
        pairs = (int64_t)a.per_rank * ((a.nqb + 1) / 2);
    }
    if (pairs == 0) return cudaSuccess;
    if (2 * pairs > INT32_MAX) return cudaErrorNotSupported;
    return d == 64 ? launch_pair_t<64>(a, stream, (int)pairs) : launch_pair_t<128>(a, stream, (int)pairs);
}

}  // namespace sfa
