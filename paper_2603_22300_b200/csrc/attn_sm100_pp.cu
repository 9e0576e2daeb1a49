// attn_sm100_pp.cu -- FlashSFA forward on sm_100a tensor cores, two query tiles in PING-PONG
// (steps 4-8 of DESIGN.md; Alg. 1, Sec. 3.2).  SFA_KERNEL_SM100_PP.
//
// Same arithmetic as attn_sm100_ot.cu (scores = dense contraction of the decompressed k-sparse rows,
// reading A1/R1 and A22; fp16 P x 2^7 against the per-head exactly scaled fp16 V copy, reading A12;
// lazy O rescale at 2^8; 1/4 of the exponentials on the FMA pipe, reading A23), arranged to spend as
// little shared-memory bandwidth as possible -- the OT kernel's binding resource (tensor-core operand
// reads + P stores + decompression ~90 % of the shared-memory data path, profiles/r02_ot_ab.txt):
//
//   * K~ tiles arrive by TMA from the decompressed key rows the prepare step writes once per key
//     (k_dense_kernel, vprep.cu) instead of being rebuilt in shared memory once per work item;
//   * P stays in TMEM (fp16 pairs over the first 64 columns of its S tile) and O_t += P_t V(j) reads it
//     there (TS-MMA): no P stores, no P operand reads;
//   per 128-key step of both tiles: S reads 1,024 wavefronts, P.V reads 512, the two TMA tiles 512,
//   against ~2,900 for the OT kernel.
//
// The price is the chain softmax_t(j) -> O_t += P_t V(j) -> S_t(j+1) -> softmax_t(j+1) per tile (S_t
// and P_t share TMEM columns).  The two tiles hide it for each other: while tile t exponentiates, the
// tensor pipe runs the other tile's P.V and next S.  The exponential phases of the two softmax
// warpgroups strictly alternate (named barriers 1 and 2), so each has the SM's MUFU units to itself
// and neither can drift into lockstep with the other.
//
// Warp roles (640 threads):
//   warps 0-7   softmax for query tile 0: warp w = TMEM lanes [32 (w % 4), +32) (thread = query row) x
//               key half (w / 4) of every tile, so each SMSP runs two warps per tile; the two halves of a
//               row exchange their partial max through shared memory (named barrier 3 + t); each half
//               rescales and writes back its d_v/2 output columns.  Warps 0-7 also build the Q~ tiles.
//   warps 8-15  softmax for query tile 1
//   warp 16     tcgen05.mma issuer (one thread) + TMEM owner
//   warp 17     TMA producer for V (fp16 copy, NV-stage ring)
//   warp 18     TMA producer for K~ (bf16 decompressed rows, NK-stage ring)
// TMEM (512 columns): S_0/P_0 [0,128), S_1/P_1 [128,256), O_0 [256, 256+DV), O_1 [256+DV, 256+2DV).
// MMA order per key tile j: O_0 += P_0(j) V(j), S_0(j+1), O_1 += P_1(j) V(j), S_1(j+1).
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

// exponentials per group of 8 pairs on the FMA pipe (exp2_poly2, reading A23)
#ifndef SFA_PP_POLY
#define SFA_PP_POLY 2
#endif
// 1: the two softmax warpgroups' exponential phases strictly alternate; 0: free running
#ifndef SFA_PP_PINGPONG
#define SFA_PP_PINGPONG 1
#endif
#ifndef SFA_PP_NK  // K~ / V ring depths (Q~ 2 x 32 KB + (NK + NV) x 32 KB <= 227 KB at d = d_v = 128)
#define SFA_PP_NK 2
#endif
#ifndef SFA_PP_NV
#define SFA_PP_NV 2
#endif

constexpr int BM = 128;  // query rows per tile (UMMA M)
constexpr int BN = 128;  // keys per tile (UMMA N of S, UMMA K of P.V)
constexpr int NTHREADS = 640;  // 16 softmax warps + MMA + 2 TMA + 1 spare
constexpr float P_SHIFT = 7.f;  // P stored as fp16 * 2^7 (reading A12)

template <int D, int DV>
struct Cfg {
    static constexpr int QT = BM * D * 2;   // one decompressed Q~ tile
    static constexpr int KT = BN * D * 2;   // one K~ stage
    static constexpr int VT = BN * DV * 2;  // one V stage
    static constexpr int NK = SFA_PP_NK;    // K~ stages
    static constexpr int NV = SFA_PP_NV;    // V stages
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + 2 * QT;
    static constexpr int OFF_V = OFF_K + NK * KT;
    static constexpr int OFF_BAR = OFF_V + NV * VT;
    static constexpr int OFF_X = OFF_BAR + 256;  // row-max exchange [2][2][2][128] + row sums [2][2][128], fp32
    static constexpr int SMEM = OFF_X + (8 + 4) * BM * 4 + 1024;  // + slack to align the base to 1024 B
    static constexpr int O_COL = 256;
};
static_assert(Cfg<128, 128>::SMEM <= 232448, "shared memory budget");

// mbarrier slots (rings up to 4 deep); the TMEM base address lives at OFF_BAR + 240
enum { KFULL = 0, KEMPTY = 4, VFULL = 8, VEMPTY = 12, SFULL = 16, PFULL = 18, OFULL = 20, QFULL = 21, NBAR = 22 };
static_assert(SFA_PP_NK <= 4 && SFA_PP_NV <= 4, "ring depth");

struct PpArgs {
    AttnParams p;
    int32_t nqb;         // ceil(n_q / BM)
    int32_t pair_heads;  // 1: tiles (2hp, 2hp+1) at one q block; 0: (h, 2p), (h, 2p+1)
    int32_t nkt;         // ceil(n_kv / BN)
    float c_scale;       // scale * log2(e)
    float *dbg;          // optional: raw S of the first key tile of work item 0, tile 0 (tests)
};

struct Tile {
    int h, qb;
    bool valid;
};

// kv-group-major work order (as attn_sm100_ot.cu): all items of one (batch, kv head) group back to
// back, heaviest causal query blocks first, so the resident CTAs share one group's K~ and V in L2
__device__ __forceinline__ void decode_item(const PpArgs &a, int item, int &b, Tile (&t)[2]) {
    const AttnParams &p = a.p;
    if (a.pair_heads) {
        const int PG = p.H / p.H_kv / 2;  // head pairs per kv group
        const int per_g = PG * a.nqb;
        const int gi = item / per_g, rem = item % per_g;
        const int qb = a.nqb - 1 - rem / PG, pl = rem % PG;
        b = gi / p.H_kv;
        const int h0 = 2 * ((gi % p.H_kv) * PG + pl);
        t[0] = {h0, qb, true};
        t[1] = {h0 + 1, qb, true};
    } else {
        const int npairs = (a.nqb + 1) / 2;
        const int bh = item / npairs, pr = npairs - 1 - item % npairs;
        b = bh / p.H;
        const int h = bh % p.H;
        t[0] = {h, 2 * pr, 2 * pr < a.nqb};
        t[1] = {h, 2 * pr + 1, 2 * pr + 1 < a.nqb};
    }
}

// Debug timeline (SFA_NVCC_FLAGS=-DSFA_TIMELINE, tools/timeline.py ... pp): CTA 0 stores (tag, clock64)
// records after the score tile in the diagnostic buffer; tag = kind << 12 | tile << 10 | j
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

__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int D, int DV, bool DBG>
__global__ void __launch_bounds__(NTHREADS, 1) attn_sm100_pp_kernel(const __grid_constant__ CUtensorMap tmap_v,
                                                                      const __grid_constant__ CUtensorMap tmap_k,
                                                                      const PpArgs a) {
    using C = Cfg<D, DV>;
    const AttnParams &p = a.p;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t sbase = (raw_s + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (sbase - raw_s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = sbase + C::OFF_BAR;
#define BAR(i) (bar0 + 8u * (uint32_t)(i))
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + C::OFF_BAR + 240);

    int b;
    Tile tl[2];
    decode_item(a, blockIdx.x, b, tl);
    const int g = tl[0].h / (p.H / p.H_kv);
    int nt = a.nkt;  // key tiles of this item: causal -> up to the diagonal of its last valid row
    if (p.causal) {
        const int qbl = tl[1].valid ? tl[1].qb : tl[0].qb;
        int64_t last = (int64_t)qbl * BM + BM - 1;
        if (last > p.n_q - 1) last = p.n_q - 1;
        const int64_t lim = (p.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i)
            mbar_init(BAR(i), (i == PFULL || i == PFULL + 1 || i == QFULL) ? 8u : 1u);
        fence_mbar_init();
    }
    if (warp == 16) tmem_alloc<512>(smem_u32(tmem_slot));
    if (warp == 17 && lane == 0) {
        tma_prefetch_desc(&tmap_v);
        tma_prefetch_desc(&tmap_k);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 16) {
        // 640 threads x 96 registers fill the register file; the softmax fits in 96 (64 scores per thread)
        // without spills, so no setmaxnreg (an .inc would wait for a .dec that no warp can afford)
        // ============================ softmax (steps 5, 6, 8) ============================
        // 8 warps per query tile: lane quarter wq = TMEM lanes [32 wq, 32 wq + 32) = rows, key half
        // h = keys [64 h, 64 h + 64) of every tile (so each SMSP runs two warps of each tile)
        const int t = warp >> 3, wq = warp & 3, h = (warp >> 2) & 1, r = wq * 32 + lane;
        const Tile mt = t ? tl[1] : tl[0];  // (a select, not a dynamically indexed local array)
        // ---- the two Q~ tiles (step 4's A operands), once: thread per row, warps 0-7
        if (warp < 8) {
            const int tq = warp >> 2, rq = (warp & 3) * 32 + lane;  // tile, row
            const Tile qt = tq ? tl[1] : tl[0];
            const int64_t iq = (int64_t)qt.qb * BM + rq;
            const bool ok = qt.valid && iq < p.n_q;
            const int64_t row = ((int64_t)b * p.H + qt.h) * p.n_q + (ok ? iq : 0);
            densify_row<D>(sbase + C::OFF_Q + tq * C::QT, BM, rq, ok, p.q_idx + row * p.k,
                           reinterpret_cast<const uint16_t *>(p.q_val) + row * p.k, p.k);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(QFULL));
        }
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_off + (uint32_t)(t * 128);
        const uint32_t tO = tmem + lane_off + (uint32_t)(C::O_COL + t * DV + h * (DV / 2));
        float *xmax = reinterpret_cast<float *>(gbase + C::OFF_X);           // [parity][tile][half][128]
        float *xsum = xmax + 2 * 2 * 2 * BM;                                  // [tile][half][128]
        const int64_t i = (int64_t)mt.qb * BM + r;
        const bool row_ok = mt.valid && i < p.n_q;
        int64_t kend = p.n_kv;
        if (p.causal && p.q_pos0 + i + 1 < kend) kend = p.q_pos0 + i + 1;
        const float cs = a.c_scale;
#if SFA_PP_PINGPONG
        if (t == 1 && nt > 0) named_bar_arrive(1, 512);  // tile 0 exponentiates first
#endif
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            mbar_wait(BAR(SFULL + t), j & 1);
            if (lane == 0 && wq == 0 && h == 0) TLREC(0x1000 | (t << 10) | (j & 1023));
            tc_fence_after();
            uint32_t s[2][32];
            tmem_ld32(tS + 64 * h, s[0]);
            tmem_ld32(tS + 64 * h + 32, s[1]);
            tmem_ld_wait();
            if (DBG && blockIdx.x == 0 && t == 0 && j == 0) {
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c) a.dbg[r * BN + 64 * h + 32 * q + c] = __uint_as_float(s[q][c]);
            }
            int64_t lim64 = kend - (int64_t)j * BN - 64 * h;  // allowed keys of this half
            const int lim = lim64 < 0 ? 0 : (lim64 > 64 ? 64 : (int)lim64);
            if (lim < 64) {  // step 5 on diagonal / ragged tiles: excluded keys -> -inf -> p = 0
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (32 * q + c >= lim) s[q][c] = 0xFF800000u;
            }
            float mq0 = -INFINITY, mq1 = -INFINITY;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                mq0 = fmaxf(mq0, __uint_as_float(s[0][c]));
                mq1 = fmaxf(mq1, __uint_as_float(s[1][c]));
            }
            // the row max over both halves: exchange through shared memory (double-buffered by parity)
            float *xm = xmax + ((j & 1) * 2 + t) * 2 * BM;
            xm[h * BM + r] = fmaxf(mq0, mq1);
            named_bar_sync(3 + t, 256);
            const float mx = fmaxf(xm[r], xm[BM + r]) * cs;  // same value in both halves
            const float m_new = fmaxf(m, mx);
            // O_t row r lives in TMEM lane r; tcgen05.ld/st are warp-wide, so a warp rescales if any of
            // its rows needs it (alpha = 1 for the others); each half rescales its DV/2 columns
            const bool need = m_new > m + 8.f;
            const bool rescale = __any_sync(0xffffffffu, need);
            float alpha = 1.f;
            if (need) {
                alpha = (m_new == -INFINITY) ? 1.f : fast_exp2(m - m_new);
                l *= alpha;
                m = m_new;
            }
            const float ms = ((m == -INFINITY) ? 0.f : m) - P_SHIFT;  // p = 2^(s - m + P_SHIFT)
            if (lane == 0 && wq == 0 && h == 0) TLREC(0x4000 | (t << 10) | (j & 1023));
#if SFA_PP_PINGPONG
            named_bar_sync(1 + t, 512);  // this tile's turn on the MUFU units
#endif
            if (lane == 0 && wq == 0 && h == 0) TLREC(0x5000 | (t << 10) | (j & 1023));
            float rs0 = 0.f, rs1 = 0.f, rs2 = 0.f, rs3 = 0.f;
#pragma unroll
            for (int q = 0; q < 2; ++q) {  // 32 keys -> 16 packed fp16 columns of P (S's first 64 columns)
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    float x0, x1, p0, p1;
                    ffma2(x0, x1, __uint_as_float(s[q][2 * c]), __uint_as_float(s[q][2 * c + 1]), cs, -ms);
                    if ((c & 7) < SFA_PP_POLY) {
                        exp2_poly2(x0, x1, p0, p1);
                    } else {
                        p0 = fast_exp2(x0);
                        p1 = fast_exp2(x1);
                    }
                    if (c & 1) fadd2(rs2, rs3, p0, p1); else fadd2(rs0, rs1, p0, p1);
                    pk[c] = pack_f16x2(p0, p1);
                }
                tmem_st16(tS + 32 * h + 16 * q, pk);
            }
#if SFA_PP_PINGPONG
            if (t == 0 || j + 1 < nt) named_bar_arrive(2 - t, 512);  // the other tile's turn
#endif
            l += (rs0 + rs1) + (rs2 + rs3);
            if (rescale && j > 0) {  // O_t holds sum_{j' < j} P V: those MMAs completed before S_t(j)'s commit
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
            if (lane == 0) mbar_arrive(BAR(PFULL + t));
            if (lane == 0 && wq == 0 && h == 0) TLREC(0x2000 | (t << 10) | (j & 1023));
        }
        // ---- epilogue (step 8): O = 2^e (sum_j P'_j V'_j) / l, V' = V 2^-e (vprep.cu); l = both halves
        xsum[(t * 2 + h) * BM + r] = l;
        named_bar_sync(3 + t, 256);
        const float lt = xsum[(t * 2) * BM + r] + xsum[(t * 2 + 1) * BM + r];
        mbar_wait(BAR(OFULL), 0);
        tc_fence_after();
        const float inv =
            lt > 0.f ? __uint_as_float((uint32_t)(127 + vprep_head_exp(__ldg(p.v_amax + b * p.H_kv + g))) << 23) / lt : 0.f;
        const int64_t orow = ((int64_t)b * p.H + mt.h) * p.n_q + i;
#pragma unroll
        for (int q = 0; q < DV / 64; ++q) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * q, o);
            tmem_ld_wait();
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.o) + orow * DV + h * (DV / 2) + 32 * q);
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
        if (row_ok && h == 0) p.lse[orow] = lt > 0.f ? (m + __log2f(lt) - P_SHIFT) * 0.69314718055994530942f : -INFINITY;
    } else {
        if (warp == 16) {
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
                    const int vs = j % C::NV, vu = j / C::NV;
                    const bool nxt = j + 1 < nt;
                    const int s1 = (j + 1) % C::NK, u1 = (j + 1) / C::NK;
                    mbar_wait(BAR(VFULL + vs), vu & 1);
                    mbar_wait(BAR(PFULL + 0), j & 1);
                    TLREC(0x3000 | (j & 1023));
                    tc_fence_after();
                    mma_O(0, vs, j > 0);
                    if (nxt) {
                        mbar_wait(BAR(KFULL + s1), u1 & 1);
                        tc_fence_after();
                        mma_S(0, s1);
                        umma_commit(BAR(SFULL + 0));
                    }
                    mbar_wait(BAR(PFULL + 1), j & 1);
                    TLREC(0x3400 | (j & 1023));
                    tc_fence_after();
                    mma_O(1, vs, j > 0);
                    umma_commit(BAR(VEMPTY + vs));
                    if (nxt) {
                        mma_S(1, s1);
                        umma_commit(BAR(SFULL + 1));
                        umma_commit(BAR(KEMPTY + s1));
                    }
                }
                umma_commit(BAR(OFULL));
            }
            __syncwarp();
        } else if (warp == 17) {
            // ============================ TMA producer for V ============================
            if (lane == 0) {
                const int bhkv = b * p.H_kv + g;
                for (int j = 0; j < nt; ++j) {
                    const int s = j % C::NV, u = j / C::NV;
                    mbar_wait(BAR(VEMPTY + s), (u & 1) ^ 1);
                    mbar_arrive_expect_tx(BAR(VFULL + s), C::VT);
                    const uint32_t dst = sbase + C::OFF_V + s * C::VT;
#pragma unroll
                    for (int cb = 0; cb < DV / 64; ++cb)
                        tma_load_3d(dst + cb * BN * 128, &tmap_v, BAR(VFULL + s), cb * 64, j * BN, bhkv);
                }
            }
            __syncwarp();
        } else if (warp == 18) {
            // ============================ TMA producer for K~ (decompressed rows) ============================
            if (lane == 0) {
                const int bhkv = b * p.H_kv + g;
                for (int j = 0; j < nt; ++j) {
                    const int s = j % C::NK, u = j / C::NK;
                    mbar_wait(BAR(KEMPTY + s), (u & 1) ^ 1);
                    mbar_arrive_expect_tx(BAR(KFULL + s), C::KT);
                    const uint32_t dst = sbase + C::OFF_K + s * C::KT;
#pragma unroll
                    for (int cb = 0; cb < D / 64; ++cb)
                        tma_load_3d(dst + cb * BN * 128, &tmap_k, BAR(KFULL + s), cb * 64, j * BN, bhkv);
                }
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 16) {
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
cudaError_t launch_t(const PpArgs &a, cudaStream_t stream, int items) {
    using C = Cfg<D, DV>;
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
    auto kern = a.dbg != nullptr ? attn_sm100_pp_kernel<D, DV, true> : attn_sm100_pp_kernel<D, DV, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<items, NTHREADS, C::SMEM, stream>>>(tv, tk, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100_pp(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg) {
    if ((d != 64 && d != 128) || (d_v != 64 && d_v != 128)) return cudaErrorNotSupported;
    if (p.k_dense == nullptr || p.edges_only || p.window > 0 || p.q_dense != nullptr) return cudaErrorNotSupported;
    PpArgs a;
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
    if (d == 64) return d_v == 64 ? launch_t<64, 64>(a, stream, (int)items) : launch_t<64, 128>(a, stream, (int)items);
    return d_v == 64 ? launch_t<128, 64>(a, stream, (int)items) : launch_t<128, 128>(a, stream, (int)items);
}

}  // namespace sfa
