// attn_sm100_wide.cu -- FlashSFA forward with 256-key score tiles (steps 4-8 of DESIGN.md; Alg. 1
// P:L701-755, Sec. 3.2).  Same method and per-row arithmetic as attn_sm100.cu (S = Q~ K~^T
// of the decompressed codes, reading A22; fp16 P x exactly scaled fp16 V, reading A12).
//
// Shaped by two measurements (tools/umma_bench.cu, profiles/r01_timeline_v1.txt): a tcgen05.mma
// costs ~100 clocks per SM whatever its N <= 128 is, while an N = 256 instruction runs at the full
// 8192 FLOP/clk; and the softmax must never wait for the tensor pipe nor the pipe for the softmax.
// So one CTA owns 128 query rows and walks the keys in tiles of 256:
//   S(j) = Q~ K~(j)^T      8 MMAs of M128 x N256 x K16 into one 256-column TMEM buffer
//   O   += P(j) V(j)       16 MMAs of M128 x N128 x K16, P read from its OWN 128-column TMEM region
// TMEM: S [0, 256), P [256, 384), O [384, 512).  Because P does not alias S, the MMA warp issues
// S(j+1) as soon as both softmax groups have read S(j) into registers (SFREE), i.e. while they are
// still computing exponentials; P(j) is written once O += P(j-1) V(j-1) has finished reading the
// previous P (PEMPTY), which is also the moment O may be rescaled.
// Warps (512 threads):
//   0-3 / 4-7   softmax groups: keys 0-127 / 128-255 of every tile for the CTA's 128 rows
//               (thread = row = TMEM lane); partial row maxima exchanged through shared memory
//   8-11        decompression: Q~ once, then the 256-key K~ tile (2 keys per thread, 1 stage)
//   12          TMEM owner + single-thread MMA issuer
//   13          TMA producer: V in 128-key chunks through a 3-slot ring
#include <cudaTypedefs.h>
#include <mutex>

#include "launch.cuh"
#include "sm100.cuh"

namespace sfa {
using namespace sm100;

namespace {

constexpr int BM = 128;         // query rows per CTA
constexpr int BN = 256;         // keys per score tile
constexpr int GK = BN / 2;      // keys per softmax group
constexpr int VC = 128;         // keys per V chunk
constexpr int NVS = 3;          // V chunk slots
constexpr int NTHREADS = 512;
constexpr float P_SHIFT = 7.f;  // P = fp16 * 2^7 (reading A12)

template <int D, int DV>
struct Cfg {
    static constexpr int QT = BM * D * 2;
    static constexpr int KT = BN * D * 2;   // the 256-key K~ tile (single stage)
    static constexpr int VT = VC * DV * 2;  // one V chunk
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + QT;
    static constexpr int OFF_V = OFF_K + KT;
    static constexpr int OFF_RED = OFF_V + NVS * VT;  // [2 tile parities][2 groups][BM] fp32
    static constexpr int OFF_BAR = OFF_RED + 4 * BM * 4;
    static constexpr int SMEM = OFF_BAR + 256 + 1024;
    static constexpr int S_COL = 0, P_COL = 256, O_COL = 384;
    static_assert(SMEM <= 232448, "shared memory budget");
};

enum {
    KFULL = 0,   // K~ tile decompressed (4 warp arrivals)
    KEMPTY = 1,  // S MMA that read K~ completed (commit)
    VFULL = 2,   // + slot (3): V chunk landed (TMA tx)
    VEMPTY = 5,  // + slot (3): P.V MMA that read it completed (commit)
    SFULL = 8,   // S computed (commit)
    SFREE = 9,   // both softmax groups hold S in registers (8 warp arrivals)
    PFULL = 10,  // P written (8 warp arrivals)
    PEMPTY = 11, // O += P V completed: P free, O stable (commit)
    OFULL = 12,  // all MMAs completed (commit)
    QFULL = 13,  // Q~ decompressed (4 warp arrivals)
    NBAR = 14
};

struct WideArgs {
    AttnParams p;
    int32_t nqb;    // ceil(n_q / BM)
    int32_t nkt;    // ceil(n_kv / BN)
    float c_scale;  // scale * log2(e)
    float *dbg;     // optional: raw S of the first key tile of CTA 0 (tests)
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
            unsigned long long *tb_ = reinterpret_cast<unsigned long long *>(a.dbg + BM * 128);       \
            const unsigned slot_ = ((((tag) >> 12) - 1) << 11) | ((tag) & 2047);                    \
            if (slot_ < 8191) tb_[1 + slot_] = ((unsigned long long)(tag) << 48) | (clock64() & 0xFFFFFFFFFFFFull); \
        }                                                                                            \
    } while (0)
#else
#define TLREC(tag) do {} while (0)
#endif

template <int D, int DV>
__global__ void __launch_bounds__(NTHREADS, 1) attn_sm100_wide_kernel(const __grid_constant__ CUtensorMap tmap_v,
                                                                        const WideArgs a) {
    using C = Cfg<D, DV>;
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

    // work item: heaviest causal query blocks first; heads of one GQA group adjacent (L2 reuse)
    const int per_qb = p.B * p.H;
    const int qb = a.nqb - 1 - (int)(blockIdx.x / per_qb);
    const int bh = (int)(blockIdx.x % per_qb);
    const int b = bh / p.H, h = bh % p.H;
    const int g = h / (p.H / p.H_kv);
    int nt = a.nkt;
    if (p.causal) {
        int64_t last = (int64_t)qb * BM + BM - 1;
        if (last > p.n_q - 1) last = p.n_q - 1;
        const int64_t lim = (p.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }
    const int nvc = (int)((p.n_kv + VC - 1) / VC);  // V chunks that exist

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i) {
            uint32_t cnt = 1;
            if (i == KFULL || i == QFULL) cnt = 4;
            if (i == SFREE || i == PFULL) cnt = 8;
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

    // register budget per warpgroup (setmaxnreg): 2 x 184 (softmax) + 64 (decompress) + 80 = 4 x 128
    const int wg = warp >> 2;
    if (wg < 2) {
        reg_alloc<184>();
        // ============================ softmax (steps 5, 6, 8) ============================
        const int grp = wg, wq = warp & 3, r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_off + (uint32_t)(C::S_COL + grp * GK);
        const uint32_t tP = tmem + lane_off + (uint32_t)(C::P_COL + grp * (GK / 2));
        const uint32_t tO = tmem + lane_off + (uint32_t)(C::O_COL + grp * (DV / 2));
        const int64_t i = (int64_t)qb * BM + r;
        const bool row_ok = i < p.n_q;
        int64_t kend = p.n_kv;
        if (p.causal && p.q_pos0 + i + 1 < kend) kend = p.q_pos0 + i + 1;
        const float cs = a.c_scale;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            mbar_wait(BAR(SFULL), j & 1);
            if (lane == 0 && wq == 0) TLREC(0x1000 | (grp << 10) | (j & 1023));
            tc_fence_after();
            uint32_t s[4][32];
#pragma unroll
            for (int q = 0; q < 4; ++q) tmem_ld32(tS + 32 * q, s[q]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(SFREE));  // S may now be overwritten by S(j+1)
            if (a.dbg != nullptr && blockIdx.x == 0 && j == 0 && grp == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c) a.dbg[r * 128 + 32 * q + c] = __uint_as_float(s[q][c]);
            }
            const int64_t lim64 = kend - (int64_t)j * BN - grp * GK;
            const int lim = lim64 < 0 ? 0 : (lim64 > GK ? GK : (int)lim64);
            if (lim < GK) {  // step 5 on diagonal / ragged tiles: excluded keys -> -inf -> p = 0
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (32 * q + c >= lim) s[q][c] = 0xFF800000u;
            }
            float pm0 = __uint_as_float(s[0][0]), pm1 = __uint_as_float(s[0][1]), pm2 = __uint_as_float(s[0][2]),
                  pm3 = __uint_as_float(s[0][3]);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    pm0 = fmaxf(pm0, __uint_as_float(s[q][c]));
                    pm1 = fmaxf(pm1, __uint_as_float(s[q][c + 1]));
                    pm2 = fmaxf(pm2, __uint_as_float(s[q][c + 2]));
                    pm3 = fmaxf(pm3, __uint_as_float(s[q][c + 3]));
                }
            float *rj = red + (j & 1) * 2 * BM;  // alternates with the tile: a group is at most one tile ahead
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
            float ps0 = 0.f, ps1 = 0.f, ps2 = 0.f, ps3 = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 32; c += 2) {  // p in place of s, packed to fp16 pairs
                    float x0, x1;
                    ffma2(x0, x1, __uint_as_float(s[q][c]), __uint_as_float(s[q][c + 1]), cs, -ms);
                    const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
                    if (c & 2) fadd2(ps2, ps3, p0, p1); else fadd2(ps0, ps1, p0, p1);
                    s[q][c >> 1] = pack_f16x2(p0, p1);  // c >> 1 < c: never overwrites an unread score
                }
            l += (ps0 + ps1) + (ps2 + ps3);
            if (j > 0) {  // O += P(j-1) V(j-1) complete: the P region is free and O is stable
                mbar_wait(BAR(PEMPTY), (j - 1) & 1);
                tc_fence_after();
                if (rescale) {
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
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // 128 keys -> 64 packed columns of this group's P
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) pk[c] = s[q][c];
                tmem_st16(tP + 16 * q, pk);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(PFULL));
            if (lane == 0 && wq == 0) TLREC(0x2000 | (grp << 10) | (j & 1023));
        }
        // ---- epilogue (step 8): combine the groups' row sums, each group stores half of O
        named_bar_sync(1, 256);
        red[grp * BM + r] = l;
        named_bar_sync(1, 256);
        const float lt = red[r] + red[BM + r];
        mbar_wait(BAR(OFULL), 0);
        tc_fence_after();
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
        reg_dealloc<64>();
        // ============================ decompression of Q~ and K~ ============================
        const int r = threadIdx.x - 256;
        const int k = p.k;
        const uint16_t *qv = reinterpret_cast<const uint16_t *>(p.q_val);
        const uint16_t *kv = reinterpret_cast<const uint16_t *>(p.k_val);
        {
            const int64_t i = (int64_t)qb * BM + r;
            const bool ok = i < p.n_q;
            const int64_t row = ((int64_t)b * p.H + h) * p.n_q + (ok ? i : 0);
            densify_row<D>(sbase + C::OFF_Q, BM, r, ok, p.q_idx + row * k, qv + row * k, k);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(QFULL));
        const int64_t kv0 = ((int64_t)b * p.H_kv + g) * p.n_kv;
        for (int j = 0; j < nt; ++j) {
            mbar_wait(BAR(KEMPTY), (j & 1) ^ 1);
#pragma unroll
            for (int half = 0; half < 2; ++half) {  // keys r and r + 128 of the tile
                const int rr = r + half * BM;
                const int64_t key = (int64_t)j * BN + rr;
                const bool ok = key < p.n_kv;
                densify_row<D>(sbase + C::OFF_K, BN, rr, ok, p.k_idx + (kv0 + (ok ? key : 0)) * k,
                               kv + (kv0 + (ok ? key : 0)) * k, k);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(KFULL));
        }
    } else {
        reg_dealloc<80>();
        if (warp == 12) {
            // ============================ tcgen05.mma issuer ============================
            if (lane == 0) {
                constexpr uint32_t idS = umma_idesc_f16kind(BM, BN, 0, 0, 1);  // bf16 Q~ x bf16 K~, N = 256
                constexpr uint32_t idO = umma_idesc_f16kind(BM, DV, 0, 1, 0);  // fp16 P (TMEM) x fp16 V
                const uint32_t qa = sbase + C::OFF_Q, ka = sbase + C::OFF_K;
                auto mma_S = [&]() {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off_q = (kk >> 2) * BM * 128 + (kk & 3) * 32;
                        const uint32_t off_k = (kk >> 2) * BN * 128 + (kk & 3) * 32;
                        umma_ss(tmem + C::S_COL, umma_desc_sw128(qa + off_q, 16, 1024),
                                umma_desc_sw128(ka + off_k, 16, 1024), idS, kk > 0);
                    }
                };
                // O += P(j) V(j): 16 K-steps over the tile's two V chunks (2j, 2j+1)
                auto mma_PV = [&](int j) {
#pragma unroll
                    for (int hc = 0; hc < 2; ++hc) {
                        const int cidx = 2 * j + hc;
                        const uint32_t va = sbase + C::OFF_V + (cidx % NVS) * C::VT;
#pragma unroll
                        for (int kk = 0; kk < VC / 16; ++kk)
                            umma_ts(tmem + C::O_COL, tmem + C::P_COL + hc * 64 + kk * 8,
                                    umma_desc_sw128(va + kk * 2048, VC * 128, 1024), idO,
                                    (j > 0 || hc > 0 || kk > 0) ? 1u : 0u);
                    }
                };
                mbar_wait(BAR(QFULL), 0);
                mbar_wait(BAR(KFULL), 0);
                tc_fence_after();
                mma_S();
                umma_commit(BAR(SFULL));
                umma_commit(BAR(KEMPTY));
                for (int j = 0; j < nt; ++j) {
                    if (j + 1 < nt) {  // S(j+1) once both groups hold S(j) and K~(j+1) is ready
                        mbar_wait(BAR(SFREE), j & 1);
                        mbar_wait(BAR(KFULL), (j + 1) & 1);
                        tc_fence_after();
                        mma_S();
                        umma_commit(BAR(SFULL));
                        umma_commit(BAR(KEMPTY));
                    }
                    for (int hc = 0; hc < 2; ++hc) {
                        const int cidx = 2 * j + hc;
                        mbar_wait(BAR(VFULL + cidx % NVS), (cidx / NVS) & 1);
                    }
                    mbar_wait(BAR(PFULL), j & 1);
                    if (threadIdx.x == 384) TLREC(0x3000 | (j & 1023));
                    tc_fence_after();
                    mma_PV(j);
                    umma_commit(BAR(PEMPTY));
                    umma_commit(BAR(VEMPTY + (2 * j) % NVS));
                    umma_commit(BAR(VEMPTY + (2 * j + 1) % NVS));
                    if (threadIdx.x == 384) TLREC(0x3400 | (j & 1023));
                }
                umma_commit(BAR(OFULL));
            }
            __syncwarp();
        } else if (warp == 13) {
            // ============================ TMA producer: V in 128-key chunks ============================
            if (lane == 0) {
                const int bhkv = b * p.H_kv + g;
                for (int cidx = 0; cidx < 2 * nt; ++cidx) {
                    const int sl = cidx % NVS, u = cidx / NVS;
                    mbar_wait(BAR(VEMPTY + sl), (u & 1) ^ 1);
                    const uint32_t dst = sbase + C::OFF_V + sl * C::VT;
                    if (cidx < nvc) {
                        mbar_arrive_expect_tx(BAR(VFULL + sl), C::VT);
#pragma unroll
                        for (int cb = 0; cb < DV / 64; ++cb)
                            tma_load_3d(dst + cb * VC * 128, &tmap_v, BAR(VFULL + sl), cb * 64, cidx * VC, bhkv);
                    } else {
                        // a chunk wholly past n_kv (last tile of a short sequence): its P is 0, but the
                        // stale slot could hold non-finite-free garbage only -- still zero it via TMA OOB
                        mbar_arrive_expect_tx(BAR(VFULL + sl), C::VT);
#pragma unroll
                        for (int cb = 0; cb < DV / 64; ++cb)
                            tma_load_3d(dst + cb * VC * 128, &tmap_v, BAR(VFULL + sl), cb * 64, cidx * VC, bhkv);
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

template <int D, int DV>
cudaError_t launch_wide_t(const WideArgs &a, cudaStream_t stream, int items) {
    using C = Cfg<D, DV>;
    const AttnParams &p = a.p;
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)DV, (cuuint64_t)p.n_kv, (cuuint64_t)p.B * p.H_kv};
    cuuint64_t strides[2] = {(cuuint64_t)DV * 2, (cuuint64_t)p.n_kv * DV * 2};
    cuuint32_t box[3] = {64, VC, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void *>(p.v16), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    auto kern = attn_sm100_wide_kernel<D, DV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<items, NTHREADS, C::SMEM, stream>>>(tm, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100_wide(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg) {
    if ((d != 64 && d != 128) || (d_v != 64 && d_v != 128)) return cudaErrorNotSupported;
    WideArgs a;
    a.p = p;
    a.nqb = (int)((p.n_q + BM - 1) / BM);
    a.nkt = (int)((p.n_kv + BN - 1) / BN);
    a.c_scale = p.scale_log2;
    a.dbg = dbg;
    const int64_t items = (int64_t)p.B * p.H * a.nqb;
    if (items == 0) return cudaSuccess;
    if (items > INT32_MAX) return cudaErrorNotSupported;
    if (d == 64) return d_v == 64 ? launch_wide_t<64, 64>(a, stream, (int)items) : launch_wide_t<64, 128>(a, stream, (int)items);
    return d_v == 64 ? launch_wide_t<128, 64>(a, stream, (int)items) : launch_wide_t<128, 128>(a, stream, (int)items);
}

}  // namespace sfa
