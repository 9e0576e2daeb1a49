// bwd.cu -- FlashSFA backward with the straight-through rule on sm_100a tensor cores
// (Sec. 3.1 "Backward computation", Eq. topk_grad).
//
// With P_ij = exp(s_ij - LSE_i) recomputed from the codes and the forward's LSE, and
// D_i = sum_c dO_ic O_ic:
//   dP = dO V^T,  dS = P (.) (dP - D),  dV = P^T dO,  dQ~ = scale dS K~,  dK~ = scale dS^T Q~,
// and the straight-through rule keeps only the selected coordinates: dq_val[i][t] = dQ~[i][q_idx[i][t]],
// dk_val[j][t] = dK~[j][k_idx[j][t]] (the dense dQ, dK of Eq. topk_grad are these scattered to the
// supports, zero elsewhere).  GQA: dK~ and dV of a kv head sum over its query heads (A15).
//
// Two kernels, no atomics, every reduction in a fixed order (S "Concurrency Model": deterministic):
//   bwd_dq_kernel    one CTA per 128-row query tile (query-stationary, like the forward):
//                    per key tile S = Q~ K~^T and dP = dO V^T (SS-MMAs, M = 128 queries), the row
//                    warps form dS in bf16 into S's TMEM columns, dQ~ += dS K~ (TS-MMA, K~ read
//                    MN-major from the same swizzled tile);
//   bwd_dkdv_kernel  one CTA per 128-key tile of a kv head (key-stationary): per (query head of the
//                    group, query tile) S^T = K~ Q~^T and dP^T = V dO^T (M = 128 keys), the key
//                    warps form P^T and dS^T in bf16 in TMEM, dV += P^T dO and dK~ += dS^T Q~
//                    (TS-MMAs, dO and Q~ read MN-major).
// Both recompute the scores exactly as the forward (bf16 products are exact in fp32); P and dS are
// rounded to bf16 for the tensor cores (reading A24: the gradient tolerance is componentwise).
// Operands: codes decompressed on chip into 128B-swizzled tiles (densify.cuh), V and dO by TMA.
#include <cudaTypedefs.h>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "densify.cuh"
#include "launch.cuh"
#include "sm100.cuh"

namespace sfa {
using namespace sm100;
using namespace dz;

namespace {

constexpr int BM = 128, BN = 128, NTH = 448;
// Thread roles (both kernels): warps 0-7 = two groups of four row warps (TMEM lane quarter = warp & 3);
// group g forms P / dS for the columns [64g, 64g + 64) of the 128-wide score tile, so every SMSP runs
// two such warps (the exponentials and the TMEM traffic of one hide the latency of the other);
// warps 8-11 decompression; warp 12 tcgen05.mma issuer + TMEM owner; warp 13 TMA.
constexpr int ROW_WARPS = 8;
// 1: Q~ and K~ tiles arrive by TMA from rows decompressed once per row (k_dense_kernel, vprep.cu) --
// the on-chip decompression (zero fill + k u16 stores per row per tile) was ~40 % of the dK/dV kernel's
// shared-memory LSU traffic and most of its 440 M bank conflicts; 0: decompression warps, as round 1
#ifndef SFA_BWD_TMA
#define SFA_BWD_TMA 1
#endif

// TMEM column of the packed bf16 operand (P, P^T, dS or dS^T) for the K-step kk (16 rows of K):
// group g writes its 64 columns' worth of bf16 pairs into [64g, 64g + 32) over scores it has read
__device__ __forceinline__ uint32_t packed_col(int kk) { return (uint32_t)(64 * (kk >> 2) + 8 * (kk & 3)); }

struct BwdArgs {
    const uint8_t *q_idx, *k_idx;
    const uint16_t *q_val, *k_val;
    const float *lse, *Dr;  // [B][H][n_q]: forward LSE, D_i = rowsum(dO . O)
    float *dq, *dk, *dv;    // [B][H][n_q][k], [B][H_kv][n_kv][k], [B][H_kv][n_kv][d_v] (fp32)
    int32_t B, H, H_kv, k;
    int64_t n_q, n_kv, q_pos0;
    int32_t causal, nqb, nkt;
    float scale, c_scale;  // scale, scale * log2(e)
};

__global__ void bwd_prep_kernel(const uint16_t *__restrict__ o, const uint16_t *__restrict__ dO, int64_t rows,
                                int d_v, float *__restrict__ Dr) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float acc = 0.f;
    for (int c = lane; c < d_v; c += 32) {
        const float a = __uint_as_float((uint32_t)__ldg(o + row * d_v + c) << 16);
        const float b = __uint_as_float((uint32_t)__ldg(dO + row * d_v + c) << 16);
        acc = fmaf(a, b, acc);
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) Dr[row] = acc;
}

// SW128 operand descriptors: K-major tile of `rows` rows, K-step kk (16 elements); MN-major view of
// the same tile (rows = the K dimension), K-step kk = 16 rows
__device__ __forceinline__ uint64_t kmaj(uint32_t base, int rows, int kk) {
    return umma_desc_sw128(base + (uint32_t)((kk >> 2) * rows * 128 + (kk & 3) * 32), 16, 1024);
}
__device__ __forceinline__ uint64_t mnmaj(uint32_t base, int rows, int kk) {
    return umma_desc_sw128(base + (uint32_t)(kk * 2048), (uint32_t)rows * 128, 1024);
}

// ---------------------------------------------------------------------------------------------
// dQ: one CTA per (b, h, query tile)
// ---------------------------------------------------------------------------------------------
template <int D, int DV>
struct DqCfg {
    static constexpr int OFF_Q = 0;                      // Q~ tile  [128][D] bf16
    static constexpr int OFF_DO = OFF_Q + BM * D * 2;    // dO tile  [128][DV] bf16
    static constexpr int NK = 3;                          // K~ ring depth (K~(j+2) decompresses while dQ(j) waits)
    static constexpr int OFF_K = OFF_DO + BM * DV * 2;    // K~ ring  NK x [128][D]
    static constexpr int OFF_V = OFF_K + NK * BN * D * 2; // V ring   2 x [128][DV]
    static constexpr int OFF_BAR = OFF_V + 2 * BN * DV * 2;
    static constexpr int SMEM = OFF_BAR + 256 + 1024;
};
static_assert(DqCfg<128, 128>::SMEM <= 232448, "dQ kernel shared memory");
// dQ TMEM: S double-buffered in columns [0,128) / [384,512) (dS written over the buffer it came from),
// dP [128,256), dQ~ [256,384).  S(j+1) is issued while the row warps still work on tile j; dP(j+1) as
// soon as they have read dP(j) (DP_FREE); dQ~ += dS(j) K~(j) after that.
enum { Q_FULL = 0, DO_FULL, K_FULL, K_EMPTY = K_FULL + 3, V_FULL = K_EMPTY + 3, V_EMPTY = V_FULL + 2, S_FULL = V_EMPTY + 2,
       DP_FULL = S_FULL + 2, DP_FREE, DS_READY, DQ_FULL, NBAR_DQ };
__device__ __forceinline__ uint32_t dq_sbuf(int j) { return (j & 1) ? 384u : 0u; }

template <int D, int DV>
__global__ void __launch_bounds__(NTH, 1) bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_v,
                                                        const __grid_constant__ CUtensorMap tm_do,
                                                        const __grid_constant__ CUtensorMap tm_q,
                                                        const __grid_constant__ CUtensorMap tm_k, const BwdArgs a) {
    using C = DqCfg<D, DV>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t sb = (raw_s + 1023u) & ~1023u;
    uint8_t *gb = smem_raw + (sb - raw_s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#define BAR(i) (sb + C::OFF_BAR + 8u * (uint32_t)(i))
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gb + C::OFF_BAR + 200);

    // kv-group-major order (as the forward): the group's R heads x query tiles, heaviest causal tiles first,
    // so resident CTAs share one group's K codes and V in L2
    const int Rg = a.H / a.H_kv;
    const int per_g = Rg * a.nqb;
    const int gi = (int)(blockIdx.x / per_g), rem = (int)(blockIdx.x % per_g);
    const int ib = a.nqb - 1 - rem / Rg;
    const int b = gi / a.H_kv, g = gi % a.H_kv, h = g * Rg + rem % Rg;
    int nt = a.nkt;
    if (a.causal) {
        int64_t last = (int64_t)ib * BM + BM - 1;
        if (last > a.n_q - 1) last = a.n_q - 1;
        const int64_t lim = (a.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR_DQ; ++i)
            mbar_init(BAR(i), (i == Q_FULL || i == K_FULL || i == K_FULL + 1 || i == K_FULL + 2) ? (SFA_BWD_TMA ? 1u : 4u)
                              : ((i == DS_READY || i == DP_FREE) ? 8u : 1u));
        fence_mbar_init();
    }
    if (warp == 12) tmem_alloc<512>(smem_u32(tmem_slot));
    if (warp == 13 && lane == 0) {
        tma_prefetch_desc(&tm_v);
        tma_prefetch_desc(&tm_do);
        if (SFA_BWD_TMA) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < ROW_WARPS) {
        // ==================== row warps: thread = query row = TMEM lane; group = key half ====================
        const int grp = warp >> 2, wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lo = (uint32_t)(wq * 32) << 16;
        const int64_t i = (int64_t)ib * BM + r;
        const bool row_ok = i < a.n_q;
        const int64_t qrow = ((int64_t)b * a.H + h) * a.n_q + i;
        const float lse2 = row_ok ? __ldg(a.lse + qrow) * 1.4426950408889634f : 0.f;
        const float Di = row_ok ? __ldg(a.Dr + qrow) : 0.f;
        int64_t kend = row_ok ? a.n_kv : 0;
        if (row_ok && a.causal && a.q_pos0 + i + 1 < kend) kend = a.q_pos0 + i + 1;
        const float cs = a.c_scale;
        for (int j = 0; j < nt; ++j) {
            const uint32_t sbuf = dq_sbuf(j);
            mbar_wait(BAR(S_FULL + (j & 1)), (j >> 1) & 1);
            tc_fence_after();
            int64_t l64 = kend - (int64_t)j * BN;
            const int lim = l64 < 0 ? 0 : (l64 > BN ? BN : (int)l64);
            // P-phase (needs S only: runs while dP(j) is still on the tensor pipe); p kept in fp32
            float pp[2][32];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int cc = 2 * grp + c;
                uint32_t s[32];
                tmem_ld32(tmem + lo + sbuf + 32 * cc, s);
                tmem_ld_wait();
                auto chunk = [&](auto masked) {  // masks only where the diagonal / ragged end cuts the chunk
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        float p = fast_exp2(fmaf(__uint_as_float(s[e]), cs, -lse2));
                        if (decltype(masked)::value && 32 * cc + e >= lim) p = 0.f;
                        pp[c][e] = p;
                    }
                };
                if (lim >= 32 * cc + 32)
                    chunk(std::false_type{});
                else
                    chunk(std::true_type{});
            }
            // dS-phase: dS = P (.) (dP - D), bf16 over the S columns this group has read
            mbar_wait(BAR(DP_FULL), j & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int cc = 2 * grp + c;
                uint32_t dp[32], pk[16];
                tmem_ld32(tmem + lo + 128 + 32 * cc, dp);
                tmem_ld_wait();
                if (c == 1) {  // this warp is done with dP(j): dP(j+1) may be issued
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(BAR(DP_FREE));
                }
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    pk[e] = pack_bf16x2(pp[c][2 * e] * (__uint_as_float(dp[2 * e]) - Di),
                                        pp[c][2 * e + 1] * (__uint_as_float(dp[2 * e + 1]) - Di));
                tmem_st16(tmem + lo + sbuf + 64 * grp + 16 * c, pk);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(DS_READY));
        }
        if (grp == 0) {
        // ---- epilogue (group 0): dQ~ row -> shared staging (the dead K~ ring) -> gather at the support
        mbar_wait(BAR(DQ_FULL), 0);
        tc_fence_after();
        // the decompression warps' last K~ stores into the ring precede DQ_FULL through the MMA chain; the
        // named barrier makes that ordering explicit (and visible to racecheck) before the ring is reused
        named_bar_sync(6, 256);
        float *st = reinterpret_cast<float *>(gb + C::OFF_K) + (size_t)r * D;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tmem + lo + 256 + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) st[(32 * c + e + r) % D] = __uint_as_float(o[e]);  // rotated: no bank conflicts
        }
        if (row_ok)
            for (int t = 0; t < a.k; ++t) {
                const int f = __ldg(a.q_idx + qrow * a.k + t);
                a.dq[qrow * a.k + t] = a.scale * st[(f + r) % D];
            }
        }
    } else if (warp < 12) {
        // ==================== Q~ once, K~ per key tile: TMA (warp 8, lane 0) or decompression ====================
        const int r = threadIdx.x - 32 * ROW_WARPS;
        const int k = a.k;
        if (SFA_BWD_TMA) {
            if (warp == ROW_WARPS && lane == 0) {
                mbar_arrive_expect_tx(BAR(Q_FULL), BM * D * 2);
#pragma unroll
                for (int cb = 0; cb < D / 64; ++cb)
                    tma_load_3d(sb + C::OFF_Q + cb * BM * 128, &tm_q, BAR(Q_FULL), cb * 64, ib * BM, b * a.H + h);
                for (int j = 0; j < nt; ++j) {
                    const int s = j % C::NK, u = j / C::NK;
                    mbar_wait(BAR(K_EMPTY + s), (u & 1) ^ 1);
                    mbar_arrive_expect_tx(BAR(K_FULL + s), BN * D * 2);
#pragma unroll
                    for (int cb = 0; cb < D / 64; ++cb)
                        tma_load_3d(sb + C::OFF_K + s * BN * D * 2 + cb * BN * 128, &tm_k, BAR(K_FULL + s), cb * 64,
                                    j * BN, b * a.H_kv + g);
                }
            }
            __syncwarp();
        } else {
        {
            const int64_t i = (int64_t)ib * BM + r;
            const bool ok = i < a.n_q;
            const int64_t row = ((int64_t)b * a.H + h) * a.n_q + (ok ? i : 0);
            densify_row<D>(sb + C::OFF_Q, BM, r, ok, a.q_idx + row * k, a.q_val + row * k, k);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(Q_FULL));
        const int64_t kv0 = ((int64_t)b * a.H_kv + g) * a.n_kv;
        for (int j = 0; j < nt; ++j) {
            const int s = j % C::NK, u = j / C::NK;
            const int64_t key = (int64_t)j * BN + r;
            const bool ok = key < a.n_kv;
            const int64_t kr = kv0 + (ok ? key : 0);
            if (j + 1 < nt && key + BN < a.n_kv) prefetch_code_row(a.k_idx + (kr + BN) * k, a.k_val + (kr + BN) * k);
            mbar_wait(BAR(K_EMPTY + s), (u & 1) ^ 1);
            densify_row<D>(sb + C::OFF_K + s * BN * D * 2, BN, r, ok, a.k_idx + kr * k, a.k_val + kr * k, k);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(K_FULL + s));
        }
        }
        asm volatile("bar.arrive 6, 256;" ::: "memory");  // done with the K~ ring (the epilogue reuses it)
    } else if (warp == 12) {
        // ==================== tcgen05.mma issuer ====================
        if (lane == 0) {
            constexpr uint32_t idS = umma_idesc_f16kind(BM, BN, 0, 0, 1);  // Q~ . K~^T
            constexpr uint32_t idQ = umma_idesc_f16kind(BM, D, 0, 1, 1);   // dS[TMEM] . K~ (K~ MN-major)
            const uint32_t qa = sb + C::OFF_Q, da = sb + C::OFF_DO;
            mbar_wait(BAR(Q_FULL), 0);
            mbar_wait(BAR(DO_FULL), 0);
            auto dq_mma = [&](int jj) {  // dQ~ += dS(jj) K~(jj)
                mbar_wait(BAR(DS_READY), jj & 1);
                tc_fence_after();
                const uint32_t ka = sb + C::OFF_K + (jj % C::NK) * BN * D * 2;
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk)
                    umma_ts(tmem + 256, tmem + dq_sbuf(jj) + packed_col(kk), mnmaj(ka, BN, kk), idQ,
                            (jj > 0 || kk > 0) ? 1u : 0u);
                umma_commit(BAR(K_EMPTY + jj % C::NK));
            };
            for (int j = 0; j < nt; ++j) {
                const int s = j & 1, u = j >> 1, sk = j % C::NK;
                mbar_wait(BAR(K_FULL + sk), (j / C::NK) & 1);
                tc_fence_after();
                const uint32_t ka = sb + C::OFF_K + sk * BN * D * 2, va = sb + C::OFF_V + s * BN * DV * 2;
                // S(j) into the buffer of tile j-2: its dS was consumed by dQ(j-2), issued before (in order)
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    umma_ss(tmem + dq_sbuf(j), kmaj(qa, BM, kk), kmaj(ka, BN, kk), idS, kk > 0);
                umma_commit(BAR(S_FULL + (j & 1)));
                mbar_wait(BAR(V_FULL + s), u & 1);
                if (j > 0) mbar_wait(BAR(DP_FREE), (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < DV / 16; ++kk)
                    umma_ss(tmem + 128, kmaj(da, BM, kk), kmaj(va, BN, kk), idS, kk > 0);
                umma_commit(BAR(V_EMPTY + s));
                umma_commit(BAR(DP_FULL));
                if (j > 0) dq_mma(j - 1);
            }
            dq_mma(nt - 1);
            umma_commit(BAR(DQ_FULL));
        }
        __syncwarp();
    } else if (warp == 13) {
        // ==================== TMA: dO tile once, V tiles ====================
        if (lane == 0) {
            mbar_arrive_expect_tx(BAR(DO_FULL), BM * DV * 2);
#pragma unroll
            for (int cb = 0; cb < DV / 64; ++cb)
                tma_load_3d(sb + C::OFF_DO + cb * BM * 128, &tm_do, BAR(DO_FULL), cb * 64, ib * BM, b * a.H + h);
            for (int j = 0; j < nt; ++j) {
                const int s = j & 1, u = j >> 1;
                mbar_wait(BAR(V_EMPTY + s), (u & 1) ^ 1);
                mbar_arrive_expect_tx(BAR(V_FULL + s), BN * DV * 2);
#pragma unroll
                for (int cb = 0; cb < DV / 64; ++cb)
                    tma_load_3d(sb + C::OFF_V + s * BN * DV * 2 + cb * BN * 128, &tm_v, BAR(V_FULL + s), cb * 64,
                                j * BN, b * a.H_kv + g);
            }
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 12) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
#undef BAR
}

// ---------------------------------------------------------------------------------------------
// dK, dV: one CTA per (b, kv head, key tile)
// ---------------------------------------------------------------------------------------------
template <int D, int DV>
struct KvCfg {
    static constexpr int OFF_K = 0;                        // K~ tile [128][D]
    static constexpr int OFF_V = OFF_K + BN * D * 2;       // V tile  [128][DV]
    static constexpr int NQ = 3;                           // Q~ (+ LSE, D) ring depth
    static constexpr int OFF_Q = OFF_V + BN * DV * 2;      // Q~ ring NQ x [128][D]
    static constexpr int OFF_DO = OFF_Q + NQ * BM * D * 2; // dO tile [128][DV] (single stage)
    static constexpr int OFF_LD = OFF_DO + BM * DV * 2;    // NQ stages x {LSE*log2e, D} x 128 fp32
    static constexpr int OFF_BAR = OFF_LD + NQ * 2 * BM * 4;
    static constexpr int SMEM = OFF_BAR + 256 + 1024;
};
static_assert(KvCfg<128, 128>::SMEM <= 232448, "dK/dV kernel shared memory");
// dK~/dV pipeline per step s (TMEM: S^T [0,128) | dP^T [128,256) | dV | dK~, all 512 columns):
//   MMA:   ... [P_READY(s)] dV += P^T(s) dO(s);  S^T(s+1)  [KDS_READY(s)] dK~ += dS^T(s) Q~(s);  dP^T(s+1)
//   warps: [SS_FULL] P-phase (P^T(s) over S^T) -> P_READY;  [KDP_FULL] dS-phase (dS^T over dP^T) -> KDS_READY
// S^T(s+1) overwrites P^T(s) and dP^T(s+1) overwrites dS^T(s) only after the MMAs reading them were
// issued (in-order tensor pipe), so the warps' dS-phase of step s overlaps S^T(s+1) and dV(s), and
// their P-phase of step s+1 overlaps dK~(s) and dP^T(s+1).
// Q~ ring of 3: Q~(s+1) lands in the slot dK~(s-2) released, so its decompression is off the
// S^T(s+1) critical path; dO needs one stage (dP^T(s+1) is issued well after dV(s) frees it).
enum { KK_FULL = 0, KV_FULL, QQ_FULL, QQ_EMPTY = QQ_FULL + 3, DOO_FULL = QQ_EMPTY + 3, DOO_EMPTY,
       SS_FULL, KDP_FULL, P_READY, KDS_READY, OUT_FULL, NBAR_KV };

template <int D, int DV>
__global__ void __launch_bounds__(NTH, 1) bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_v,
                                                          const __grid_constant__ CUtensorMap tm_do,
                                                          const __grid_constant__ CUtensorMap tm_q,
                                                          const __grid_constant__ CUtensorMap tm_k, const BwdArgs a) {
    using C = KvCfg<D, DV>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t sb = (raw_s + 1023u) & ~1023u;
    uint8_t *gb = smem_raw + (sb - raw_s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#define BAR(i) (sb + C::OFF_BAR + 8u * (uint32_t)(i))
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gb + C::OFF_BAR + 200);
    float *ldv = reinterpret_cast<float *>(gb + C::OFF_LD);  // [stage][{lse2, D}][128]

    // kv-group-major order: one group's key tiles back to back, low key tiles (most query tiles) first,
    // so resident CTAs share the group's query codes and dO in L2
    const int bg = (int)(blockIdx.x / a.nkt), jb = (int)(blockIdx.x % a.nkt);
    const int b = bg / a.H_kv, g = bg % a.H_kv;
    const int R = a.H / a.H_kv;
    int ib0 = 0;
    if (a.causal) {  // first query tile holding a query at or after this tile's first key
        const int64_t first = (int64_t)jb * BN - a.q_pos0;
        ib0 = first <= 0 ? 0 : (int)(first / BM);
    }
    const int nib = a.nqb > ib0 ? a.nqb - ib0 : 0;
    const int ns = R * nib;  // steps: (query head of the group, query tile)

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR_KV; ++i)
            mbar_init(BAR(i), i == KK_FULL ? (SFA_BWD_TMA ? 1u : 4u)
                              : (i == QQ_FULL || i == QQ_FULL + 1 || i == QQ_FULL + 2) ? 4u
                              : ((i == P_READY || i == KDS_READY) ? 8u : 1u));
        fence_mbar_init();
    }
    if (warp == 12) tmem_alloc<512>(smem_u32(tmem_slot));
    if (warp == 13 && lane == 0) {
        tma_prefetch_desc(&tm_v);
        tma_prefetch_desc(&tm_do);
        if (SFA_BWD_TMA) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t DV_COL = 256, DK_COL = 256 + DV;

    if (warp < ROW_WARPS) {
        // ==================== key warps: thread = key = TMEM lane; group = query half ====================
        const int grp = warp >> 2, wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lo = (uint32_t)(wq * 32) << 16;
        const int64_t kj = (int64_t)jb * BN + r;
        const bool key_ok = kj < a.n_kv;
        const float cs = a.c_scale;
        for (int s = 0; s < ns; ++s) {
            const int st = s % C::NQ, ib = ib0 + s % nib;
            mbar_wait(BAR(SS_FULL), s & 1);
            mbar_wait(BAR(QQ_FULL + st), (s / C::NQ) & 1);  // LSE / D of this step visible (generic stores)
            tc_fence_after();
            const float *lse2 = ldv + st * 2 * BM, *Dq = lse2 + BM;
            // query q of this tile may use key kj iff q < n_q and (non-causal or kj <= q_pos0 + q)
            int64_t qmin = a.causal ? kj - a.q_pos0 - (int64_t)ib * BM : 0;  // first allowed local query
            if (qmin < 0) qmin = 0;
            int64_t qmax = a.n_q - (int64_t)ib * BM;                          // one past the last valid
            if (!key_ok) qmax = 0;
            // P-phase: p from S^T and LSE (kept in fp32 for the dS-phase), P^T in bf16 over S^T
            float pk[2][32];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int cc = 2 * grp + c;
                uint32_t sv[32], pp[16];
                tmem_ld32(tmem + lo + 32 * cc, sv);
                tmem_ld_wait();
                // LSE of 4 queries per 16-byte shared load; the mask tests only on chunks the causal
                // diagonal or the ragged end cuts (most steps have every pair allowed)
                auto pchunk = [&](auto masked) {
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4) {
                        const int qb = 32 * cc + 4 * e4;
                        const float4 L = *reinterpret_cast<const float4 *>(lse2 + qb);
                        const float lv[4] = {L.x, L.y, L.z, L.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            float p = fast_exp2(fmaf(__uint_as_float(sv[4 * e4 + u]), cs, -lv[u]));
                            if (decltype(masked)::value && !(qb + u >= qmin && qb + u < qmax)) p = 0.f;
                            pk[c][4 * e4 + u] = p;
                        }
                    }
                };
                if (qmin <= 32 * cc && qmax >= 32 * cc + 32)
                    pchunk(std::false_type{});
                else
                    pchunk(std::true_type{});
#pragma unroll
                for (int e = 0; e < 16; ++e) pp[e] = pack_bf16x2(pk[c][2 * e], pk[c][2 * e + 1]);
                tmem_st16(tmem + lo + 64 * grp + 16 * c, pp);  // P^T over S^T columns this group read
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(P_READY));
            // dS-phase: dS^T = P^T (.) (dP^T - D), bf16 over dP^T
            mbar_wait(BAR(KDP_FULL), s & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int cc = 2 * grp + c;
                uint32_t dp[32], pd[16];
                tmem_ld32(tmem + lo + 128 + 32 * cc, dp);
                tmem_ld_wait();
#pragma unroll
                for (int e4 = 0; e4 < 8; ++e4) {
                    const float4 Dv = *reinterpret_cast<const float4 *>(Dq + 32 * cc + 4 * e4);
                    pd[2 * e4] = pack_bf16x2(pk[c][4 * e4] * (__uint_as_float(dp[4 * e4]) - Dv.x),
                                             pk[c][4 * e4 + 1] * (__uint_as_float(dp[4 * e4 + 1]) - Dv.y));
                    pd[2 * e4 + 1] = pack_bf16x2(pk[c][4 * e4 + 2] * (__uint_as_float(dp[4 * e4 + 2]) - Dv.z),
                                                 pk[c][4 * e4 + 3] * (__uint_as_float(dp[4 * e4 + 3]) - Dv.w));
                }
                tmem_st16(tmem + lo + 128 + 64 * grp + 16 * c, pd);  // dS^T over dP^T's
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(KDS_READY));
        }
        // ---- epilogue: group 0 writes the dV row (fp32) straight out; group 1 stages the dK~ row
        // (dead Q~ ring) and gathers it at the support
        const int64_t krow = ((int64_t)b * a.H_kv + g) * a.n_kv + kj;
        float *stg = reinterpret_cast<float *>(gb + C::OFF_Q) + (size_t)r * D;
        if (ns > 0) {
            mbar_wait(BAR(OUT_FULL), 0);
            tc_fence_after();
        }
        if (grp == 0) {
#pragma unroll 1
        for (int c = 0; c < DV / 32; ++c) {
            uint32_t o[32];
            if (ns > 0) {
                tmem_ld32(tmem + lo + DV_COL + 32 * c, o);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = 0u;
            }
            if (key_ok) {
                float4 *dst = reinterpret_cast<float4 *>(a.dv + krow * DV + 32 * c);
#pragma unroll
                for (int v4 = 0; v4 < 8; ++v4)
                    dst[v4] = make_float4(__uint_as_float(o[4 * v4]), __uint_as_float(o[4 * v4 + 1]),
                                          __uint_as_float(o[4 * v4 + 2]), __uint_as_float(o[4 * v4 + 3]));
            }
        }
        } else {
        // the decompression warps' last Q~ stores precede the MMAs' completion; the named barrier makes the
        // ordering explicit (and visible to racecheck) before the dead Q~ ring is reused as staging
        named_bar_sync(6, 256);
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            if (ns > 0) {
                tmem_ld32(tmem + lo + DK_COL + 32 * c, o);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = 0u;
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) stg[(32 * c + e + r) % D] = __uint_as_float(o[e]);
        }
        if (key_ok)
            for (int t = 0; t < a.k; ++t) {
                const int f = __ldg(a.k_idx + krow * a.k + t);
                a.dk[krow * a.k + t] = a.scale * stg[(f + r) % D];
            }
        }
    } else if (warp < 12) {
        // ============ K~ once, Q~ (+ LSE, D staging) per step: TMA (warp 8, lane 0) or decompression ============
        const int r = threadIdx.x - 32 * ROW_WARPS;
        const int k = a.k;
        const int64_t kv0 = ((int64_t)b * a.H_kv + g) * a.n_kv;
        if (SFA_BWD_TMA) {
            if (warp == ROW_WARPS && lane == 0) {
                mbar_arrive_expect_tx(BAR(KK_FULL), BN * D * 2);
#pragma unroll
                for (int cb = 0; cb < D / 64; ++cb)
                    tma_load_3d(sb + C::OFF_K + cb * BN * 128, &tm_k, BAR(KK_FULL), cb * 64, jb * BN, b * a.H_kv + g);
            }
        } else {
            {
                const int64_t key = (int64_t)jb * BN + r;
                const bool ok = key < a.n_kv;
                const int64_t kr = kv0 + (ok ? key : 0);
                densify_row<D>(sb + C::OFF_K, BN, r, ok, a.k_idx + kr * k, a.k_val + kr * k, k);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(KK_FULL));
        }
        for (int s = 0; s < ns; ++s) {
            const int st = s % C::NQ, u = s / C::NQ;
            const int h = g * R + s / nib, ib = ib0 + s % nib;
            const int64_t i = (int64_t)ib * BM + r;
            const bool ok = i < a.n_q;
            const int64_t row = ((int64_t)b * a.H + h) * a.n_q + (ok ? i : 0);
            if (!SFA_BWD_TMA && s + 1 < ns) {  // next step's query codes (and LSE, D) into L1
                const int h1 = g * R + (s + 1) / nib, ib1 = ib0 + (s + 1) % nib;
                const int64_t i1 = (int64_t)ib1 * BM + r;
                if (i1 < a.n_q) {
                    const int64_t row1 = ((int64_t)b * a.H + h1) * a.n_q + i1;
                    prefetch_code_row(a.q_idx + row1 * k, a.q_val + row1 * k);
                }
            }
            mbar_wait(BAR(QQ_EMPTY + st), (u & 1) ^ 1);
            if (SFA_BWD_TMA) {  // the Q~ tile by TMA; its bytes join this stage's four warp arrivals
                if (warp == ROW_WARPS && lane == 0) {
                    mbar_expect_tx(BAR(QQ_FULL + st), BM * D * 2);
#pragma unroll
                    for (int cb = 0; cb < D / 64; ++cb)
                        tma_load_3d(sb + C::OFF_Q + st * BM * D * 2 + cb * BM * 128, &tm_q, BAR(QQ_FULL + st), cb * 64,
                                    ib * BM, b * a.H + h);
                }
            } else {
                densify_row<D>(sb + C::OFF_Q + st * BM * D * 2, BM, r, ok, a.q_idx + row * k, a.q_val + row * k, k);
            }
            ldv[st * 2 * BM + r] = ok ? __ldg(a.lse + row) * 1.4426950408889634f : 0.f;
            ldv[st * 2 * BM + BM + r] = ok ? __ldg(a.Dr + row) : 0.f;
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(QQ_FULL + st));
        }
        asm volatile("bar.arrive 6, 256;" ::: "memory");  // done with the Q~ ring (the dK~ epilogue reuses it)
    } else if (warp == 12) {
        // ==================== tcgen05.mma issuer ====================
        if (lane == 0 && ns > 0) {
            constexpr uint32_t idS = umma_idesc_f16kind(BN, BM, 0, 0, 1);  // K~ . Q~^T and V . dO^T
            constexpr uint32_t idV = umma_idesc_f16kind(BN, DV, 0, 1, 1);  // P^T[TMEM] . dO (MN-major)
            constexpr uint32_t idK = umma_idesc_f16kind(BN, D, 0, 1, 1);   // dS^T[TMEM] . Q~ (MN-major)
            const uint32_t ka = sb + C::OFF_K, va = sb + C::OFF_V;
            mbar_wait(BAR(KK_FULL), 0);
            mbar_wait(BAR(KV_FULL), 0);
            auto issue_S = [&](int ss) {  // S^T = K~ Q~(ss)^T
                const uint32_t qa = sb + C::OFF_Q + (ss % C::NQ) * BM * D * 2;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) umma_ss(tmem, kmaj(ka, BN, kk), kmaj(qa, BM, kk), idS, kk > 0);
                umma_commit(BAR(SS_FULL));
            };
            auto issue_dP = [&](int ss) {  // dP^T = V dO(ss)^T
                const uint32_t da = sb + C::OFF_DO;
                mbar_wait(BAR(DOO_FULL), ss & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < DV / 16; ++kk) umma_ss(tmem + 128, kmaj(va, BN, kk), kmaj(da, BM, kk), idS, kk > 0);
                umma_commit(BAR(KDP_FULL));
            };
            mbar_wait(BAR(QQ_FULL), 0);
            tc_fence_after();
            issue_S(0);
            issue_dP(0);
            for (int s = 0; s < ns; ++s) {
                const int st = s % C::NQ;
                const uint32_t qa = sb + C::OFF_Q + st * BM * D * 2, da = sb + C::OFF_DO;
                mbar_wait(BAR(P_READY), s & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < BM / 16; ++kk)  // dV += P^T dO
                    umma_ts(tmem + DV_COL, tmem + packed_col(kk), mnmaj(da, BM, kk), idV, (s > 0 || kk > 0) ? 1u : 0u);
                umma_commit(BAR(DOO_EMPTY));
                if (s + 1 < ns) {
                    const int s1 = s + 1;
                    mbar_wait(BAR(QQ_FULL + s1 % C::NQ), (s1 / C::NQ) & 1);
                    tc_fence_after();
                    issue_S(s1);  // over P^T(s): dV(s), issued above, reads it first
                }
                mbar_wait(BAR(KDS_READY), s & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < BM / 16; ++kk)  // dK~ += dS^T Q~
                    umma_ts(tmem + DK_COL, tmem + 128 + packed_col(kk), mnmaj(qa, BM, kk), idK,
                            (s > 0 || kk > 0) ? 1u : 0u);
                umma_commit(BAR(QQ_EMPTY + st));
                if (s + 1 < ns) issue_dP(s + 1);  // over dS^T(s): dK~(s), issued above, reads it first
            }
            umma_commit(BAR(OUT_FULL));
        }
        __syncwarp();
    } else if (warp == 13) {
        // ==================== TMA: V tile once, dO tiles per step ====================
        if (lane == 0 && ns > 0) {
            mbar_arrive_expect_tx(BAR(KV_FULL), BN * DV * 2);
#pragma unroll
            for (int cb = 0; cb < DV / 64; ++cb)
                tma_load_3d(sb + C::OFF_V + cb * BN * 128, &tm_v, BAR(KV_FULL), cb * 64, jb * BN, b * a.H_kv + g);
            for (int s = 0; s < ns; ++s) {
                const int h = g * R + s / nib, ib = ib0 + s % nib;
                mbar_wait(BAR(DOO_EMPTY), (s & 1) ^ 1);
                mbar_arrive_expect_tx(BAR(DOO_FULL), BM * DV * 2);
#pragma unroll
                for (int cb = 0; cb < DV / 64; ++cb)
                    tma_load_3d(sb + C::OFF_DO + cb * BM * 128, &tm_do, BAR(DOO_FULL), cb * 64, ib * BM, b * a.H + h);
            }
        }
        __syncwarp();
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

// bf16 [planes][rows][dv] as 3-D TMA map, box 64 x 128 rows, 128B swizzle (zero fill past `rows`)
bool make_map(CUtensorMap *tm, const void *base, int dv, int64_t rows, int64_t planes) {
    auto encode = get_encode();
    if (!encode) return false;
    cuuint64_t dims[3] = {(cuuint64_t)dv, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)dv * 2, (cuuint64_t)rows * dv * 2};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int DV>
cudaError_t launch_bwd_t(const BwdArgs &a, const CUtensorMap &tv, const CUtensorMap &tdo, const CUtensorMap &tq,
                         const CUtensorMap &tk, cudaStream_t st) {
    using CQ = DqCfg<D, DV>;
    using CK = KvCfg<D, DV>;
    auto kq = bwd_dq_kernel<D, DV>;
    auto kk = bwd_dkdv_kernel<D, DV>;
    cudaError_t e = cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, CQ::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, CK::SMEM);
    if (e != cudaSuccess) return e;
    const int64_t nq_items = (int64_t)a.B * a.H * a.nqb, nk_items = (int64_t)a.B * a.H_kv * a.nkt;
    if (nq_items > INT32_MAX || nk_items > INT32_MAX) return cudaErrorNotSupported;
    if (nk_items > 0) kk<<<(unsigned)nk_items, NTH, CK::SMEM, st>>>(tv, tdo, tq, tk, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (nq_items > 0) kq<<<(unsigned)nq_items, NTH, CQ::SMEM, st>>>(tv, tdo, tq, tk, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd(const AttnParams &p, int d, int d_v, const void *dO, float *Dws, void *qd, void *kd,
                            float *dq, float *dk, float *dv, cudaStream_t st) {
    if ((d != 64 && d != 128) || (d_v != 64 && d_v != 128)) return cudaErrorNotSupported;
    if (SFA_BWD_TMA) {  // Q~ and K~ rows, decompressed once per row for the kernels' TMA
        cudaError_t e = launch_kdense(p.q_idx, p.q_val, (int64_t)p.B * p.H * p.n_q, d, p.k, qd, st);
        if (e == cudaSuccess) e = launch_kdense(p.k_idx, p.k_val, (int64_t)p.B * p.H_kv * p.n_kv, d, p.k, kd, st);
        if (e != cudaSuccess) return e;
    }
    const int64_t rows = (int64_t)p.B * p.H * p.n_q;
    if (rows > 0) {
        bwd_prep_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(static_cast<const uint16_t *>(p.o),
                                                                   static_cast<const uint16_t *>(dO), rows, d_v, Dws);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    BwdArgs a;
    a.q_idx = p.q_idx;
    a.k_idx = p.k_idx;
    a.q_val = static_cast<const uint16_t *>(p.q_val);
    a.k_val = static_cast<const uint16_t *>(p.k_val);
    a.lse = p.lse;
    a.Dr = Dws;
    a.dq = dq;
    a.dk = dk;
    a.dv = dv;
    a.B = p.B;
    a.H = p.H;
    a.H_kv = p.H_kv;
    a.k = p.k;
    a.n_q = p.n_q;
    a.n_kv = p.n_kv;
    a.q_pos0 = p.q_pos0;
    a.causal = p.causal;
    a.nqb = (int)((p.n_q + BM - 1) / BM);
    a.nkt = (int)((p.n_kv + BN - 1) / BN);
    a.c_scale = p.scale_log2;
    a.scale = p.scale_log2 / 1.4426950408889634f;
    CUtensorMap tv, tdo, tq, tk;
    memset(&tq, 0, sizeof(tq));
    memset(&tk, 0, sizeof(tk));
    if (!make_map(&tv, p.v, d_v, p.n_kv, (int64_t)p.B * p.H_kv) || !make_map(&tdo, dO, d_v, p.n_q, (int64_t)p.B * p.H))
        return cudaErrorInvalidValue;
    if (SFA_BWD_TMA &&
        (!make_map(&tq, qd, d, p.n_q, (int64_t)p.B * p.H) || !make_map(&tk, kd, d, p.n_kv, (int64_t)p.B * p.H_kv)))
        return cudaErrorInvalidValue;
    if (d == 64) return d_v == 64 ? launch_bwd_t<64, 64>(a, tv, tdo, tq, tk, st) : launch_bwd_t<64, 128>(a, tv, tdo, tq, tk, st);
    return d_v == 64 ? launch_bwd_t<128, 64>(a, tv, tdo, tq, tk, st) : launch_bwd_t<128, 128>(a, tv, tdo, tq, tk, st);
}

}  // namespace sfa
