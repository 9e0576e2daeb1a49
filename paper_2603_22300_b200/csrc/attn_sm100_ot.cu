// attn_sm100_ot.cu -- FlashSFA forward on sm_100a tensor cores with a TRANSPOSED output accumulator
// (steps 4-8 of DESIGN.md; Alg. 1, Sec. 3.2).  SFA_KERNEL_SM100_OT.
//
// Same computation as attn_sm100.cu (scores = dense contraction of the decompressed k-sparse rows,
// reading A1/R1; fp16 P x 2^7 against the per-head scaled fp16 V copy, reading A12; lazy O rescale),
// laid out so that every P.V tensor-core instruction has N = 256:
//
//   S_t(j)   = Q~_t K~(j)^T             M = 128 query rows, N = 128 keys, K = d        (SS, per tile t)
//   O^T     += V(j)^T [P_0(j) ; P_1(j)]^T  M = d_v = 128,  N = 256 queries of BOTH tiles, K = 128 keys
//
// tools/umma_bench.cu: an M = 128 instruction costs ~75-100 clocks for any N <= 128 but N = 256 runs
// at the full 8192 FLOP/clk/SM (profiles/r01_umma_microbench.txt), so the P.V half of the tensor
// work drops from 16 x ~100 to 8 x 128 clocks per key tile; each tile's S MMAs are issued as soon as
// that tile has read its previous scores (issuing both tiles' S interleaved, two accumulators, was
// ~2 % slower).  P goes to shared memory (the B operand of the
// transposed product), so S_t's TMEM columns are free as soon as the softmax has read them and
// S_t(j+1) runs on the tensor pipe while the softmax of tile j computes its exponentials: no
// softmax -> MMA -> softmax chain per tile as in attn_sm100.cu.
//
// Warp roles (512 threads):
//   warps 0-3   softmax for query tile 0 (thread = query row = TMEM lane of S_0); with warps 4-7
//   warps 4-7   softmax for query tile 1        they also rescale O^T columns and run the epilogue
//   warps 8-11  decompression of Q~ (once) and K~(j) from the key codes into a 2-stage ring
//   warp 12     tcgen05.mma issuer (one thread) + TMEM owner
//   warp 13     TMA producer for V (single stage)
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O^T [256,512) (lane = output feature, column =
// query: tile 0's 128 queries then tile 1's).
// Shared memory (d = 128): Q~ 2 x 32 KB, K~ 2 x 32 KB, V 32 KB, P 64 KB (256 rows x 128 keys fp16,
// K-major SW128), 1 KB per-query factors; 226 KB of the 227 KB.
#include <cudaTypedefs.h>
#include <cstring>
#include <mutex>

#include "densify.cuh"
#include "topk_row.cuh"
#include "launch.cuh"
#include "sm100.cuh"

namespace sfa {
using namespace sm100;
using namespace dz;

namespace {

// exponentials per group of 8 pairs computed by exp2_poly2 on the FMA pipe instead of MUFU.EX2
// (16 ex2 / clk / SM on B200, tools/mufu_bench.cu): 2 of 8 (25 %) is fastest at Qwen3-32K (1: +4 %,
// 3: +2 %, 4: +15 %; none: +8 %)
#ifndef SFA_OT_POLY
#define SFA_OT_POLY 2
#endif
// P is handed to the tensor core once per 128-key tile (two 64-key hand-offs measured slower: attention
// 7.51-7.59 vs 7.08-7.12 ms, profiles/r02_ot_ab.txt).  The K~ ring is filled by TMA from the key rows
// the prepare step decompresses once per key (k_dense_kernel, vprep.cu): rebuilding every K~ tile in
// shared memory once per work item cost ~630 of the ~3,200 shared-memory wavefronts of a key-tile
// iteration (6.93 -> 6.53 ms, profiles/r02_ot_ab.txt).
//
// Tile scheduler: persistent CTAs (one per SM) take work items dynamically -- CTA c starts with item c,
// then its K~ producer warp claims the next unclaimed item (atomicAdd on a counter in the workspace)
// and publishes it to the CTA's other roles through a 4-slot ring in shared memory.  The item list is
// in kv-group-major, heaviest-causal-first order, so this is greedy LPT (simulated 98 % balance at
// Qwen3-32K vs 94 % for a static snake order, which measured 2 % slower than one item per CTA).
// Every pipeline counter runs across items: the next
// item's Q~ is built as soon as the current item's last S MMA has completed (QEMPTY), its first S MMAs
// are issued during the current item's last softmax, its K~ / V tiles stream in meanwhile, and only
// its first P.V waits for the current item's epilogue to have read O^T out of TMEM (OEMPTY).




constexpr int BM = 128;  // query rows per tile (UMMA M of S)
constexpr int BN = 128;  // keys per tile (UMMA N of S, UMMA K of P.V)
constexpr int DV = 128;  // output features (UMMA M of O^T)
constexpr int NTHREADS = 512;

template <int D>
struct Cfg {
    static constexpr int QT = BM * D * 2;  // one decompressed Q~ tile
    static constexpr int KT = BN * D * 2;  // one K~ stage
    static constexpr int VT = BN * DV * 2; // the V stage
    static constexpr int PT = 2 * BM * BN * 2;  // P of both query tiles
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + 2 * QT;
    static constexpr int NV = 1;  // V stages
    static constexpr int NK = 2;  // K~ stages
    static constexpr int NP = 1;  // P stages
    static constexpr int OFF_V = OFF_K + NK * KT;
    static constexpr int OFF_P = OFF_V + NV * VT;
    static constexpr int OFF_BAR = OFF_P + NP * PT;
    static constexpr int OFF_F = OFF_BAR + 256;  // 2 x 128 fp32 per-query factors (alpha, then 1/l)
    static constexpr int SMEM = OFF_F + 1024 + 1024;  // + slack to align the base to 1024 B
    static constexpr int O_COL = 256;
};
static_assert(Cfg<128>::SMEM <= 232448, "shared memory budget");

// mbarrier slots
enum {
    KFULL = 0, KEMPTY = 2, VFULL = 4, VEMPTY = 6, SFULL = 8, SEMPTY = 10, PFULL = 12, PEMPTY = 14, OFULL = 16,
    QFULL = 17, QEMPTY = 18, OEMPTY = 19, IFULL = 20, IEMPTY = 24, NBAR = 28
};
constexpr int NRING = 4;  // work-item ring slots

struct OtArgs {
    AttnParams p;
    int32_t nqb;         // ceil(n_q / BM)
    int32_t pair_heads;  // 1: tiles (2hp, 2hp+1) at one q block; 0: (h, 2p), (h, 2p+1)
    int32_t per_rank;    // work items per q-block rank
    int32_t nkt;         // ceil(n_kv / BN)
    int32_t items;       // work items (the persistent CTAs walk them, sched_item)
    int32_t dv_out;      // d_v of O (64: V's fp16 copy is zero-padded to DV = 128 columns, vprep.cu)
    float c_scale;       // scale * log2(e)
    float *dbg;          // optional: raw S of the first key tile of work item 0, tile 0 (tests)
};

constexpr float P_SHIFT = 7.f;  // P stored as fp16 * 2^7 (attn_sm100.cu, reading A12)



struct Tile {
    int h, qb;
    bool valid;
};

// Work-item order.  SFA_OT_ORDER 1 (default): kv-group major -- all work items of one (batch, kv head)
// group run back to back (heaviest causal query blocks of the group first), so the ~148 resident CTAs
// share one group's K codes and V in L2 instead of streaming all groups' at once.  0: query-block
// major across every head (global LPT order, the earlier version).
#ifndef SFA_OT_ORDER
#define SFA_OT_ORDER 1
#endif
// 1: one work item per CTA (grid = items, the round-1 launch) instead of the persistent tile scheduler
#ifndef SFA_OT_ONE_ITEM_PER_CTA
#define SFA_OT_ONE_ITEM_PER_CTA 0
#endif
__device__ __forceinline__ void decode_item(const OtArgs &a, int item, int &b, Tile (&t)[2]) {
    const AttnParams &p = a.p;
#if SFA_OT_ORDER
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
    return;
#endif
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

// one work item's geometry: batch, kv group, its key tiles j0, j0 + 1, ..., j0 + nt - 1 -- or, with a
// block selection (BSEL, NSA-style token sparsity), the tiles bl[0 .. nt) (none: no selected tile at or
// below the causal limit -> one fully masked tile, O = 0, LSE = -inf)
struct ItemGeo {
    int b, g, nt, j0;
    Tile tl[2];
    const int32_t *bl;
    bool none;
};
template <bool WIN, bool BSEL = false>
__device__ __forceinline__ ItemGeo item_geo(const OtArgs &a, int item) {
    const AttnParams &p = a.p;
    ItemGeo G;
    decode_item(a, item, G.b, G.tl);
    G.g = G.tl[0].h / (p.H / p.H_kv);
    int nt = a.nkt;
    if (p.causal) {  // up to the diagonal of the item's last valid row
        const int qbl = G.tl[1].valid ? G.tl[1].qb : G.tl[0].qb;
        int64_t last = (int64_t)qbl * BM + BM - 1;
        if (last > p.n_q - 1) last = p.n_q - 1;
        const int64_t lim = (p.q_pos0 + last) / BN + 1;
        if (lim < nt) nt = (int)lim;
    }
    // sliding window (N4): key tiles before the window of the item's first row are skipped
    int j0 = 0;
    if (WIN) {
        const int64_t kb = p.q_pos0 + (int64_t)G.tl[0].qb * BM - p.window + 1;
        if (kb > 0) j0 = (int)(kb / BN);
        if (j0 > nt - 1) j0 = nt - 1;  // no key left: one fully masked tile (O = 0, LSE = -inf)
        nt -= j0;
    }
    G.bl = nullptr;
    G.none = false;
    if (BSEL) {  // the selected key tiles of the item's query block (both tiles share it: pair_heads)
        G.bl = p.bsel + ((int64_t)(G.b * p.H_kv + G.g) * a.nqb + G.tl[0].qb) * p.max_sel;
        int cnt = 0;
        while (cnt < p.max_sel) {
            const int t = __ldg(G.bl + cnt);
            if (t < 0 || t >= nt) break;  // ascending list: the rest is padding or above the causal limit
            ++cnt;
        }
        G.none = cnt == 0;
        nt = cnt > 0 ? cnt : 1;
    }
    G.nt = nt;
    G.j0 = j0;
    return G;
}
// the key tile of iteration j of an item
template <bool BSEL>
__device__ __forceinline__ int key_tile(const ItemGeo &G, int j) {
    return BSEL ? (G.none ? 0 : __ldg(G.bl + j)) : G.j0 + j;
}
// the m-th work item of this CTA (-1: none left), from the ring the K~ producer fills; every consumer
// warp reads each slot once and releases it (one arrive per warp; single-lane roles call with
// whole_warp = false)
__device__ __forceinline__ int ring_get(volatile int *ring, uint32_t ifull, uint32_t iempty, int m, bool whole_warp) {
    const int slot = m & (NRING - 1);
    mbar_wait(ifull + 8u * slot, (m / NRING) & 1);
    const int item = ring[slot];
    if (whole_warp) __syncwarp();
    if (!whole_warp || (threadIdx.x & 31) == 0) mbar_arrive(iempty + 8u * slot);
    return item;
}

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

__device__ __forceinline__ void prefetch_l1(const void *ptr) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
}

// EDGE (reading A1/R2, edges.cu): a pair enters the softmax only if the supports intersect.  Per key
// tile each softmax thread ORs the tile's feature bitsets kf[f] over the k features of its row:
// eh[q] bit c = "key 32q+c shares a feature with this row" (k 16-byte loads, issued before the
// wait for S), ANDs in the causal / ragged bound, and excludes the other keys like the causal mask.
// FUSEQ: step 1 on Q fused into the prologue -- the softmax thread of query row r
// of tile t loads the DENSE bf16 Q row, selects its top-k with the same code as the stand-alone kernel
// (topk_row.cuh), writes the masked row straight into the swizzled Q~ tile and (optionally) the row's
// code to q_idx_out / q_val_out; the decompression warps then only build K~.
// WIN: causal sliding window (N4) -- a template flag so the full-causal kernel carries none of its work.
// BSEL: NSA-style block selection (N4): per (b, kv head, query block) an ascending list of the key tiles
// the block may attend (p.bsel), intersected with the causal mask; EDGE / FUSEQ / WIN off.
template <int D, bool DBG, bool EDGE, bool FUSEQ, bool WIN, bool BSEL>
__global__ void __launch_bounds__(NTHREADS, 1) attn_sm100_ot_kernel(const __grid_constant__ CUtensorMap tmap_v,
                                                                      const __grid_constant__ CUtensorMap tmap_k,
                                                                      const OtArgs a) {
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
    volatile int *ring = reinterpret_cast<volatile int *>(gbase + C::OFF_BAR + 240);  // NRING item ids
    float *fac = reinterpret_cast<float *>(gbase + C::OFF_F);

#define ITEM_LOOP_BEGIN(WHOLE_WARP)                                                                 \
    for (int m_ = 0;; ++m_) {                                                                      \
        const int item_ = ring_get(ring, BAR(IFULL), BAR(IEMPTY), m_, WHOLE_WARP);                 \
        if (item_ < 0) break;                                                                      \
        const ItemGeo G_ = item_geo<WIN, BSEL>(a, item_);                                                \
        const int b = G_.b, g = G_.g, nt = G_.nt, j0 = G_.j0;                                      \
        const Tile tl[2] = {G_.tl[0], G_.tl[1]};                                                   \
        (void)b; (void)g; (void)tl;
#define ITEM_LOOP_END }

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBAR; ++i) {
            uint32_t cnt = 1;
            if (i == SEMPTY || i == SEMPTY + 1 || i == QFULL) cnt = 4;
            if (FUSEQ && i == QFULL) cnt = 8;  // the eight softmax warps build Q~
            if (i == PFULL || i == PFULL + 1 || i == OEMPTY) cnt = 8;
            if (i >= IEMPTY && i < IEMPTY + NRING) cnt = FUSEQ ? 10 : 14;  // V, MMA, 8 softmax (+ 4 Q~) warps
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
        const uint32_t tS = tmem + lane_off + (uint32_t)(t * 128);
        // O^T: this thread's TMEM lane is output feature r; tile t's queries are columns [128t, 128t+128)
        const uint32_t tO = tmem + lane_off + (uint32_t)(C::O_COL + t * BM);
        uint32_t sc = 0;  // S tiles of this query tile consumed so far, over all items (phase of SFULL / PFULL)
        ITEM_LOOP_BEGIN(true)
        const int64_t i = (int64_t)tl[t].qb * BM + r;
        const bool row_ok = tl[t].valid && i < p.n_q;
        int64_t kend = p.n_kv;
        if (p.causal && p.q_pos0 + i + 1 < kend) kend = p.q_pos0 + i + 1;
#ifdef SFA_FAULT_CAUSAL_PLUS1  // negative control: the diagonal's next key also allowed
        if (p.causal && kend < p.n_kv) kend += 1;
#endif
        const int64_t kbeg = WIN ? p.q_pos0 + i - p.window + 1 : 0;  // N4 sliding window
        const float cs = a.c_scale;
        if (FUSEQ) {
            // ---- step 1 on this row: dense Q row -> top-k masks -> masked row into the Q~ tile
            constexpr int NW = D / 2, NC = D / 8;  // words / 16-byte chunks per row
            const int64_t qrow = ((int64_t)b * p.H + tl[t].h) * p.n_q + (row_ok ? i : 0);
            {   // coalesced loads of the CTA's 256 dense rows into the (still unused) P buffer, 16-byte
                // chunks XOR-swizzled by row so each thread then reads its own row conflict-free
                const int tid = threadIdx.x;  // 0..255 = the eight softmax warps
                uint8_t *stage = gbase + C::OFF_P;
                for (int v = tid; v < 2 * BM * NC; v += 2 * BM) {
                    const int rr = v / NC, c = v % NC, tt = rr / BM, ri = rr % BM;
                    const int64_t ii = (int64_t)tl[tt].qb * BM + ri;
                    uint4 w = make_uint4(0u, 0u, 0u, 0u);
                    if (tl[tt].valid && ii < p.n_q)
                        w = __ldcs(reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(p.q_dense) +
                                                                   (((int64_t)b * p.H + tl[tt].h) * p.n_q + ii) * D) + c);
                    *reinterpret_cast<uint4 *>(stage + rr * D * 2 + ((c ^ (rr & 15) & (NC - 1)) << 4)) = w;
                }
                named_bar_sync(3, 2 * BM);
            }
            uint32_t raw[NW], ab[NW];
            {
                const int rr = t * BM + r;
                const uint8_t *stage = gbase + C::OFF_P + rr * D * 2;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const uint4 w = *reinterpret_cast<const uint4 *>(stage + ((c ^ (rr & 15) & (NC - 1)) << 4));
                    raw[4 * c] = w.x; raw[4 * c + 1] = w.y; raw[4 * c + 2] = w.z; raw[4 * c + 3] = w.w;
                }
            }
#pragma unroll
            for (int q = 0; q < NW; ++q) ab[q] = raw[q] & 0x7FFF7FFFu;
            const uint32_t mx = tk::row_max_key(ab);
            if (row_ok && p.status_word != nullptr && mx >= 0x7F80u) atomicOr(p.status_word, 1u);
            uint32_t gm[D / 32];
            tk::select_masks(ab, p.k, gm, mx);
            if (!row_ok) {
#pragma unroll
                for (int w = 0; w < D / 32; ++w) gm[w] = 0u;
            }
            const uint32_t qt = sbase + C::OFF_Q + t * C::QT;
#pragma unroll
            for (int kb = 0; kb < D / 64; ++kb)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint32_t o4[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int W = 4 * (8 * kb + c) + q;  // word = features 2W, 2W + 1
                        const uint32_t b2 = (gm[W >> 4] >> (2 * (W & 15))) & 3u;
                        o4[q] = raw[W] & (((b2 & 1u) * 0xFFFFu) | ((b2 >> 1) * 0xFFFF0000u));
                    }
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(qt + kb * BM * 128 + r * 128 +
                                                                                    ((c ^ (r & 7)) << 4)),
                                 "r"(o4[0]), "r"(o4[1]), "r"(o4[2]), "r"(o4[3])
                                 : "memory");
                }
            if (row_ok && p.q_idx_out != nullptr) {  // the row's code, ascending (A4)
                uint8_t *oi = p.q_idx_out + qrow * p.k;
                uint16_t *ov = static_cast<uint16_t *>(p.q_val_out) + qrow * p.k;
                int pos = 0;
#pragma unroll
                for (int w = 0; w < D / 32; ++w) {
                    uint32_t mm = gm[w];
                    while (mm != 0u) {
                        const int f = 32 * w + (__ffs(mm) - 1);
                        mm &= mm - 1u;
                        oi[pos] = (uint8_t)f;
                        uint16_t vbits;  // re-read from the Q~ row just written (no dynamic register index)
                        asm volatile("ld.shared.u16 %0, [%1];"
                                     : "=h"(vbits)
                                     : "r"(qt + (f >> 6) * BM * 128 + r * 128 + ((((f >> 3) & 7) ^ (r & 7)) << 4) +
                                           (f & 7) * 2));
                        ov[pos] = vbits;
                        ++pos;
                    }
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(QFULL));
        }
        float *f_t = fac + t * BM;
        const uint32_t prow = sbase + C::OFF_P + (uint32_t)(t * BM + r) * 128u;  // row t*128+r, key atom 0
        const int bar_id = 1 + t;
        const uint8_t *qi_row = p.q_idx + (((int64_t)b * p.H + tl[t].h) * p.n_q + (row_ok ? i : 0)) * p.k;
        const uint4 *kf_head = reinterpret_cast<const uint4 *>(p.kfmask) + (int64_t)(b * p.H_kv + g) * a.nkt * D;
        // EDGE, k <= 16: the row's feature indices stay in registers (4 x 4 bytes), so the k bitset
        // loads of a tile are independent and issue back to back
        uint32_t qw[4] = {0u, 0u, 0u, 0u};
        if (EDGE && row_ok && p.k <= 16)
            for (int u = 0; u < p.k; ++u) qw[u >> 2] |= (uint32_t)__ldg(qi_row + u) << (8 * (u & 3));
        if (EDGE && lane < 2 * (D / 16)) prefetch_l1(kf_head + lane * 8);  // tile 0: D x 16 bytes of bitsets
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            const int kt = key_tile<BSEL>(G_, j);
            int64_t lim64 = (BSEL && G_.none) ? 0 : kend - (int64_t)kt * BN;
            const int lim = lim64 < 0 ? 0 : (lim64 > BN ? BN : (int)lim64);
            int lo = 0;  // first allowed key of the window in this tile
            if (WIN) {
                const int64_t lo64 = kbeg - (int64_t)kt * BN;
                lo = lo64 < 0 ? 0 : (lo64 > BN ? BN : (int)lo64);
            }
            uint32_t eh[4];
            if (EDGE) {
                const uint4 *kf = kf_head + (int64_t)kt * D;
                uint4 h = make_uint4(0u, 0u, 0u, 0u);
                if (row_ok && p.k <= 16) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        if (u < p.k) {
                            const uint4 x = __ldg(kf + ((qw[u >> 2] >> (8 * (u & 3))) & 0xFFu));
                            h.x |= x.x;
                            h.y |= x.y;
                            h.z |= x.z;
                            h.w |= x.w;
                        }
                    }
                } else if (row_ok) {
#pragma unroll 4
                    for (int u = 0; u < p.k; ++u) {
                        const uint4 x = __ldg(kf + __ldg(qi_row + u));
                        h.x |= x.x;
                        h.y |= x.y;
                        h.z |= x.z;
                        h.w |= x.w;
                    }
                }
                // the next tile's bitsets into L1 while this tile's softmax runs
                if (j + 1 < nt && lane < 2 * (D / 16)) prefetch_l1(kf + D + lane * 8);
                const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rem = lim - 32 * q;  // step 5 folded in: keys at or past lim are excluded
                    const int rlo = lo - 32 * q;   // and keys before the window
                    eh[q] = hw[q] & (rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : ((1u << rem) - 1u))) &
                            (rlo <= 0 ? 0xFFFFFFFFu : (rlo >= 32 ? 0u : ~((1u << rlo) - 1u)));
                }
            }
            mbar_wait(BAR(SFULL + t), sc & 1);
            if (lane == 0 && wq == 0) TLREC(0x1000 | (t << 10) | (sc & 511));
            tc_fence_after();
            uint32_t s[4][32];
            float mq[4];  // four independent max chains; keys 64-127 load while 0-63 are reduced
            tmem_ld32(tS, s[0]);
            tmem_ld32(tS + 32, s[1]);
            tmem_ld_wait();
            tmem_ld32(tS + 64, s[2]);
            tmem_ld32(tS + 96, s[3]);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (EDGE) {
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (!((eh[q] >> c) & 1u)) s[q][c] = 0xFF800000u;
                }
                mq[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < 32; ++c) mq[q] = fmaxf(mq[q], __uint_as_float(s[q][c]));
            }
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(SEMPTY + t));  // S_t may be overwritten by S_t(j+1)
#pragma unroll
            for (int q = 2; q < 4; ++q) {
                if (EDGE) {
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (!((eh[q] >> c) & 1u)) s[q][c] = 0xFF800000u;
                }
                mq[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < 32; ++c) mq[q] = fmaxf(mq[q], __uint_as_float(s[q][c]));
            }
            if (DBG && blockIdx.x == 0 && m_ == 0 && t == 0 && j == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 32; ++c) a.dbg[r * BN + 32 * q + c] = __uint_as_float(s[q][c]);
            }
            if (!EDGE && (lim < BN || (WIN && lo > 0))) {  // step 5 on diagonal / ragged / window-edge tiles: excluded -> -inf
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    mq[q] = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        if (32 * q + c >= lim || 32 * q + c < lo) s[q][c] = 0xFF800000u;
                        mq[q] = fmaxf(mq[q], __uint_as_float(s[q][c]));
                    }
                }
            }
            const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * cs;
            if (lane == 0 && wq == 0) TLREC(0x5000 | (t << 10) | (sc & 511));
            const float m_new = fmaxf(m, mx);
            // O^T columns are shared by the whole warpgroup: rescale all of tile t or none of it
            const bool rescale = named_bar_or(bar_id, 128, m_new > m + 8.f);
#ifdef SFA_FAULT_NO_O_RESCALE  // negative control: alpha applied to l but never to O^T
            const bool rescale_o = false;
#else
            const bool rescale_o = rescale;
#endif
            if (lane == 0 && wq == 0) TLREC(0x6000 | (t << 10) | (sc & 511));
            if (rescale) {
                const float alpha = (m_new == -INFINITY) ? 1.f : fast_exp2(m - m_new);
                l *= alpha;
                m = m_new;
                if (j > 0) f_t[r] = alpha;
            }
            const float ms = ((m == -INFINITY) ? 0.f : m) - P_SHIFT;  // p = 2^(s - m + P_SHIFT)
            float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // keys [64h, 64h + 64) = P atom h
                uint32_t pk[32];
#pragma unroll
                for (int q = 2 * h; q < 2 * h + 2; ++q) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        float x0, x1, p0, p1;
                        ffma2(x0, x1, __uint_as_float(s[q][2 * c]), __uint_as_float(s[q][2 * c + 1]), cs, -ms);
                        if ((c & 7) < SFA_OT_POLY) {  // SFA_OT_POLY pairs in 8 on the FMA pipe (exp2_poly2)
                            exp2_poly2(x0, x1, p0, p1);
                        } else
                        {
                            p0 = fast_exp2(x0);
                            p1 = fast_exp2(x1);
                        }
                        fadd2(rs0, rs1, p0, p1);
                        pk[16 * (q - 2 * h) + c] = pack_f16x2(p0, p1);
                    }
                }
                if (h == 0) {
                    if (lane == 0 && wq == 0) TLREC(0x4000 | (t << 10) | (sc & 511));
                    // the P buffer is free (the previous P.V, over all items, has read it)
                    mbar_wait(BAR(PEMPTY), (sc & 1) ^ 1);
                    if (lane == 0 && wq == 0) TLREC(0x7000 | (t << 10) | (sc & 511));
                    if (rescale_o && j > 0) {
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
                }
                // P row (t*128 + r), atom h: 16-byte chunk c8 swizzled by row
#pragma unroll
                for (int c8 = 0; c8 < 8; ++c8)
                    sts_v4(prow + (uint32_t)h * (2 * BM * 128) + ((uint32_t)(c8 ^ (r & 7)) << 4), pk[4 * c8], pk[4 * c8 + 1],
                           pk[4 * c8 + 2], pk[4 * c8 + 3]);
            }
            l += rs0 + rs1;
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(PFULL));
            if (lane == 0 && wq == 0) TLREC(0x2000 | (t << 10) | (sc & 511));
            ++sc;
        }
        // ---- epilogue (step 8): O = 2^e (sum_j P'_j V'_j) / l, V' = V 2^-e (vprep.cu)
        mbar_wait(BAR(OFULL), m_ & 1);
        if (lane == 0 && wq == 0) TLREC(0x8000 | (t << 10) | ((2 * m_) & 511));
        tc_fence_after();
        const float inv = l > 0.f ? __uint_as_float((uint32_t)(127 + vprep_head_exp(__ldg(p.v_amax + b * p.H_kv + g))) << 23) / l : 0.f;
        f_t[r] = inv;
        named_bar_sync(bar_id, 128);
        // O^T lane r = feature r: scale column c by 1/l of query c, transpose through shared memory
        // (the dead P buffer; row = query, 16-byte chunk swizzled by row) for row-contiguous stores
        const uint32_t so = sbase + C::OFF_P + (uint32_t)t * (BM * DV * 2);
        // per element: one FMUL, one cvt, one LOP3 (the chunk swizzle; (qq & 15) = (c & 15) is a constant of
        // the unrolled loop) and one STS with the row offset as an immediate; 1/l four queries per LDS.128;
        // the TMEM loads two 32-column blocks at a time (one wait per pair)
        const uint32_t rbase = so + (uint32_t)(r & 7) * 2, rh = (uint32_t)(r >> 3) << 4;
#pragma unroll 1
        for (int q = 0; q < BM / 32; q += 2) {
            uint32_t o[2][32];
            tmem_ld32(tO + 32 * q, o[0]);
            tmem_ld32(tO + 32 * q + 32, o[1]);
            tmem_ld_wait();
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
                const uint32_t qb = rbase + (uint32_t)(32 * (q + hq)) * (DV * 2);
#pragma unroll
                for (int c4 = 0; c4 < 32; c4 += 4) {
                    const float4 iv = *reinterpret_cast<const float4 *>(f_t + 32 * (q + hq) + c4);
                    const float ivs[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int c = c4 + u;
                        const float v = __uint_as_float(o[hq][c]) * ivs[u];
                        sts_u16(qb + (uint32_t)c * (DV * 2) + (rh ^ ((uint32_t)(c & 15) << 4)),
                                __bfloat16_as_ushort(__float2bfloat16_rn(v)));
                    }
                }
            }
        }
        // O^T is read out: the next item's first P.V may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(OEMPTY));
        named_bar_sync(bar_id, 128);
        const int64_t orow = ((int64_t)b * p.H + tl[t].h) * p.n_q + i;
        if (row_ok) {
            uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.o) + orow * a.dv_out);
            if (a.dv_out == DV) {
#pragma unroll
                for (int c = 0; c < DV / 8; ++c) dst[c] = lds_v4(so + (uint32_t)r * (DV * 2) + ((uint32_t)(c ^ (r & 15)) << 4));
            } else {  // d_v = 64: the padded features 64..127 of O^T are zero and not stored
#pragma unroll
                for (int c = 0; c < DV / 16; ++c) dst[c] = lds_v4(so + (uint32_t)r * (DV * 2) + ((uint32_t)(c ^ (r & 15)) << 4));
            }
            p.lse[orow] = l > 0.f ? (m + __log2f(l) - P_SHIFT) * 0.69314718055994530942f : -INFINITY;
        }
        if (lane == 0 && wq == 0) TLREC(0x8000 | (t << 10) | ((2 * m_ + 1) & 511));
        // both tiles' staging (the dead P buffer, where the other tile's rows interleave) is read before
        // either tile stores the next item's P
        named_bar_sync(5, 2 * BM);
        ITEM_LOOP_END
    } else if (wg == 2) {
        reg_dealloc<64>();
        // ============================ decompression of Q~ (per item) ============================
        const int r = threadIdx.x - 256;
        const int k = p.k;
        const uint16_t *qv = reinterpret_cast<const uint16_t *>(p.q_val);
        if (!FUSEQ) {
            ITEM_LOOP_BEGIN(true)
            if (m_ > 0) mbar_wait(BAR(QEMPTY), (m_ - 1) & 1);  // the previous item's S MMAs are complete
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int64_t i = (int64_t)tl[t].qb * BM + r;
                const bool ok = tl[t].valid && i < p.n_q;
                const int64_t row = ((int64_t)b * p.H + tl[t].h) * p.n_q + (ok ? i : 0);
                densify_row<D>(sbase + C::OFF_Q + t * C::QT, BM, r, ok, p.q_idx + row * k, qv + row * k, k);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(QFULL));
            ITEM_LOOP_END
        }
    } else {
        reg_dealloc<80>();
        if (warp == 12) {
            // ============================ tcgen05.mma issuer ============================
            if (lane == 0) {
                constexpr uint32_t idS = umma_idesc_f16kind(BM, BN, 0, 0, 1);      // bf16 Q~ x bf16 K~
                constexpr uint32_t idO = umma_idesc_f16kind(DV, 2 * BM, 1, 0, 0);  // fp16 V^T (MN-major) x fp16 P
                auto mma_O = [&](bool acc, int vs, int ps) {
                    const uint32_t va = sbase + C::OFF_V + vs * C::VT, pa = sbase + C::OFF_P + ps * C::PT;
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk)
                        umma_ss(tmem + C::O_COL, umma_desc_sw128(va + kk * 2048, BN * 128, 1024),
                                umma_desc_sw128(pa + (kk >> 2) * (2 * BM * 128) + (kk & 3) * 32, 16, 1024), idO,
                                (acc || kk > 0) ? 1u : 0u);
                };
                // one stream of key tiles over all items of this CTA: the S of the next tile (of this item,
                // or the next item's first) is issued before the P.V of the current one
                uint32_t kc = 0, gs = 0, vc = 0;  // K~ tiles consumed, S tiles issued (per query tile), V tiles
                auto next_S = [&](bool last_of_item) {
                    const int s1 = (int)(kc % C::NK);
                    mbar_wait(BAR(KFULL + s1), (kc / C::NK) & 1);
                    const uint32_t ka = sbase + C::OFF_K + s1 * C::KT;
#pragma unroll
                    for (int t = 0; t < 2; ++t) {  // each tile's S as soon as that tile has read its last one
                        if (gs > 0) mbar_wait(BAR(SEMPTY + t), (gs - 1) & 1);
                        tc_fence_after();
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            umma_ss(tmem + t * 128,
                                    umma_desc_sw128(sbase + C::OFF_Q + t * C::QT + (kk >> 2) * BM * 128 + (kk & 3) * 32, 16, 1024),
                                    umma_desc_sw128(ka + (kk >> 2) * BN * 128 + (kk & 3) * 32, 16, 1024), idS, kk > 0);
                        umma_commit(BAR(SFULL + t));
                    }
                    umma_commit(BAR(KEMPTY + s1));
                    if (last_of_item) umma_commit(BAR(QEMPTY));  // Q~ may be rebuilt for the next item
                    ++kc;
                    ++gs;
                };
                int m = 0, item = ring_get(ring, BAR(IFULL), BAR(IEMPTY), 0, false);
                if (item >= 0) {
                    ItemGeo G = item_geo<WIN, BSEL>(a, item);
                    mbar_wait(BAR(QFULL), 0);
                    next_S(G.nt == 1);
                    for (;;) {
                        int item_n = -1;
                        ItemGeo Gn = G;
                        for (int j = 0; j < G.nt; ++j) {
                            if (j + 1 < G.nt) {
                                next_S(j + 2 == G.nt);
                            } else {  // the next item's first S overlaps this item's tail.  Read only now:
                                // the K~ producer publishes the next item after this item's last K~ load
                                item_n = ring_get(ring, BAR(IFULL), BAR(IEMPTY), m + 1, false);
                                if (item_n >= 0) {
                                    Gn = item_geo<WIN, BSEL>(a, item_n);
                                    mbar_wait(BAR(QFULL), (m + 1) & 1);
                                    next_S(Gn.nt == 1);
                                }
                            }
                            mbar_wait(BAR(VFULL), vc & 1);  // one V stage
                            mbar_wait(BAR(PFULL), vc & 1);  // one P per key tile
                            TLREC(0x3000 | (vc & 511));
                            if (j == 0 && m > 0) mbar_wait(BAR(OEMPTY), (m - 1) & 1);  // O^T read out
                            tc_fence_after();
                            mma_O(j > 0, 0, 0);
                            umma_commit(BAR(PEMPTY));
                            umma_commit(BAR(VEMPTY));
                            ++vc;
                        }
                        umma_commit(BAR(OFULL));
                        if (item_n < 0) break;
                        G = Gn;
                        ++m;
                    }
                }
            }
            __syncwarp();
        } else if (warp == 13) {
            // ============================ TMA producer for V ============================
            if (lane == 0) {
                uint32_t vc = 0;
                ITEM_LOOP_BEGIN(false)
                const int bhkv = b * p.H_kv + g;
                for (int j = 0; j < nt; ++j, ++vc) {
                    const int vs = (int)(vc % C::NV);
                    mbar_wait(BAR(VEMPTY + vs), ((vc / C::NV) & 1) ^ 1);
                    mbar_arrive_expect_tx(BAR(VFULL + vs), C::VT);
                    const uint32_t dst = sbase + C::OFF_V + vs * C::VT;
#pragma unroll
                    for (int cb = 0; cb < DV / 64; ++cb)
                        tma_load_3d(dst + cb * BN * 128, &tmap_v, BAR(VFULL + vs), cb * 64, key_tile<BSEL>(G_, j) * BN, bhkv);
                }
                ITEM_LOOP_END
            }
            __syncwarp();
        } else if (warp == 14) {
            // ============================ TMA producer for K~ (decompressed rows) ============================
            if (lane == 0) {
                uint32_t kc = 0;
                for (int m_ = 0;; ++m_) {
                    // claim the next item and publish it to the other roles
                    const int slot = m_ & (NRING - 1);
                    mbar_wait(BAR(IEMPTY + slot), ((m_ / NRING) & 1) ^ 1);
                    int item_ = m_ == 0 ? (int)blockIdx.x : (int)atomicAdd(p.sched, 1u) + (int)gridDim.x;
                    if (item_ >= a.items) item_ = -1;
                    ring[slot] = item_;
                    mbar_arrive(BAR(IFULL + slot));
                    if (item_ < 0) break;
                    const ItemGeo G_ = item_geo<WIN, BSEL>(a, item_);
                    const int b = G_.b, g = G_.g, nt = G_.nt, j0 = G_.j0;
                const int bhkv = b * p.H_kv + g;
                for (int j = 0; j < nt; ++j, ++kc) {
                    const int s = (int)(kc % C::NK);
                    mbar_wait(BAR(KEMPTY + s), ((kc / C::NK) & 1) ^ 1);
                    mbar_arrive_expect_tx(BAR(KFULL + s), C::KT);
                    const uint32_t dst = sbase + C::OFF_K + s * C::KT;
#pragma unroll
                    for (int cb = 0; cb < D / 64; ++cb)
                        tma_load_3d(dst + cb * BN * 128, &tmap_k, BAR(KFULL + s), cb * 64, key_tile<BSEL>(G_, j) * BN, bhkv);
                }
                ITEM_LOOP_END
            }
            __syncwarp();
        }
    }
#undef ITEM_LOOP_BEGIN
#undef ITEM_LOOP_END
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
cudaError_t launch_t(const OtArgs &a, cudaStream_t stream, int items) {
    using C = Cfg<D>;
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
    CUtensorMap tk;  // K~ rows (bf16 [B*H_kv][n_kv][D]), same box shape and swizzle as the decompression wrote
    memset(&tk, 0, sizeof(tk));
    {
        if (p.k_dense == nullptr) return cudaErrorInvalidValue;
        cuuint64_t kdims[3] = {(cuuint64_t)D, (cuuint64_t)p.n_kv, (cuuint64_t)p.B * p.H_kv};
        cuuint64_t kstrides[2] = {(cuuint64_t)D * 2, (cuuint64_t)p.n_kv * D * 2};
        cuuint32_t kbox[3] = {64, BN, 1};
        cr = encode(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(p.k_dense), kdims, kstrides, kbox, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    const bool win = p.window > 0;
    auto kern = p.bsel != nullptr ? attn_sm100_ot_kernel<D, false, false, false, false, true>
                : p.q_dense != nullptr ? attn_sm100_ot_kernel<D, false, false, true, false, false>
                : win ? (p.edges_only ? attn_sm100_ot_kernel<D, false, true, false, true, false>
                                      : attn_sm100_ot_kernel<D, false, false, false, true, false>)
                : p.edges_only ? (a.dbg != nullptr ? attn_sm100_ot_kernel<D, true, true, false, false, false>
                                                   : attn_sm100_ot_kernel<D, false, true, false, false, false>)
                               : (a.dbg != nullptr ? attn_sm100_ot_kernel<D, true, false, false, false, false>
                                                   : attn_sm100_ot_kernel<D, false, false, false, false, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    // persistent: one CTA per SM takes items from the work counter; the fused-Q prologue keeps one item
    // per CTA (grid = items: every CTA's second claim is past the end)
    if (p.sched == nullptr) return cudaErrorInvalidValue;
    cudaError_t me = cudaMemsetAsync(p.sched, 0, sizeof(uint32_t), stream);
    if (me != cudaSuccess) return me;
    int grid = items;
    if (p.q_dense == nullptr && !SFA_OT_ONE_ITEM_PER_CTA) {
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (grid > sms) grid = sms;
    }
    kern<<<grid, NTHREADS, C::SMEM, stream>>>(tm, tk, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100_ot(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg) {
    // d_v = 64 runs the same kernel over V's fp16 copy zero-padded to DV = 128 columns (vprep.cu): the
    // extra half of the P.V is free next to the fixed costs of the small heads that have d_v = 64
    if ((d != 64 && d != 128) || (d_v != DV && d_v != 64)) return cudaErrorNotSupported;
    if (p.edges_only && p.kfmask == nullptr) return cudaErrorInvalidValue;
    if (p.q_dense != nullptr && (p.edges_only || dbg != nullptr || p.window > 0)) return cudaErrorNotSupported;
    if (p.window > 0 && dbg != nullptr) return cudaErrorNotSupported;
    // block selection: R1, no window, no fused Q; both tiles of an item must share the query block
    if (p.bsel != nullptr && (p.edges_only || p.window > 0 || p.q_dense != nullptr || dbg != nullptr ||
                              (p.H / p.H_kv) % 2 != 0 || p.max_sel < 1))
        return cudaErrorNotSupported;
    OtArgs a;
    a.p = p;
    a.nqb = (int)((p.n_q + BM - 1) / BM);
    a.nkt = (int)((p.n_kv + BN - 1) / BN);
    a.c_scale = p.scale_log2;
#ifdef SFA_FAULT_SCALE  // negative control: logit scale off by 2^-9 relative
    a.c_scale *= 1.f + 1.f / 512.f;
#endif
    a.dbg = dbg;
    a.dv_out = d_v;
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
    a.items = (int)items;
    return d == 64 ? launch_t<64>(a, stream, (int)items) : launch_t<128>(a, stream, (int)items);
}

}  // namespace sfa
