// bucket.cu -- step 3: key-tile feature bucketing (our form of the paper's CSC_feat,
// P:L786-795 "Feature-wise CSC Format"; replaces Alg. 1's per-tile BinarySearchRange,
// L723 / P:L757-758, because every tile gets its own posting lists).
//
// One warp per (batch, kv head, key tile of BK keys): a counting sort of the tile's BK*k
// (key, value) pairs by feature, each bucket padded to a multiple of 4 entries with
// (trash row, +0) pads (layout in common.cuh).  Integer-only, O(nk), deterministic: the
// placement order inside a bucket is fixed (key chunk, code slot, lane) via match.any, so
// the workspace is bitwise reproducible.  The order inside a bucket never changes O: each
// key appears at most once per bucket.
#include "launch.cuh"

namespace sfa {

template <int D, bool BF16>
__global__ void __launch_bounds__(128) bucket_keys_kernel(const uint8_t *__restrict__ k_idx,
                                                          const void *__restrict__ k_val, int64_t n_kv, int k,
                                                          BucketLayout L, int64_t total_tiles,
                                                          uint8_t *__restrict__ ws) {
    __shared__ int s_cnt[4][D];
    __shared__ int s_cur[4][D];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = (int64_t)blockIdx.x * 4 + w;
    if (tile >= total_tiles) return;  // warp-uniform
    const int64_t bh = tile / L.ntiles;
    const int t = (int)(tile % L.ntiles);
    const int64_t key0 = (int64_t)t * L.bk;
    const int nkeys = (int)((n_kv - key0) < L.bk ? (n_kv - key0) : L.bk);
    int *cnt = s_cnt[w], *cur = s_cur[w];
    uint8_t *tb = ws + tile * L.tile_bytes;
    uint16_t *off = reinterpret_cast<uint16_t *>(tb);

    for (int f = lane; f < D; f += 32) cnt[f] = 0;
    __syncwarp();
    const uint8_t *ki = k_idx + (bh * n_kv + key0) * k;
    for (int jl = lane; jl < nkeys; jl += 32)
        for (int tt = 0; tt < k; ++tt) atomicAdd(&cnt[ki[(int64_t)jl * k + tt]], 1);
    __syncwarp();
    // exclusive scan of the 4-padded counts; lane owns features [lane*FPL, lane*FPL+FPL)
    constexpr int FPL = D / 32;
    int loc[FPL], sum = 0;
#pragma unroll
    for (int i = 0; i < FPL; ++i) {
        loc[i] = sum;
        sum += (cnt[lane * FPL + i] + 3) & ~3;
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int base = incl - sum;
#pragma unroll
    for (int i = 0; i < FPL; ++i) {
        cur[lane * FPL + i] = base + loc[i];
        off[lane * FPL + i] = (uint16_t)(base + loc[i]);
    }
    if (lane == 31) {
        off[D] = (uint16_t)incl;
        for (int x = D + 1; x < L.off_bytes / 2; ++x) off[x] = 0;  // alignment padding (copied as 16-byte vectors)
    }
    __syncwarp();

    // deterministic stable placement
    for (int c = 0; c < L.bk; c += 32) {
        const int jl = c + lane;
        const bool valid = jl < nkeys;
        for (int tt = 0; tt < k; ++tt) {
            const int f = valid ? (int)ki[(int64_t)jl * k + tt] : 0xFFFF;
            const uint32_t peers = __match_any_sync(0xffffffffu, f);
            const int rank = __popc(peers & lanemask_lt());
            int pos = 0;
            if (valid) pos = cur[f] + rank;
            __syncwarp();
            if (valid) {
                const int64_t vi = (bh * n_kv + key0 + jl) * k + tt;
                if (BF16) {
                    const uint32_t vb = reinterpret_cast<const uint16_t *>(k_val)[vi];
                    reinterpret_cast<uint32_t *>(tb + L.off_bytes)[pos] = (vb << 16) | (uint32_t)(jl * SLAB_ROW_BYTES);
                } else {
                    const uint32_t vb = reinterpret_cast<const uint32_t *>(k_val)[vi];
                    reinterpret_cast<uint2 *>(tb + L.off_bytes)[pos] = make_uint2((uint32_t)(jl * SLAB_ROW_BYTES), vb);
                }
                if (rank == 0) cur[f] += __popc(peers);
            }
            __syncwarp();
        }
    }
    // pads: (trash row BK, +0) fill [off[f] + cnt[f], off[f] + pad4(cnt[f]))
    const uint32_t trash = (uint32_t)(L.bk * SLAB_ROW_BYTES);
#pragma unroll
    for (int i = 0; i < FPL; ++i) {
        const int f = lane * FPL + i;
        const int end = base + loc[i] + ((cnt[f] + 3) & ~3);
        for (int p = cur[f]; p < end; ++p) {
            if (BF16)
                reinterpret_cast<uint32_t *>(tb + L.off_bytes)[p] = trash;
            else
                reinterpret_cast<uint2 *>(tb + L.off_bytes)[p] = make_uint2(trash, 0u);
        }
    }
}

cudaError_t launch_bucket(const uint8_t *k_idx, const void *k_val, bool bf16, int d, int k, int64_t bh_kv,
                          int64_t n_kv, const BucketLayout &L, void *ws, cudaStream_t stream) {
    const int64_t total = bh_kv * L.ntiles;
    if (total == 0) return cudaSuccess;
    const int64_t grid = (total + 3) / 4;
    uint8_t *w = (uint8_t *)ws;
    if (bf16) {
        if (d == 64) bucket_keys_kernel<64, true><<<(unsigned)grid, 128, 0, stream>>>(k_idx, k_val, n_kv, k, L, total, w);
        else bucket_keys_kernel<128, true><<<(unsigned)grid, 128, 0, stream>>>(k_idx, k_val, n_kv, k, L, total, w);
    } else {
        if (d == 64) bucket_keys_kernel<64, false><<<(unsigned)grid, 128, 0, stream>>>(k_idx, k_val, n_kv, k, L, total, w);
        else bucket_keys_kernel<128, false><<<(unsigned)grid, 128, 0, stream>>>(k_idx, k_val, n_kv, k, L, total, w);
    }
    return cudaGetLastError();
}

}  // namespace sfa
