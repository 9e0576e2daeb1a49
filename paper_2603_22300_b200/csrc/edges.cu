// edges.cu -- per-key-tile feature bitsets for the edge-only semantics (reading A1/R2, SURVEY 8(f)
// N4; "Traversing active coordinates yields only the nonzero attention edges").
//
// Under R2 a pair (i, j) enters the softmax only if the supports share a feature index.  This is
// the paper's feature-wise inverted index CSC_feat in bitset form: for each
// (batch, kv head, key tile of 128 keys) and each feature f,
//   kf[f] = 128-bit set of the tile's keys whose code selects f       (4 u32, bit j%32 of word j/32)
// (index equality only: a selected entry with value 0 is support, reading A8).  The tensor-core
// kernel (attn_sm100_ot.cu) then gets the edge set of query row i in the tile as
//   OR_{f in S_i} kf[f]   -- k 16-byte loads per row and tile instead of a test per pair.
// Layout: [B*H_kv][ceil(n_kv/128)][d][4] u32.  One CTA per tile, one thread per key: shared-memory
// atomicOr per selected feature, then a coalesced write.  Integer only; O(n k) work.
#include "launch.cuh"

namespace sfa {

namespace {

__global__ void __launch_bounds__(128) kfmask_kernel(const uint8_t *__restrict__ k_idx, int64_t n_kv, int k, int d,
                                                     int ntiles, uint32_t *__restrict__ out) {
    __shared__ uint32_t m[256 * 4];
    const int tile = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    for (int i = tid; i < d * 4; i += 128) m[i] = 0u;
    __syncthreads();
    const int64_t key = (int64_t)tile * 128 + tid;
    if (key < n_kv) {
        const uint8_t *src = k_idx + ((int64_t)bh * n_kv + key) * k;
        const uint32_t bit = 1u << (tid & 31);
        for (int t = 0; t < k; ++t) atomicOr(&m[(int)__ldg(src + t) * 4 + (tid >> 5)], bit);
    }
    __syncthreads();
    uint32_t *dst = out + ((int64_t)bh * ntiles + tile) * d * 4;
    for (int i = tid; i < d * 4; i += 128) dst[i] = m[i];
}

}  // namespace

size_t kfmask_bytes(int64_t bh_kv, int64_t n_kv, int d) { return (size_t)bh_kv * ((n_kv + 127) / 128) * d * 16; }

cudaError_t launch_kfmask(const uint8_t *k_idx, int64_t bh_kv, int64_t n_kv, int d, int k, uint32_t *out,
                          cudaStream_t stream) {
    if (d > 256) return cudaErrorNotSupported;
    const int64_t ntiles = (n_kv + 127) / 128;
    if (bh_kv == 0 || ntiles == 0) return cudaSuccess;
    if (ntiles > INT32_MAX || bh_kv > 65535) return cudaErrorNotSupported;
    kfmask_kernel<<<dim3((unsigned)ntiles, (unsigned)bh_kv), 128, 0, stream>>>(k_idx, n_kv, k, d, (int)ntiles, out);
    return cudaGetLastError();
}

}  // namespace sfa
