// dist.cu -- step 9 (sharded path only): query-block sharding of one long sequence over P GPUs
// (the paper runs long contexts on one GPU and has no sequence parallelism).
//
// Zig-zag partition: the sequence is cut into 2P chunks of c tokens; rank p owns chunks p and
// 2P-1-p, so the causal work of every rank is exactly equal.  A rank computes the codes (stage 1)
// of its own tokens, and one all-gather of the key codes and V gives every rank the whole
// sequence.  Local tensors are
// chunk-major, [2][B][H(_kv)][c][.] (chunk p, then chunk 2P-1-p), so each query chunk's codes and
// outputs are contiguous for the attention call.  NCCL's all-gather is rank-major, so the received
// blocks [P][2][B][H_kv][c][.] are unpacked into sequence order [B][H_kv][2Pc][.] by
// `zigzag_unpack_kernel` (a pure copy).  Each rank then runs the attention
// for its two query chunks with q_pos0 = chunk start (reading A9): outputs stay sharded.
//
// NCCL is loaded with dlopen("libnccl.so.2") when a communicator is created, so the library loads
// (and every single-GPU entry point works) on a machine without NCCL, and a process that already
// loaded PyTorch's NCCL shares that copy.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "../../include/sfa.h"
#include "launch.cuh"

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    bool ok = false;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GroupStart &&
                 api.GroupEnd;
    });
    return api;
}

// out[b][h][chunk q][i] <- in[rank r][half][b][h][i], q = half ? 2P-1-r : r  (one row = row_bytes,
// moved as 16-byte words when row_bytes % 16 == 0, else as bytes)
template <typename W>
__global__ void zigzag_unpack_kernel(const W *__restrict__ in, W *__restrict__ out, int P, int64_t bh, int64_t c,
                                     int64_t words_per_row) {
    const int64_t per_chunk = c * words_per_row;  // one (b, h) chunk
    const int64_t per_half = bh * per_chunk;
    const int64_t total = (int64_t)P * 2 * per_half;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rh = x / per_half;  // rank * 2 + half
        const int64_t y = x - rh * per_half;
        const int64_t hb = y / per_chunk;
        const int64_t w = y - hb * per_chunk;
        const int64_t r = rh >> 1;
        const int64_t q = (rh & 1) ? 2 * P - 1 - r : r;
        out[(hb * 2 * P + q) * per_chunk + w] = in[x];
    }
}

cudaError_t launch_unpack(const void *in, void *out, int P, int64_t bh, int64_t c, int64_t row_bytes,
                          cudaStream_t st) {
    const int64_t bytes = (int64_t)P * bh * 2 * c * row_bytes;
    if (bytes == 0) return cudaSuccess;
    int64_t grid = 148 * 8;
    if (row_bytes % 16 == 0) {
        const int64_t wpr = row_bytes / 16, words = bytes / 16;
        if ((words + 255) / 256 < grid) grid = (words + 255) / 256;
        zigzag_unpack_kernel<uint4><<<(unsigned)grid, 256, 0, st>>>((const uint4 *)in, (uint4 *)out, P, bh, c, wpr);
    } else {
        if ((bytes + 255) / 256 < grid) grid = (bytes + 255) / 256;
        zigzag_unpack_kernel<uint8_t><<<(unsigned)grid, 256, 0, st>>>((const uint8_t *)in, (uint8_t *)out, P, bh, c,
                                                                      row_bytes);
    }
    return cudaGetLastError();
}

size_t esize(sfa_dtype t) { return t == SFA_BF16 ? 2 : 4; }

}  // namespace

struct sfa_dist {
    ncclComm_t comm;
    int rank, world;
};

extern "C" {

sfa_status sfa_dist_unique_id(void *out) {
    if (!out) return SFA_ERR_INVALID_ARGUMENT;
    const NcclApi &api = nccl();
    if (!api.ok) return SFA_ERR_UNSUPPORTED;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return SFA_ERR_CUDA;
    memcpy(out, &id, sizeof(id));
    return SFA_OK;
}

sfa_status sfa_dist_init(int rank, int world, const void *nccl_unique_id, sfa_dist_t *out) {
    if (!out || !nccl_unique_id || world < 1 || rank < 0 || rank >= world) return SFA_ERR_INVALID_ARGUMENT;
    const NcclApi &api = nccl();
    if (!api.ok) return SFA_ERR_UNSUPPORTED;
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    sfa_dist *h = new sfa_dist;
    h->rank = rank;
    h->world = world;
    if (api.CommInitRank(&h->comm, world, id, rank) != ncclSuccess) {
        delete h;
        return SFA_ERR_CUDA;
    }
    *out = h;
    return SFA_OK;
}

sfa_status sfa_dist_destroy(sfa_dist_t h) {
    if (!h) return SFA_ERR_INVALID_ARGUMENT;
    const ncclResult_t r = nccl().CommDestroy(h->comm);
    delete h;
    return r == ncclSuccess ? SFA_OK : SFA_ERR_CUDA;
}

sfa_status sfa_dist_kv_plan(const sfa_attn_desc *local_desc, int32_t world, sfa_dist_kv_plan_t *plan) {
    const sfa_attn_desc *d = local_desc;
    if (!d || !plan || world < 1 || d->B < 1 || d->H_kv < 1 || d->n_kv < 2 || (d->n_kv & 1) || d->k < 1 ||
        d->d_v < 1)
        return SFA_ERR_INVALID_ARGUMENT;
    if (d->dtype != SFA_F32 && d->dtype != SFA_BF16) return SFA_ERR_INVALID_ARGUMENT;
    const size_t es = esize(d->dtype);
    const size_t rows_local = (size_t)d->B * d->H_kv * d->n_kv;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    plan->bh = (int64_t)d->B * d->H_kv;
    plan->chunk = d->n_kv / 2;
    plan->row_bytes[0] = d->k;                   // k_idx rows (u8)
    plan->row_bytes[1] = (int64_t)d->k * es;     // k_val rows
    plan->row_bytes[2] = (int64_t)d->d_v * es;   // V rows
    size_t off = 0;
    for (int t = 0; t < 3; ++t) {
        plan->bytes_per_rank[t] = (int64_t)(rows_local * plan->row_bytes[t]);
        plan->staging_offset[t] = (int64_t)off;
        off += al((size_t)plan->bytes_per_rank[t] * world);
    }
    plan->staging_bytes = (int64_t)off;
    return SFA_OK;
}

size_t sfa_dist_staging_bytes(const sfa_attn_desc *local_desc, int32_t world) {
    sfa_dist_kv_plan_t pl;
    return sfa_dist_kv_plan(local_desc, world, &pl) == SFA_OK ? (size_t)pl.staging_bytes : 0;
}

sfa_status sfa_dist_zigzag_chunk(int64_t n, int32_t world, int32_t rank, int32_t half, int64_t *chunk_len,
                                 int64_t *q_pos0) {
    if (world < 1 || rank < 0 || rank >= world || (half != 0 && half != 1) || n < 2 * (int64_t)world ||
        n % (2 * (int64_t)world))
        return SFA_ERR_INVALID_ARGUMENT;
    const int64_t c = n / (2 * (int64_t)world);
    const int64_t q = half ? 2 * (int64_t)world - 1 - rank : rank;
    if (chunk_len) *chunk_len = c;
    if (q_pos0) *q_pos0 = q * c;
    return SFA_OK;
}

sfa_status sfa_dist_head_shard(const sfa_attn_desc *full, int32_t world, int32_t rank, sfa_attn_desc *sub,
                               int64_t *unit0) {
    if (!full || !sub || !unit0 || world < 1 || rank < 0 || rank >= world) return SFA_ERR_INVALID_ARGUMENT;
    if (full->B < 1 || full->H < 1 || full->H_kv < 1 || full->H % full->H_kv) return SFA_ERR_INVALID_ARGUMENT;
    const int64_t units = (int64_t)full->B * full->H_kv;
    if (units < world) return SFA_ERR_UNSUPPORTED;  // a rank would get no (batch, kv head) unit
    const int64_t u0 = units * rank / world, u1 = units * (rank + 1) / world;
    if (u1 - u0 > INT32_MAX) return SFA_ERR_UNSUPPORTED;
    *sub = *full;
    sub->B = (int32_t)(u1 - u0);  // each unit is its own batch element of H/H_kv query heads, 1 kv head
    sub->H = full->H / full->H_kv;
    sub->H_kv = 1;
    *unit0 = u0;
    return SFA_OK;
}

sfa_status sfa_dist_unpack_zigzag(const void *in, void *out, int32_t world, int64_t bh, int64_t chunk,
                                  int64_t row_bytes, sfa_stream_t stream) {
    if (world < 1 || bh < 0 || chunk < 0 || row_bytes < 1) return SFA_ERR_INVALID_ARGUMENT;
    if ((int64_t)world * bh * chunk == 0) return SFA_OK;
    if (!in || !out) return SFA_ERR_INVALID_ARGUMENT;
    if (row_bytes % 16 == 0 && ((((uintptr_t)in) | ((uintptr_t)out)) & 15u)) return SFA_ERR_INVALID_ARGUMENT;
    return launch_unpack(in, out, world, bh, chunk, row_bytes, (cudaStream_t)stream) == cudaSuccess ? SFA_OK
                                                                                                   : SFA_ERR_CUDA;
}

sfa_status sfa_dist_allgather_kv(sfa_dist_t h, const sfa_attn_desc *local_desc, const uint8_t *k_idx_local,
                                 const void *k_val_local, const void *v_local, uint8_t *k_idx_full, void *k_val_full,
                                 void *v_full, void *staging, size_t staging_bytes, sfa_stream_t stream) {
    if (!h || !local_desc) return SFA_ERR_INVALID_ARGUMENT;
    sfa_dist_kv_plan_t pl;
    if (sfa_dist_kv_plan(local_desc, h->world, &pl) != SFA_OK) return SFA_ERR_INVALID_ARGUMENT;
    const size_t need = (size_t)pl.staging_bytes;
    if (!k_idx_local || !k_val_local || !v_local || !k_idx_full || !k_val_full || !v_full || !staging)
        return SFA_ERR_INVALID_ARGUMENT;
    // every tensor 16-byte aligned (include/sfa.h conventions): the unpack moves 16-byte words when a
    // row is a multiple of 16 bytes, so a misaligned buffer must be rejected here, before any launch
    if ((((uintptr_t)k_idx_local) | ((uintptr_t)k_val_local) | ((uintptr_t)v_local) | ((uintptr_t)k_idx_full) |
         ((uintptr_t)k_val_full) | ((uintptr_t)v_full) | ((uintptr_t)staging)) & 15u)
        return SFA_ERR_INVALID_ARGUMENT;
    if (staging_bytes < need) return SFA_ERR_RESOURCE;
    const NcclApi &api = nccl();
    cudaStream_t st = (cudaStream_t)stream;
    const int P = h->world;
    // one grouped all-gather of the three rank-major blocks, then the unpack into sequence order; the
    // offsets and sizes come from sfa_dist_kv_plan (also what the CPU multi-process tests execute)
    const void *src[3] = {k_idx_local, k_val_local, v_local};
    void *dst[3] = {k_idx_full, k_val_full, v_full};
    if (api.GroupStart() != ncclSuccess) return SFA_ERR_CUDA;
    bool ok = true;
    for (int t = 0; t < 3; ++t)
        ok = ok && api.AllGather(src[t], (uint8_t *)staging + pl.staging_offset[t], (size_t)pl.bytes_per_rank[t],
                                 ncclUint8, h->comm, st) == ncclSuccess;
    if (api.GroupEnd() != ncclSuccess || !ok) return SFA_ERR_CUDA;
    for (int t = 0; t < 3; ++t)
        if (launch_unpack((uint8_t *)staging + pl.staging_offset[t], dst[t], P, pl.bh, pl.chunk, pl.row_bytes[t],
                          st) != cudaSuccess)
            return SFA_ERR_CUDA;
    return SFA_OK;
}

}  // extern "C"
