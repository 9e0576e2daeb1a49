// launch.cuh -- internal launcher declarations shared by the kernels and the C-ABI layer.
#pragma once
#include "common.cuh"

namespace sfa {

struct AttnParams {
    const uint8_t *q_idx;
    const void *q_val;
    const uint8_t *k_idx;  // key codes (sm100 kernel decompresses them on chip; SIMT reads buckets)
    const void *k_val;
    const void *v;
    const void *v16;         // sm100: fp16 copy of V scaled by 2^-e per (b, kv head) (vprep.cu)
    const uint32_t *v_amax;  // sm100: per (b, kv head) max|V| bits, e = vprep_head_exp(bits)
    const void *k_dense = nullptr;  // SM100_OT: decompressed K~ rows, bf16 [B][H_kv][n_kv][d] (vprep.cu)
    uint32_t *sched = nullptr;      // SM100_OT: the persistent tile scheduler's work counter (workspace)
    // N4 block selection (SM100_OT): [B][H_kv][ceil(n_q/128)][max_sel] ascending key-tile indices, -1 padded
    const int32_t *bsel = nullptr;
    int32_t max_sel = 0;
    void *o;
    float *lse;
    const uint8_t *ws;
    int32_t B, H, H_kv, k;
    int64_t n_q, n_kv, q_pos0;
    int32_t causal;
    float scale_log2;  // scale * log2(e): logits live in the log2 domain inside the kernels
    BucketLayout L;
    int32_t edges_only;      // reading A1/R2: only pairs whose supports intersect enter the softmax
    int64_t window = 0;      // N4: causal sliding window, key j also needs j > q_pos0 + i - window (0 = off)
    const uint32_t *kfmask;  // R2, SM100_OT: per key tile, per feature, the 128-bit set of keys selecting it
    // fused step 1 on Q (SM100_OT, N3(ii)): dense bf16 Q [B][H][n_q][d] instead of q codes; the kernel
    // optionally writes the codes it selected (q_idx_out / q_val_out) and flags non-finite Q
    const void *q_dense = nullptr;
    uint8_t *q_idx_out = nullptr;
    void *q_val_out = nullptr;
    uint32_t *status_word = nullptr;
};

// R2 feature bitsets of the key tiles (edges.cu): [B*H_kv][ceil(n_kv/128)][d][4] u32
size_t kfmask_bytes(int64_t bh_kv, int64_t n_kv, int d);
cudaError_t launch_kfmask(const uint8_t *k_idx, int64_t bh_kv, int64_t n_kv, int d, int k, uint32_t *out,
                          cudaStream_t stream);

cudaError_t launch_topk(const void *x, bool bf16, int64_t rows, int d, int64_t ld, int k, uint8_t *idx, void *val,
                        uint32_t *status_word, cudaStream_t stream);
cudaError_t launch_topk_pair(const void *x0, int64_t rows0, int64_t ld0, uint8_t *idx0, void *val0, const void *x1,
                             int64_t rows1, int64_t ld1, uint8_t *idx1, void *val1, int d, int k,
                             uint32_t *status_word, cudaStream_t stream);
cudaError_t launch_bucket(const uint8_t *k_idx, const void *k_val, bool bf16, int d, int k, int64_t bh_kv,
                          int64_t n_kv, const BucketLayout &L, void *ws, cudaStream_t stream);
// P.V operand prep for the sm100 kernel: amax[bh] = max|V| bits, v16 = fp16(V * 2^-e) (vprep.cu), rows of
// dvp >= d_v features (zeros past d_v)
cudaError_t launch_vprep(const void *v, int64_t bh_kv, int64_t n_kv, int d_v, int dvp, uint32_t *amax, void *v16,
                         cudaStream_t stream);
// the same plus the K~ rows (k_dense != null) in ONE launch without a memset, one block per (batch, kv
// head) (vprep.cu prep_small_kernel): for heads of at most 128 KB of V (prep_small_ok)
bool prep_small_ok(int64_t bh_kv, int64_t n_kv, int d_v, int64_t krows);
cudaError_t launch_prep_small(const void *v, int64_t bh_kv, int64_t n_kv, int d_v, int dvp, uint32_t *amax, void *v16,
                              const uint8_t *k_idx, const void *k_val, int d, int k, void *k_dense, cudaStream_t stream);
// e with max|V| * 2^-e in [2^14, 2^15) (fp16-safe and clear of fp16's subnormal range, in either
// direction: small heads are scaled UP), clamped to e >= -126 so that 2^-e and 2^e are both normal
// floats; e = 0 for an all-zero head.  Shared by vprep.cu and the attention epilogues.
__device__ __forceinline__ int vprep_head_exp(uint32_t amax_bits) {
    if (amax_bits == 0u) return 0;
    const int e = (int)((amax_bits >> 23) & 0xFF) - 127 - 14;
    return e < -126 ? -126 : e;
}
// K~ rows from the key codes, bf16 [rows][d] (vprep.cu k_dense_kernel), for the SM100_OT K~ TMA
cudaError_t launch_kdense(const uint8_t *k_idx, const void *k_val, int64_t rows, int d, int k, void *out,
                          cudaStream_t stream);
// decode shape (rows = n_q * H / H_kv <= 16 per kv head): split-KV CUDA-core kernel + LSE merge
// (decode.cu); ws >= decode_workspace_bytes
cudaError_t launch_decode(const AttnParams &p, int d, int d_v, cudaStream_t st, void *ws);
size_t decode_workspace_bytes(int64_t bh_kv, int64_t n_kv, int d_v);
cudaError_t launch_attn_simt(const AttnParams &p, bool bf16, int d, int d_v, cudaStream_t stream);
// sm_100a tcgen05 kernel (bf16); returns cudaErrorNotSupported for shapes it does not cover.
// dbg (tests only, may be null): receives the raw 128x128 fp32 score tile S = Q~ K~^T of the
// first key tile of work item 0, query tile 0.
cudaError_t launch_attn_sm100(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg);
cudaError_t launch_attn_sm100_ot(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg);
// two query tiles in ping-pong, K~ by TMA from p.k_dense, P in TMEM (attn_sm100_pp.cu); R1, no window
cudaError_t launch_attn_sm100_pp(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg);
// SM100_OT with Q~ in TMEM and 64-key score halves (attn_sm100_oth.cu); R1, no window, d_v = 128
cudaError_t launch_attn_sm100_oth(const AttnParams &p, int d, int d_v, cudaStream_t stream, float *dbg);
// backward with the straight-through rule (bwd.cu): D = rowsum(dO . O) into Dws [B*H*n_q], then the
// dK~/dV and dQ~ tensor-core kernels; gradients w.r.t. the code values and V, fp32
// qd / kd: workspace for the decompressed Q~ / K~ rows (bf16 [rows][d]) the kernels' TMA reads
cudaError_t launch_attn_bwd(const AttnParams &p, int d, int d_v, const void *dO, float *Dws, void *qd, void *kd,
                            float *dq, float *dk, float *dv, cudaStream_t st);

}  // namespace sfa
