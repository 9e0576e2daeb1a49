// launch.cuh -- internal launcher declarations shared by the kernels and the C-ABI layer.
#pragma once
#include "common.cuh"

namespace sfa {

struct AttnParams {
    const uint8_t *q_idx;
    const void *q_val;
    const void *v;
    void *o;
    float *lse;
    const uint8_t *ws;
    int32_t B, H, H_kv, k;
    int64_t n_q, n_kv, q_pos0;
    int32_t causal;
    float scale_log2;  // scale * log2(e): logits live in the log2 domain inside the kernels
    BucketLayout L;
};

cudaError_t launch_topk(const void *x, bool bf16, int64_t rows, int d, int64_t ld, int k, uint8_t *idx, void *val,
                        uint32_t *status_word, cudaStream_t stream);
cudaError_t launch_bucket(const uint8_t *k_idx, const void *k_val, bool bf16, int d, int k, int64_t bh_kv,
                          int64_t n_kv, const BucketLayout &L, void *ws, cudaStream_t stream);
cudaError_t launch_attn_simt(const AttnParams &p, bool bf16, int d, int d_v, cudaStream_t stream);
// sm_100a tcgen05 kernel; returns cudaErrorNotSupported for shapes it does not cover
cudaError_t launch_attn_sm100(const AttnParams &p, int d, int d_v, cudaStream_t stream);

}  // namespace sfa
