/*
 * include/sfa.h -- C ABI of the B200 (sm_100a) FlashSFA hot path.
 *
 * Sparse Feature Attention (arXiv 2603.22300).  Citations: "P:Lnnn" = PAPER.md line nnn,
 * "S:Lnnn" = SPEC.md line nnn; readings A1..A21 are listed in DESIGN.md.
 *
 * The path has two stages:
 *   stage 1  sfa_topk_codes  -- row-wise Top-k coding of Q and of K (Eq. topk_QK):
 *            keep the k entries of largest |x|, sign kept; ties -> lower index (A2);
 *            indices ascending (A4); always exactly k entries (A8).
 *   stage 2  sfa_attn_fwd    -- the exact attention forward over those codes (P:L97-101 Eq. s_ij,
 *            P:L126-135 Sec. 3.2, Alg. 1):
 *              s_ij = scale * sum_{u in S_i and S_j} q~_iu k~_ju   (0 when disjoint: A1/R1)
 *              O_i  = sum_j softmax_j(s_ij, j allowed) V_j ;  LSE_i = ln sum_j exp(s_ij)  (A11)
 *            computed tile by tile with an online softmax; no n x n matrix is ever stored.
 *
 * Conventions for every call:
 *   - Tensor pointers are DEVICE pointers owned by the caller (the Python layer allocates them
 *     with PyTorch), except in sfa_forward_host, whose inputs/outputs are HOST pointers.
 *   - The library never allocates device memory, never frees, never synchronises the device
 *     (sfa_forward_host synchronises its stream), and keeps no mutable global state: calls are
 *     thread-safe and ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Argument errors are detected on the host BEFORE any launch and leave outputs untouched.
 *   - Data errors (non-finite inputs) are reported asynchronously through `status_word`.
 *   - All tensors are dense, row-major, last index fastest, 16-byte aligned.
 */
#ifndef SFA_H
#define SFA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SFA_API __attribute__((visibility("default")))
#else
#define SFA_API
#endif

typedef struct CUstream_st *sfa_stream_t; /* == cudaStream_t */

typedef enum {
    SFA_OK = 0,
    SFA_ERR_INVALID_ARGUMENT = 1, /* bad shape / k / scale / null or misaligned pointer */
    SFA_ERR_INVALID_INPUT = 2,    /* non-finite input values (reading A14)                      */
    SFA_ERR_UNSUPPORTED = 3,      /* valid but not compiled (d, d_v not in {64,128}), or no sm_100 GPU */
    SFA_ERR_RESOURCE = 4,         /* workspace / scratch too small (S:L180 resource-limit)             */
    SFA_ERR_CUDA = 5              /* a CUDA launch or copy failed                                      */
} sfa_status;

typedef enum { SFA_F32 = 0, SFA_BF16 = 1 } sfa_dtype;

/* Kernel selection for sfa_attn_fwd (desc.kernel). */
typedef enum {
    SFA_KERNEL_AUTO = 0, /* SIMT for fp32; for bf16 DECODE when n_q * H / H_kv <= 16, else SM100_OT for
                            d_v = 128 and SM100 for d_v = 64; bf16 with edges_only or a window: SM100_OT */
    SFA_KERNEL_SIMT = 1, /* CUDA-core kernel: key-tile feature buckets, shared-memory scatter of the
                            support overlaps, FFMA P.V (the only fp32 path: reading A12)             */
    SFA_KERNEL_SM100 = 2, /* sm_100a kernel (bf16 only): key codes decompressed on chip, S = Q~ K~^T and
                            O += P V on tcgen05 tensor cores, S/P/O in TMEM, V by TMA    */
    SFA_KERNEL_SM100_PAIR = 3, /* round-1 ablations (M = 256 CTA-pair MMAs; 256-key score tiles), measured   */
    SFA_KERNEL_SM100_WIDE = 4, /* slower and removed in round 2: SFA_ERR_UNSUPPORTED (numbers kept reserved)  */
    SFA_KERNEL_DECODE = 5,     /* few query rows over a long cache (n_q * H / H_kv <= 16, bf16): split-KV
                                  CUDA-core kernel reading codes + V, LSE merge.  AUTO picks
                                  it for such shapes.                                                      */
    SFA_KERNEL_SM100_OT = 6,   /* SM100 with a transposed output accumulator: O^T += V^T P^T as N = 256 MMAs
                                  over both query tiles, P in shared memory (bf16; d_v = 64 runs the same
                                  d_v = 128 product over V's zero-padded fp16 copy)                        */
    SFA_KERNEL_SM100_PP = 7,   /* two query tiles in ping-pong: K~ tiles by TMA from key rows decompressed
                                  once per key (prepare step), P in TMEM (TS-MMA P.V), exponential phases
                                  of the two softmax warpgroups alternating (bf16, R1, no window)          */
    SFA_KERNEL_SM100_OTH = 8   /* SM100_OT with Q~ in TMEM (TS-MMA scores over 64-key halves, P handed over
                                  per half): fewer shared-memory bytes per key (bf16, d_v = 128, R1, no
                                  window)                                                                */
} sfa_kernel;

SFA_API const char *sfa_status_string(sfa_status s);

/* ------------------------------------------------------------------------------------------
 * Stage 1: Top-k codes.
 *   x    [rows][d] with row stride `ld` elements (ld >= d); dtype SFA_F32 or SFA_BF16.
 *        rows = B*H*n for Q, B*H_kv*n for K (the same operator on Q and on K).
 *   idx  [rows][k] uint8, ascending feature indices (A4, A6: u8 covers d <= 256).
 *   val  [rows][k] same dtype as x, bit copies of the selected entries (A7; -0 kept).
 *   Ranking key |x| compared exactly (IEEE magnitude bits; no flush-to-zero, A21); ties -> lower index.
 *   status_word (nullable, device): bit 0 is OR-ed in when any non-finite x is seen; the outputs
 *        are then unspecified and the caller reports SFA_ERR_INVALID_INPUT (A14).
 *   Requires 1 <= k <= d, d in {64, 128}, rows >= 0.  Stream-ordered, no allocation.
 * ------------------------------------------------------------------------------------------ */
SFA_API sfa_status sfa_topk_codes(const void *x, sfa_dtype dtype, int64_t rows, int32_t d, int64_t ld, int32_t k,
                          uint8_t *idx, void *val, uint32_t *status_word, sfa_stream_t stream);

/* Stage 1 on Q and on K of one step in ONE launch (the same operator and arguments as two
 * sfa_topk_codes calls; results bit-identical to them).  bf16 only takes the fused launch;
 * fp32, k = d or unaligned rows fall back to two launches.  Argument errors of either tensor are
 * reported before any launch. */
SFA_API sfa_status sfa_topk_codes_qk(const void *q, int64_t q_rows, int64_t q_ld, uint8_t *q_idx, void *q_val,
                                     const void *k, int64_t k_rows, int64_t k_ld, uint8_t *k_idx, void *k_val,
                                     sfa_dtype dtype, int32_t d, int32_t kk, uint32_t *status_word,
                                     sfa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Stage 2: attention forward over the codes.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
    int32_t B, H, H_kv;  /* batch, query heads, kv heads; H % H_kv == 0; head h reads kv head h/(H/H_kv) (A15) */
    int32_t d, k, d_v;   /* head dim (64|128), code size (1..d), value dim (64|128)                       */
    int64_t n_q, n_kv;   /* query rows and keys per head (n_q >= 1, n_kv >= 1)                             */
    int64_t q_pos0;      /* query i sits at global position q_pos0 + i (A9); >= 0                          */
    int32_t causal;      /* 1: key j allowed iff j <= q_pos0 + i ("masking for causality"); 0: all */
    float scale;         /* logit multiplier; > 0 and finite; the paper's is 1/sqrt(d) (A5)         */
    sfa_dtype dtype;     /* dtype of q_val, k_val, v and o (LSE is always fp32)                            */
    int32_t kernel;      /* sfa_kernel; SFA_KERNEL_AUTO unless benchmarking an ablation                   */
    int32_t edges_only;  /* 0: reading A1/R1 (default) -- every allowed pair enters the softmax, a pair with
                            disjoint supports with logit 0 ("mathematically identical
                            to softmax(Q~K~^T/sqrt d)V").  1: R2 -- only the "nonzero
                            attention edges": pair (i, j) enters iff the supports share
                            a feature index (zero-valued selected entries count, A8); a row with no edge
                            gets O = 0, LSE = -inf.  R2 runs on SM100_OT (bf16) and SIMT (AUTO picks
                            them); other explicit kernels -> SFA_ERR_UNSUPPORTED.                      */
    int64_t window;      /* 0: off.  > 0 (requires causal = 1): causal sliding window -- SFA composed with
                            token-level sparsity: key j is allowed only if
                            also j > q_pos0 + i - window.  Key tiles before a query block's window are
                            skipped, so the work is ~ n * window.  Runs on SM100_OT and SIMT (AUTO picks
                            them); DECODE / SM100 / PAIR / WIDE and the backward -> SFA_ERR_UNSUPPORTED. */
} sfa_attn_desc;

/* Bytes of device workspace sfa_attn_fwd needs (0 on an invalid desc):
 *   SIMT kernel : the key-tile feature buckets (our form of the
 *                 paper's CSC_feat);
 *   SM100 kernel: max|V| per (b, kv head) + an fp16 copy of V scaled by a power of two per
 *                 (b, kv head) -- the exact fp16 P.V operand (reading A12); with
 *                 edges_only also, per 128-key tile, a 128-bit key set per feature (edges.cu);
 *   DECODE kernel: one fp32 partial (max, sum, O) per (b, kv head, key split) for the merge. */
SFA_API size_t sfa_attn_workspace_bytes(const sfa_attn_desc *desc);

/* O, LSE = FlashSFA forward.
 *   q_idx [B][H][n_q][k] u8,  q_val [B][H][n_q][k]   (stage-1 codes of Q: every row's indices distinct and
 *                                                      ascending, as sfa_topk_codes writes them (A4); with
 *                                                      k = d the kernels rely on idx[t] = t)
 *   k_idx [B][H_kv][n_kv][k] u8, k_val [B][H_kv][n_kv][k]
 *   v     [B][H_kv][n_kv][d_v]       o [B][H][n_q][d_v] (dtype)       lse [B][H][n_q] fp32, natural log
 *   workspace: >= sfa_attn_workspace_bytes(desc) device bytes (else SFA_ERR_RESOURCE), 16-aligned.
 *   Code and value pointers must be 16-byte aligned.
 *   Launches (SIMT) the bucketing kernel + the attention kernel, or (SM100) the two V-prep kernels
 *   + the attention kernel, on `stream`.
 *   O is rounded to the output dtype with round-to-nearest-even (A21). Rows with no allowed key
 *   (impossible when q_pos0 >= 0) get O = 0, LSE = -inf (A10). */
SFA_API sfa_status sfa_attn_fwd(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                        const void *k_val, const void *v, void *o, float *lse, void *workspace,
                        size_t workspace_bytes, sfa_stream_t stream);

/* sfa_attn_fwd in two calls (the sharded path prepares the gathered keys once; the bench times
 * the attention kernel alone):
 *   sfa_attn_prepare      -- step 3 for the kernel desc selects: key-tile buckets (SIMT) or max|V|
 *                            and the scaled fp16 V (SM100), written into `workspace`;
 *   sfa_attn_fwd_prepared -- steps 4-8 over that workspace (same desc, codes and V). */
SFA_API sfa_status sfa_attn_prepare(const sfa_attn_desc *desc, const uint8_t *k_idx, const void *k_val, const void *v,
                                    void *workspace, size_t workspace_bytes, sfa_stream_t stream);
SFA_API sfa_status sfa_attn_fwd_prepared(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                         const uint8_t *k_idx, const void *k_val, const void *v, void *o, float *lse,
                                         const void *workspace, size_t workspace_bytes, sfa_stream_t stream);

/* FlashSFA forward composed with block-level token selection (NSA-style "each query
 * block attends the key blocks it selected", "SFA is orthogonal to token-level sparsity").
 *   block_sel [B][H_kv][ceil(n_q/128)][max_sel] int32, device: for each (batch, kv head, block of 128
 *             query rows) the indices of the 128-key blocks it may attend, ASCENDING, padded with -1
 *             (entries past the first negative one are ignored); intersected with the causal mask.
 *   Key j is allowed for query row i iff j <= q_pos0 + i (if causal) and j / 128 is listed for the
 *   row's query block i / 128; rows without an allowed key get O = 0, LSE = -inf.  Runs steps 3-8 on
 *   the default tensor-core kernel (persistent tile scheduler over the listed tiles only).
 *   Supported: bf16, H / H_kv even, edges_only = 0, window = 0, and the desc resolving to SM100_OT
 *   (kernel AUTO with d_v = 128, or SFA_KERNEL_SM100_OT with d_v = 64 or 128); else SFA_ERR_UNSUPPORTED.  max_sel >= 1; block_sel 4-byte aligned.  Workspace as sfa_attn_fwd. */
SFA_API sfa_status sfa_attn_fwd_blocksel(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                         const uint8_t *k_idx, const void *k_val, const void *v,
                                         const int32_t *block_sel, int32_t max_sel, void *o, float *lse,
                                         void *workspace, size_t workspace_bytes, sfa_stream_t stream);

/* Steps 1 (on Q) to 8 in one kernel: the attention prologue selects the top-k of
 * every DENSE query row itself (the same selection code as sfa_topk_codes, so the support and the result
 * are bit-identical to sfa_topk_codes + sfa_attn_fwd_prepared), builds Q~ on chip and, if q_idx_out /
 * q_val_out are non-null (both or neither), also writes the codes [B][H][n_q][k] it selected.
 *   q: dense bf16 [B][H][n_q][d], 16-byte aligned.  k codes, v, workspace as sfa_attn_fwd_prepared
 *   (workspace prepared by sfa_attn_prepare).  status_word (nullable): bit 0 OR-ed on non-finite q (A14).
 *   Supported when the desc resolves to SFA_KERNEL_SM100_OT (bf16, d_v = 128) with edges_only = 0;
 *   otherwise SFA_ERR_UNSUPPORTED.  Measured slower than the two-kernel path at Qwen3-32K (the per-CTA
 *   top-k prologue sits on every CTA's critical path), so sfa_forward does not use it. */
SFA_API sfa_status sfa_attn_fwd_fused_q(const sfa_attn_desc *desc, const void *q, const uint8_t *k_idx,
                                        const void *k_val, const void *v, void *o, float *lse, uint8_t *q_idx_out,
                                        void *q_val_out, uint32_t *status_word, const void *workspace,
                                        size_t workspace_bytes, sfa_stream_t stream);
/* ------------------------------------------------------------------------------------------
 * Backward: the straight-through rule of P:L103-112 (Sec. 3.1 "Backward
 * computation", Eq. topk_grad) composed with the softmax-attention backward.
 *   Inputs: the forward's codes, v, o and lse (same desc; bf16 only) and the upstream gradient
 *   dO [B][H][n_q][d_v] bf16.  Outputs (fp32, device, caller-owned, fully overwritten):
 *     dq_val [B][H][n_q][k]     = dL/dq~ at the selected coordinates q_idx (the dense dQ of
 *                                 Eq. topk_grad is this scattered to the support, 0 elsewhere)
 *     dk_val [B][H_kv][n_kv][k] = dL/dk~ at k_idx, summed over the kv head's query heads
 *     dv     [B][H_kv][n_kv][d_v]
 *   workspace >= sfa_attn_bwd_workspace_bytes(desc) (D_i = rowsum(dO . O), fp32 per query row).
 *   P is recomputed from the codes and lse (never stored); P and dS enter the tensor cores in
 *   bf16 (reading A24).  Deterministic: no atomics, fixed reduction order.
 *   Errors: fp32 desc or d, d_v not in {64, 128} -> SFA_ERR_UNSUPPORTED; null / misaligned
 *   pointers -> SFA_ERR_INVALID_ARGUMENT; short workspace -> SFA_ERR_RESOURCE. */
SFA_API size_t sfa_attn_bwd_workspace_bytes(const sfa_attn_desc *desc);
SFA_API sfa_status sfa_attn_bwd(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                const uint8_t *k_idx, const void *k_val, const void *v, const void *o,
                                const float *lse, const void *dO, float *dq_val, float *dk_val, float *dv,
                                void *workspace, size_t workspace_bytes, sfa_stream_t stream);

/* SIMT only -- step 3 alone (exposed for the bucket-layout tests):
 * builds the buckets of every key tile into `workspace` (layout in DESIGN.md).  sfa_attn_fwd calls it. */
SFA_API sfa_status sfa_bucket_keys(const sfa_attn_desc *desc, const uint8_t *k_idx, const void *k_val, void *workspace,
                           size_t workspace_bytes, sfa_stream_t stream);

/* SIMT only -- attention over buckets already built by sfa_bucket_keys (same desc, same workspace).
 * Both return SFA_ERR_UNSUPPORTED for a desc that selects the SM100 kernel. */
SFA_API sfa_status sfa_attn_fwd_bucketed(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                 const void *v, void *o, float *lse, const void *workspace,
                                 size_t workspace_bytes, sfa_stream_t stream);

/* Key tile size the bucket layout and kernels use for this desc (128, or 64 when k > 32). */
SFA_API int32_t sfa_key_tile(const sfa_attn_desc *desc);

/* ------------------------------------------------------------------------------------------
 * The whole hot path in one call: codes of Q and K (stage 1) then the attention (stage 2).
 *   q [B][H][n_q][d], k [B][H_kv][n_kv][d], v [B][H_kv][n_kv][d_v], o, lse as above.
 *   scratch: >= sfa_forward_scratch_bytes(desc) device bytes; holds the codes, buckets and
 *   the status word.  Non-finite q/k are detected asynchronously (status word in scratch;
 *   sfa_forward_host checks it and returns SFA_ERR_INVALID_INPUT).
 * ------------------------------------------------------------------------------------------ */
SFA_API size_t sfa_forward_scratch_bytes(const sfa_attn_desc *desc);
SFA_API sfa_status sfa_forward(const sfa_attn_desc *desc, const void *q, const void *k, const void *v, void *o, float *lse,
                       void *scratch, size_t scratch_bytes, sfa_stream_t stream);

/* Same, end to end from HOST buffers: copies q, k, v (pinned host memory recommended) into the
 * caller's device buffers q_dev/k_dev/v_dev, runs sfa_forward, copies o and lse back into
 * o_host/lse_host, and synchronises `stream` before returning (so the host outputs are valid). */
SFA_API sfa_status sfa_forward_host(const sfa_attn_desc *desc, const void *q_host, const void *k_host, const void *v_host,
                            void *o_host, float *lse_host, void *q_dev, void *k_dev, void *v_dev, void *o_dev,
                            float *lse_dev, void *scratch, size_t scratch_bytes, sfa_stream_t stream);

/* Same as sfa_forward_host, pipelined: the B*H_kv independent (batch, kv head) units -- contiguous in
 * every tensor -- are split into `chunks` (1..64) groups; group c's host->device copies, its stage 1+2
 * kernels (on `stream`) and its device->host copies run on three streams, so copies of one group
 * overlap the kernels of its neighbours.  Host buffers must be pinned for the copies to overlap.
 * Results are identical to sfa_forward_host (each unit is computed by the same kernels). Creates and
 * destroys two internal streams and 2*chunks events per call; synchronises before returning. */
SFA_API sfa_status sfa_forward_host_pipelined(const sfa_attn_desc *desc, const void *q_host, const void *k_host,
                                              const void *v_host, void *o_host, float *lse_host, void *q_dev,
                                              void *k_dev, void *v_dev, void *o_dev, float *lse_dev, void *scratch,
                                              size_t scratch_bytes, int32_t chunks, sfa_stream_t stream);

/* Diagnostic (tests only): runs sfa_attn_fwd with the sm_100a kernel (desc->dtype must be bf16 and
 * desc->kernel not SIMT) and also writes the raw fp32 score tile S = Q~ K~^T (unscaled sums of
 * support overlaps) of the first key tile of work item 0 -- query tile 0, the last
 * query block of head 0 (batch 0) -- to `scores` [128][128] (device).  Lets a test check the
 * tensor-core score contraction apart from the softmax and P.V. */
SFA_API sfa_status sfa_debug_sm100_scores(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                          const uint8_t *k_idx, const void *k_val, const void *v, void *o,
                                          float *lse, void *workspace, size_t workspace_bytes, float *scores,
                                          sfa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Step 9 (sharded path only): query-block sharding of one sequence over P GPUs.
 * Zig-zag partition: the sequence is cut into 2P chunks of c tokens; rank p owns chunks p and
 * 2P-1-p (equal causal work), held chunk-major as [2][B][H(_kv)][c][.] (chunk p, then chunk
 * 2P-1-p), so each query chunk's codes and outputs are contiguous.
 * NCCL is loaded at run time (dlopen "libnccl.so.2"); without it these return SFA_ERR_UNSUPPORTED.
 *   sfa_dist_unique_id  -- rank 0 creates the 128-byte ncclUniqueId (shared by the caller, e.g. via
 *                          torch.distributed.broadcast_object_list);
 *   sfa_dist_init       -- every rank joins; the handle owns the communicator (sfa_dist_destroy).
 *   sfa_dist_allgather_kv -- local_desc describes the LOCAL keys (n_kv = 2c, even; B, H_kv, k, d_v,
 *                          dtype as in the full problem); gathers every
 *                          rank's key codes and V (one grouped NCCL all-gather, staged in
 *                          `staging` >= sfa_dist_staging_bytes) and unpacks them into sequence
 *                          order: k_idx_full [B][H_kv][2Pc][k], k_val_full, v_full [B][H_kv][2Pc][d_v].
 *                          The caller then runs sfa_attn_fwd for each of its two query chunks with
 *                          q_pos0 = chunk start over the full keys (reading A9).  Stream-ordered.
 *   sfa_dist_unpack_zigzag -- the unpack alone (device buffers; rank-major [P][2][bh][chunk][row_bytes]
 *                          -> [bh][2P][chunk][row_bytes]); used by sfa_dist_allgather_kv, exposed for tests.
 * ------------------------------------------------------------------------------------------ */
typedef struct sfa_dist *sfa_dist_t;
SFA_API sfa_status sfa_dist_unique_id(void *nccl_unique_id_out /* 128 B */);
SFA_API sfa_status sfa_dist_init(int rank, int world, const void *nccl_unique_id, sfa_dist_t *out);
SFA_API sfa_status sfa_dist_destroy(sfa_dist_t h);
SFA_API size_t sfa_dist_staging_bytes(const sfa_attn_desc *local_desc, int32_t world);
SFA_API sfa_status sfa_dist_allgather_kv(sfa_dist_t h, const sfa_attn_desc *local_desc, const uint8_t *k_idx_local,
                                         const void *k_val_local, const void *v_local, uint8_t *k_idx_full,
                                         void *k_val_full, void *v_full, void *staging, size_t staging_bytes,
                                         sfa_stream_t stream);
SFA_API sfa_status sfa_dist_unpack_zigzag(const void *in, void *out, int32_t world, int64_t bh, int64_t chunk,
                                          int64_t row_bytes, sfa_stream_t stream);

/* Host-only partition plans (no device, no NCCL; the CPU multi-process tests call them too):
 *   sfa_dist_kv_plan    -- what sfa_dist_allgather_kv does for local_desc at `world` ranks: the three
 *                          gathered tensors t = 0 (k_idx), 1 (k_val), 2 (V) each send bytes_per_rank[t]
 *                          bytes per rank into staging at staging_offset[t] (rank-major), then are
 *                          unpacked with sfa_dist_unpack_zigzag(world, bh, chunk, row_bytes[t]);
 *                          staging_bytes = sfa_dist_staging_bytes.  Invalid desc -> INVALID_ARGUMENT.
 *   sfa_dist_zigzag_chunk -- the zig-zag partition of n tokens: chunk length c = n/(2P)
 *                          and the start q_pos0 of rank's chunk half (0: chunk rank, 1: chunk 2P-1-rank).
 *                          n must be a positive multiple of 2P.
 *   sfa_dist_head_shard -- the (batch, kv head) partition (no communication): the B*H_kv
 *                          units of `full` (contiguous in every tensor: unit u = b*H_kv + g holds query heads
 *                          [g*R, g*R+R), R = H/H_kv) split into `world` contiguous ranges whose sizes differ
 *                          by at most one.  Rank `rank` gets units [unit0, unit0 + sub->B): *sub is the same
 *                          problem with B = that count, H = R, H_kv = 1, so its tensors start at unit0 times
 *                          the per-unit size of each tensor.  Fewer units than ranks -> UNSUPPORTED. */
typedef struct {
    int64_t bh, chunk;            /* (batch, kv head) rows and chunk length of the local desc            */
    int64_t row_bytes[3];         /* bytes of one row of k_idx, k_val, V                                  */
    int64_t bytes_per_rank[3];    /* bytes each rank contributes to each gather                           */
    int64_t staging_offset[3];    /* 256-aligned offsets of the three rank-major blocks in the staging    */
    int64_t staging_bytes;
} sfa_dist_kv_plan_t;
SFA_API sfa_status sfa_dist_kv_plan(const sfa_attn_desc *local_desc, int32_t world, sfa_dist_kv_plan_t *plan);
SFA_API sfa_status sfa_dist_zigzag_chunk(int64_t n, int32_t world, int32_t rank, int32_t half, int64_t *chunk_len,
                                         int64_t *q_pos0);
SFA_API sfa_status sfa_dist_head_shard(const sfa_attn_desc *full, int32_t world, int32_t rank, sfa_attn_desc *sub,
                                       int64_t *unit0);

/* Build / device info: 1 if the calling thread's current device is sm_100 and the kernels load. */
SFA_API int32_t sfa_device_supported(void);

#ifdef __cplusplus
}
#endif
#endif /* SFA_H */
