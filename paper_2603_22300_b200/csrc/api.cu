// api.cu -- the C ABI (include/sfa.h): host-side validation, workspace layout, kernel selection.
// Every argument check runs before any launch, so a rejected call leaves all outputs untouched.
#include <math.h>
#include <string.h>

#include "../../include/sfa.h"
#include "launch.cuh"

using namespace sfa;

namespace {

constexpr float kLog2e = 1.4426950408889634f;

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

sfa_status from_cuda(cudaError_t e) { return e == cudaSuccess ? SFA_OK : SFA_ERR_CUDA; }

int key_tile(int k) { return k <= 32 ? 128 : 64; }

int resolve_kernel(const sfa_attn_desc *d);

sfa_status validate_desc(const sfa_attn_desc *d) {
    if (!d) return SFA_ERR_INVALID_ARGUMENT;
    if (d->B < 1 || d->H < 1 || d->H_kv < 1 || d->H % d->H_kv) return SFA_ERR_INVALID_ARGUMENT;
    if (d->d < 1 || d->d > 256 || d->k < 1 || d->k > d->d || d->d_v < 1) return SFA_ERR_INVALID_ARGUMENT;
    if (d->n_q < 1 || d->n_kv < 1 || d->q_pos0 < 0) return SFA_ERR_INVALID_ARGUMENT;
    if (d->causal != 0 && d->causal != 1) return SFA_ERR_INVALID_ARGUMENT;
    if (!(d->scale > 0.f) || !isfinite(d->scale)) return SFA_ERR_INVALID_ARGUMENT;
    if (d->dtype != SFA_F32 && d->dtype != SFA_BF16) return SFA_ERR_INVALID_ARGUMENT;
    if (d->kernel < SFA_KERNEL_AUTO || d->kernel > SFA_KERNEL_SM100_OTH) return SFA_ERR_INVALID_ARGUMENT;
    if (d->kernel == SFA_KERNEL_SM100_PAIR || d->kernel == SFA_KERNEL_SM100_WIDE) return SFA_ERR_UNSUPPORTED;  // removed
    if (d->d != 64 && d->d != 128) return SFA_ERR_UNSUPPORTED;
    if (d->d_v != 64 && d->d_v != 128) return SFA_ERR_UNSUPPORTED;
    if ((d->kernel == SFA_KERNEL_SM100 || d->kernel == SFA_KERNEL_SM100_PAIR || d->kernel == SFA_KERNEL_SM100_WIDE ||
         d->kernel == SFA_KERNEL_SM100_OT || d->kernel == SFA_KERNEL_SM100_PP || d->kernel == SFA_KERNEL_SM100_OTH) &&
        d->dtype != SFA_BF16)
        return SFA_ERR_UNSUPPORTED;
    if ((d->kernel == SFA_KERNEL_SM100_PAIR || d->kernel == SFA_KERNEL_SM100_OTH) && d->d_v != 128)
        return SFA_ERR_UNSUPPORTED;
    if (d->kernel == SFA_KERNEL_DECODE &&
        (d->dtype != SFA_BF16 || (int64_t)(d->H / d->H_kv) * d->n_q > 16))
        return SFA_ERR_UNSUPPORTED;
    if ((d->n_kv + 63) / 64 > (int64_t)INT32_MAX) return SFA_ERR_UNSUPPORTED;
    if (d->edges_only != 0 && d->edges_only != 1) return SFA_ERR_INVALID_ARGUMENT;
    if (d->window < 0 || (d->window > 0 && !d->causal)) return SFA_ERR_INVALID_ARGUMENT;
    if (d->window > 0 && d->kernel != SFA_KERNEL_AUTO && d->kernel != SFA_KERNEL_SIMT &&
        d->kernel != SFA_KERNEL_SM100_OT)
        return SFA_ERR_UNSUPPORTED;  // the window is built into the OT and SIMT kernels only
    if (d->edges_only && d->kernel != SFA_KERNEL_AUTO && d->kernel != SFA_KERNEL_SIMT &&
        d->kernel != SFA_KERNEL_SM100_OT)
        return SFA_ERR_UNSUPPORTED;  // R2 is built into the OT and SIMT kernels only
    // grid.y limits, checked before any launch: the SIMT kernel puts B*H on grid.y, the R2 bitset
    // kernel (edges.cu) B*H_kv (the V prep strides heads over grid.y and has no limit)
    const int kern = resolve_kernel(d);
    if (kern == SFA_KERNEL_SIMT && (int64_t)d->B * d->H > 65535) return SFA_ERR_UNSUPPORTED;
    if (d->edges_only && kern == SFA_KERNEL_SM100_OT && (int64_t)d->B * d->H_kv > 65535) return SFA_ERR_UNSUPPORTED;
    return SFA_OK;
}

BucketLayout layout_of(const sfa_attn_desc *d) {
    return make_layout(d->d, d->k, d->n_kv, key_tile(d->k), d->dtype == SFA_BF16);
}

// Which attention kernel a desc runs.  AUTO: the CUDA-core kernel for fp32 (reading A12); for bf16
// the split-KV decode kernel when a kv head has at most 16 query rows (n_q * H / H_kv), else the
// sm_100a tensor-core kernel: the transposed-output one (SM100_OT) for d_v = 128, SM100 for d_v = 64 (at the
// GPT-2 shape SM100 is faster: 0.054 vs 0.070 ms, profiles/r02_gpt2_ot_dv64.txt), except that R2 and the
// sliding window are built into SM100_OT only (d_v = 64 over the zero-padded V copy).
int resolve_kernel(const sfa_attn_desc *d) {
    if (d->kernel == SFA_KERNEL_SIMT || d->dtype == SFA_F32) return SFA_KERNEL_SIMT;
    if (d->kernel != SFA_KERNEL_AUTO) return d->kernel;
    if (d->edges_only || d->window > 0) return SFA_KERNEL_SM100_OT;  // R2 / window: built into SM100_OT only
    if ((int64_t)(d->H / d->H_kv) * d->n_q <= 16) return SFA_KERNEL_DECODE;
    return d->d_v == 128 ? SFA_KERNEL_SM100_OT : SFA_KERNEL_SM100;
}
bool uses_simt(const sfa_attn_desc *d) { return resolve_kernel(d) == SFA_KERNEL_SIMT; }

size_t bucket_bytes(const sfa_attn_desc *d) {
    const BucketLayout L = layout_of(d);
    return (size_t)d->B * d->H_kv * L.ntiles * L.tile_bytes;
}

// sm100 workspace: [max|V| per (b, kv head), 256-aligned][fp16 copy of V scaled by 2^-e] (vprep.cu);
// the sm100 kernel decompresses key codes on chip and needs no buckets
size_t vprep_amax_bytes(const sfa_attn_desc *d) { return align_up((int64_t)d->B * d->H_kv * 4, 256); }
// features per row of the fp16 V copy: SM100_OT's P.V is d_v = 128 wide, so a d_v = 64 head is padded
int v16_cols(const sfa_attn_desc *d) { return resolve_kernel(d) == SFA_KERNEL_SM100_OT ? 128 : d->d_v; }
size_t vprep_bytes(const sfa_attn_desc *d) {
    return vprep_amax_bytes(d) + (size_t)d->B * d->H_kv * d->n_kv * v16_cols(d) * 2;
}
// SM100_OT: the decompressed K~ rows (bf16, read by TMA) follow the V prep, 256-aligned; then, for R2,
// the key-tile feature bitsets (edges.cu)
bool uses_kdense(const sfa_attn_desc *d) {
    const int k = resolve_kernel(d);
    return k == SFA_KERNEL_SM100_OT || k == SFA_KERNEL_SM100_PP || k == SFA_KERNEL_SM100_OTH;
}
size_t kdense_off(const sfa_attn_desc *d) { return align_up(vprep_bytes(d), 256); }
size_t kdense_bytes(const sfa_attn_desc *d) {
    return uses_kdense(d) ? align_up((int64_t)d->B * d->H_kv * d->n_kv * d->d * 2, 256) : 0;
}
bool uses_kmask(const sfa_attn_desc *d) { return d->edges_only && resolve_kernel(d) == SFA_KERNEL_SM100_OT; }
// ... and last, 256 bytes for the persistent tile scheduler's work counter (SM100_OT)
size_t sched_off(const sfa_attn_desc *d) {
    const size_t o = kdense_off(d) + kdense_bytes(d);
    return uses_kmask(d) ? align_up(o + kfmask_bytes((int64_t)d->B * d->H_kv, d->n_kv, d->d), 256) : o;
}
size_t ws_bytes(const sfa_attn_desc *d) {
    const int kern = resolve_kernel(d);
    if (kern == SFA_KERNEL_SIMT) return bucket_bytes(d);
    if (kern == SFA_KERNEL_DECODE) return decode_workspace_bytes((int64_t)d->B * d->H_kv, d->n_kv, d->d_v);
    if (uses_kdense(d)) return sched_off(d) + 256;
    return vprep_bytes(d);
}

size_t esize(sfa_dtype t) { return t == SFA_BF16 ? 2 : 4; }

// scratch of sfa_forward: [status 256 B][q_idx][q_val][k_idx][k_val][buckets], each 256-aligned
struct Scratch {
    size_t status, q_idx, q_val, k_idx, k_val, ws, total;
};
Scratch scratch_layout(const sfa_attn_desc *d) {
    Scratch s;
    const size_t rq = (size_t)d->B * d->H * d->n_q, rk = (size_t)d->B * d->H_kv * d->n_kv;
    size_t o = 0;
    s.status = o; o += 256;
    s.q_idx = o; o += align_up(rq * d->k, 256);
    s.q_val = o; o += align_up(rq * d->k * esize(d->dtype), 256);
    s.k_idx = o; o += align_up(rk * d->k, 256);
    s.k_val = o; o += align_up(rk * d->k * esize(d->dtype), 256);
    s.ws = o; o += align_up(ws_bytes(d), 256);
    s.total = o;
    return s;
}

AttnParams make_params(const sfa_attn_desc *d, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                       const void *k_val, const void *v, void *o, float *lse, const void *ws) {
    AttnParams p;
    p.q_idx = q_idx; p.q_val = q_val; p.k_idx = k_idx; p.k_val = k_val;
    p.v = v; p.o = o; p.lse = lse; p.ws = (const uint8_t *)ws;
    p.v_amax = (const uint32_t *)ws;
    p.v16 = ws ? (const uint8_t *)ws + vprep_amax_bytes(d) : nullptr;
    p.B = d->B; p.H = d->H; p.H_kv = d->H_kv; p.k = d->k;
    p.n_q = d->n_q; p.n_kv = d->n_kv; p.q_pos0 = d->q_pos0; p.causal = d->causal;
    p.scale_log2 = d->scale * kLog2e;
    p.L = layout_of(d);
    p.edges_only = d->edges_only;
    p.window = d->window;
    p.k_dense = (ws && uses_kdense(d)) ? (const uint8_t *)ws + kdense_off(d) : nullptr;
    p.sched = (ws && uses_kdense(d)) ? (uint32_t *)((uint8_t *)const_cast<void *>(ws) + sched_off(d)) : nullptr;
    p.kfmask = (ws && uses_kmask(d)) ? (const uint32_t *)((const uint8_t *)ws + kdense_off(d) + kdense_bytes(d)) : nullptr;
    return p;
}

sfa_status from_launch(cudaError_t e) {
    if (e == cudaSuccess) return SFA_OK;
    (void)cudaGetLastError();
    return e == cudaErrorNotSupported ? SFA_ERR_UNSUPPORTED : SFA_ERR_CUDA;
}

// step 3: what the chosen attention kernel reads besides the codes -- key-tile buckets (SIMT) or
// max|V| + the scaled fp16 V (SM100)
sfa_status run_prepare(const sfa_attn_desc *d, const uint8_t *k_idx, const void *k_val, const void *v, void *ws,
                       cudaStream_t st) {
    const AttnParams p = make_params(d, nullptr, nullptr, k_idx, k_val, v, nullptr, nullptr, ws);
    if (resolve_kernel(d) == SFA_KERNEL_DECODE) return SFA_OK;  // reads the codes and bf16 V as they are
    if (uses_simt(d))
        return from_cuda(launch_bucket(k_idx, k_val, d->dtype == SFA_BF16, d->d, d->k, (int64_t)d->B * d->H_kv,
                                       d->n_kv, p.L, ws, st));
    const int64_t bh_kv = (int64_t)d->B * d->H_kv;
    cudaError_t e;
    if (prep_small_ok(bh_kv, d->n_kv, d->d_v, uses_kdense(d) ? bh_kv * d->n_kv : 0)) {
        // small heads: max|V|, the fp16 V copy and the K~ rows in one launch
        e = launch_prep_small(v, bh_kv, d->n_kv, d->d_v, v16_cols(d), (uint32_t *)p.v_amax, (void *)p.v16, k_idx, k_val,
                              d->d, d->k, uses_kdense(d) ? (void *)p.k_dense : nullptr, st);
    } else {
        e = launch_vprep(v, bh_kv, d->n_kv, d->d_v, v16_cols(d), (uint32_t *)p.v_amax, (void *)p.v16, st);
        if (e == cudaSuccess && uses_kdense(d))
            e = launch_kdense(k_idx, k_val, bh_kv * d->n_kv, d->d, d->k, (void *)p.k_dense, st);
    }
    if (e == cudaSuccess && uses_kmask(d))
        e = launch_kfmask(k_idx, (int64_t)d->B * d->H_kv, d->n_kv, d->d, d->k, (uint32_t *)p.kfmask, st);
    return from_cuda(e);
}

// steps 4-8 over a prepared workspace
sfa_status run_attn_prepared(const sfa_attn_desc *d, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                             const void *k_val, const void *v, void *o, float *lse, void *ws, cudaStream_t st,
                             float *dbg = nullptr) {
    const AttnParams p = make_params(d, q_idx, q_val, k_idx, k_val, v, o, lse, ws);
    const int kern = resolve_kernel(d);
    if (kern == SFA_KERNEL_DECODE) return from_launch(launch_decode(p, d->d, d->d_v, st, ws));
    if (kern == SFA_KERNEL_SM100_OT) return from_launch(launch_attn_sm100_ot(p, d->d, d->d_v, st, dbg));
    if (kern == SFA_KERNEL_SM100_PP) return from_launch(launch_attn_sm100_pp(p, d->d, d->d_v, st, dbg));
    if (kern == SFA_KERNEL_SM100_OTH) return from_launch(launch_attn_sm100_oth(p, d->d, d->d_v, st, dbg));
    if (kern == SFA_KERNEL_SM100) return from_launch(launch_attn_sm100(p, d->d, d->d_v, st, dbg));
    return from_cuda(launch_attn_simt(p, d->dtype == SFA_BF16, d->d, d->d_v, st));
}

sfa_status run_attn(const sfa_attn_desc *d, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                    const void *k_val, const void *v, void *o, float *lse, void *ws, cudaStream_t st) {
    sfa_status s = run_prepare(d, k_idx, k_val, v, ws, st);
    if (s != SFA_OK) return s;
    return run_attn_prepared(d, q_idx, q_val, k_idx, k_val, v, o, lse, ws, st);
}

bool codes_aligned(const void *a, const void *b) { return aligned16(a) && aligned16(b); }

// the fused step-1-on-Q path (N3(ii)) exists for the SM100_OT kernel with R1 semantics
bool fusable(const sfa_attn_desc *d) {
    return d->dtype == SFA_BF16 && !d->edges_only && d->window == 0 && resolve_kernel(d) == SFA_KERNEL_SM100_OT;
}

}  // namespace

extern "C" {

const char *sfa_status_string(sfa_status s) {
    switch (s) {
        case SFA_OK: return "ok";
        case SFA_ERR_INVALID_ARGUMENT: return "invalid-argument";
        case SFA_ERR_INVALID_INPUT: return "invalid-input";
        case SFA_ERR_UNSUPPORTED: return "unsupported";
        case SFA_ERR_RESOURCE: return "resource-limit";
        case SFA_ERR_CUDA: return "cuda-error";
    }
    return "unknown-status";
}

sfa_status sfa_topk_codes(const void *x, sfa_dtype dtype, int64_t rows, int32_t d, int64_t ld, int32_t k,
                          uint8_t *idx, void *val, uint32_t *status_word, sfa_stream_t stream) {
    if (dtype != SFA_F32 && dtype != SFA_BF16) return SFA_ERR_INVALID_ARGUMENT;
    if (rows < 0 || d < 1 || d > 256 || k < 1 || k > d || ld < d) return SFA_ERR_INVALID_ARGUMENT;
    if (d != 64 && d != 128) return SFA_ERR_UNSUPPORTED;
    if (rows == 0) return SFA_OK;
    if (!x || !idx || !val) return SFA_ERR_INVALID_ARGUMENT;
    // every lane issues one vector load of d/32 elements: the row starts must be vector aligned
    const size_t vec = (size_t)(d / 32) * esize(dtype);
    if (((uintptr_t)x % vec) || ((size_t)ld * esize(dtype)) % vec) return SFA_ERR_INVALID_ARGUMENT;
    if (status_word && ((uintptr_t)status_word & 3u)) return SFA_ERR_INVALID_ARGUMENT;
    return from_cuda(launch_topk(x, dtype == SFA_BF16, rows, d, ld, k, idx, val, status_word, (cudaStream_t)stream));
}

sfa_status sfa_topk_codes_qk(const void *q, int64_t q_rows, int64_t q_ld, uint8_t *q_idx, void *q_val, const void *k,
                             int64_t k_rows, int64_t k_ld, uint8_t *k_idx, void *k_val, sfa_dtype dtype, int32_t d,
                             int32_t kk, uint32_t *status_word, sfa_stream_t stream) {
    if (dtype != SFA_BF16) {  // the fp32 path has no fused launch: two stage-1 calls
        sfa_status s = sfa_topk_codes(q, dtype, q_rows, d, q_ld, kk, q_idx, q_val, status_word, stream);
        return s != SFA_OK ? s : sfa_topk_codes(k, dtype, k_rows, d, k_ld, kk, k_idx, k_val, status_word, stream);
    }
    // same argument rules as sfa_topk_codes, for each tensor, before any launch
    for (int t = 0; t < 2; ++t) {
        const void *x = t ? k : q;
        const int64_t rows = t ? k_rows : q_rows, ld = t ? k_ld : q_ld;
        const void *ix = t ? (const void *)k_idx : (const void *)q_idx, *vx = t ? k_val : q_val;
        if (rows < 0 || d < 1 || d > 256 || kk < 1 || kk > d || ld < d) return SFA_ERR_INVALID_ARGUMENT;
        if (d != 64 && d != 128) return SFA_ERR_UNSUPPORTED;
        if (rows > 0 && (!x || !ix || !vx)) return SFA_ERR_INVALID_ARGUMENT;
        const size_t vec = (size_t)(d / 32) * 2;
        if (rows > 0 && (((uintptr_t)x % vec) || ((size_t)ld * 2) % vec)) return SFA_ERR_INVALID_ARGUMENT;
    }
    if (status_word && ((uintptr_t)status_word & 3u)) return SFA_ERR_INVALID_ARGUMENT;
    if (q_rows == 0 || k_rows == 0) {
        sfa_status s = sfa_topk_codes(q, dtype, q_rows, d, q_ld, kk, q_idx, q_val, status_word, stream);
        return s != SFA_OK ? s : sfa_topk_codes(k, dtype, k_rows, d, k_ld, kk, k_idx, k_val, status_word, stream);
    }
    return from_cuda(launch_topk_pair(q, q_rows, q_ld, q_idx, q_val, k, k_rows, k_ld, k_idx, k_val, d, kk, status_word,
                                      (cudaStream_t)stream));
}

size_t sfa_attn_workspace_bytes(const sfa_attn_desc *desc) {
    if (validate_desc(desc) != SFA_OK) return 0;
    return ws_bytes(desc);
}

int32_t sfa_key_tile(const sfa_attn_desc *desc) {
    if (validate_desc(desc) != SFA_OK) return 0;
    return key_tile(desc->k);
}

sfa_status sfa_bucket_keys(const sfa_attn_desc *desc, const uint8_t *k_idx, const void *k_val, void *workspace,
                           size_t workspace_bytes, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!uses_simt(desc)) return SFA_ERR_UNSUPPORTED;  // buckets feed the CUDA-core kernel only
    if (!k_idx || !k_val || !workspace || !aligned16(workspace)) return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    return from_cuda(launch_bucket(k_idx, k_val, desc->dtype == SFA_BF16, desc->d, desc->k,
                                   (int64_t)desc->B * desc->H_kv, desc->n_kv, layout_of(desc), workspace,
                                   (cudaStream_t)stream));
}

sfa_status sfa_attn_fwd_bucketed(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val, const void *v,
                                 void *o, float *lse, const void *workspace, size_t workspace_bytes,
                                 sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!q_idx || !q_val || !v || !o || !lse || !workspace) return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(v) || !aligned16(o) || !aligned16(workspace) || ((uintptr_t)lse & 3u))
        return SFA_ERR_INVALID_ARGUMENT;
    if (!uses_simt(desc)) return SFA_ERR_UNSUPPORTED;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    const AttnParams p = make_params(desc, q_idx, q_val, nullptr, nullptr, v, o, lse, workspace);
    return from_cuda(launch_attn_simt(p, desc->dtype == SFA_BF16, desc->d, desc->d_v, (cudaStream_t)stream));
}

sfa_status sfa_attn_fwd(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                        const void *k_val, const void *v, void *o, float *lse, void *workspace,
                        size_t workspace_bytes, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!q_idx || !q_val || !k_idx || !k_val || !v || !o || !lse) return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(v) || !aligned16(o) || ((uintptr_t)lse & 3u) || !codes_aligned(q_idx, q_val) ||
        !codes_aligned(k_idx, k_val))
        return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    if (!workspace || !aligned16(workspace)) return SFA_ERR_INVALID_ARGUMENT;
    return run_attn(desc, q_idx, q_val, k_idx, k_val, v, o, lse, workspace, (cudaStream_t)stream);
}

sfa_status sfa_attn_prepare(const sfa_attn_desc *desc, const uint8_t *k_idx, const void *k_val, const void *v,
                            void *workspace, size_t workspace_bytes, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!k_idx || !k_val || !v || !workspace) return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(v) || !aligned16(workspace) || !codes_aligned(k_idx, k_val)) return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    return run_prepare(desc, k_idx, k_val, v, workspace, (cudaStream_t)stream);
}

sfa_status sfa_attn_fwd_prepared(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                 const uint8_t *k_idx, const void *k_val, const void *v, void *o, float *lse,
                                 const void *workspace, size_t workspace_bytes, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!q_idx || !q_val || !k_idx || !k_val || !v || !o || !lse || !workspace) return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(v) || !aligned16(o) || ((uintptr_t)lse & 3u) || !aligned16(workspace) ||
        !codes_aligned(q_idx, q_val) || !codes_aligned(k_idx, k_val))
        return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    return run_attn_prepared(desc, q_idx, q_val, k_idx, k_val, v, o, lse, (void *)workspace, (cudaStream_t)stream);
}

sfa_status sfa_attn_fwd_blocksel(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                 const uint8_t *k_idx, const void *k_val, const void *v, const int32_t *block_sel,
                                 int32_t max_sel, void *o, float *lse, void *workspace, size_t workspace_bytes,
                                 sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (desc->dtype != SFA_BF16 || (desc->H / desc->H_kv) % 2 != 0 || desc->edges_only ||
        desc->window > 0 || resolve_kernel(desc) != SFA_KERNEL_SM100_OT)
        return SFA_ERR_UNSUPPORTED;
    if (!q_idx || !q_val || !k_idx || !k_val || !v || !o || !lse || !workspace || !block_sel || max_sel < 1)
        return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(v) || !aligned16(o) || ((uintptr_t)lse & 3u) || !aligned16(workspace) ||
        ((uintptr_t)block_sel & 3u) || !codes_aligned(q_idx, q_val) || !codes_aligned(k_idx, k_val))
        return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    cudaStream_t st = (cudaStream_t)stream;
    s = run_prepare(desc, k_idx, k_val, v, workspace, st);
    if (s != SFA_OK) return s;
    AttnParams p = make_params(desc, q_idx, q_val, k_idx, k_val, v, o, lse, workspace);
    p.bsel = block_sel;
    p.max_sel = max_sel;
    return from_launch(launch_attn_sm100_ot(p, desc->d, desc->d_v, st, nullptr));
}

sfa_status sfa_attn_fwd_fused_q(const sfa_attn_desc *desc, const void *q, const uint8_t *k_idx, const void *k_val,
                                const void *v, void *o, float *lse, uint8_t *q_idx_out, void *q_val_out,
                                uint32_t *status_word, const void *workspace, size_t workspace_bytes,
                                sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!fusable(desc)) return SFA_ERR_UNSUPPORTED;
    if (!q || !k_idx || !k_val || !v || !o || !lse || !workspace) return SFA_ERR_INVALID_ARGUMENT;
    if ((q_idx_out == nullptr) != (q_val_out == nullptr)) return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !codes_aligned(k_idx, k_val) || !aligned16(v) || !aligned16(o) || ((uintptr_t)lse & 3u) ||
        (q_idx_out && !codes_aligned(q_idx_out, q_val_out)) || ((uintptr_t)status_word & 3u))
        return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    AttnParams p = make_params(desc, nullptr, nullptr, k_idx, k_val, v, o, lse, workspace);
    p.q_dense = q;
    p.q_idx_out = q_idx_out;
    p.q_val_out = q_val_out;
    p.status_word = status_word;
    return from_launch(launch_attn_sm100_ot(p, desc->d, desc->d_v, (cudaStream_t)stream, nullptr));
}

// backward workspace: D_i [B*H*n_q] fp32, then (256-aligned) the decompressed Q~ rows [B*H*n_q][d] and K~
// rows [B*H_kv*n_kv][d], bf16, for the kernels' TMA
struct BwdWs {
    size_t qd, kd, total;
};
BwdWs bwd_ws(const sfa_attn_desc *d) {
    BwdWs w;
    w.qd = align_up((int64_t)d->B * d->H * d->n_q * sizeof(float), 256);
    w.kd = w.qd + align_up((int64_t)d->B * d->H * d->n_q * d->d * 2, 256);
    w.total = w.kd + align_up((int64_t)d->B * d->H_kv * d->n_kv * d->d * 2, 256);
    return w;
}
size_t sfa_attn_bwd_workspace_bytes(const sfa_attn_desc *desc) {
    if (validate_desc(desc) != SFA_OK) return 0;
    return bwd_ws(desc).total;
}

sfa_status sfa_attn_bwd(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                        const void *k_val, const void *v, const void *o, const float *lse, const void *dO,
                        float *dq_val, float *dk_val, float *dv, void *workspace, size_t workspace_bytes,
                        sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (desc->dtype != SFA_BF16 || desc->edges_only || desc->window > 0) return SFA_ERR_UNSUPPORTED;
    if (!q_idx || !q_val || !k_idx || !k_val || !v || !o || !lse || !dO || !dq_val || !dk_val || !dv || !workspace)
        return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(v) || !aligned16(o) || !aligned16(dO) || !aligned16(dv) || !aligned16(workspace) ||
        ((uintptr_t)lse & 3u) || ((uintptr_t)dq_val & 3u) || ((uintptr_t)dk_val & 3u) ||
        !codes_aligned(q_idx, q_val) || !codes_aligned(k_idx, k_val))
        return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < sfa_attn_bwd_workspace_bytes(desc)) return SFA_ERR_RESOURCE;
    const AttnParams p = make_params(desc, q_idx, q_val, k_idx, k_val, v, const_cast<void *>(o),
                                     const_cast<float *>(lse), workspace);
    const BwdWs w = bwd_ws(desc);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    return from_launch(launch_attn_bwd(p, desc->d, desc->d_v, dO, static_cast<float *>(workspace), ws + w.qd, ws + w.kd,
                                       dq_val, dk_val, dv, (cudaStream_t)stream));
}

sfa_status sfa_debug_sm100_scores(const sfa_attn_desc *desc, const uint8_t *q_idx, const void *q_val,
                                  const uint8_t *k_idx, const void *k_val, const void *v, void *o, float *lse,
                                  void *workspace, size_t workspace_bytes, float *scores, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    const int kern = resolve_kernel(desc);
    if (kern == SFA_KERNEL_SIMT || kern == SFA_KERNEL_DECODE) return SFA_ERR_UNSUPPORTED;
    if (!q_idx || !q_val || !k_idx || !k_val || !v || !o || !lse || !scores || !workspace) return SFA_ERR_INVALID_ARGUMENT;
    if (workspace_bytes < ws_bytes(desc)) return SFA_ERR_RESOURCE;
    cudaStream_t st = (cudaStream_t)stream;
    s = run_prepare(desc, k_idx, k_val, v, workspace, st);
    if (s != SFA_OK) return s;
    return run_attn_prepared(desc, q_idx, q_val, k_idx, k_val, v, o, lse, workspace, st, scores);
}

size_t sfa_forward_scratch_bytes(const sfa_attn_desc *desc) {
    if (validate_desc(desc) != SFA_OK) return 0;
    return scratch_layout(desc).total;
}

// stages 1 + 2 with the non-finite flag OR-ed into `status` (not reset here)
static sfa_status forward_impl(const sfa_attn_desc *desc, const void *q, const void *k, const void *v, void *o,
                               float *lse, uint8_t *S, uint32_t *status, cudaStream_t st) {
    const Scratch L = scratch_layout(desc);
    const bool bf16 = desc->dtype == SFA_BF16;
    cudaError_t e;
    // step 1 on Q as its own kernel (measured faster than the fused prologue, N3(ii)), Q and K
    // rows in one launch when both take the bf16 row kernel
    const bool fuse = false;
    if (bf16 && desc->k < desc->d) {
        e = launch_topk_pair(q, (int64_t)desc->B * desc->H * desc->n_q, desc->d, S + L.q_idx, S + L.q_val, k,
                             (int64_t)desc->B * desc->H_kv * desc->n_kv, desc->d, S + L.k_idx, S + L.k_val, desc->d,
                             desc->k, status, st);
        if (e != cudaSuccess) return SFA_ERR_CUDA;
    } else {
        e = launch_topk(q, bf16, (int64_t)desc->B * desc->H * desc->n_q, desc->d, desc->d, desc->k, S + L.q_idx,
                        S + L.q_val, status, st);
        if (e != cudaSuccess) return SFA_ERR_CUDA;
        e = launch_topk(k, bf16, (int64_t)desc->B * desc->H_kv * desc->n_kv, desc->d, desc->d, desc->k, S + L.k_idx,
                        S + L.k_val, status, st);
        if (e != cudaSuccess) return SFA_ERR_CUDA;
    }
    if (!fuse || !fusable(desc))
        return run_attn(desc, S + L.q_idx, S + L.q_val, S + L.k_idx, S + L.k_val, v, o, lse, S + L.ws, st);
    sfa_status s = run_prepare(desc, S + L.k_idx, S + L.k_val, v, S + L.ws, st);
    if (s != SFA_OK) return s;
    AttnParams p = make_params(desc, nullptr, nullptr, S + L.k_idx, S + L.k_val, v, o, lse, S + L.ws);
    p.q_dense = q;
    p.q_idx_out = S + L.q_idx;  // the codes of Q stay available (e.g. for the backward)
    p.q_val_out = S + L.q_val;
    p.status_word = status;
    return from_launch(launch_attn_sm100_ot(p, desc->d, desc->d_v, st, nullptr));
}

sfa_status sfa_forward(const sfa_attn_desc *desc, const void *q, const void *k, const void *v, void *o, float *lse,
                       void *scratch, size_t scratch_bytes, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!q || !k || !v || !o || !lse || !scratch) return SFA_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(scratch) ||
        ((uintptr_t)lse & 3u))
        return SFA_ERR_INVALID_ARGUMENT;
    const Scratch L = scratch_layout(desc);
    if (scratch_bytes < L.total) return SFA_ERR_RESOURCE;
    uint8_t *S = (uint8_t *)scratch;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *status = (uint32_t *)(S + L.status);
    if (cudaMemsetAsync(status, 0, 4, st) != cudaSuccess) return SFA_ERR_CUDA;
    return forward_impl(desc, q, k, v, o, lse, S, status, st);
}

sfa_status sfa_forward_host(const sfa_attn_desc *desc, const void *q_host, const void *k_host, const void *v_host,
                            void *o_host, float *lse_host, void *q_dev, void *k_dev, void *v_dev, void *o_dev,
                            float *lse_dev, void *scratch, size_t scratch_bytes, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!q_host || !k_host || !v_host || !o_host || !lse_host) return SFA_ERR_INVALID_ARGUMENT;
    if (!q_dev || !k_dev || !v_dev || !o_dev || !lse_dev || !scratch) return SFA_ERR_INVALID_ARGUMENT;
    const Scratch L = scratch_layout(desc);
    if (scratch_bytes < L.total) return SFA_ERR_RESOURCE;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t es = esize(desc->dtype);
    const size_t qb = (size_t)desc->B * desc->H * desc->n_q * desc->d * es;
    const size_t kb = (size_t)desc->B * desc->H_kv * desc->n_kv * desc->d * es;
    const size_t vb = (size_t)desc->B * desc->H_kv * desc->n_kv * desc->d_v * es;
    const size_t ob = (size_t)desc->B * desc->H * desc->n_q * desc->d_v * es;
    const size_t lb = (size_t)desc->B * desc->H * desc->n_q * 4;
    if (cudaMemcpyAsync(q_dev, q_host, qb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SFA_ERR_CUDA;
    if (cudaMemcpyAsync(k_dev, k_host, kb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SFA_ERR_CUDA;
    if (cudaMemcpyAsync(v_dev, v_host, vb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SFA_ERR_CUDA;
    s = sfa_forward(desc, q_dev, k_dev, v_dev, o_dev, lse_dev, scratch, scratch_bytes, stream);
    if (s != SFA_OK) return s;
    uint32_t status = 0;
    if (cudaMemcpyAsync(o_host, o_dev, ob, cudaMemcpyDeviceToHost, st) != cudaSuccess) return SFA_ERR_CUDA;
    if (cudaMemcpyAsync(lse_host, lse_dev, lb, cudaMemcpyDeviceToHost, st) != cudaSuccess) return SFA_ERR_CUDA;
    if (cudaMemcpyAsync(&status, (uint8_t *)scratch + L.status, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return SFA_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return SFA_ERR_CUDA;
    return status ? SFA_ERR_INVALID_INPUT : SFA_OK;
}

sfa_status sfa_forward_host_pipelined(const sfa_attn_desc *desc, const void *q_host, const void *k_host,
                                      const void *v_host, void *o_host, float *lse_host, void *q_dev, void *k_dev,
                                      void *v_dev, void *o_dev, float *lse_dev, void *scratch, size_t scratch_bytes,
                                      int32_t chunks, sfa_stream_t stream) {
    sfa_status s = validate_desc(desc);
    if (s != SFA_OK) return s;
    if (!q_host || !k_host || !v_host || !o_host || !lse_host) return SFA_ERR_INVALID_ARGUMENT;
    if (!q_dev || !k_dev || !v_dev || !o_dev || !lse_dev || !scratch || chunks < 1) return SFA_ERR_INVALID_ARGUMENT;
    if (scratch_bytes < scratch_layout(desc).total) return SFA_ERR_RESOURCE;
    const int R = desc->H / desc->H_kv;
    const int64_t units = (int64_t)desc->B * desc->H_kv;  // (b, kv head): independent, contiguous everywhere
    const int64_t nch = chunks < units ? chunks : units;
    const size_t es = esize(desc->dtype);
    // bytes of one unit in each tensor
    const size_t uq = (size_t)R * desc->n_q * desc->d * es, uk = (size_t)desc->n_kv * desc->d * es;
    const size_t uv = (size_t)desc->n_kv * desc->d_v * es, uo = (size_t)R * desc->n_q * desc->d_v * es;
    const size_t ul = (size_t)R * desc->n_q * 4;
    cudaStream_t st = (cudaStream_t)stream, s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_in[64], ev_done[64];
    if (nch > 64) return SFA_ERR_INVALID_ARGUMENT;
    if (cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking) != cudaSuccess) return SFA_ERR_CUDA;
    if (cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking) != cudaSuccess) {
        cudaStreamDestroy(s_in);
        return SFA_ERR_CUDA;
    }
    int nev = 0;
    sfa_status res = SFA_OK;
    for (; nev < nch; ++nev) {
        if (cudaEventCreateWithFlags(&ev_in[nev], cudaEventDisableTiming) != cudaSuccess) break;
        if (cudaEventCreateWithFlags(&ev_done[nev], cudaEventDisableTiming) != cudaSuccess) {
            cudaEventDestroy(ev_in[nev]);
            break;
        }
    }
    if (nev < nch) res = SFA_ERR_CUDA;
    // the caller's stream may carry prior work on the device buffers: the copies start after it
    cudaEvent_t ev_start;
    if (res == SFA_OK && cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(ev_start, st);
        cudaStreamWaitEvent(s_in, ev_start, 0);
        cudaEventDestroy(ev_start);
    }
    // one status word per chunk (the 256-byte status area holds 64): no host sync inside the pipeline
    const Scratch L = scratch_layout(desc);
    uint32_t *status_dev = (uint32_t *)((uint8_t *)scratch + L.status);
    if (res == SFA_OK && cudaMemsetAsync(status_dev, 0, 256, st) != cudaSuccess) res = SFA_ERR_CUDA;
    for (int64_t c = 0; c < nch && res == SFA_OK; ++c) {
        const int64_t u0 = units * c / nch, u1 = units * (c + 1) / nch, nu = u1 - u0;
        sfa_attn_desc sub = *desc;  // the chunk as its own problem: nu batches of R query heads, 1 kv head
        sub.B = (int32_t)nu;
        sub.H = R;
        sub.H_kv = 1;
        auto q8 = [](const void *p, size_t off) { return (const uint8_t *)p + off; };
        auto w8 = [](void *p, size_t off) { return (uint8_t *)p + off; };
        bool ok = cudaMemcpyAsync(w8(q_dev, u0 * uq), q8(q_host, u0 * uq), nu * uq, cudaMemcpyHostToDevice, s_in) ==
                  cudaSuccess;
        ok = ok && cudaMemcpyAsync(w8(k_dev, u0 * uk), q8(k_host, u0 * uk), nu * uk, cudaMemcpyHostToDevice, s_in) ==
                       cudaSuccess;
        ok = ok && cudaMemcpyAsync(w8(v_dev, u0 * uv), q8(v_host, u0 * uv), nu * uv, cudaMemcpyHostToDevice, s_in) ==
                       cudaSuccess;
        ok = ok && cudaEventRecord(ev_in[c], s_in) == cudaSuccess;
        ok = ok && cudaStreamWaitEvent(st, ev_in[c], 0) == cudaSuccess;
        if (!ok) {
            res = SFA_ERR_CUDA;
            break;
        }
        res = forward_impl(&sub, w8(q_dev, u0 * uq), w8(k_dev, u0 * uk), w8(v_dev, u0 * uv), w8(o_dev, u0 * uo),
                           (float *)w8(lse_dev, u0 * ul), (uint8_t *)scratch, status_dev + c, st);
        if (res != SFA_OK) break;
        ok = cudaEventRecord(ev_done[c], st) == cudaSuccess && cudaStreamWaitEvent(s_out, ev_done[c], 0) == cudaSuccess;
        ok = ok && cudaMemcpyAsync(w8(o_host, u0 * uo), w8(o_dev, u0 * uo), nu * uo, cudaMemcpyDeviceToHost, s_out) ==
                       cudaSuccess;
        ok = ok && cudaMemcpyAsync(w8(lse_host, u0 * ul), w8(lse_dev, u0 * ul), nu * ul, cudaMemcpyDeviceToHost,
                                   s_out) == cudaSuccess;
        if (!ok) res = SFA_ERR_CUDA;
    }
    uint32_t status_h[64] = {0};
    if (res == SFA_OK && cudaMemcpyAsync(status_h, status_dev, 256, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        res = SFA_ERR_CUDA;
    uint32_t status = 0;
    if (cudaStreamSynchronize(s_out) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) res = SFA_ERR_CUDA;
    for (int i = 0; i < nev; ++i) {
        cudaEventDestroy(ev_in[i]);
        cudaEventDestroy(ev_done[i]);
    }
    cudaStreamDestroy(s_in);
    cudaStreamDestroy(s_out);
    if (res != SFA_OK) return res;
    for (int i = 0; i < 64; ++i) status |= status_h[i];
    return status ? SFA_ERR_INVALID_INPUT : SFA_OK;
}

int32_t sfa_device_supported(void) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0;
}

}  // extern "C"
