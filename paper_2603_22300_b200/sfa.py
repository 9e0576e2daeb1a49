"""Thin Python binding of the C ABI in include/sfa.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of ``libsfa.so``; this module only
allocates outputs with PyTorch, checks dtypes/devices/contiguity, and passes raw pointers
and the current CUDA stream.  There is no CPU fallback: if the library is missing the
import of the library fails loudly (build it with ``python -m paper_2603_22300_b200.build``).
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsfa.so")

SFA_F32, SFA_BF16 = 0, 1
(KERNEL_AUTO, KERNEL_SIMT, KERNEL_SM100, KERNEL_SM100_PAIR, KERNEL_SM100_WIDE, KERNEL_DECODE, KERNEL_SM100_OT,
 KERNEL_SM100_PP, KERNEL_SM100_OTH) = range(9)
GEN_IID, GEN_LATTICE, GEN_SKEWED = 0, 1, 2
_STATUS = {0: "ok", 1: "invalid-argument", 2: "invalid-input", 3: "unsupported", 4: "resource-limit",
           5: "cuda-error"}


class SfaError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {_STATUS.get(code, code)}")
        self.code = code


class KvPlan(ctypes.Structure):
    """sfa_dist_kv_plan_t (include/sfa.h)."""
    _fields_ = [("bh", ctypes.c_int64), ("chunk", ctypes.c_int64), ("row_bytes", ctypes.c_int64 * 3),
                ("bytes_per_rank", ctypes.c_int64 * 3), ("staging_offset", ctypes.c_int64 * 3),
                ("staging_bytes", ctypes.c_int64)]


class AttnDesc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("H_kv", ctypes.c_int32),
                ("d", ctypes.c_int32), ("k", ctypes.c_int32), ("d_v", ctypes.c_int32),
                ("n_q", ctypes.c_int64), ("n_kv", ctypes.c_int64), ("q_pos0", ctypes.c_int64),
                ("causal", ctypes.c_int32), ("scale", ctypes.c_float), ("dtype", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("edges_only", ctypes.c_int32), ("window", ctypes.c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2603_22300_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        D = ctypes.POINTER(AttnDesc)
        sig = {
            "sfa_status_string": ([I32], ctypes.c_char_p),
            "sfa_topk_codes": ([P, I32, I64, I32, I64, I32, P, P, P, P], I32),
            "sfa_topk_codes_qk": ([P, I64, I64, P, P, P, I64, I64, P, P, I32, I32, I32, P, P], I32),
            "sfa_attn_workspace_bytes": ([D], SZ),
            "sfa_attn_fwd": ([D, P, P, P, P, P, P, P, P, SZ, P], I32),
            "sfa_bucket_keys": ([D, P, P, P, SZ, P], I32),
            "sfa_attn_fwd_bucketed": ([D, P, P, P, P, P, P, SZ, P], I32),
            "sfa_attn_prepare": ([D, P, P, P, P, SZ, P], I32),
            "sfa_dist_unique_id": ([P], I32),
            "sfa_dist_init": ([I32, I32, P, P], I32),
            "sfa_dist_destroy": ([P], I32),
            "sfa_dist_staging_bytes": ([D, I32], SZ),
            "sfa_dist_allgather_kv": ([P, D, P, P, P, P, P, P, P, SZ, P], I32),
            "sfa_dist_unpack_zigzag": ([P, P, I32, I64, I64, I64, P], I32),
            "sfa_attn_fwd_prepared": ([D, P, P, P, P, P, P, P, P, SZ, P], I32),
            "sfa_key_tile": ([D], I32),
            "sfa_forward_scratch_bytes": ([D], SZ),
            "sfa_forward": ([D, P, P, P, P, P, P, SZ, P], I32),
            "sfa_forward_host": ([D, P, P, P, P, P, P, P, P, P, P, P, SZ, P], I32),
            "sfa_forward_host_pipelined": ([D, P, P, P, P, P, P, P, P, P, P, P, SZ, I32, P], I32),
            "sfa_device_supported": ([], I32),
            "sfa_debug_sm100_scores": ([D, P, P, P, P, P, P, P, P, SZ, P, P], I32),
            "sfa_gen_fill": ([P, I32, I64, I64, ctypes.c_uint64, I32, I32, I64, I32, I32, P], I32),
            "sfa_attn_bwd_workspace_bytes": ([D], SZ),
            "sfa_attn_bwd": ([D, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P], I32),
            "sfa_attn_fwd_fused_q": ([D, P, P, P, P, P, P, P, P, P, P, SZ, P], I32),
            "sfa_attn_fwd_blocksel": ([D, P, P, P, P, P, P, I32, P, P, P, SZ, P], I32),
            "sfa_dist_kv_plan": ([D, I32, ctypes.POINTER(KvPlan)], I32),
            "sfa_dist_zigzag_chunk": ([I64, I32, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)], I32),
            "sfa_dist_head_shard": ([D, I32, I32, D, ctypes.POINTER(I64)], I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


EXPORTS = ("sfa_status_string", "sfa_topk_codes", "sfa_topk_codes_qk", "sfa_attn_workspace_bytes", "sfa_attn_fwd", "sfa_bucket_keys",
           "sfa_attn_fwd_bucketed", "sfa_key_tile", "sfa_forward_scratch_bytes", "sfa_forward",
           "sfa_forward_host", "sfa_device_supported", "sfa_gen_fill", "sfa_debug_sm100_scores",
           "sfa_attn_prepare", "sfa_attn_fwd_prepared", "sfa_dist_unique_id", "sfa_dist_init", "sfa_dist_destroy",
           "sfa_dist_staging_bytes", "sfa_dist_allgather_kv", "sfa_dist_unpack_zigzag", "sfa_forward_host_pipelined",
           "sfa_attn_bwd_workspace_bytes", "sfa_attn_bwd", "sfa_attn_fwd_fused_q", "sfa_attn_fwd_blocksel", "sfa_dist_kv_plan",
           "sfa_dist_zigzag_chunk", "sfa_dist_head_shard")


def _check(code: int, where: str):
    if code != 0:
        raise SfaError(code, where)


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return SFA_BF16
    if t.dtype == torch.float32:
        return SFA_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _dev(*ts):
    for t in ts:
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("tensors must be contiguous CUDA tensors")


def _expect(t, shape, dtype, name):
    """The C ABI sees raw pointers only: every shape / dtype it relies on is checked here."""
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")


def _check_codes(q_idx, q_val, k_idx, k_val, v, d):
    """Codes and V of one attention call: q [B,H,n_q,k], k [B,H_kv,n_kv,k], v [B,H_kv,n_kv,d_v]; the value
    tensors share v's dtype (bf16 or fp32), indices are u8."""
    _dt(v)
    if q_idx.dim() != 4 or k_idx.dim() != 4 or v.dim() != 4:
        raise ValueError("q_idx, k_idx and v must be 4-D ([B, heads, n, .])")
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    if not 1 <= k <= d:
        raise ValueError(f"code size k={k} must lie in [1, d={d}]")
    _expect(q_idx, (B, H, n_q, k), torch.uint8, "q_idx")
    _expect(q_val, (B, H, n_q, k), v.dtype, "q_val")
    _expect(k_idx, (B, H_kv, n_kv, k), torch.uint8, "k_idx")
    _expect(k_val, (B, H_kv, n_kv, k), v.dtype, "k_val")
    _expect(v, (B, H_kv, n_kv, v.shape[-1]), v.dtype, "v")
    if H_kv < 1 or H % H_kv:
        raise ValueError(f"H={H} must be a multiple of H_kv={H_kv}")


def _check_out(out, B, H, n_q, d_v, dtype):
    o, lse = out
    _dev(o, lse)
    _expect(o, (B, H, n_q, d_v), dtype, "out[0] (O)")
    _expect(lse, (B, H, n_q), torch.float32, "out[1] (LSE)")


def _check_ws(ws, nbytes):
    _dev(ws)
    if ws.dtype != torch.uint8 or ws.numel() < nbytes:
        raise ValueError(f"workspace must be a uint8 tensor of >= {nbytes} bytes")


def make_desc(*, B, H, H_kv, d, k, d_v, n_q, n_kv, q_pos0=0, causal=True, scale=None, dtype=SFA_BF16,
              kernel=KERNEL_AUTO, edges_only=False, window=0) -> AttnDesc:
    """edges_only: reading A1/R2 (include/sfa.h) -- only pairs whose supports intersect.
    window > 0: causal sliding window (N4) -- key j also needs j > q_pos0 + i - window."""
    if scale is None:
        scale = 1.0 / math.sqrt(d)  # P:L99, reading A5
    return AttnDesc(B, H, H_kv, d, k, d_v, n_q, n_kv, q_pos0, int(bool(causal)), scale, dtype, kernel,
                    int(bool(edges_only)), int(window))


def topk_codes(x: torch.Tensor, k: int, status: torch.Tensor | None = None):
    """Stage 1: x [..., d] -> (idx u8 [..., k], val [..., k])."""
    _dev(x)
    d = x.shape[-1]
    rows = x.numel() // d
    idx = torch.empty(x.shape[:-1] + (k,), dtype=torch.uint8, device=x.device)
    val = torch.empty(x.shape[:-1] + (k,), dtype=x.dtype, device=x.device)
    _check(lib().sfa_topk_codes(_p(x), _dt(x), rows, d, d, k, _p(idx), _p(val), _p(status), _stream()),
           "sfa_topk_codes")
    return idx, val


def topk_codes_qk(q: torch.Tensor, kx: torch.Tensor, k: int, status: torch.Tensor | None = None):
    """Stage 1 on Q and on K in one launch (sfa_topk_codes_qk): the same codes as two topk_codes calls."""
    _dev(q)
    _dev(kx)
    if q.dtype != kx.dtype or q.shape[-1] != kx.shape[-1] or not q.is_contiguous() or not kx.is_contiguous():
        raise ValueError("topk_codes_qk: q and k need the same dtype and d, contiguous")
    d = q.shape[-1]
    out = []
    for x in (q, kx):
        out.append((torch.empty(x.shape[:-1] + (k,), dtype=torch.uint8, device=x.device),
                    torch.empty(x.shape[:-1] + (k,), dtype=x.dtype, device=x.device)))
    (qi, qv), (ki, kv) = out
    _check(lib().sfa_topk_codes_qk(_p(q), q.numel() // d, d, _p(qi), _p(qv), _p(kx), kx.numel() // d, d, _p(ki),
                                   _p(kv), _dt(q), d, k, _p(status), _stream()), "sfa_topk_codes_qk")
    return qi, qv, ki, kv


def _desc_from_codes(q_idx, k_idx, v, d, causal, scale, q_pos0, kernel, dtype, edges_only=False, window=0):
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    return make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k, d_v=v.shape[-1], n_q=n_q, n_kv=n_kv, q_pos0=q_pos0,
                     causal=causal, scale=scale, dtype=dtype, kernel=kernel, edges_only=edges_only, window=window)


def workspace_bytes(desc: AttnDesc) -> int:
    return int(lib().sfa_attn_workspace_bytes(ctypes.byref(desc)))


def key_tile(desc: AttnDesc) -> int:
    return int(lib().sfa_key_tile(ctypes.byref(desc)))


def attn_fwd(q_idx, q_val, k_idx, k_val, v, *, d, causal=True, scale=None, q_pos0=0, kernel=KERNEL_AUTO,
             workspace=None, out=None, edges_only=False, window=0):
    """Stage 2: (O, LSE) = FlashSFA forward over the codes (bucketing + attention kernels).
    edges_only: reading A1/R2 -- only the pairs whose supports intersect enter the softmax."""
    _dev(q_idx, q_val, k_idx, k_val, v)
    _check_codes(q_idx, q_val, k_idx, k_val, v, d)
    desc = _desc_from_codes(q_idx, k_idx, v, d, causal, scale, q_pos0, kernel, _dt(v), edges_only, window)
    B, H, n_q, _ = q_idx.shape
    nb = workspace_bytes(desc)
    if workspace is None:
        workspace = torch.empty(max(nb, 16), dtype=torch.uint8, device=v.device)
    _check_ws(workspace, nb)
    if out is not None:
        _check_out(out, B, H, n_q, v.shape[-1], v.dtype)
    if out is None:
        o = torch.empty((B, H, n_q, v.shape[-1]), dtype=v.dtype, device=v.device)
        lse = torch.empty((B, H, n_q), dtype=torch.float32, device=v.device)
    else:
        o, lse = out
    _check(lib().sfa_attn_fwd(ctypes.byref(desc), _p(q_idx), _p(q_val), _p(k_idx), _p(k_val), _p(v), _p(o),
                              _p(lse), _p(workspace), workspace.numel(), _stream()), "sfa_attn_fwd")
    return o, lse


def attn_fwd_blocksel(q_idx, q_val, k_idx, k_val, v, block_sel, *, d, causal=True, scale=None, q_pos0=0,
                      workspace=None):
    """Stage 2 composed with NSA-style block selection (sfa_attn_fwd_blocksel):
    block_sel int32 [B, H_kv, ceil(n_q/128), max_sel], ascending key-block indices padded with -1."""
    _dev(q_idx, q_val, k_idx, k_val, v, block_sel)
    _check_codes(q_idx, q_val, k_idx, k_val, v, d)
    B, H, n_q, _ = q_idx.shape
    H_kv = k_idx.shape[1]
    if block_sel.dtype != torch.int32 or block_sel.dim() != 4 or not block_sel.is_contiguous() or \
            tuple(block_sel.shape[:3]) != (B, H_kv, (n_q + 127) // 128):
        raise ValueError("block_sel: contiguous int32 [B, H_kv, ceil(n_q/128), max_sel]")
    # block selection runs on SM100_OT (named explicitly: AUTO would pick SM100 for d_v = 64)
    desc = _desc_from_codes(q_idx, k_idx, v, d, causal, scale, q_pos0, KERNEL_SM100_OT, _dt(v))
    nb = workspace_bytes(desc)
    if workspace is None:
        workspace = torch.empty(max(nb, 16), dtype=torch.uint8, device=v.device)
    _check_ws(workspace, nb)
    o = torch.empty((B, H, n_q, v.shape[-1]), dtype=v.dtype, device=v.device)
    lse = torch.empty((B, H, n_q), dtype=torch.float32, device=v.device)
    _check(lib().sfa_attn_fwd_blocksel(ctypes.byref(desc), _p(q_idx), _p(q_val), _p(k_idx), _p(k_val), _p(v),
                                       _p(block_sel), int(block_sel.shape[3]), _p(o), _p(lse), _p(workspace),
                                       workspace.numel(), _stream()), "sfa_attn_fwd_blocksel")
    return o, lse


def attn_fwd_fused_q(q, k_idx, k_val, v, *, causal=True, scale=None, q_pos0=0, kernel=KERNEL_AUTO, codes_out=True,
                     status=None):
    """Steps 1 (on Q) to 8 in one kernel (include/sfa.h sfa_attn_fwd_fused_q): dense bf16 q, key codes and
    v -> (O, LSE, q_idx, q_val); the codes are None when codes_out is False."""
    _dev(q, k_idx, k_val, v)
    B, H, n_q, d = q.shape
    _, H_kv, n_kv, k = k_idx.shape
    if q.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
        raise TypeError("the fused path takes bf16 q and v")
    _expect(k_val, (B, H_kv, n_kv, k), v.dtype, "k_val")
    _expect(k_idx, (B, H_kv, n_kv, k), torch.uint8, "k_idx")
    _expect(v, (B, H_kv, n_kv, v.shape[-1]), v.dtype, "v")
    desc = make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k, d_v=v.shape[-1], n_q=n_q, n_kv=n_kv, q_pos0=q_pos0,
                     causal=causal, scale=scale, dtype=_dt(v), kernel=kernel)
    ws = torch.empty(max(workspace_bytes(desc), 16), dtype=torch.uint8, device=v.device)
    _check(lib().sfa_attn_prepare(ctypes.byref(desc), _p(k_idx), _p(k_val), _p(v), _p(ws), ws.numel(), _stream()),
           "sfa_attn_prepare")
    o = torch.empty((B, H, n_q, v.shape[-1]), dtype=v.dtype, device=v.device)
    lse = torch.empty((B, H, n_q), dtype=torch.float32, device=v.device)
    qi = torch.empty((B, H, n_q, k), dtype=torch.uint8, device=v.device) if codes_out else None
    qv = torch.empty((B, H, n_q, k), dtype=q.dtype, device=v.device) if codes_out else None
    _check(lib().sfa_attn_fwd_fused_q(ctypes.byref(desc), _p(q), _p(k_idx), _p(k_val), _p(v), _p(o), _p(lse), _p(qi),
                                      _p(qv), _p(status), _p(ws), ws.numel(), _stream()), "sfa_attn_fwd_fused_q")
    return o, lse, qi, qv


def bucket_keys(k_idx, k_val, *, d, n_q=1, H=None, d_v=64, causal=True, workspace=None):
    """Step 3 alone: the key-tile feature buckets (uint8 workspace tensor)."""
    _dev(k_idx, k_val)
    B, H_kv, n_kv, k = k_idx.shape
    _expect(k_val, (B, H_kv, n_kv, k), k_val.dtype, "k_val")
    _dt(k_val)
    desc = make_desc(B=B, H=H or H_kv, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=n_q, n_kv=n_kv, causal=causal,
                     dtype=_dt(k_val), kernel=KERNEL_SIMT)  # buckets feed the CUDA-core kernel
    nb = workspace_bytes(desc)
    if workspace is None:
        workspace = torch.zeros(max(nb, 16), dtype=torch.uint8, device=k_idx.device)
    _check(lib().sfa_bucket_keys(ctypes.byref(desc), _p(k_idx), _p(k_val), _p(workspace), workspace.numel(),
                                 _stream()), "sfa_bucket_keys")
    return workspace, desc


def attn_fwd_bucketed(desc: AttnDesc, q_idx, q_val, v, workspace, out=None):
    _dev(q_idx, q_val, v, workspace)
    _expect(q_idx, (desc.B, desc.H, desc.n_q, desc.k), torch.uint8, "q_idx")
    _expect(q_val, (desc.B, desc.H, desc.n_q, desc.k), v.dtype, "q_val")
    _expect(v, (desc.B, desc.H_kv, desc.n_kv, desc.d_v), v.dtype, "v")
    if _dt(v) != desc.dtype:
        raise TypeError("v's dtype differs from the desc the buckets were built for")
    _check_ws(workspace, workspace_bytes(desc))
    if out is not None:
        _check_out(out, desc.B, desc.H, desc.n_q, desc.d_v, v.dtype)
    if out is None:
        o = torch.empty((desc.B, desc.H, desc.n_q, desc.d_v), dtype=v.dtype, device=v.device)
        lse = torch.empty((desc.B, desc.H, desc.n_q), dtype=torch.float32, device=v.device)
    else:
        o, lse = out
    _check(lib().sfa_attn_fwd_bucketed(ctypes.byref(desc), _p(q_idx), _p(q_val), _p(v), _p(o), _p(lse),
                                       _p(workspace), workspace.numel(), _stream()), "sfa_attn_fwd_bucketed")
    return o, lse


def debug_sm100_scores(q_idx, q_val, k_idx, k_val, v, *, d, causal=True, scale=None, kernel=KERNEL_SM100):
    """Diagnostic: run the sm_100a kernel and return (O, LSE, S) where S [128, 128] fp32 is the raw
    score tile Q~ K~^T of the first key tile of work item 0 / query tile 0 (include/sfa.h)."""
    _dev(q_idx, q_val, k_idx, k_val, v)
    _check_codes(q_idx, q_val, k_idx, k_val, v, d)
    desc = _desc_from_codes(q_idx, k_idx, v, d, causal, scale, 0, kernel, _dt(v))
    B, H, n_q, _ = q_idx.shape
    o = torch.empty((B, H, n_q, v.shape[-1]), dtype=v.dtype, device=v.device)
    lse = torch.empty((B, H, n_q), dtype=torch.float32, device=v.device)
    # score tile [128 x 128] fp32, then room for the debug-build timeline (SFA_TIMELINE)
    S = torch.full((128 * 128 + 2 * 8192,), float("nan"), dtype=torch.float32, device=v.device)
    S[128 * 128:] = 0
    ws = torch.empty(max(workspace_bytes(desc), 16), dtype=torch.uint8, device=v.device)
    _check(lib().sfa_debug_sm100_scores(ctypes.byref(desc), _p(q_idx), _p(q_val), _p(k_idx), _p(k_val), _p(v),
                                        _p(o), _p(lse), _p(ws), ws.numel(), _p(S), _stream()),
           "sfa_debug_sm100_scores")
    return o, lse, S[:128 * 128].view(128, 128), S[128 * 128:]


def attn_bwd(q_idx, q_val, k_idx, k_val, v, o, lse, dO, *, d, causal=True, scale=None, q_pos0=0, workspace=None,
             out=None):
    """Backward with the straight-through rule (include/sfa.h sfa_attn_bwd): returns fp32
    (dq_val [B,H,n_q,k], dk_val [B,H_kv,n_kv,k], dv [B,H_kv,n_kv,d_v])."""
    _dev(q_idx, q_val, k_idx, k_val, v, o, lse, dO)
    _check_codes(q_idx, q_val, k_idx, k_val, v, d)
    desc = _desc_from_codes(q_idx, k_idx, v, d, causal, scale, q_pos0, KERNEL_AUTO, _dt(v))
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    d_v = v.shape[-1]
    if v.dtype != torch.bfloat16:
        raise TypeError("the backward takes bf16 codes, v, o and dO")
    _check_out((o, lse), B, H, n_q, d_v, v.dtype)
    _expect(dO, (B, H, n_q, d_v), torch.bfloat16, "dO")
    nb = int(lib().sfa_attn_bwd_workspace_bytes(ctypes.byref(desc)))
    if workspace is None:
        workspace = torch.empty(max(nb, 16), dtype=torch.uint8, device=v.device)
    _check_ws(workspace, nb)
    if out is not None:
        _dev(*out)
        _expect(out[0], (B, H, n_q, k), torch.float32, "dq_val")
        _expect(out[1], (B, H_kv, n_kv, k), torch.float32, "dk_val")
        _expect(out[2], (B, H_kv, n_kv, d_v), torch.float32, "dv")
    if out is None:
        f32 = dict(dtype=torch.float32, device=v.device)
        out = (torch.empty((B, H, n_q, k), **f32), torch.empty((B, H_kv, n_kv, k), **f32),
               torch.empty((B, H_kv, n_kv, v.shape[-1]), **f32))
    dq, dk, dv = out
    _check(lib().sfa_attn_bwd(ctypes.byref(desc), _p(q_idx), _p(q_val), _p(k_idx), _p(k_val), _p(v), _p(o), _p(lse),
                              _p(dO), _p(dq), _p(dk), _p(dv), _p(workspace), workspace.numel(), _stream()),
           "sfa_attn_bwd")
    return dq, dk, dv


def scratch_bytes(desc: AttnDesc) -> int:
    return int(lib().sfa_forward_scratch_bytes(ctypes.byref(desc)))


def forward(q, k, v, *, k_code, causal=True, scale=None, q_pos0=0, kernel=KERNEL_AUTO, scratch=None, out=None,
            edges_only=False, window=0):
    """The whole hot path (stage 1 on Q and K, then stage 2): dense q, k, v -> (O, LSE)."""
    _dev(q, k, v)
    B, H, n_q, d = q.shape
    _, H_kv, n_kv, _ = k.shape
    _dt(v)
    _expect(q, (B, H, n_q, d), v.dtype, "q")
    _expect(k, (B, H_kv, n_kv, d), v.dtype, "k")
    _expect(v, (B, H_kv, n_kv, v.shape[-1]), v.dtype, "v")
    desc = make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k_code, d_v=v.shape[-1], n_q=n_q, n_kv=n_kv, q_pos0=q_pos0,
                     causal=causal, scale=scale, dtype=_dt(v), kernel=kernel, edges_only=edges_only, window=window)
    nb = scratch_bytes(desc)
    if scratch is None:
        scratch = torch.empty(max(nb, 16), dtype=torch.uint8, device=v.device)
    _check_ws(scratch, nb)
    if out is not None:
        _check_out(out, B, H, n_q, v.shape[-1], v.dtype)
    if out is None:
        o = torch.empty((B, H, n_q, v.shape[-1]), dtype=v.dtype, device=v.device)
        lse = torch.empty((B, H, n_q), dtype=torch.float32, device=v.device)
    else:
        o, lse = out
    _check(lib().sfa_forward(ctypes.byref(desc), _p(q), _p(k), _p(v), _p(o), _p(lse), _p(scratch),
                             scratch.numel(), _stream()), "sfa_forward")
    return o, lse


def forward_host(desc: AttnDesc, q_host, k_host, v_host, o_host, lse_host, dev_bufs, scratch, chunks=0):
    """End to end from host (pinned) tensors: H2D copies, the hot path, D2H copies, stream sync.
    chunks > 0: the pipelined variant (copies of one chunk overlap the kernels of the others)."""
    qd, kd, vd, od, ld = dev_bufs
    if chunks:
        _check(lib().sfa_forward_host_pipelined(ctypes.byref(desc), _p(q_host), _p(k_host), _p(v_host), _p(o_host),
                                                _p(lse_host), _p(qd), _p(kd), _p(vd), _p(od), _p(ld), _p(scratch),
                                                scratch.numel(), chunks, _stream()), "sfa_forward_host_pipelined")
        return
    _check(lib().sfa_forward_host(ctypes.byref(desc), _p(q_host), _p(k_host), _p(v_host), _p(o_host),
                                  _p(lse_host), _p(qd), _p(kd), _p(vd), _p(od), _p(ld), _p(scratch),
                                  scratch.numel(), _stream()), "sfa_forward_host")


def gen_fill(t: torch.Tensor, seed: int, tensor_id: int, variant: int = GEN_IID, offset: int = 0, skew_span: int = 3):
    """Fill a CUDA tensor [..., n, d] with the seeded generator (bit-identical to inputs.py)."""
    _dev(t)
    n = t.shape[-2] if t.dim() >= 2 else 1
    d = t.shape[-1]
    _check(lib().sfa_gen_fill(_p(t), _dt(t), t.numel(), offset, seed, tensor_id, variant, n, d, skew_span,
                              _stream()), "sfa_gen_fill")
    return t


def device_supported() -> bool:
    return bool(lib().sfa_device_supported())
