"""fp64 CPU oracle for Sparse Feature Attention -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2603_22300_b200``) never imports it, and the two share no code.

``build()`` compiles ``sfa_oracle.c`` with gcc into ``liboracle.so`` next to it;
the wrappers below only marshal numpy arrays (see sfa_oracle.c for the definitions
and the PAPER.md passages each function follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sfa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

F32, BF16, F64 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2, no fast-math) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math", "-ffp-contract=off",
             "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, I, L, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        _lib.ref_topk_codes.argtypes = [P, I, L, I, I, P, P]
        _lib.ref_topk_codes.restype = I
        _lib.ref_attn_fwd.argtypes = [I, I, I, I, I, I, L, L, L, I, D, I, P, P, P, P, P, P, L, P, P, I]
        _lib.ref_attn_fwd_ex.argtypes = [I, I, I, I, I, I, L, L, L, I, D, I, P, P, P, P, P, P, L, P, P, I, I, L, P, I]
        _lib.ref_attn_fwd.restype = I
        _lib.ref_scores_row.argtypes = [I, I, I, I, I, L, L, L, I, D, I, P, P, P, P, L, P]
        _lib.ref_scores_row.restype = I
        _lib.ref_attn_bwd.argtypes = [I, I, I, I, I, I, L, L, L, I, D, I, P, P, P, P, P, P, P, P, P, P, P, P, I]
        _lib.ref_attn_bwd.restype = I
        _lib.ref_edge_count.argtypes = [I, I, I, I, L, L, L, I, P, P]
        _lib.ref_edge_count.restype = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__({1: "invalid-argument", 2: "invalid-input"}.get(code, f"status {code}"))
        self.code = code


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _dtype_code(vals: np.ndarray) -> int:
    if vals.dtype == np.float32:
        return F32
    if vals.dtype == np.uint16:  # bf16 bit patterns
        return BF16
    if vals.dtype == np.float64:  # finite-difference pins of attn_bwd only
        return F64
    raise TypeError(f"oracle takes float32, float64 or uint16 (bf16 bits), got {vals.dtype}")


def topk_codes(x: np.ndarray, k: int):
    """x: [rows, d] float32 or uint16 (bf16 bits).  Returns (idx u8 [rows,k], val [rows,k])."""
    x = np.ascontiguousarray(x)
    rows, d = x.shape
    idx = np.zeros((rows, k), np.uint8)
    val = np.zeros((rows, k), x.dtype)
    st = _load().ref_topk_codes(_ptr(x), _dtype_code(x), rows, d, k, _ptr(idx), _ptr(val))
    if st:
        raise OracleError(st)
    return idx, val


def attn_fwd(q_idx, q_val, k_idx, k_val, v, *, d, causal=True, scale=None, q_pos0=0, rows=None,
             threads=None, edges_only=False, window=0, block_sel=None):
    """Plain fp64 SFA attention forward on the decompressed codes (sfa_oracle.c ref_attn_fwd).

    q_idx/q_val [B,H,n_q,k]; k_idx/k_val [B,H_kv,n_kv,k]; v [B,H_kv,n_kv,d_v] (vals and v share a
    dtype: float32 or uint16 bf16 bits).  ``d`` is the full head dimension.  ``rows``: optional
    int64 flat row ids into [B,H,n_q].  ``edges_only``: reading A1/R2 --
    only pairs whose supports intersect enter the softmax.  ``window`` > 0: causal sliding window (SURVEY
    8(f) N4), key j also needs j > q_pos0 + i - window.  ``block_sel`` int32 [B,H_kv,ceil(n_q/128),max_sel]
    (NSA-style block selection): key j also needs its block j // 128 in the list of the
    row's query block i // 128 (entries < 0 are padding).  Returns fp64 (o, lse), shaped [B,H,n_q,(d_v)]
    or [nsel,(d_v)].
    """
    q_idx = np.ascontiguousarray(q_idx); q_val = np.ascontiguousarray(q_val)
    k_idx = np.ascontiguousarray(k_idx); k_val = np.ascontiguousarray(k_val)
    v = np.ascontiguousarray(v)
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    d_v = v.shape[-1]
    dt = _dtype_code(q_val)
    assert _dtype_code(k_val) == dt and _dtype_code(v) == dt
    if scale is None:
        scale = 1.0 / np.sqrt(d)  # A5: 1/sqrt(d), d the full head dimension
    if rows is None:
        sel, nsel = None, B * H * n_q
        o = np.zeros((B, H, n_q, d_v), np.float64)
        lse = np.zeros((B, H, n_q), np.float64)
    else:
        sel = np.ascontiguousarray(rows, dtype=np.int64)
        nsel = sel.size
        o = np.zeros((nsel, d_v), np.float64)
        lse = np.zeros((nsel,), np.float64)
    threads = threads or os.cpu_count() or 1
    bs, max_sel = None, 0
    if block_sel is not None:
        bs = np.ascontiguousarray(block_sel, dtype=np.int32)
        assert bs.shape[:3] == (B, H_kv, (n_q + 127) // 128), bs.shape
        max_sel = bs.shape[3]
    st = _load().ref_attn_fwd_ex(B, H, H_kv, d, k, d_v, n_q, n_kv, q_pos0, int(bool(causal)), float(scale), dt,
                                 _ptr(q_idx), _ptr(q_val), _ptr(k_idx), _ptr(k_val), _ptr(v), _ptr(sel), nsel,
                                 _ptr(o), _ptr(lse), int(threads), int(bool(edges_only)), int(window), _ptr(bs),
                                 int(max_sel))
    if st:
        raise OracleError(st)
    return o, lse


def attn_bwd(q_idx, q_val, k_idx, k_val, v, dO, *, d, causal=True, scale=None, q_pos0=0, bounds=False,
             threads=None):
    """Plain fp64 SFA backward with the straight-through rule (sfa_oracle.c ref_attn_bwd).

    Inputs as attn_fwd plus dO [B,H,n_q,d_v] (any float dtype, used as fp64).  Returns fp64
    (dq_val [B,H,n_q,k], dk_val [B,H_kv,n_kv,k], dv [B,H_kv,n_kv,d_v]) -- the gradients with respect
    to the code values and V -- and, with ``bounds=True``, their componentwise magnitude sums
    (bq, bk, bv) used by the GPU tolerance (reading A24)."""
    q_idx = np.ascontiguousarray(q_idx); q_val = np.ascontiguousarray(q_val)
    k_idx = np.ascontiguousarray(k_idx); k_val = np.ascontiguousarray(k_val)
    v = np.ascontiguousarray(v)
    dO = np.ascontiguousarray(dO, dtype=np.float64)
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    d_v = v.shape[-1]
    dt = _dtype_code(q_val)
    assert _dtype_code(k_val) == dt and _dtype_code(v) == dt
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    dq = np.zeros((B, H, n_q, k)); dk = np.zeros((B, H_kv, n_kv, k)); dv = np.zeros((B, H_kv, n_kv, d_v))
    bq = np.zeros_like(dq) if bounds else None
    bk = np.zeros_like(dk) if bounds else None
    bv = np.zeros_like(dv) if bounds else None
    threads = threads or os.cpu_count() or 1
    st = _load().ref_attn_bwd(B, H, H_kv, d, k, d_v, n_q, n_kv, q_pos0, int(bool(causal)), float(scale), dt,
                              _ptr(q_idx), _ptr(q_val), _ptr(k_idx), _ptr(k_val), _ptr(v), _ptr(dO), _ptr(dq),
                              _ptr(dk), _ptr(dv), _ptr(bq), _ptr(bk), _ptr(bv), int(threads))
    if st:
        raise OracleError(st)
    return (dq, dk, dv, bq, bk, bv) if bounds else (dq, dk, dv)


def scores_row(q_idx, q_val, k_idx, k_val, flat_row, *, d, causal=True, scale=None, q_pos0=0):
    q_idx = np.ascontiguousarray(q_idx); q_val = np.ascontiguousarray(q_val)
    k_idx = np.ascontiguousarray(k_idx); k_val = np.ascontiguousarray(k_val)
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    s = np.zeros((n_kv,), np.float64)
    st = _load().ref_scores_row(B, H, H_kv, d, k, n_q, n_kv, q_pos0, int(bool(causal)), float(scale),
                                _dtype_code(q_val), _ptr(q_idx), _ptr(q_val), _ptr(k_idx), _ptr(k_val),
                                int(flat_row), _ptr(s))
    if st:
        raise OracleError(st)
    return s


def edge_count(q_idx, k_idx, *, causal=True, q_pos0=0) -> int:
    q_idx = np.ascontiguousarray(q_idx); k_idx = np.ascontiguousarray(k_idx)
    B, H, n_q, k = q_idx.shape
    _, H_kv, n_kv, _ = k_idx.shape
    return int(_load().ref_edge_count(B, H, H_kv, k, n_q, n_kv, q_pos0, int(bool(causal)),
                                      _ptr(q_idx), _ptr(k_idx)))
