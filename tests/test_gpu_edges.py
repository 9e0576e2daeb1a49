"""GPU parity of the edge-only semantics (reading A1/R2) against the oracle.

R2 keeps a pair only if the supports share a feature index.  It runs in the tensor-core kernel
SM100_OT (bf16, d_v = 128: key support bitmasks from edges.cu, per-pair test in the softmax) and
in the CUDA-core kernel SIMT (the scatter marks the pairs it touches).  Both are compared with
oracle.attn_fwd(edges_only=True), which is pinned in tests/test_oracle_edges.py.
"""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu

OT, SIMT, AUTO = 6, 1, 0


def gpu_attn(lib, qi, qv, ki, kv, v, dtype, d, **kw):
    import torch
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, dtype), to_torch(ki, "u8"), to_torch(kv, dtype),
                          to_torch(v, dtype), d=d, edges_only=True, **kw)
    torch.cuda.synchronize()
    return from_torch(o), from_torch(lse)


def run_case(lib, seed, B, H, H_kv, n, d, d_v, k, dtype, kernel, causal=True, n_kv=None, q_pos0=0,
             variant="iid"):
    q, kx, v = host_qkv(seed, B, H, H_kv, n, d, d_v, dtype, n_kv=n_kv, variant=variant)
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, q_pos0=q_pos0, edges_only=True)
    o, lse = gpu_attn(lib, qi, qv, ki, kv, v, dtype, d, causal=causal, kernel=kernel, q_pos0=q_pos0)
    return assert_attn_close(o, lse, o_ref, l_ref, dtype)


@pytest.mark.parametrize("kernel", [OT, SIMT])
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("shape", [
    (1, 4, 2, 300, 128, 128, 4),     # GQA, ragged n, k = 4: most pairs are non-edges (12 % overlap)
    (1, 2, 1, 385, 128, 128, 16),    # 3 tiles + 1
    (2, 2, 2, 257, 64, 128, 8),      # d = 64
    (2, 3, 3, 300, 64, 64, 8),       # GPT-2 head shape: d = d_v = 64 (OT over the zero-padded V copy)
    (1, 2, 2, 1, 128, 128, 2),       # single token
    (1, 2, 1, 200, 128, 128, 1),     # k = 1: edge iff the same single feature (many empty rows)
])
def test_parity(lib, kernel, causal, shape):
    B, H, H_kv, n, d, d_v, k = shape
    run_case(lib, 51, B, H, H_kv, n, d, d_v, k, "bf16", kernel, causal=causal)


def test_fp32_simt(lib):
    run_case(lib, 52, 1, 1, 1, 256, 64, 64, 8, "f32", AUTO)     # tiny config shape, fp32 -> SIMT
    run_case(lib, 53, 1, 2, 1, 130, 128, 64, 2, "f32", SIMT, causal=False)


@pytest.mark.parametrize("kernel", [OT, SIMT])
def test_q_pos0_and_skewed(lib, kernel):
    run_case(lib, 54, 1, 2, 2, 140, 128, 128, 8, "bf16", kernel, n_kv=400, q_pos0=260)
    run_case(lib, 55, 1, 2, 1, 300, 128, 128, 16, "bf16", kernel, variant="skewed")


@pytest.mark.parametrize("kernel", [OT, SIMT])
def test_k_equals_d_equals_r1(lib, kernel):
    """k = d: every pair is an edge, so R2 must reproduce the R1 result bit for bit."""
    import torch
    q, kx, v = host_qkv(56, 1, 2, 1, 200, 64, 128, "bf16")
    qi, qv = oracle_codes(q, 64)
    ki, kv = oracle_codes(kx, 64)
    args = [to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"), to_torch(v, "bf16")]
    o2, l2 = lib.attn_fwd(*args, d=64, kernel=kernel, edges_only=True)
    o1, l1 = lib.attn_fwd(*args, d=64, kernel=kernel, edges_only=False)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("kernel", [OT, SIMT])
def test_disjoint_supports_no_edges(lib, kernel):
    """No pair shares a feature: every row has O = 0 and LSE = -inf (R1 would give the prefix mean)."""
    n, d, k, d_v = 300, 128, 16, 128
    qi = np.tile(np.arange(k, dtype=np.uint8), (1, 1, n, 1))
    ki = np.tile(np.arange(64, 64 + k, dtype=np.uint8), (1, 1, n, 1))
    qv = inputs.gen(1, 1, (1, 1, n, k), "bf16")
    kv = inputs.gen(1, 2, (1, 1, n, k), "bf16")
    v = inputs.gen(1, 3, (1, 1, n, d_v), "bf16")
    o, lse = gpu_attn(lib, qi, qv, ki, kv, v, "bf16", d, kernel=kernel)
    assert np.all(inputs.bf16_bits_to_f32(o) == 0.0) and np.all(np.isneginf(lse))


def test_unsupported_kernels(lib):
    q, kx, v = host_qkv(57, 1, 2, 1, 64, 128, 128, "bf16")
    qi, qv = oracle_codes(q, 8)
    ki, kv = oracle_codes(kx, 8)
    for kern in (2, 3, 4, 5):  # SM100, PAIR, WIDE, DECODE: R2 not built there
        with pytest.raises(lib.SfaError):
            gpu_attn(lib, qi, qv, ki, kv, v, "bf16", 128, kernel=kern)


def test_qwen3_sampled_rows(lib):
    """BASELINE Qwen3 shape at n = 32K with R2 (AUTO -> SM100_OT): sampled rows vs the oracle."""
    import torch
    B, H, H_kv, n, d, d_v, k = 1, 32, 8, 32768, 128, 128, 16
    q, kx, v = host_qkv(21, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o, lse = gpu_attn(lib, qi, qv, ki, kv, v, "bf16", d)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([[0, 1, 127, 128, n - 1, n * H - 1],
                                     rng.integers(0, n * H, 120)])).astype(np.int64)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, rows=rows, edges_only=True)
    assert_attn_close(o.reshape(-1, d_v)[rows], lse.reshape(-1)[rows], o_ref, l_ref, "bf16")
