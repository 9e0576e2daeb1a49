"""GPU checks specific to the sm_100a tensor-core kernel (attn_sm100.cu).

The score contraction S = Q~ K~^T is checked on its own through the diagnostic hook
sfa_debug_sm100_scores (include/sfa.h) against the exact overlap sums computed on the host
from the oracle's codes (s_ij / scale = sum over the shared support); then the whole
kernel against the oracle on shapes that exercise the work-item pairing (GQA head pairs,
consecutive query blocks for MHA / odd groups, an empty second tile), ragged tails and k = d.
"""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu


def dense_from_codes(idx, val_bits, d):
    """Decompress k-sparse codes [rows, k] into [rows, d] float64 (zeros off the support)."""
    rows, k = idx.shape
    out = np.zeros((rows, d), np.float64)
    vals = inputs.bf16_bits_to_f32(val_bits).astype(np.float64)
    np.put_along_axis(out, idx.astype(np.int64), vals, axis=1)
    return out


@pytest.mark.parametrize("d,k", [(128, 16), (64, 8), (128, 128), (128, 3), (64, 4)])
def test_score_tile_is_exact_overlap_sum(lib, d, k):
    import torch
    B, H, H_kv, n, d_v = 1, 2, 1, 128, 64
    q, kx, v = host_qkv(101 + k, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o, lse, S, _ = lib.debug_sm100_scores(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"),
                                       to_torch(kv, "bf16"), to_torch(v, "bf16"), d=d)
    torch.cuda.synchronize()
    S = S.cpu().numpy().astype(np.float64)
    Qd = dense_from_codes(qi[0, 0], qv[0, 0], d)
    Kd = dense_from_codes(ki[0, 0], kv[0, 0], d)
    ref = Qd @ Kd.T
    # bf16 x bf16 products are exact in fp32; only the fp32 summation order differs
    np.testing.assert_allclose(S, ref, rtol=1e-6, atol=1e-6 * np.abs(ref).max())


@pytest.mark.parametrize("shape", [
    (1, 4, 2, 256, 128, 128, 16),   # GQA pairs of heads, 2 q blocks
    (1, 3, 1, 256, 128, 128, 16),   # odd group (R=3): consecutive q-block pairs
    (2, 2, 2, 384, 128, 64, 16),    # MHA, 3 q blocks -> last pair has an empty second tile
    (1, 2, 2, 100, 64, 64, 8),      # single partial tile
    (1, 8, 8, 1000, 64, 64, 8),     # GPT-2-like heads, ragged
    (1, 2, 1, 515, 128, 128, 32),
])
@pytest.mark.parametrize("causal", [True, False])
def test_sm100_against_oracle(lib, shape, causal):
    import torch
    B, H, H_kv, n, d, d_v, k = shape
    q, kx, v = host_qkv(55, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                          to_torch(v, "bf16"), d=d, causal=causal, kernel=lib.KERNEL_SM100)
    torch.cuda.synchronize()
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")


def test_peaked_rows_trigger_rescale(lib):
    """Large logits (lattice values x 4) make the running max jump by more than 2^8 between key
    tiles, exercising the lazy O rescale in TMEM; still within tolerance of the oracle."""
    import torch
    B, H, H_kv, n, d, d_v, k = 1, 2, 1, 640, 128, 128, 16
    q, kx, v = host_qkv(8, B, H, H_kv, n, d, d_v, "bf16", variant="lattice")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, scale=0.5)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                          to_torch(v, "bf16"), d=d, scale=0.5, kernel=lib.KERNEL_SM100)
    torch.cuda.synchronize()
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")


# ---------------------------------------------------------------------------------------------
# the other tensor-core kernels (attn_sm100_ot.cu default, _pp / _oth ablations): same checks
# ---------------------------------------------------------------------------------------------
VARIANTS = ["ot", "pp", "oth"]  # SFA_KERNEL_SM100_OT / _PP / _OTH


def _kern(lib, name):
    return {"ot": lib.KERNEL_SM100_OT, "pp": lib.KERNEL_SM100_PP, "oth": lib.KERNEL_SM100_OTH}[name]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("d,k", [(128, 16), (64, 8), (128, 128)])
def test_variant_score_tile_is_exact_overlap_sum(lib, variant, d, k):
    import torch
    B, H, H_kv, n, d_v = 1, 2, 1, 128, 128
    q, kx, v = host_qkv(201 + k, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o, lse, S, _ = lib.debug_sm100_scores(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"),
                                          to_torch(kv, "bf16"), to_torch(v, "bf16"), d=d,
                                          kernel=_kern(lib, variant))
    torch.cuda.synchronize()
    S = S.cpu().numpy().astype(np.float64)
    ref = dense_from_codes(qi[0, 0], qv[0, 0], d) @ dense_from_codes(ki[0, 0], kv[0, 0], d).T
    np.testing.assert_allclose(S, ref, rtol=1e-6, atol=1e-6 * np.abs(ref).max())


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("shape", [
    (1, 4, 2, 256, 128, 128, 16),   # GQA: pairs of heads
    (1, 3, 1, 384, 128, 128, 16),   # odd group: pairs of consecutive q blocks, last pair half empty
    (2, 2, 2, 300, 64, 128, 8),     # MHA, d = 64, ragged
    (1, 2, 1, 515, 128, 128, 32),
    (1, 2, 2, 1, 128, 128, 4),      # a single token
    (1, 2, 2, 700, 64, 64, 8),      # d_v = 64 (pp; ot over the zero-padded V copy)
    (1, 4, 2, 333, 128, 64, 16),    # d_v = 64, d = 128, GQA, ragged
])
@pytest.mark.parametrize("causal", [True, False])
def test_variant_against_oracle(lib, variant, shape, causal):
    import torch
    B, H, H_kv, n, d, d_v, k = shape
    if variant == "oth" and d_v != 128:
        pytest.skip("the oth kernel needs d_v = 128 (M of the transposed product)")
    q, kx, v = host_qkv(56, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                          to_torch(v, "bf16"), d=d, causal=causal, kernel=_kern(lib, variant))
    torch.cuda.synchronize()
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")


@pytest.mark.parametrize("variant", VARIANTS)
def test_variant_peaked_rows_and_q_pos0(lib, variant):
    import torch
    B, H, H_kv, n, d, d_v, k = 1, 2, 1, 640, 128, 128, 16
    q, kx, v = host_qkv(8, B, H, H_kv, n, d, d_v, "bf16", variant="lattice")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi[:, :, 200:], qv[:, :, 200:], ki, kv, v, d=d, scale=0.5, q_pos0=200)
    o, lse = lib.attn_fwd(to_torch(qi[:, :, 200:], "u8"), to_torch(qv[:, :, 200:], "bf16"), to_torch(ki, "u8"),
                          to_torch(kv, "bf16"), to_torch(v, "bf16"), d=d, scale=0.5, q_pos0=200,
                          kernel=_kern(lib, variant))
    torch.cuda.synchronize()
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")


def test_ot_gpt2_config_dv64(lib):
    """BASELINE configs[1] (B=8, H=12, n=1024, d=64, d_v=64, k=8, causal) on SM100_OT: d_v = 64 runs the
    d_v = 128 transposed P.V over V's zero-padded fp16 copy; every element against the oracle."""
    import torch
    B, H, H_kv, n, d, d_v, k = 8, 12, 12, 1024, 64, 64, 8
    q, kx, v = host_qkv(11, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=True)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                          to_torch(v, "bf16"), d=d, causal=True, kernel=lib.KERNEL_SM100_OT)
    torch.cuda.synchronize()
    assert o.shape[-1] == 64
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")
