"""GPU parity of the fused step-1-on-Q forward (include/sfa.h sfa_attn_fwd_fused_q).

The attention prologue selects the top-k of every dense query row with the same selection code as
the stand-alone top-k kernel, so: its codes must equal the oracle's bit for bit, and its (O, LSE)
must be bit-identical to sfa_topk_codes + sfa_attn_fwd (SM100_OT) and within the bar of the oracle.
"""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu
OT = 6


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("shape", [
    (1, 4, 2, 300, 128, 128, 16),    # GQA, ragged n
    (2, 2, 2, 257, 64, 128, 8),      # d = 64, MHA (odd-free pairing), 3 tiles + 1
    (1, 2, 1, 1, 128, 128, 4),       # single token
    (1, 6, 2, 130, 128, 128, 128),   # k = d
])
def test_fused_matches_oracle_and_unfused(lib, causal, shape):
    import torch
    B, H, H_kv, n, d, d_v, k = shape
    q, kx, v = host_qkv(61, B, H, H_kv, n, d, d_v, "bf16", variant="lattice" if k == 4 else "iid")
    qi_ref, qv_ref = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    qt, kit, kvt, vt = to_torch(q, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"), to_torch(v, "bf16")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    o, lse, qi, qv = lib.attn_fwd_fused_q(qt, kit, kvt, vt, causal=causal, status=status, kernel=OT)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    np.testing.assert_array_equal(from_torch(qi), qi_ref)
    np.testing.assert_array_equal(from_torch(qv), qv_ref)
    o_ref, l_ref = oracle.attn_fwd(qi_ref, qv_ref, ki, kv, v, d=d, causal=causal)
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")
    o2, l2 = lib.attn_fwd(to_torch(qi_ref, "u8"), to_torch(qv_ref, "bf16"), kit, kvt, vt, d=d, causal=causal, kernel=OT)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(lse, l2)


def test_fused_flags_nonfinite_and_forward_uses_it(lib):
    import torch
    B, H, H_kv, n, d, d_v, k = 1, 2, 1, 200, 128, 128, 16
    q, kx, v = host_qkv(62, B, H, H_kv, n, d, d_v, "bf16")
    qt, kt, vt = to_torch(q, "bf16"), to_torch(kx, "bf16"), to_torch(v, "bf16")
    ki, kv = lib.topk_codes(kt, k)
    # sfa_forward (two-kernel path) and the fused call give bit-identical results
    o1, l1 = lib.forward(qt, kt, vt, k_code=k)
    o2, l2, _, _ = lib.attn_fwd_fused_q(qt, ki, kv, vt, codes_out=False)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    qbad = qt.clone()
    qbad[0, 1, 77, 5] = float("inf")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.attn_fwd_fused_q(qbad, ki, kv, vt, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) & 1


def test_fused_unsupported(lib):
    import torch
    q, kx, v = host_qkv(63, 1, 2, 1, 64, 128, 64, "bf16")   # d_v = 64: not the OT kernel
    ki, kv = oracle_codes(kx, 8)
    with pytest.raises(lib.SfaError):
        lib.attn_fwd_fused_q(to_torch(q, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"), to_torch(v, "bf16"))


def test_fused_qwen3_sampled_rows(lib):
    """Qwen3-32K through the fused path: codes of every row bit-exact, sampled rows vs the oracle."""
    import torch
    B, H, H_kv, n, d, d_v, k = 1, 32, 8, 32768, 128, 128, 16
    q, kx, v = host_qkv(21, B, H, H_kv, n, d, d_v, "bf16")
    qi_ref, qv_ref = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o, lse, qi, qv = lib.attn_fwd_fused_q(to_torch(q, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                                          to_torch(v, "bf16"))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(from_torch(qi), qi_ref)
    np.testing.assert_array_equal(from_torch(qv), qv_ref)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([[0, 127, 128, n - 1, n * H - 1], rng.integers(0, n * H, 100)])).astype(np.int64)
    o_ref, l_ref = oracle.attn_fwd(qi_ref, qv_ref, ki, kv, v, d=d, rows=rows)
    assert_attn_close(from_torch(o).reshape(-1, d_v)[rows], from_torch(lse).reshape(-1)[rows], o_ref, l_ref, "bf16")
