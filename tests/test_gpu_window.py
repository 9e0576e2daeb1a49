"""GPU parity of the causal sliding window (SFA composed with token sparsity) against
the oracle (pinned in tests/test_oracle_window.py).  Runs on SM100_OT (tiles before a block's window
are skipped, lower-bound mask in the softmax) and SIMT."""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch

pytestmark = pytest.mark.gpu
OT, SIMT, AUTO = 6, 1, 0


def run_case(lib, seed, B, H, H_kv, n, d, d_v, k, dtype, kernel, window, n_kv=None, q_pos0=0, edges_only=False):
    import torch
    q, kx, v = host_qkv(seed, B, H, H_kv, n, d, d_v, dtype, n_kv=n_kv)
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, q_pos0=q_pos0, window=window, edges_only=edges_only)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, dtype), to_torch(ki, "u8"), to_torch(kv, dtype),
                          to_torch(v, dtype), d=d, q_pos0=q_pos0, kernel=kernel, window=window, edges_only=edges_only)
    torch.cuda.synchronize()
    return assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, dtype)


@pytest.mark.parametrize("kernel", [OT, SIMT])
@pytest.mark.parametrize("window", [1, 37, 128, 129, 300, 5000])
def test_parity(lib, kernel, window):
    run_case(lib, 71, 1, 4, 2, 600, 128, 128, 16, "bf16", kernel, window)


@pytest.mark.parametrize("kernel", [OT, SIMT])
def test_shapes(lib, kernel):
    run_case(lib, 72, 2, 2, 2, 257, 64, 128, 8, "bf16", kernel, 100)            # d = 64, MHA pairing
    run_case(lib, 77, 2, 3, 3, 300, 64, 64, 8, "bf16", kernel, 90)              # d = d_v = 64 (GPT-2 heads)
    run_case(lib, 73, 1, 2, 1, 200, 128, 128, 16, "bf16", kernel, 64, n_kv=700, q_pos0=500)  # chunk at q_pos0
    run_case(lib, 74, 1, 2, 1, 400, 128, 128, 4, "bf16", kernel, 150, edges_only=True)       # + R2


def test_fp32_simt(lib):
    run_case(lib, 75, 1, 1, 1, 256, 64, 64, 8, "f32", AUTO, 50)


def test_unsupported(lib):
    q, kx, v = host_qkv(76, 1, 2, 1, 64, 128, 128, "bf16")
    qi, qv = oracle_codes(q, 8)
    ki, kv = oracle_codes(kx, 8)
    args = [to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"), to_torch(v, "bf16")]
    for kern in (2, 3, 4, 5):
        with pytest.raises(lib.SfaError):
            lib.attn_fwd(*args, d=128, kernel=kern, window=16)
    with pytest.raises(lib.SfaError):  # a window needs the causal mask
        lib.attn_fwd(*args, d=128, causal=False, window=16)


def test_qwen3_window_sampled_rows(lib):
    """Qwen3-32K with a 4096-token window (AUTO -> SM100_OT): sampled rows vs the oracle."""
    import torch
    B, H, H_kv, n, d, d_v, k, w = 1, 32, 8, 32768, 128, 128, 16, 4096
    q, kx, v = host_qkv(21, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                          to_torch(v, "bf16"), d=d, window=w)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    rows = np.unique(np.concatenate([[0, 4095, 4096, 4200, n - 1, n * H - 1], rng.integers(0, n * H, 100)])).astype(np.int64)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, rows=rows, window=w)
    assert_attn_close(from_torch(o).reshape(-1, d_v)[rows], from_torch(lse).reshape(-1)[rows], o_ref, l_ref, "bf16")
