"""GPU parity of the decode-shape kernel (csrc/decode.cu) against the oracle.

Few query rows per kv head (n_q * H / H_kv <= 16) over a long key/value cache: the same
definition as the full forward (the oracle is unchanged), with the queries at the END of the
sequence (q_pos0 = n_kv - n_q, reading A9) for causal decode, or anywhere for non-causal."""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch

pytestmark = pytest.mark.gpu


def run(lib, seed, B, H, H_kv, n_q, n_kv, d, d_v, k, causal=True, kernel=None):
    import torch
    q, _, _ = host_qkv(seed, B, H, H_kv, n_q, d, d_v, "bf16")
    _, kx, v = host_qkv(seed + 1, B, H, H_kv, n_kv, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    q_pos0 = n_kv - n_q if causal else 0
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, q_pos0=q_pos0)
    o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                          to_torch(v, "bf16"), d=d, causal=causal, q_pos0=q_pos0,
                          kernel=lib.KERNEL_DECODE if kernel is None else kernel)
    torch.cuda.synchronize()
    return assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16"), (o, lse)


@pytest.mark.parametrize("shape", [
    (1, 32, 8, 1, 32768, 128, 128, 16),  # Qwen3 decode step over a 32K cache
    (2, 8, 8, 1, 5000, 64, 64, 8),       # GPT-2-like heads (R = 1), ragged cache
    (1, 8, 2, 4, 3001, 128, 128, 16),    # speculative decode: 4 query rows x R = 4 -> 16 rows
    (1, 4, 1, 2, 700, 128, 64, 4),       # R = 4, n_q = 2, k = 4 (sweep's smallest)
    (1, 2, 2, 1, 1, 128, 128, 16),       # a cache of one key
    (1, 2, 1, 3, 257, 64, 128, 5),       # k not a multiple of 8 (scalar code loads)
    (1, 4, 4, 1, 100000, 128, 128, 128), # k = d
])
@pytest.mark.parametrize("causal", [True, False])
def test_decode_against_oracle(lib, shape, causal):
    run(lib, 61, *shape, causal=causal)


def test_auto_selects_decode_and_matches(lib):
    """AUTO picks the decode kernel for decode shapes; the tensor-core kernel agrees within the bar."""
    import torch
    _, (o_auto, l_auto) = run(lib, 71, 1, 8, 2, 1, 2000, 128, 128, 16, kernel=lib.KERNEL_AUTO)
    _, (o_dec, l_dec) = run(lib, 71, 1, 8, 2, 1, 2000, 128, 128, 16, kernel=lib.KERNEL_DECODE)
    assert torch.equal(o_auto, o_dec) and torch.equal(l_auto, l_dec)
    _, (o_tc, l_tc) = run(lib, 71, 1, 8, 2, 1, 2000, 128, 128, 16, kernel=lib.KERNEL_SM100)


def test_decode_rejects_too_many_rows(lib):
    import ctypes
    d = lib.make_desc(B=1, H=32, H_kv=1, d=128, k=16, d_v=128, n_q=1, n_kv=100, kernel=lib.KERNEL_DECODE)
    P = ctypes.c_void_p(16)
    assert lib.lib().sfa_attn_fwd(ctypes.byref(d), *([P] * 8), 1 << 30, None) == 3  # 32 rows > 16
