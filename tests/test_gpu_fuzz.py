"""Seeded random shapes through every forward kernel the library dispatches to, against the oracle.

The hand-picked parity cases cover the tile boundaries and the BASELINE configs; this sweep draws
160 further shapes from a fixed seed (batch, heads and GQA ratio, ragged lengths, decode shapes with a
few query rows over up to 5K keys, a query chunk at an offset of the key sequence, d and d_v in
{64, 128}, k anywhere in 1..d, causal or not, a sliding window or the edge-only semantics now and then)
so that combinations nobody wrote down still meet the bar.
Each case runs AUTO (which may pick DECODE, SM100 or SM100_OT) and, where it applies, SM100_OT
explicitly; the oracle regenerates everything on the host.
"""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch

pytestmark = pytest.mark.gpu


def draw(i):
    rng = np.random.default_rng(1000 + i)
    B = int(rng.integers(1, 3))
    H_kv = int(rng.integers(1, 3))
    R = int(rng.choice([1, 2, 4]))
    d = int(rng.choice([64, 128]))
    d_v = int(rng.choice([64, 128]))
    k = int(rng.integers(1, d + 1)) if rng.random() < 0.3 else int(rng.choice([4, 8, 16]))
    n_kv = int(rng.integers(1, 700))
    u = rng.random()
    if u < 0.2:  # decode shape: a few query rows at the end of the cache (AUTO -> DECODE when rows <= 16)
        n_kv = int(rng.integers(1, 5000))
        n_q = int(rng.integers(1, min(4, n_kv) + 1))
    else:
        n_q = n_kv if u < 0.65 else int(rng.integers(1, n_kv + 1))
    q_pos0 = n_kv - n_q if rng.random() < 0.7 else int(rng.integers(0, n_kv - n_q + 1))
    causal = bool(rng.random() < 0.75)
    window = int(rng.integers(1, 400)) if causal and rng.random() < 0.2 else 0
    edges = bool(rng.random() < 0.15)
    return B, R * H_kv, H_kv, n_q, n_kv, q_pos0, d, d_v, k, causal, window, edges


@pytest.mark.parametrize("i", range(160))
def test_random_shape(lib, i):
    import torch
    B, H, H_kv, n_q, n_kv, q_pos0, d, d_v, k, causal, window, edges = draw(i)
    _, kx, v = host_qkv(500 + i, B, H, H_kv, n_kv, d, d_v, "bf16")
    q, _, _ = host_qkv(700 + i, B, H, H_kv, n_q, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, q_pos0=q_pos0, window=window,
                                   edges_only=edges)
    kernels = [lib.KERNEL_AUTO]
    if not (window or edges) and (H // H_kv) * n_q > 16:
        kernels.append(lib.KERNEL_SM100_OT)
    for kern in kernels:
        o, lse = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                              to_torch(v, "bf16"), d=d, causal=causal, q_pos0=q_pos0, kernel=kern, window=window,
                              edges_only=edges)
        torch.cuda.synchronize()
        assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")


def draw_bwd(i):
    rng = np.random.default_rng(5000 + i)
    B = int(rng.integers(1, 3))
    H_kv = int(rng.integers(1, 3))
    R = int(rng.choice([1, 2, 3, 4]))
    d = int(rng.choice([64, 128]))
    d_v = int(rng.choice([64, 128]))
    k = int(rng.integers(1, d + 1)) if rng.random() < 0.3 else int(rng.choice([4, 8, 16]))
    n_kv = int(rng.integers(1, 500))
    n = n_kv if rng.random() < 0.6 else int(rng.integers(1, n_kv + 1))
    q_pos0 = n_kv - n if rng.random() < 0.7 else int(rng.integers(0, n_kv - n + 1))
    causal = bool(rng.random() < 0.75)
    return B, R * H_kv, H_kv, n, n_kv, q_pos0, d, d_v, k, causal


@pytest.mark.parametrize("i", range(32))
def test_random_shape_backward(lib, i):
    """The backward (straight-through rule) on 32 seeded random shapes, with test_gpu_bwd's componentwise
    and normwise bounds (reading A24) and its bitwise determinism check."""
    from test_gpu_bwd import check, run_bwd
    B, H, H_kv, n, n_kv, q_pos0, d, d_v, k, causal = draw_bwd(i)
    gpu, ref = run_bwd(lib, 900 + i, B, H, H_kv, n, d, d_v, k, causal=causal, q_pos0=q_pos0, n_kv=n_kv)
    check(gpu, ref)
