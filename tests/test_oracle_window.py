"""Pins for the oracle's causal sliding window (SFA composed with token sparsity,
P:L918-1087 -- Longformer / Mistral-style local attention over the feature-sparse scores).

Key j is allowed for query i iff j <= q_pos0 + i (causal, A9) and j > q_pos0 + i - window.  Pinned by:
  - an independent torch fp64 formulation at k = d (Topk is the identity): dense SDPA with a banded
    boolean mask;
  - window >= q_pos0 + n covers every causal key: identical to the plain causal oracle;
  - window = 1: only the key at the query's own position -> O_i = V_{q_pos0+i}, LSE_i = s_{i,q_pos0+i};
  - the same band on top of R2 (edges only) against torch with both masks.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2603_22300_b200 import inputs


def codes(x, k):
    shp = x.shape
    idx, val = oracle.topk_codes(x.reshape(-1, shp[-1]), k)
    return idx.reshape(shp[:-1] + (k,)), val.reshape(shp[:-1] + (k,))


def f64(a):
    return a.astype(np.float64) if a.dtype != np.uint16 else inputs.bf16_bits_to_f32(a).astype(np.float64)


def band(n_q, n_kv, q_pos0, window):
    i = torch.arange(n_q)[:, None] + q_pos0
    j = torch.arange(n_kv)[None, :]
    return (j <= i) & (j > i - window)


@pytest.mark.parametrize("window", [1, 5, 16, 40])
@pytest.mark.parametrize("q_pos0", [0, 7])
def test_k_equals_d_matches_banded_sdpa(window, q_pos0):
    B, H, H_kv, n_q, d, d_v = 1, 4, 2, 33, 16, 8
    n_kv = n_q + q_pos0
    q, kx, v = inputs.qkv(17, B, H, H_kv, n_q, d, d_v, "f32", n_kv=n_kv)
    qi, qv = codes(q, d)
    ki, kv = codes(kx, d)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, q_pos0=q_pos0, window=window)
    Q = torch.from_numpy(q.astype(np.float64))
    K = torch.from_numpy(kx.astype(np.float64)).repeat_interleave(2, 1)
    V = torch.from_numpy(v.astype(np.float64)).repeat_interleave(2, 1)
    m = band(n_q, n_kv, q_pos0, window)
    ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V, attn_mask=m, scale=1 / math.sqrt(d))
    np.testing.assert_allclose(o, ref.numpy(), rtol=0, atol=1e-12)
    S = (Q @ K.transpose(-1, -2)) / math.sqrt(d)
    np.testing.assert_allclose(lse, torch.logsumexp(S.masked_fill(~m, -math.inf), -1).numpy(), rtol=0, atol=1e-12)


def test_wide_window_is_plain_causal():
    q, kx, v = inputs.qkv(18, 1, 2, 1, 50, 64, 16, "bf16")
    qi, qv = codes(q, 8)
    ki, kv = codes(kx, 8)
    o0, l0 = oracle.attn_fwd(qi, qv, ki, kv, v, d=64)
    for w in (50, 51, 10 ** 9):
        o1, l1 = oracle.attn_fwd(qi, qv, ki, kv, v, d=64, window=w)
        np.testing.assert_array_equal(o0, o1)
        np.testing.assert_array_equal(l0, l1)


def test_window_one_is_the_own_key():
    q, kx, v = inputs.qkv(19, 1, 2, 2, 30, 64, 16, "f32")
    qi, qv = codes(q, 8)
    ki, kv = codes(kx, 8)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=64, window=1)
    for h in range(2):
        np.testing.assert_array_equal(o[0, h], v[0, h].astype(np.float64))
        for i in (0, 13, 29):
            s = oracle.scores_row(qi, qv, ki, kv, h * 30 + i, d=64)
            assert lse[0, h, i] == s[i]


def test_window_with_edges_only():
    B, H, n, d, k, d_v, w = 1, 2, 60, 64, 4, 16, 9
    q, kx, v = inputs.qkv(20, B, H, H, n, d, d_v, "f32")
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, window=w, edges_only=True)

    def dense(idx, val):
        out = np.zeros(idx.shape[:-1] + (d,))
        np.put_along_axis(out, idx.astype(np.int64), f64(val), axis=-1)
        return torch.from_numpy(out)

    def ind(idx):
        out = np.zeros(idx.shape[:-1] + (d,))
        np.put_along_axis(out, idx.astype(np.int64), 1.0, axis=-1)
        return torch.from_numpy(out)

    Q, K = dense(qi, qv), dense(ki, kv)
    allowed = band(n, n, 0, w) & ((ind(qi) @ ind(ki).transpose(-1, -2)) > 0)
    S = ((Q @ K.transpose(-1, -2)) / math.sqrt(d)).masked_fill(~allowed, -math.inf)
    L = torch.logsumexp(S, -1)
    P = torch.exp(S - L[..., None]).nan_to_num(0.0)
    np.testing.assert_allclose(o, (P @ torch.from_numpy(f64(v))).numpy(), rtol=0, atol=1e-12)
    fin = torch.isfinite(L).numpy()
    assert (~fin).any() and fin.any()
    np.testing.assert_allclose(lse[fin], L.numpy()[fin], rtol=0, atol=1e-12)
    assert np.all(lse[~fin] == -np.inf) and np.all(o[~fin] == 0.0)
