"""Pins for the oracle's edge-only mode (reading A1/R2).

R2 ("Traversing active coordinates yields only the nonzero attention edges"; P:L122
"O(E + E d_v)"; Alg. 1 "iterate nonzeros P_ij"): a query-key pair enters the softmax
only if the two supports share a feature index.  Each pin is fixed by something other than the
oracle's C code:
  - an independent torch fp64 formulation: dense Q~ K~^T with the mask built from the indicator
    product 1[S_i] 1[S_j]^T > 0 (a library matmul, not index comparison);
  - the exact identity between R2 and R1 (pinned in test_oracle_attn.py), with the non-edge set
    counted by Python set intersection: e^{LSE1} = e^{LSE2} + |N_i| and
    e^{LSE1} O1 = e^{LSE2} O2 + sum_{j in N_i} V_j  (non-edges have logit 0 under R1);
  - k = d (every pair is an edge): R2 equals dense SDPA;
  - constructed disjoint supports: no edges -> O = 0, LSE = -inf (as A10);
  - a hand example with one zero-valued selected entry (A8: zeros count as support).
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


def dense(idx, val, d):
    out = np.zeros(idx.shape[:-1] + (d,), np.float64)
    np.put_along_axis(out, idx.astype(np.int64), f64(val), axis=-1)
    return out


def indicator(idx, d):
    out = np.zeros(idx.shape[:-1] + (d,), np.float64)
    np.put_along_axis(out, idx.astype(np.int64), 1.0, axis=-1)
    return out


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,H,H_kv,n,d,k,d_v", [(1, 2, 1, 40, 64, 4, 16), (2, 4, 2, 33, 128, 8, 32),
                                                (1, 1, 1, 70, 64, 2, 8)])
def test_matches_torch_masked_softmax(causal, dtype, B, H, H_kv, n, d, k, d_v):
    q, kx, v = inputs.qkv(5, B, H, H_kv, n, d, d_v, dtype)
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, edges_only=True)
    rep = H // H_kv
    Q = torch.from_numpy(dense(qi, qv, d))
    K = torch.from_numpy(dense(ki, kv, d)).repeat_interleave(rep, 1)
    V = torch.from_numpy(f64(v)).repeat_interleave(rep, 1)
    IQ = torch.from_numpy(indicator(qi, d))
    IK = torch.from_numpy(indicator(ki, d)).repeat_interleave(rep, 1)
    allowed = (IQ @ IK.transpose(-1, -2)) > 0
    if causal:
        allowed &= ~torch.triu(torch.ones(n, n, dtype=torch.bool), 1)
    S = (Q @ K.transpose(-1, -2)) / math.sqrt(d)
    S = S.masked_fill(~allowed, -math.inf)
    L = torch.logsumexp(S, -1)
    P = torch.exp(S - L[..., None]).nan_to_num(0.0)  # rows with no edge: all -inf -> 0
    O = P @ V
    assert (~allowed).any(), "the case must contain non-edges"
    np.testing.assert_allclose(o, O.numpy(), rtol=0, atol=1e-12)
    fin = torch.isfinite(L).numpy()
    np.testing.assert_allclose(lse[fin], L.numpy()[fin], rtol=0, atol=1e-12)
    assert np.all(lse[~fin] == -np.inf)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_identity_with_r1(k):
    """Non-edges have logit exactly 0 under R1, so R1 = R2 + |N_i| unit weights on V_j, j in N_i."""
    B, H, H_kv, n, d, d_v = 1, 2, 1, 48, 64, 16
    q, kx, v = inputs.qkv(8, B, H, H_kv, n, d, d_v, "f32")
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    o1, l1 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, edges_only=False)
    o2, l2 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, edges_only=True)
    vf = v.astype(np.float64)
    n_non = 0
    for h in range(H):
        for i in range(n):
            sq = set(qi[0, h, i].tolist())
            non = [j for j in range(i + 1) if not (sq & set(ki[0, 0, j].tolist()))]
            n_non += len(non)
            e2 = math.exp(l2[0, h, i]) if np.isfinite(l2[0, h, i]) else 0.0
            assert math.exp(l1[0, h, i]) == pytest.approx(e2 + len(non), rel=1e-12)
            rhs = e2 * o2[0, h, i] + vf[0, 0, non].sum(0)
            np.testing.assert_allclose(math.exp(l1[0, h, i]) * o1[0, h, i], rhs, rtol=0, atol=1e-11)
    assert n_non > 0


def test_k_equals_d_is_dense():
    """k = d: every support is the full feature set, so every pair is an edge (R2 = R1 = SDPA)."""
    q, kx, v = inputs.qkv(3, 1, 2, 1, 30, 16, 8, "f32")
    qi, qv = codes(q, 16)
    ki, kv = codes(kx, 16)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=16, edges_only=True)
    K = torch.from_numpy(kx.astype(np.float64)).repeat_interleave(2, 1)
    V = torch.from_numpy(v.astype(np.float64)).repeat_interleave(2, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(torch.from_numpy(q.astype(np.float64)), K, V,
                                                           is_causal=True, scale=0.25)
    np.testing.assert_allclose(o, ref.numpy(), rtol=0, atol=1e-12)


def test_disjoint_supports_have_no_edges():
    n, d, k, d_v = 20, 64, 8, 16
    qi = np.tile(np.arange(k, dtype=np.uint8), (1, 1, n, 1))
    ki = np.tile(np.arange(32, 32 + k, dtype=np.uint8), (1, 1, n, 1))
    qv = inputs.gen(1, 1, (1, 1, n, k), "f32")
    kv = inputs.gen(1, 2, (1, 1, n, k), "f32")
    v = inputs.gen(1, 3, (1, 1, n, d_v), "f32")
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, edges_only=True)
    assert np.all(o == 0.0) and np.all(lse == -np.inf)


def test_zero_valued_support_is_an_edge():
    """Hand example (A8): the only shared feature carries q~ = 0, so s = 0 -- but it IS an edge.
    Row 0 sees key 0 (edge, s = 0) -> O = v0, LSE = 0.  Row 1 sees key 0 and key 1, key 1 disjoint
    -> still O = v0, LSE = 0 (R1 would give the mean of v0, v1 and LSE = ln 2)."""
    d = 8
    qi = np.array([[[[1, 2], [1, 2]]]], np.uint8)
    qv = np.array([[[[0.0, 3.0], [0.0, 3.0]]]], np.float32)
    ki = np.array([[[[1, 5], [6, 7]]]], np.uint8)
    kv = np.array([[[[2.0, 4.0], [1.0, 1.0]]]], np.float32)
    v = np.array([[[[1.0, -2.0], [5.0, 7.0]]]], np.float32)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, edges_only=True)
    np.testing.assert_array_equal(o[0, 0], [[1.0, -2.0], [1.0, -2.0]])
    np.testing.assert_array_equal(lse[0, 0], [0.0, 0.0])
    o1, l1 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, edges_only=False)
    np.testing.assert_allclose(o1[0, 0, 1], [3.0, 2.5], rtol=0, atol=1e-15)
    assert l1[0, 0, 1] == pytest.approx(math.log(2.0), abs=1e-15)
