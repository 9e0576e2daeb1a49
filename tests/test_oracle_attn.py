"""Pins for the oracle's attention forward (oracle/sfa_oracle.c ref_attn_fwd / ref_scores_row).

O = softmax(scale * Q~ K~^T (.) M) V on the decompressed codes (P:L97-101 Eq. s_ij,
P:L43-50 Sec. 2, "mathematically identical to computing softmax(Q~K~^T/sqrt d)V").
Each pin is fixed by something other than the oracle's code: a library routine (torch
fp64 scaled_dot_product_attention at k = d, where Topk is the identity), closed forms
(n = 1, disjoint supports, Q = K = V = I), the paper's hand example, the softmax
normalisation identity, and causality.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2603_22300_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def codes(x, k):
    shp = x.shape
    idx, val = oracle.topk_codes(x.reshape(-1, shp[-1]), k)
    return idx.reshape(shp[:-1] + (k,)), val.reshape(shp[:-1] + (k,))


def test_hand_example_score():
    g = GOLD["score_hand_example"]
    d = g["d"]
    qi = np.array([[[[g["q"][0][0]]]]], np.uint8)
    qv = np.array([[[[g["q"][0][1]]]]], np.float32)
    ki = np.array([[[[g["k"][0][0]]]]], np.uint8)
    kv = np.array([[[[g["k"][0][1]]]]], np.float32)
    s = oracle.scores_row(qi, qv, ki, kv, 0, d=d, causal=False)
    assert s[0] == g["s"]
    # disjoint supports -> exactly 0 (reading A1: logit 0)
    ki2 = np.array([[[[1]]]], np.uint8)
    assert oracle.scores_row(qi, qv, ki2, kv, 0, d=d, causal=False)[0] == 0.0


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,H,H_kv,n,d,d_v", [(1, 1, 1, 33, 16, 8), (2, 4, 2, 40, 8, 16), (1, 2, 1, 17, 64, 64)])
def test_k_equals_d_is_dense_sdpa(causal, dtype, B, H, H_kv, n, d, d_v):
    """k = d: Topk is the identity, so SFA is textbook softmax attention."""
    q, k, v = inputs.qkv(3, B, H, H_kv, n, d, d_v, dtype)
    qi, qv = codes(q, d)
    ki, kv = codes(k, d)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal)
    tof = (lambda a: torch.from_numpy(a.astype(np.float64))) if dtype == "f32" else \
          (lambda a: torch.from_numpy(inputs.bf16_bits_to_f32(a).astype(np.float64)))
    Q, K, V = tof(q), tof(k), tof(v)
    rep = H // H_kv
    K = K.repeat_interleave(rep, dim=1)
    V = V.repeat_interleave(rep, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V, is_causal=causal, scale=1 / math.sqrt(d))
    np.testing.assert_allclose(o, ref.numpy(), rtol=0, atol=1e-12)
    S = (Q @ K.transpose(-1, -2)) / math.sqrt(d)
    if causal:
        S = S.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool), 1), -math.inf)
    np.testing.assert_allclose(lse, torch.logsumexp(S, -1).numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_single_key(dtype):
    """n = 1: softmax over one key is 1, so O = v and LSE = s_00."""
    q, k, v = inputs.qkv(4, 1, 3, 1, 1, 64, 64, dtype)
    qi, qv = codes(q, 8)
    ki, kv = codes(k, 8)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=64)
    vf = v.astype(np.float64) if dtype == "f32" else inputs.bf16_bits_to_f32(v).astype(np.float64)
    for h in range(3):
        np.testing.assert_array_equal(o[0, h, 0], vf[0, 0, 0])
        s = oracle.scores_row(qi, qv, ki, kv, h, d=64)
        assert lse[0, h, 0] == s[0]


@pytest.mark.parametrize("q_pos0", [0, 5])
def test_disjoint_supports_prefix_mean(q_pos0):
    """Disjoint supports -> every logit 0 (reading A1) -> O_i = mean(V[0..q_pos0+i]), LSE_i = ln(#keys)."""
    n_q, n_kv, d, k, d_v = 24, 24 + q_pos0, 64, 8, 16
    rng = np.random.default_rng(0)
    qi = np.sort(rng.permutation(32)[:k])[None, None, None, :].repeat(n_q, 2).astype(np.uint8)
    ki = (32 + np.sort(rng.permutation(32)[:k]))[None, None, None, :].repeat(n_kv, 2).astype(np.uint8)
    qv = rng.standard_normal((1, 1, n_q, k)).astype(np.float32)
    kv = rng.standard_normal((1, 1, n_kv, k)).astype(np.float32)
    v = rng.standard_normal((1, 1, n_kv, d_v)).astype(np.float32)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=True, q_pos0=q_pos0)
    cm = np.cumsum(v[0, 0].astype(np.float64), 0) / np.arange(1, n_kv + 1)[:, None]
    np.testing.assert_allclose(o[0, 0], cm[q_pos0:], rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse[0, 0], np.log(np.arange(q_pos0 + 1, n_kv + 1)), rtol=0, atol=1e-13)


def test_identity_closed_form():
    """Q = K = V = I (n = d = d_v), no mask: O_ii = e^{1/sqrt d}/(e^{1/sqrt d}+n-1)."""
    n = d = 16
    eye = np.eye(n, dtype=np.float32)[None, None]
    qi, qv = codes(eye, 1)
    o, lse = oracle.attn_fwd(qi, qv, qi, qv, eye, d=d, causal=False)
    e = math.exp(1 / math.sqrt(d))
    want = np.full((n, n), 1 / (e + n - 1))
    np.fill_diagonal(want, e / (e + n - 1))
    np.testing.assert_allclose(o[0, 0], want, rtol=0, atol=1e-15)
    np.testing.assert_allclose(lse[0, 0], math.log(e + n - 1), rtol=0, atol=1e-14)


@pytest.mark.parametrize("causal", [True, False])
def test_rows_of_p_sum_to_one(causal):
    """sum_j exp(s_ij - LSE_i) = 1 over allowed keys (softmax normalisation)."""
    q, k, v = inputs.qkv(9, 1, 2, 1, 50, 64, 32, "bf16")
    qi, qv = codes(q, 8)
    ki, kv = codes(k, 8)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=64, causal=causal)
    for flat in (0, 1, 17, 49, 50, 99):
        s = oracle.scores_row(qi, qv, ki, kv, flat, d=64, causal=causal)
        tot = np.exp(s - lse.reshape(-1)[flat]).sum()
        assert abs(tot - 1.0) < 1e-12


def test_causality_perturbation():
    """Perturbing key/value j > i leaves row i bit-identical."""
    q, k, v = inputs.qkv(12, 1, 1, 1, 40, 64, 16, "f32")
    qi, qv = codes(q, 8)
    ki, kv = codes(k, 8)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=64)
    i = 20
    k2, v2 = k.copy(), v.copy()
    k2[0, 0, i + 1:] = inputs.gen_f32(99, 2, k2[0, 0, i + 1:].shape)
    v2[0, 0, i + 1:] = -7.0
    ki2, kv2 = codes(k2, 8)
    o2, lse2 = oracle.attn_fwd(qi, qv, ki2, kv2, v2, d=64)
    np.testing.assert_array_equal(o[0, 0, :i + 1], o2[0, 0, :i + 1])
    np.testing.assert_array_equal(lse[0, 0, :i + 1], lse2[0, 0, :i + 1])
    assert not np.array_equal(o[0, 0, i + 1:], o2[0, 0, i + 1:])


def test_sampled_rows_and_q_pos0_match_full():
    q, k, v = inputs.qkv(13, 2, 4, 2, 64, 64, 32, "bf16")
    qi, qv = codes(q, 8)
    ki, kv = codes(k, 8)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=64)
    rows = np.array([0, 5, 63, 64, 200, 511], np.int64)
    os_, ls_ = oracle.attn_fwd(qi, qv, ki, kv, v, d=64, rows=rows)
    np.testing.assert_array_equal(os_, o.reshape(-1, 32)[rows])
    np.testing.assert_array_equal(ls_, lse.reshape(-1)[rows])
    # a query chunk at global offset q_pos0 sees the same keys as in the full run (reading A9)
    oc, lc = oracle.attn_fwd(qi[:, :, 40:], qv[:, :, 40:], ki, kv, v, d=64, q_pos0=40)
    np.testing.assert_array_equal(oc, o[:, :, 40:])
    np.testing.assert_array_equal(lc, lse[:, :, 40:])


def test_gqa_mapping():
    """Query head h reads kv head h // (H/H_kv) (reading A15): equal to H_kv=H with repeated kv."""
    q, k, v = inputs.qkv(14, 1, 4, 2, 30, 64, 16, "f32")
    qi, qv = codes(q, 8)
    ki, kv = codes(k, 8)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=64)
    o2, lse2 = oracle.attn_fwd(qi, qv, ki.repeat(2, 1), kv.repeat(2, 1), v.repeat(2, 1), d=64)
    np.testing.assert_array_equal(o, o2)
    np.testing.assert_array_equal(lse, lse2)


def test_errors():
    q, k, v = inputs.qkv(1, 1, 1, 1, 4, 8, 8, "f32")
    qi, qv = codes(q, 2)
    ki, kv = codes(k, 2)
    with pytest.raises(oracle.OracleError):
        oracle.attn_fwd(qi, qv, ki, kv, v, d=8, scale=-1.0)
    with pytest.raises(oracle.OracleError):
        oracle.attn_fwd(qi, qv, ki, kv, v, d=1)  # k > d
