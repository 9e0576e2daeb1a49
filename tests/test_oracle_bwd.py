"""Pins for the oracle's backward pass (oracle/sfa_oracle.c ref_attn_bwd), SURVEY 8(f) N1.

The backward of O = softmax(scale * Q~ K~^T (.) M) V with the straight-through rule of P:L103-112
(Sec. 3.1 "Backward computation", Eq. topk_grad: the gradient reaches q_{i,u} / k_{j,u} only for
u in the support, where it equals the gradient w.r.t. the decompressed entry).  Pinned by things
other than the oracle's own code:
  * central finite differences of the oracle FORWARD (ref_attn_fwd on fp64 values) with the
    supports held fixed, loss = <dO, O>;
  * torch fp64 autograd of dense attention at k = d (Topk is the identity there), with GQA;
  * closed forms: dO = 0 -> 0; n = 1 -> dV = dO (summed over the group), dq = dk = 0;
  * linearity in dO; the bounds dominate the gradients.
"""
import numpy as np
import pytest
import torch

import oracle


def _codes(x, k):
    shp = x.shape
    idx, _ = oracle.topk_codes(x.reshape(-1, shp[-1]).astype(np.float32), k)
    idx = idx.reshape(shp[:-1] + (k,))
    val = np.take_along_axis(x, idx.astype(np.int64), axis=-1)  # fp64 values at the fp32-chosen support
    return idx, np.ascontiguousarray(val)


def _case(seed, B, H, H_kv, n, d, k, d_v):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, n, d))
    kx = rng.standard_normal((B, H_kv, n, d))
    v = rng.standard_normal((B, H_kv, n, d_v))
    dO = rng.standard_normal((B, H, n, d_v))
    qi, qv = _codes(q, k)
    ki, kv = _codes(kx, k)
    return qi, qv, ki, kv, v, dO


def _loss(qi, qv, ki, kv, v, dO, d, causal):
    o, _ = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, threads=1)
    return float(np.sum(o * dO))


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("shape", [(1, 2, 1, 12, 6, 2, 4), (1, 3, 3, 9, 8, 3, 5)])
def test_finite_differences(shape, causal):
    """Every on-support gradient entry = central difference of <dO, O> (step 1e-5), rel <= 1e-5."""
    B, H, H_kv, n, d, k, d_v = shape
    qi, qv, ki, kv, v, dO = _case(7 + n, *shape)
    dq, dk, dv = oracle.attn_bwd(qi, qv, ki, kv, v, dO, d=d, causal=causal, threads=1)
    eps = 1e-5
    for name, arr, grad in (("q", qv, dq), ("k", kv, dk), ("v", v, dv)):
        fd = np.zeros_like(arr)
        flat = arr.reshape(-1)
        for e in range(flat.size):
            keep = flat[e]
            flat[e] = keep + eps
            lp = _loss(qi, qv, ki, kv, v, dO, d, causal)
            flat[e] = keep - eps
            lm = _loss(qi, qv, ki, kv, v, dO, d, causal)
            flat[e] = keep
            fd.reshape(-1)[e] = (lp - lm) / (2 * eps)
        scale = max(1.0, np.abs(grad).max())
        assert np.abs(fd - grad).max() <= 1e-5 * scale, name


@pytest.mark.parametrize("causal", [True, False])
def test_k_equals_d_is_dense_autograd(causal):
    """k = d: Topk is the identity, so the gradients are torch's dense fp64 attention gradients."""
    B, H, H_kv, n, d, d_v = 2, 4, 2, 20, 8, 6
    rng = np.random.default_rng(3)
    q = rng.standard_normal((B, H, n, d))
    kx = rng.standard_normal((B, H_kv, n, d))
    v = rng.standard_normal((B, H_kv, n, d_v))
    dO = rng.standard_normal((B, H, n, d_v))
    qi = np.broadcast_to(np.arange(d, dtype=np.uint8), (B, H, n, d)).copy()
    ki = np.broadcast_to(np.arange(d, dtype=np.uint8), (B, H_kv, n, d)).copy()
    dq, dk, dv = oracle.attn_bwd(qi, q.copy(), ki, kx.copy(), v, dO, d=d, causal=causal)

    tq = torch.tensor(q, requires_grad=True)
    tk = torch.tensor(kx, requires_grad=True)
    tv = torch.tensor(v, requires_grad=True)
    R = H // H_kv
    s = (tq @ tk.repeat_interleave(R, dim=1).transpose(-1, -2)) / np.sqrt(d)
    if causal:
        s = s.masked_fill(torch.ones(n, n, dtype=torch.bool).triu(1), float("-inf"))
    o = torch.softmax(s, dim=-1) @ tv.repeat_interleave(R, dim=1)
    (o * torch.tensor(dO)).sum().backward()
    np.testing.assert_allclose(dq, tq.grad.numpy(), rtol=0, atol=1e-10)
    np.testing.assert_allclose(dk, tk.grad.numpy(), rtol=0, atol=1e-10)
    np.testing.assert_allclose(dv, tv.grad.numpy(), rtol=0, atol=1e-10)


def test_zero_upstream_and_single_key():
    qi, qv, ki, kv, v, dO = _case(11, 1, 4, 2, 10, 8, 3, 4)
    dq, dk, dv = oracle.attn_bwd(qi, qv, ki, kv, v, np.zeros_like(dO), d=8)
    assert not dq.any() and not dk.any() and not dv.any()
    # n = 1: one allowed key, P = 1, so dV = sum of the group's dO and the score gradients vanish
    qi, qv, ki, kv, v, dO = _case(12, 1, 4, 2, 1, 8, 3, 4)
    dq, dk, dv = oracle.attn_bwd(qi, qv, ki, kv, v, dO, d=8)
    assert not dq.any() and not dk.any()
    np.testing.assert_allclose(dv, dO.reshape(1, 2, 2, 1, 4).sum(axis=2), rtol=0, atol=1e-15)


def test_linearity_and_bounds():
    qi, qv, ki, kv, v, dO1 = _case(13, 1, 2, 1, 16, 8, 3, 5)
    dO2 = np.random.default_rng(14).standard_normal(dO1.shape)
    a, b = 0.75, -1.5
    g1 = oracle.attn_bwd(qi, qv, ki, kv, v, dO1, d=8)
    g2 = oracle.attn_bwd(qi, qv, ki, kv, v, dO2, d=8)
    g12 = oracle.attn_bwd(qi, qv, ki, kv, v, a * dO1 + b * dO2, d=8, bounds=True)
    for x1, x2, x12 in zip(g1, g2, g12[:3]):
        np.testing.assert_allclose(x12, a * x1 + b * x2, rtol=0, atol=1e-12)
    for grad, bound in zip(g12[:3], g12[3:]):
        assert (bound >= 0).all() and (np.abs(grad) <= bound + 1e-12).all()
