"""Pins for the oracle's block-selection mode (SFA composed with NSA-style block-level
token selection, "SFA is orthogonal to token-level sparsity").

With key blocks of 128 positions, query row i of (batch b, kv group g) may attend key j only if j is
causally allowed AND j // 128 is in the list block_sel[b][g][i // 128].  Each pin is fixed by something
other than the oracle's C code:
  - every block selected: the plain causal forward, bit for bit (the mask is the identity);
  - an independent torch fp64 formulation: dense Q~ K~^T with the block mask built by numpy indexing
    from the lists, masked softmax;
  - an empty list: the query block's rows get O = 0, LSE = -inf (as A10); padding entries (< 0) and
    duplicate or unordered entries do not change the set;
  - the heads of one GQA group share their kv head's lists.
"""
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


def random_sel(rng, B, H_kv, n_q, n_kv, max_sel, p=0.5):
    nqb, nkb = (n_q + 127) // 128, (n_kv + 127) // 128
    sel = np.full((B, H_kv, nqb, max_sel), -1, np.int32)
    for b in range(B):
        for g in range(H_kv):
            for qb in range(nqb):
                chosen = [t for t in range(nkb) if rng.random() < p][:max_sel]
                sel[b, g, qb, :len(chosen)] = chosen
    return sel


def block_mask(sel, n_q, n_kv):
    """[B, H_kv, n_q, n_kv] bool: key block j // 128 listed for query block i // 128."""
    B, H_kv, nqb, _ = sel.shape
    nkb = (n_kv + 127) // 128
    m = np.zeros((B, H_kv, nqb, nkb), bool)
    for b in range(B):
        for g in range(H_kv):
            for qb in range(nqb):
                for t in sel[b, g, qb]:
                    if 0 <= t < nkb:
                        m[b, g, qb, t] = True
    return m[:, :, np.arange(n_q) // 128][:, :, :, np.arange(n_kv) // 128]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_all_blocks_selected_is_the_causal_forward(dtype):
    B, H, H_kv, n, d, k, d_v = 1, 4, 2, 300, 64, 8, 32
    q, kx, v = inputs.qkv(3, B, H, H_kv, n, d, d_v, dtype)
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    nb = (n + 127) // 128
    sel = np.broadcast_to(np.arange(nb, dtype=np.int32), (B, H_kv, nb, nb)).copy()
    o1, l1 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d)
    o2, l2 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, block_sel=sel)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(l1, l2)


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("B,H,H_kv,n,d,k,d_v", [(1, 2, 1, 300, 64, 8, 16), (2, 4, 2, 400, 128, 16, 32)])
def test_matches_torch_block_masked_softmax(causal, B, H, H_kv, n, d, k, d_v):
    q, kx, v = inputs.qkv(9, B, H, H_kv, n, d, d_v, "f32")
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    sel = random_sel(np.random.default_rng(4), B, H_kv, n, n, 3)
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, block_sel=sel)
    rep = H // H_kv
    Q = torch.from_numpy(dense(qi, qv, d))
    K = torch.from_numpy(dense(ki, kv, d)).repeat_interleave(rep, 1)
    V = torch.from_numpy(f64(v)).repeat_interleave(rep, 1)
    S = Q @ K.transpose(-1, -2) / np.sqrt(d)
    M = torch.from_numpy(block_mask(sel, n, n)).repeat_interleave(rep, 1)
    if causal:
        M = M & torch.ones(n, n, dtype=torch.bool).tril()
    S = S.masked_fill(~M, float("-inf"))
    lse_ref = torch.logsumexp(S, -1)
    P = torch.softmax(S, -1)
    O_ref = torch.nan_to_num(P, nan=0.0) @ V
    empty = ~M.any(-1)
    O_ref[empty] = 0.0
    lse_ref[empty] = float("-inf")
    np.testing.assert_allclose(o, O_ref.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(np.isneginf(lse), empty.numpy())
    fin = ~empty.numpy()
    np.testing.assert_allclose(lse[fin], lse_ref.numpy()[fin], rtol=1e-12, atol=1e-12)


def test_empty_list_padding_and_order():
    B, H, H_kv, n, d, k, d_v = 1, 2, 1, 384, 64, 8, 16
    q, kx, v = inputs.qkv(6, B, H, H_kv, n, d, d_v, "f32")
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    sel = np.full((1, 1, 3, 4), -1, np.int32)
    sel[0, 0, 0] = [0, -1, -1, -1]   # block 0: its own diagonal block
    sel[0, 0, 1] = [-1, -1, -1, -1]  # block 1: nothing -> O = 0, LSE = -inf
    sel[0, 0, 2] = [2, 0, 0, -5]     # unordered, duplicated, negative padding == {0, 2}
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, block_sel=sel)
    assert np.all(np.isneginf(lse[:, :, 128:256])) and np.all(o[:, :, 128:256] == 0.0)
    sel2 = sel.copy()
    sel2[0, 0, 2] = [0, 2, -1, -1]
    o2, lse2 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, block_sel=sel2)
    np.testing.assert_array_equal(o, o2)
    np.testing.assert_array_equal(lse, lse2)
    # block 0 with only its diagonal block selected is the causal forward of its rows
    o3, lse3 = oracle.attn_fwd(qi, qv, ki, kv, v, d=d)
    np.testing.assert_array_equal(o[:, :, :128], o3[:, :, :128])


def test_gqa_heads_share_the_kv_head_lists():
    B, H, H_kv, n, d, k, d_v = 1, 4, 2, 256, 64, 8, 16
    q, kx, v = inputs.qkv(8, B, H, H_kv, n, d, d_v, "f32")
    qi, qv = codes(q, k)
    ki, kv = codes(kx, k)
    sel = np.full((1, 2, 2, 2), -1, np.int32)
    sel[0, 0, 1] = [1, -1]  # kv head 0, query block 1: only its diagonal block
    sel[0, 1, 1] = [0, 1]   # kv head 1: both blocks (= causal)
    sel[0, :, 0] = [0, -1]
    o, lse = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, block_sel=sel)
    oc, lc = oracle.attn_fwd(qi, qv, ki, kv, v, d=d)
    np.testing.assert_array_equal(o[:, 2:], oc[:, 2:])  # heads 2, 3 -> kv head 1: causal
    assert not np.allclose(o[:, :2, 128:], oc[:, :2, 128:])  # heads 0, 1: block 0 excluded for rows 128+
