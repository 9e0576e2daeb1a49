"""Pins for the oracle's edge count and for the bench's accounting formulas.

E = number of structural intersections (P:L114-120 Eq. E ~ sum_u deg(u)^2 ~ n^2k^2/d).
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2603_22300_b200 import accounting, inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def prefix_count_edges(q_idx, k_idx, d, causal=True):
    """E = sum_f sum_i [f in S_i] * #{j <= i : f in S_j}, by one-hot prefix counts in O(n d)."""
    B, H, n, k = q_idx.shape
    H_kv = k_idx.shape[1]
    E = 0
    for b in range(B):
        for h in range(H):
            g = h // (H // H_kv)
            oq = np.zeros((n, d), np.int64)
            ok = np.zeros((k_idx.shape[2], d), np.int64)
            np.put_along_axis(oq, q_idx[b, h].astype(np.int64), 1, 1)
            np.put_along_axis(ok, k_idx[b, g].astype(np.int64), 1, 1)
            cnt = np.cumsum(ok, 0) if causal else np.broadcast_to(ok.sum(0), ok.shape)
            E += int((oq * cnt[:n]).sum())
    return E


@pytest.mark.parametrize("causal", [True, False])
def test_edge_count_prefix_formula(causal):
    q, k, _ = inputs.qkv(21, 2, 4, 2, 96, 64, 8, "bf16", variant="skewed")
    qi, _ = oracle.topk_codes(q.reshape(-1, 64), 8)
    ki, _ = oracle.topk_codes(k.reshape(-1, 64), 8)
    qi = qi.reshape(2, 4, 96, 8)
    ki = ki.reshape(2, 2, 96, 8)
    assert oracle.edge_count(qi, ki, causal=causal) == prefix_count_edges(qi, ki, 64, causal)


def test_balanced_supports_closed_form():
    """Balanced supports (deg(u) = nk/d for every u) give exactly E = n^2 k^2 / d."""
    n, d, k = 256, 64, 8
    sup = ((np.arange(n)[:, None] * k + np.arange(k)[None, :]) % d).astype(np.uint8)
    sup.sort(1)
    qi = sup[None, None]
    assert oracle.edge_count(qi, qi, causal=False) == n * n * k * k // d


def test_predicted_edges_golden():
    g = GOLD["predicted_edges"]
    assert accounting.predicted_edges(g["n"], g["d"], g["k"]) == g["E"]
    r = GOLD["flop_ratio"]
    assert (r["k"] / r["d"]) ** 2 == r["ratio"]


def test_appb_flop_table():
    """Our FLOP convention reproduces every App.-B table entry to < 1%."""
    t = GOLD["appB_flops_table"]
    worst = 0.0
    for name, row in t["rows"].items():
        for n, want in zip(t["n"], row["tflops"]):
            got = accounting.appb_flops(t["BH"], n, row["d"], row["d"], row["k"]) / 1e12
            worst = max(worst, abs(got - want) / want)
    assert worst < 0.01, worst


@pytest.mark.parametrize("n_q,n_kv,q_pos0", [(7, 7, 0), (5, 9, 4), (9, 5, 0), (3, 10, 2), (1, 1, 0)])
def test_causal_pairs(n_q, n_kv, q_pos0):
    brute = sum(1 for i in range(n_q) for j in range(n_kv) if j <= q_pos0 + i)
    assert accounting.causal_pairs(n_q, n_kv, q_pos0) == brute


@pytest.mark.parametrize("causal,q_pos0", [(True, 0), (False, 0), (True, 37)])
def test_exact_edges_torch_prefix_count_equals_oracle(causal, q_pos0):
    """The bench's exact interaction count (accounting.exact_edges, torch prefix counts) equals the
    oracle's explicit pair-by-pair overlap count, GQA and skewed supports included."""
    import torch
    q, k, _ = inputs.qkv(5, 2, 4, 2, 80, 64, 8, "bf16", variant="skewed", n_kv=80 + q_pos0)
    qi, _ = oracle.topk_codes(q.reshape(-1, 64), 8)
    ki, _ = oracle.topk_codes(k.reshape(-1, 64), 8)
    qi = qi.reshape(2, 4, 80, 8)
    ki = ki.reshape(2, 2, 80 + q_pos0, 8)
    E = accounting.exact_edges(torch.from_numpy(qi), torch.from_numpy(ki), 64, q_pos0=q_pos0, causal=causal)
    assert E == oracle.edge_count(qi, ki, causal=causal, q_pos0=q_pos0)
