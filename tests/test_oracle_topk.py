"""Pins for the oracle's top-k coding (oracle/sfa_oracle.c ref_topk_codes).

Topk_k(x)_u = x_u if u in arg topk(|x|) else 0   (Sec. 3.1 Eq. topk_QK).
Readings: ties -> lower index (A2), ascending output (A4), exactly k entries (A8).
The pins are independent of the oracle's code: the paper/SPEC worked examples
(tests/golden/paper_examples.json), brute force over all C(d,k) subsets with exact
rational sums, and the SPEC S:L95-99 invariants.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2603_22300_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


@pytest.mark.parametrize("case", GOLD["topk"], ids=lambda c: c["cite"][:20])
def test_paper_vectors(case):
    x = np.array([case["x"]], np.float32)
    idx, val = oracle.topk_codes(x, case["k"])
    assert idx[0].tolist() == case["idx"]
    assert val[0].tolist() == case["val"]


def brute_force_support(x_row, k):
    """Lexicographically smallest index set among those maximising sum |x| (exact rationals).

    A set maximises sum |x| iff it holds k largest magnitudes; among the tied choices the
    lexicographically smallest sorted tuple is the lowest-index one (reading A2)."""
    mags = [abs(Fraction(float(v))) for v in x_row]
    best, best_set = None, None
    for comb in itertools.combinations(range(len(x_row)), k):  # generated in lexicographic order
        s = sum(mags[u] for u in comb)
        if best is None or s > best:
            best, best_set = s, comb
    return list(best_set)


@pytest.mark.parametrize("variant", ["iid", "lattice"])
@pytest.mark.parametrize("d,k", [(4, 1), (6, 2), (8, 3), (8, 4), (10, 5), (9, 9)])
def test_brute_force(variant, d, k):
    x = inputs.gen_f32(5 + d * 10 + k, 1, (64, d), variant=variant)
    idx, val = oracle.topk_codes(x, k)
    for r in range(x.shape[0]):
        sup = brute_force_support(x[r], k)
        assert idx[r].tolist() == sup
        assert val[r].tolist() == [float(x[r, u]) for u in sup]


def test_brute_force_bf16():
    bits = inputs.gen(7, 2, (64, 8), "bf16", variant="lattice")
    idx, val = oracle.topk_codes(bits, 3)
    xf = inputs.bf16_bits_to_f32(bits)
    for r in range(bits.shape[0]):
        sup = brute_force_support(xf[r], 3)
        assert idx[r].tolist() == sup
        assert val[r].tolist() == [int(bits[r, u]) for u in sup]  # bit copies


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("d,k", [(64, 8), (128, 16), (128, 1), (128, 128)])
def test_invariants(dtype, d, k):
    """max outside <= min inside; determinism; ascending; scale equivariance."""
    x = inputs.gen(11, 1, (200, d), dtype)
    idx, val = oracle.topk_codes(x, k)
    xf = x if dtype == "f32" else inputs.bf16_bits_to_f32(x)
    for r in range(0, 200, 7):
        sel = set(idx[r].tolist())
        assert len(sel) == k and sorted(sel) == idx[r].tolist()
        inside = np.abs(xf[r, list(sel)])
        outside = np.abs(np.delete(xf[r], list(sel)))
        if outside.size:
            assert outside.max() <= inside.min()
    idx2, val2 = oracle.topk_codes(x, k)
    assert np.array_equal(idx, idx2) and np.array_equal(val, val2)
    if dtype == "f32":  # c = 4 is exact in fp32
        idx4, val4 = oracle.topk_codes(x * np.float32(4.0), k)
        assert np.array_equal(idx, idx4)
        assert np.array_equal(val4, val * np.float32(4.0))


def test_signed_zero_and_denormal():
    tiny = np.float32(1e-45)  # fp32 denormal: must outrank +-0 (no flush-to-zero in the definition)
    x = np.array([[-0.0, 0.0, tiny, -tiny, 0.0, 0.0]], np.float32)
    idx, val = oracle.topk_codes(x, 3)
    assert idx[0].tolist() == [0, 2, 3]
    assert np.signbit(val[0, 0]) and val[0, 1] == tiny and val[0, 2] == -tiny


def test_errors():
    x = np.ones((2, 8), np.float32)
    for k in (0, 9):
        with pytest.raises(oracle.OracleError) as e:
            oracle.topk_codes(x, k)
        assert e.value.code == 1  # invalid-argument
    x[1, 3] = np.inf
    with pytest.raises(oracle.OracleError) as e:
        oracle.topk_codes(x, 2)
    assert e.value.code == 2  # invalid-input (A14)
    x[1, 3] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.topk_codes(x, 2)
