"""Shared test helpers: seeded inputs on host and device, oracle-side codes, tolerance checks.

The tolerances are the north star's (BASELINE.json): top-k indices bit-exact; O and LSE
within max-abs 2e-3 with bf16 V, or 1e-5 relative with fp32.  Reading A13:
bf16 -- the 2e-3 bar applies to the arithmetic; the GPU's O is additionally rounded to the
bf16 output dtype (RNE, unit roundoff 2^-8), so elementwise |dO| <= 2e-3 + 2^-8 |O_ref|;
LSE is fp32 and must meet 2e-3 outright.  fp32 -- |dO| <= 1e-5 max(1, |O_ref|), LSE likewise.
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_2603_22300_b200 import inputs

TOL_BF16 = 2e-3
TOL_F32_REL = 1e-5
BF16_U = 2.0 ** -8  # unit roundoff of the bf16 output rounding


def host_qkv(seed, B, H, H_kv, n, d, d_v, dtype, variant="iid", n_kv=None):
    return inputs.qkv(seed, B, H, H_kv, n, d, d_v, dtype, variant=variant, n_kv=n_kv)


def to_torch(a, dtype, device="cuda"):
    import torch
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def from_torch(t):
    import torch
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def oracle_codes(x, k):
    shp = x.shape
    idx, val = oracle.topk_codes(x.reshape(-1, shp[-1]), k)
    return idx.reshape(shp[:-1] + (k,)), val.reshape(shp[:-1] + (k,))


def o_as_f64(o, dtype):
    return (inputs.bf16_bits_to_f32(o) if dtype == "bf16" else o).astype(np.float64)


def _log_parity(err_o, plain, err_l, n_el, n_small):
    """SFA_PARITY_LOG=<file>: one JSON line per bf16 comparison (test id, errors) -- the committed parity
    headroom summary (profiles/) is made from it."""
    import json
    import os
    path = os.environ.get("SFA_PARITY_LOG")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0],
                            "max_excess_o": float(err_o), "max_abs_o_small": plain, "max_abs_lse": float(err_l),
                            "elements": int(n_el), "elements_abs_o_lt_0.5": n_small}) + "\n")


def assert_attn_close(o_gpu, lse_gpu, o_ref, lse_ref, dtype):
    """o_gpu/lse_gpu: numpy (o in storage dtype); refs fp64."""
    og = o_as_f64(o_gpu, dtype)
    lg = lse_gpu.astype(np.float64)
    assert og.shape == o_ref.shape and lg.shape == lse_ref.shape
    # rows with no allowed key / no edge (A10, R2): LSE must be -inf exactly, O exactly 0
    dead = np.isneginf(lse_ref)
    assert np.array_equal(np.isneginf(lg), dead), "rows with LSE = -inf differ"
    assert np.all(og[dead] == 0.0), "rows with no allowed key must have O = 0"
    lg = np.where(dead, 0.0, lg)
    lse_ref = np.where(dead, 0.0, lse_ref)
    if dtype == "bf16":
        excess = np.abs(og - o_ref) - BF16_U * np.abs(o_ref)
        err_o = excess.max()
        err_l = np.abs(lg - lse_ref).max()
        # the north star's plain max-abs bar where it applies outright (|O| < 0.5: the bf16 output rounding
        # is <= 2^-10 there), so the headroom is visible
        small = np.abs(o_ref) < 0.5
        plain = float(np.abs(og - o_ref)[small].max()) if small.any() else 0.0
        _log_parity(err_o, plain, err_l, og.size, int(small.sum()))
        assert err_o <= TOL_BF16, f"max (|dO| - 2^-8|O_ref|) = {err_o}"
        assert plain <= TOL_BF16, f"max |dO| over |O_ref| < 0.5 = {plain}"
        assert err_l <= TOL_BF16, f"max |dLSE| = {err_l}"
    else:
        err_o = (np.abs(og - o_ref) / np.maximum(1.0, np.abs(o_ref))).max()
        err_l = (np.abs(lg - lse_ref) / np.maximum(1.0, np.abs(lse_ref))).max()
        assert err_o <= TOL_F32_REL, f"max rel |dO| = {err_o}"
        assert err_l <= TOL_F32_REL, f"max rel |dLSE| = {err_l}"
    return err_o, err_l


def gen_big(seed, tensor_id, shape, dtype, chunk=1 << 24):
    """inputs.gen for tensors too large to hash in one numpy call (256K-1M configs): the same values,
    generated chunk by chunk of flat indices (bounded temporary memory)."""
    total = int(np.prod(shape))
    out = np.empty(total, np.uint16 if dtype == "bf16" else np.float32)
    for s in range(0, total, chunk):
        e = min(total, s + chunk)
        out[s:e] = inputs.gen(seed, tensor_id, shape, dtype, flat=np.arange(s, e, dtype=np.int64))
    return out.reshape(shape)
