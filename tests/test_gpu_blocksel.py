"""GPU parity of SFA composed with NSA-style block selection (sfa_attn_fwd_blocksel)
against the oracle's block-selection mode (pinned in test_oracle_blocksel.py): random ascending key-block
lists, empty lists (O = 0, LSE = -inf), diagonal-only lists, ragged n, GQA, d = 64 keys, and the
all-blocks list, which must reproduce the plain forward bit for bit (same kernel, same tile order)."""
import numpy as np
import pytest

import oracle
from helpers import assert_attn_close, from_torch, host_qkv, oracle_codes, to_torch

pytestmark = pytest.mark.gpu


def make_sel(rng, B, H_kv, n_q, n_kv, max_sel, mode):
    nqb, nkb = (n_q + 127) // 128, (n_kv + 127) // 128
    sel = np.full((B, H_kv, nqb, max_sel), -1, np.int32)
    for b in range(B):
        for g in range(H_kv):
            for qb in range(nqb):
                if mode == "all":
                    chosen = list(range(nkb))
                elif mode == "diag":
                    chosen = [min(qb, nkb - 1)]
                elif mode == "nsa":  # the diagonal block + a few earlier ones, some query blocks empty
                    if rng.random() < 0.15:
                        chosen = []
                    else:
                        earlier = sorted(rng.choice(max(qb, 1), size=min(2, qb), replace=False).tolist()) if qb else []
                        chosen = earlier + [min(qb, nkb - 1)]
                else:  # random subsets, ascending
                    chosen = [t for t in range(nkb) if rng.random() < 0.5]
                chosen = chosen[:max_sel]
                sel[b, g, qb, :len(chosen)] = chosen
    return sel


@pytest.mark.parametrize("mode", ["random", "nsa", "diag", "all"])
@pytest.mark.parametrize("shape", [
    (1, 4, 2, 1000, 128, 128, 16),   # GQA R = 2, ragged
    (2, 8, 2, 700, 64, 128, 8),      # d = 64 keys, R = 4
    (1, 2, 1, 384, 128, 128, 4),
    (1, 4, 2, 500, 64, 64, 8),       # d = d_v = 64 (OT over the zero-padded V copy)
])
@pytest.mark.parametrize("causal", [True, False])
def test_blocksel_against_oracle(lib, mode, shape, causal):
    import torch
    B, H, H_kv, n, d, d_v, k = shape
    q, kx, v = host_qkv(71, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    nkb = (n + 127) // 128
    sel = make_sel(np.random.default_rng(hash((mode, n, d, causal)) % 2 ** 32), B, H_kv, n, n, nkb, mode)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, causal=causal, block_sel=sel)
    o, lse = lib.attn_fwd_blocksel(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"),
                                   to_torch(kv, "bf16"), to_torch(v, "bf16"),
                                   torch.from_numpy(sel).cuda(), d=d, causal=causal)
    torch.cuda.synchronize()
    assert_attn_close(from_torch(o), from_torch(lse), o_ref, l_ref, "bf16")
    if mode == "all":  # every tile listed: the plain forward, bit for bit
        o2, l2 = lib.attn_fwd(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"), to_torch(kv, "bf16"),
                              to_torch(v, "bf16"), d=d, causal=causal, kernel=lib.KERNEL_SM100_OT)
        torch.cuda.synchronize()
        assert torch.equal(o, o2) and torch.equal(lse, l2)


def test_blocksel_qwen3_shape_sampled_rows(lib):
    """Qwen3 heads at n = 8192 with an NSA-like selection (diagonal + 2 earlier blocks), sampled rows."""
    import torch
    B, H, H_kv, n, d, d_v, k = 1, 32, 8, 8192, 128, 128, 16
    q, kx, v = host_qkv(72, B, H, H_kv, n, d, d_v, "bf16")
    qi, qv = oracle_codes(q, k)
    ki, kv = oracle_codes(kx, k)
    sel = make_sel(np.random.default_rng(5), B, H_kv, n, n, 4, "nsa")
    o, lse = lib.attn_fwd_blocksel(to_torch(qi, "u8"), to_torch(qv, "bf16"), to_torch(ki, "u8"),
                                   to_torch(kv, "bf16"), to_torch(v, "bf16"), torch.from_numpy(sel).cuda(), d=d)
    torch.cuda.synchronize()
    rows = np.random.default_rng(6).choice(B * H * n, size=512, replace=False)
    o_ref, l_ref = oracle.attn_fwd(qi, qv, ki, kv, v, d=d, rows=rows, block_sel=sel)
    og = from_torch(o).reshape(-1, d_v)[rows]
    lg = from_torch(lse).reshape(-1)[rows]
    assert_attn_close(og, lg, o_ref, l_ref, "bf16")
