"""GPU parity of stage 1 (sfa_topk_codes) against the oracle: indices AND values bit-exact."""
import numpy as np
import pytest

from helpers import from_torch, oracle_codes, to_torch
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu


def run(lib, x_np, dtype, k):
    import torch
    x = to_torch(x_np, dtype)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    idx, val = lib.topk_codes(x, k, status)
    torch.cuda.synchronize()
    return from_torch(idx), from_torch(val), int(status.item())


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("variant", ["iid", "lattice", "skewed"])
def test_random_rows(lib, dtype, d, variant):
    x = inputs.gen(3 + d, 1, (2, 3, 333, d), dtype, variant=variant)  # ragged row count
    for k in sorted({1, 4, 8, 16, d // 2, d - 1, d}):
        gi, gv, st = run(lib, x, dtype, k)
        oi, ov = oracle_codes(x, k)
        assert st == 0
        np.testing.assert_array_equal(gi, oi)
        np.testing.assert_array_equal(gv, ov)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_special_values(lib, dtype):
    """+-0 ties, denormals (no flush-to-zero, A21), max finite, all-equal rows."""
    d = 128
    rows = []
    if dtype == "f32":
        specials = np.array([0.0, -0.0, 1e-45, -1e-45, 1.1754942e-38, -3.4028235e38, 3.4028235e38, 1.0, -1.0],
                            np.float32)
    else:
        specials = inputs.bf16_bits_to_f32(np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x007F, 0xFF7F, 0x7F7F,
                                                      0x3F80, 0xBF80], np.uint16))
    rng = np.random.default_rng(0)
    for _ in range(64):
        rows.append(rng.choice(specials, d))
    rows.append(np.zeros(d, np.float32))
    rows.append(np.full(d, -0.0, np.float32))
    rows.append(np.ones(d, np.float32))
    x = np.stack(rows).astype(np.float32)
    if dtype == "bf16":
        x = inputs.f32_to_bf16_bits(x)
    for k in (1, 3, 16, 64, 128):
        gi, gv, st = run(lib, x, dtype, k)
        oi, ov = oracle_codes(x, k)
        assert st == 0
        np.testing.assert_array_equal(gi, oi)
        np.testing.assert_array_equal(gv.view(np.uint32 if dtype == "f32" else np.uint16),
                                      ov.view(np.uint32 if dtype == "f32" else np.uint16))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_nonfinite_flag(lib, dtype):
    x = inputs.gen(5, 1, (40, 64), "f32")
    x[17, 5] = np.inf
    x[30, 2] = np.nan
    if dtype == "bf16":
        x = inputs.f32_to_bf16_bits(x)
    for k in (8, 64):  # k = d takes the identity kernel: it must flag too
        _, _, st = run(lib, x, dtype, k)
        assert st & 1
        x2 = inputs.gen(5, 1, (40, 64), dtype)
        assert run(lib, x2, dtype, k)[2] == 0


def test_qwen3_shape_all_rows(lib):
    """Every row of a Qwen3-shaped K (B=1, H_kv=8, n=32768, d=128, k=16), generated on the
    device, is bit-exact against the oracle on the host-regenerated K."""
    import torch
    shape = (1, 8, 32768, 128)
    kt = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    lib.gen_fill(kt, 21, inputs.TID_K)
    gi, gv = lib.topk_codes(kt, 16)
    torch.cuda.synchronize()
    k_host = inputs.gen(21, inputs.TID_K, shape, "bf16")
    oi, ov = oracle_codes(k_host, 16)
    np.testing.assert_array_equal(from_torch(gi), oi)
    np.testing.assert_array_equal(from_torch(gv), ov)


@pytest.mark.slow
def test_qwen3_q_codes_all_rows(lib):
    """Every row of a Qwen3-shaped Q (B=1, H=32, n=32768, d=128, k=16: 1M rows), generated on the
    device and coded by sfa_topk_codes, is bit-exact against the oracle on the host-regenerated Q."""
    import torch
    from helpers import gen_big
    shape = (1, 32, 32768, 128)
    qt = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    lib.gen_fill(qt, 21, inputs.TID_Q)
    gi, gv = lib.topk_codes(qt, 16)
    torch.cuda.synchronize()
    del qt
    q_host = gen_big(21, inputs.TID_Q, shape, "bf16")
    oi, ov = oracle_codes(q_host, 16)
    np.testing.assert_array_equal(from_torch(gi), oi)
    np.testing.assert_array_equal(from_torch(gv), ov)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("d,kk", [(64, 8), (128, 16), (128, 4), (128, 127), (128, 128)])
def test_qk_pair_launch_equals_oracle(lib, dtype, d, kk):
    """sfa_topk_codes_qk (Q and K rows in ONE launch, segment per tensor) gives the oracle's codes for
    both tensors, including ragged row counts that end mid-CTA in either segment."""
    q = inputs.gen(77 + d, inputs.TID_Q, (1, 3, 301, d), dtype)
    kx = inputs.gen(77 + d, inputs.TID_K, (1, 1, 173, d), dtype, variant="lattice")
    qi, qv, ki, kv = lib.topk_codes_qk(to_torch(q, dtype), to_torch(kx, dtype), kk)
    import torch
    torch.cuda.synchronize()
    for (gi, gv), x in (((qi, qv), q), ((ki, kv), kx)):
        oi, ov = oracle_codes(x, kk)
        np.testing.assert_array_equal(from_torch(gi), oi)
        np.testing.assert_array_equal(from_torch(gv), ov)
