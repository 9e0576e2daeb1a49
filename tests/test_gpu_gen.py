"""The device input generator (sfa_gen_fill) is bit-identical to the host one (inputs.py)."""
import numpy as np
import pytest

from helpers import from_torch
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("variant,code", [("iid", 0), ("lattice", 1), ("skewed", 2)])
def test_gen_matches_host(lib, dtype, variant, code):
    import torch
    shape = (2, 3, 257, 128)
    t = torch.empty(shape, dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device="cuda")
    lib.gen_fill(t, 1234, inputs.TID_K, variant=code)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(from_torch(t), inputs.gen(1234, inputs.TID_K, shape, dtype, variant=variant))
