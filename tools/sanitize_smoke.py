"""Small end-to-end runs of every product kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_22300_b200 import inputs, sfa  # noqa: E402


def run(B, H, H_kv, n, d, d_v, k, dtype, kernel):
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=dt, device="cuda"), 1, inputs.TID_Q)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=dt, device="cuda"), 1, inputs.TID_K)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=dt, device="cuda"), 1, inputs.TID_V)
    o, lse = sfa.forward(Q, K, V, k_code=k, kernel=kernel)
    torch.cuda.synchronize()
    assert torch.isfinite(lse).all()


if __name__ == "__main__":
    run(1, 1, 1, 256, 64, 64, 8, "f32", sfa.KERNEL_SIMT)          # tiny config, CUDA-core path
    run(1, 4, 2, 300, 128, 128, 16, "bf16", sfa.KERNEL_SIMT)
    run(1, 4, 2, 300, 128, 128, 16, "bf16", sfa.KERNEL_SM100)     # default tensor-core path
    run(2, 3, 3, 200, 64, 64, 8, "bf16", sfa.KERNEL_SM100)        # MHA pairing, d = 64
    run(1, 4, 2, 520, 128, 128, 16, "bf16", sfa.KERNEL_SM100_PAIR)
    run(1, 4, 2, 520, 128, 128, 16, "bf16", sfa.KERNEL_SM100_WIDE)
    print("sanitize smoke ok")
