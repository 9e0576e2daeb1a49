"""Small end-to-end runs of every product kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_22300_b200 import inputs, sfa  # noqa: E402


def run(B, H, H_kv, n, d, d_v, k, dtype, kernel, edges_only=False, n_q=None):
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    Q = sfa.gen_fill(torch.empty((B, H, n_q or n, d), dtype=dt, device="cuda"), 1, inputs.TID_Q)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=dt, device="cuda"), 1, inputs.TID_K)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=dt, device="cuda"), 1, inputs.TID_V)
    o, lse = sfa.forward(Q, K, V, k_code=k, kernel=kernel, edges_only=edges_only,
                         q_pos0=(n - n_q) if n_q else 0)
    torch.cuda.synchronize()
    if not edges_only:
        assert torch.isfinite(lse).all()


def run_bwd(B, H, H_kv, n, d, d_v, k):
    dt = torch.bfloat16
    Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=dt, device="cuda"), 2, inputs.TID_Q)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=dt, device="cuda"), 2, inputs.TID_K)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=dt, device="cuda"), 2, inputs.TID_V)
    dO = sfa.gen_fill(torch.empty((B, H, n, d_v), dtype=dt, device="cuda"), 2, 7)
    qi, qv = sfa.topk_codes(Q, k)
    ki, kv = sfa.topk_codes(K, k)
    o, lse = sfa.attn_fwd(qi, qv, ki, kv, V, d=d)
    dq, dk, dv = sfa.attn_bwd(qi, qv, ki, kv, V, o, lse, dO, d=d)
    torch.cuda.synchronize()
    assert torch.isfinite(dq).all() and torch.isfinite(dk).all() and torch.isfinite(dv).all()


if __name__ == "__main__":
    run(1, 1, 1, 256, 64, 64, 8, "f32", sfa.KERNEL_SIMT)          # tiny config, CUDA-core path
    run(1, 4, 2, 300, 128, 128, 16, "bf16", sfa.KERNEL_SIMT)
    run(1, 4, 2, 300, 128, 128, 16, "bf16", sfa.KERNEL_AUTO)       # AUTO = SM100_OT (d_v = 128), the default
    run(1, 4, 2, 300, 128, 128, 16, "bf16", sfa.KERNEL_SM100)      # SM100 (default for d_v = 64)
    run(2, 3, 3, 200, 64, 64, 8, "bf16", sfa.KERNEL_SM100)         # MHA pairing, d = 64
    run(1, 4, 2, 300, 128, 128, 4, "bf16", sfa.KERNEL_AUTO, edges_only=True)   # R2 on SM100_OT
    run(1, 2, 1, 200, 64, 64, 2, "f32", sfa.KERNEL_SIMT, edges_only=True)      # R2 on SIMT
    run(2, 8, 2, 3000, 128, 128, 16, "bf16", sfa.KERNEL_DECODE, n_q=1)         # decode shape
    run_bwd(1, 4, 2, 300, 128, 128, 16)                                        # backward kernels
    # round 2: the persistent OT scheduler with more items than SMs (256 items: every CTA claims several),
    # d = 64 keys, the fused Q + K top-k launch and the K~ rows, then the ablation kernels
    run(4, 16, 4, 1024, 128, 128, 16, "bf16", sfa.KERNEL_AUTO)
    run(2, 8, 2, 700, 64, 128, 8, "bf16", sfa.KERNEL_SM100_OT)
    run(1, 4, 2, 300, 128, 128, 16, "bf16", sfa.KERNEL_SM100_PP)
    run(1, 4, 2, 300, 128, 64, 16, "bf16", sfa.KERNEL_SM100_PP)
    run(2, 8, 2, 700, 128, 128, 16, "bf16", sfa.KERNEL_SM100_OTH)
    print("sanitize smoke ok")
