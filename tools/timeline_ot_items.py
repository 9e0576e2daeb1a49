"""Hand-off timeline of the persistent SM100_OT kernel's CTA 0 over several work items (library built with
SFA_NVCC_FLAGS=-DSFA_TIMELINE): per cumulative key tile u, when each softmax warpgroup saw S(u) ready and
stored P(u), and when the MMA warp saw P(u); per item, when the epilogue saw O^T complete (OFULL) and
when it finished its global stores.  Shape: GPT-2 heads (H = 12, d = d_v = 64, k = 8, causal) at B, n."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_22300_b200 import inputs, sfa  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
H, d, k = 12, 64, 8
dev = "cuda"
Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device=dev), 11, inputs.TID_Q)
K = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device=dev), 11, inputs.TID_K)
V = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device=dev), 11, inputs.TID_V)
qi, qv = sfa.topk_codes(Q, k)
ki, kv = sfa.topk_codes(K, k)
for _ in range(3):
    o, lse, S, tlb = sfa.debug_sm100_scores(qi, qv, ki, kv, V, d=d, causal=True, kernel=sfa.KERNEL_SM100_OT)
torch.cuda.synchronize()
raw = tlb.cpu().numpy().view(np.uint64)[1:]
raw = raw[raw != 0]
tag = (raw >> np.uint64(48)).astype(np.int64)
clk = (raw & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
clk -= clk.min()
ev = {}
for tg, c in zip(tag, clk):
    ev[(tg >> 12, (tg >> 10) & 1, tg & 511)] = int(c)
nu = 1 + max(u for (kd, _, u) in ev if kd in (1, 2, 3))
print(f"B={B} n={n}: {len(raw)} records, {nu} key tiles on CTA 0 (clocks from the first record)")
print("   u | S0rdy  P0st | S1rdy  P1st | mmaP | P0-S0 P1-S1 | period")
prev = None
for u in range(nu):
    r = [ev.get((1, 0, u), -1), ev.get((2, 0, u), -1), ev.get((1, 1, u), -1), ev.get((2, 1, u), -1), ev.get((3, 0, u), -1)]
    per = r[0] - prev if prev is not None and r[0] >= 0 else 0
    prev = r[0] if r[0] >= 0 else prev
    print(f"{u:4d} | {r[0]:6d} {r[1]:6d} | {r[2]:6d} {r[3]:6d} | {r[4]:6d} | {r[1]-r[0]:5d} {r[3]-r[2]:5d} | {per}")
print("item | t0: OFULL  stored | t1: OFULL  stored")
m = 0
while (8, 0, 2 * m) in ev:
    print(f"{m:4d} | {ev.get((8, 0, 2 * m), -1):6d} {ev.get((8, 0, 2 * m + 1), -1):6d} | "
          f"{ev.get((8, 1, 2 * m), -1):6d} {ev.get((8, 1, 2 * m + 1), -1):6d}")
    m += 1
