"""Hand-off timeline of the sm100 kernel's CTA 0 (library built with SFA_NVCC_FLAGS=-DSFA_TIMELINE).

Runs one non-causal forward whose work item 0 has NT key tiles and prints, per 64-key sub-tile u,
when each softmax group saw S(u) ready and stored P(u), and when the MMA warp saw P(u)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_22300_b200 import inputs, sfa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kern = {"sm100": sfa.KERNEL_SM100, "ot": sfa.KERNEL_SM100_OT,
        "pp": sfa.KERNEL_SM100_PP, "oth": sfa.KERNEL_SM100_OTH}[sys.argv[2] if len(sys.argv) > 2 else "sm100"]
qwen = len(sys.argv) > 3 and sys.argv[3] == "qwen"  # bench config: causal, H=32, H_kv=8 (item 0 = last q block)
B, H, H_kv, d, d_v, k = (1, 32, 8, 128, 128, 16) if qwen else (1, 2, 1, 128, 128, 16)
dev = "cuda"
Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device=dev), 3, inputs.TID_Q)
K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=torch.bfloat16, device=dev), 3, inputs.TID_K)
V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=torch.bfloat16, device=dev), 3, inputs.TID_V)
qi, qv = sfa.topk_codes(Q, k)
ki, kv = sfa.topk_codes(K, k)
for _ in range(2):
    o, lse, S, tlb = sfa.debug_sm100_scores(qi, qv, ki, kv, V, d=d, causal=qwen, kernel=kern)
torch.cuda.synchronize()
raw = tlb.cpu().numpy().view(np.uint64)
rec = raw[1:]
rec = rec[rec != 0]
cnt = len(rec)
tag = (rec >> np.uint64(48)).astype(np.int64)
clk = (rec & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
clk -= clk.min()
names = {1: "S_ready", 2: "P_stored", 3: "mma_sawP", 4: "max_done", 5: "max", 6: "bar", 7: "pempty"}
ev = {}
for tg, c in zip(tag, clk):
    kind, t, u = tg >> 12, (tg >> 10) & 3, tg & 1023
    ev[(names[kind], t, u)] = c
nu = max(u for (_, _, u) in ev) + 1
if len(sys.argv) > 2 and sys.argv[2] == "oth":  # 64-key halves u: S ready, max/bar done, P computed, P slot free, P stored, MMA saw P
    print(f"{cnt} records, {nu} score halves; clocks relative to the first record")
    print("  u | tile 0: Srdy   bar  exps  Pfree  Pst | tile 1: Srdy   bar  exps  Pfree  Pst | mmaP | period")
    prev = None
    for u in range(nu):
        r = [[ev.get((nm, t, u), -1) for nm in ("S_ready", "max", "max_done", "pempty", "P_stored")] for t in (0, 1)]
        mp = ev.get(("mma_sawP", 0, u), -1)
        per = r[0][0] - prev if prev is not None else 0
        prev = r[0][0]
        print(f"{u:3d} | " + " ".join(f"{x:6d}" for x in r[0]) + " | " + " ".join(f"{x:6d}" for x in r[1]) + f" | {mp:6d} | {per}")
    sys.exit(0)
if len(sys.argv) > 2 and sys.argv[2] == "pp":  # ping-pong kernel: S ready, max done, turn, P stored, MMA saw P
    print(f"{cnt} records, {nu} key tiles; clocks relative to the first record")
    print("  j | tile 0: Srdy  maxd  turn  Pst   mmaP  | tile 1: Srdy  maxd  turn  Pst   mmaP  | exp0  exp1 | period")
    prev = None
    for u in range(nu):
        r0 = [ev.get((nm, 0, u), -1) for nm in ("S_ready", "max_done", "max", "P_stored", "mma_sawP")]
        r1 = [ev.get((nm, 1, u), -1) for nm in ("S_ready", "max_done", "max", "P_stored")] + [ev.get(("mma_sawP", 1, u), -1)]
        per = r0[0] - prev if prev is not None else 0
        prev = r0[0]
        print(f"{u:3d} | " + " ".join(f"{x:6d}" for x in r0) + " | " + " ".join(f"{x:6d}" for x in r1) +
              f" | {r0[3]-r0[2]:5d} {r1[3]-r1[2]:5d} | {per}")
    sys.exit(0)
print(f"{cnt} records, {nu} key tiles; clocks relative to the first record")
print(" j | S0rdy  P0st  mmaP  | S1rdy  P1st  issued | softmax0 softmax1 | max0 max1 | period(S0rdy)")
prev = None
for u in range(nu):
    row = [ev.get(("S_ready", 0, u), -1), ev.get(("P_stored", 0, u), -1), ev.get(("mma_sawP", 0, u), -1),
           ev.get(("S_ready", 1, u), -1), ev.get(("P_stored", 1, u), -1), ev.get(("mma_sawP", 1, u), -1)]
    per = row[0] - prev if prev is not None else 0
    prev = row[0]
    print(f"{u:3d} | {row[0]:6d} {row[1]:6d} {row[2]:6d} | {row[3]:6d} {row[4]:6d} {row[5]:6d} | "
          f"{row[1]-row[0]:6d} {row[4]-row[3]:6d} | {ev.get(('max_done', 0, u), row[0]) - row[0]:5d} "
          f"{ev.get(('max_done', 1, u), row[3]) - row[3]:5d} | {per}" +
          ("" if ("max", 0, u) not in ev else
           " | t0 max %5d bar %5d half0 %5d pempty %5d stored %5d" % tuple(ev.get((n_, 0, u), 0) - row[0] for n_ in
                                                                      ("max", "bar", "max_done", "pempty", "P_stored"))))
