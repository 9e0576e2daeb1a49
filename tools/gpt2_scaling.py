"""GPT-2-shaped attention (H=12, n=1024, d=d_v=64, k=8, causal) vs batch size: prepared attention only
(sfa_attn_fwd_prepared), CUDA events, median of 50 -- separates the per-tile cost from fixed costs."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_22300_b200 import inputs, sfa  # noqa: E402

L = sfa.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())
H, d, k = 12, 64, 8
shapes = [(B, 1024) for B in (1, 2, 4, 8, 16, 32)] + [(8, 2048), (2, 4096), (1, 8192), (1, 16384)]
for kern_name in sys.argv[1:] or ["sm100", "ot"]:
    kern = {"sm100": sfa.KERNEL_SM100, "ot": sfa.KERNEL_SM100_OT}[kern_name]
    for B, n in shapes:
        q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device="cuda"), 11, inputs.TID_Q)
        kx = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device="cuda"), 11, inputs.TID_K)
        v = sfa.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device="cuda"), 11, inputs.TID_V)
        qi, qv = sfa.topk_codes(q, k)
        ki, kv = sfa.topk_codes(kx, k)
        desc = sfa.make_desc(B=B, H=H, H_kv=H, d=d, k=k, d_v=d, n_q=n, n_kv=n, kernel=kern)
        ws = torch.empty(sfa.workspace_bytes(desc), dtype=torch.uint8, device="cuda")
        o = torch.empty((B, H, n, d), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((B, H, n), dtype=torch.float32, device="cuda")
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert L.sfa_attn_prepare(ctypes.byref(desc), P(ki), P(kv), P(v), P(ws), ws.numel(), st) == 0
        ts = []
        for it in range(60):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = L.sfa_attn_fwd_prepared(ctypes.byref(desc), P(qi), P(qv), P(ki), P(kv), P(v), P(o), P(lse), P(ws),
                                        ws.numel(), st)
            e1.record()
            torch.cuda.synchronize()
            assert r == 0
            if it >= 10:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        tiles = B * H * sum(2 * p + 2 for p in range(n // 256))  # 2-tile items (h, 2p, 2p+1): 2p+2 key tiles
        print(f"{kern_name} B={B:3d} n={n:6d} attention {ts[len(ts) // 2]:8.1f} us  item-tile-steps {tiles:6d}  "
              f"per SM {tiles / 148:7.1f}  us/step/SM {ts[len(ts) // 2] / (tiles / 148):6.2f}", flush=True)
