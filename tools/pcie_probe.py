"""PCIe copy-rate probe for the e2e leg: pinned H2D of the Qwen3 step inputs, D2H of its outputs,
alone and concurrently (CUDA events)."""
import torch

def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

hin = torch.empty(402653184, dtype=torch.uint8).pin_memory()
din = torch.empty_like(hin, device="cuda")
hout = torch.empty(272629764, dtype=torch.uint8).pin_memory()
dout = torch.empty_like(hout, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2d = t(lambda: din.copy_(hin, non_blocking=True))
d2h = t(lambda: hout.copy_(dout, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bo = t(both)
print(f"H2D {h2d:.2f} ms ({402653184/h2d/1e6:.1f} GB/s)  D2H {d2h:.2f} ms ({272629764/d2h/1e6:.1f} GB/s)  concurrent {bo:.2f} ms")
