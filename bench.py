#!/usr/bin/env python
"""FlashSFA forward benchmark (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen3] [--kernel auto|simt|sm100]
    python bench.py --impl reference ...      # the fp64 CPU oracle on this box's host cores

One step = one pass of the whole hot path over the workload: top-k codes of Q
and of K (stage 1), the key-side preparation (step 3), FlashSFA attention (stage 2), inputs resident
in HBM.  Multi-GPU (one process per GPU; `--gpus N` re-launches itself under torch.distributed.run
when no launcher set WORLD_SIZE): the config's problem is split by (batch, kv head) units over the
ranks (SURVEY 8(e)-1, strong scaling, no data-path collective), and the `long_context` block of the
same line runs one 128K-token sequence query-block sharded over the same ranks with the NCCL
all-gather of key codes + V.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2603_22300_b200 import accounting  # noqa: E402

METRIC = "FlashSFA fwd ms & tokens/s at n=32K,d=128,k=16; HBM GB/s vs peak; 1/2/4/8 GPU"
L2_BYTES = 126 * 2 ** 20
MUFU_EX2_PER_CLK_SM = 16  # B200 SFU ex2 rate (sm_100; the B300 guide's 2x SFU is sm_103-only)
N_SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen3", choices=sorted(accounting.CONFIGS))
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "sm100", "ot", "pp", "oth"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--window", type=int, default=0,
                    help="causal sliding window (N4: SFA composed with token sparsity); 0 = full causal")
    ap.add_argument("--edges-only", action="store_true",
                    help="reading A1/R2 (SURVEY 8(f) N4): only pairs whose supports intersect enter the softmax")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--separate-topk", action="store_true",
                    help="stage 1 as two launches (Q, then K) instead of one sfa_topk_codes_qk launch")
    ap.add_argument("--graph", action="store_true",
                    help="time the step as one CUDA graph replay (stage split from an extra eager pass)")
    ap.add_argument("--concurrent-stages", action="store_true",
                    help="stage 1 on K and step 3 on a second stream concurrently with stage 1 on Q (measured: no "
                         "gain, the top-k kernels compete for the SMs); default: back to back on one stream")
    ap.add_argument("--no-dense-context", action="store_true", help="skip the dense SDPA context timing")
    ap.add_argument("--fused-q", action="store_true",
                    help="step 1 on Q inside the attention prologue (sfa_attn_fwd_fused_q, N3(ii) ablation)")
    ap.add_argument("--k", type=int, default=None, help="override the code size k (sweep)")
    ap.add_argument("--blocks", type=int, default=8,
                    help="--mode blocksel: key blocks (of 128) each query block selects (its diagonal + earlier ones)")
    ap.add_argument("--mode", default="forward", choices=["forward", "decode", "bwd", "blocksel"],
                    help="decode: SURVEY 8(f) N2, one new query row per sequence over a cached K/V of the config's n")
    ap.add_argument("--decode-batch", type=int, default=8, help="sequences per GPU in --mode decode")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): the config's problem split by (batch, kv head) over the GPUs; weak: "
                         "B = config B x GPUs, one batch element's heads per GPU group")
    ap.add_argument("--seq-len", type=int, default=None, help="override n (e.g. --config long --seq-len 1048576)")
    ap.add_argument("--no-long", action="store_true",
                    help="skip the long_context block (128K tokens query-block sharded over the same GPUs)")
    ap.add_argument("--shard-seq", action="store_true",
                    help="query-block sharding of one sequence (default for --config long under torchrun, N>1; "
                         "with N=1 it exercises the same NCCL path on one GPU)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=d["hbm_gbs"], bf16_tflops=d["bf16_tflops"], sm_max_mhz=d.get("sm_max_mhz", 1965.0),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, sm_max_mhz=1965.0, source="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# --------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference): the oracle as it stands, on a bounded sample
# --------------------------------------------------------------------------------------------
def oracle_sample(W, seed, n_rows, n_topk_rows, threads):
    """Time the oracle on a bounded sample of the workload, extrapolated to tokens/s.

    Sample: top-k of n_topk_rows Q rows and n_topk_rows K rows, plus the attention of n_rows
    uniformly random (head, position) query rows over all of their allowed keys (the causal
    row cost is linear in the position, so a uniform sample is unbiased)."""
    import numpy as np

    import oracle
    from paper_2603_22300_b200 import inputs
    rng = np.random.default_rng(seed)
    B, H, H_kv, n, d, d_v, k = 1, W.H, W.H_kv, W.n, W.d, W.d_v, W.k
    # inputs for the sample (generation is not timed)
    kx = inputs.gen(seed, inputs.TID_K, (B, H_kv, n, d), W.dtype)
    v = inputs.gen(seed, inputs.TID_V, (B, H_kv, n, d_v), W.dtype)
    rows = np.sort(rng.choice(B * H * n, n_rows, replace=False)).astype(np.int64)
    qflat = rows[:, None] * d + np.arange(d)[None, :]
    q_rows = inputs.gen(seed, inputs.TID_Q, (B, H, n, d), W.dtype, flat=qflat)
    q_top = inputs.gen(seed, inputs.TID_Q, (n_topk_rows, d), W.dtype)
    # --- timed: top-k sample
    t0 = time.perf_counter()
    oracle.topk_codes(q_top, k)
    oracle.topk_codes(kx.reshape(-1, d)[:n_topk_rows], k)
    t_topk = time.perf_counter() - t0
    # codes the attention sample needs (all keys of the kv heads, the sampled query rows): untimed
    ki, kv = oracle.topk_codes(kx.reshape(-1, d), k)
    qi_r, qv_r = oracle.topk_codes(q_rows, k)
    qi = np.zeros((B, H, n, k), np.uint8)
    qv = np.zeros((B, H, n, k), qv_r.dtype)
    qi.reshape(-1, k)[rows] = qi_r
    qv.reshape(-1, k)[rows] = qv_r
    t0 = time.perf_counter()
    oracle.attn_fwd(qi, qv, ki.reshape(B, H_kv, n, k), kv.reshape(B, H_kv, n, k), v, d=d, rows=rows,
                    threads=threads)
    t_attn = time.perf_counter() - t0
    total_rows_q = B * H * n
    total_rows_topk = B * (H + H_kv) * n
    t_full = t_attn * total_rows_q / n_rows + t_topk * total_rows_topk / (2 * n_topk_rows)
    return {"tokens_per_s": B * n / t_full, "t_sample": t_topk + t_attn, "t_full_extrapolated": t_full,
            "sample": f"{n_rows} uniformly random (head, position) query rows of the {W.H}x{W.n} grid over all "
                      f"their allowed keys + top-k of {n_topk_rows} Q and {n_topk_rows} K rows; "
                      f"linear extrapolation to the full {B}x{H}x{n} workload"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, W, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # size each step so warmup+steps finish in about 2-3 minutes on this host
    budget_s = 150.0 / max(1, args.steps + args.warmup)
    n_rows = 64
    probe = oracle_sample(W, 7, n_rows, 256, threads)
    per_row = probe["t_sample"] / n_rows
    n_rows = int(max(16, min(4096, budget_s / max(per_row, 1e-6))))
    for i in range(args.warmup):
        oracle_sample(W, 100 + i, n_rows, 256, threads)
    vals, ts = [], []
    for i in range(args.steps):
        r = oracle_sample(W, 200 + i, n_rows, 256, threads)
        vals.append(r["tokens_per_s"])
        ts.append(r["t_full_extrapolated"])
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(ts),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based generator, DESIGN.md input recipe)",
            "config": config_of(args, W),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": r["sample"]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(args, W, B_glob=None, world=1):
    B_glob = W.B if B_glob is None else B_glob
    units = B_glob * W.H_kv
    par = (f"(batch, kv head) sharding (SURVEY 8(e)-1, sfa_dist_head_shard): the {units} units of the "
           f"B={B_glob} problem in {world} contiguous range{'s' if world > 1 else ''}, "
           f"{units // world}{'-' + str(-(-units // world)) if units % world else ''} per GPU; "
           "no data-path collective")
    return {"workload": f"{args.config}: B={B_glob}, H={W.H}, H_kv={W.H_kv}, n={W.n}, d={W.d}, d_v={W.d_v}, "
                        f"k={W.k}, {'causal' if W.causal else 'non-causal'}, {W.dtype} V",
            "global_batch": B_glob, "seq_len": W.n,
            "parallelism": par + (" (weak: B grows with the GPU count)" if getattr(args, "scaling", "strong") == "weak"
                                  else " (strong: fixed global problem)"),
            "kernel": args.kernel,
            "semantics": ("R2 edges-only (A1/R2)" if getattr(args, "edges_only", False) else "R1 (A1)")
                         + (f", causal sliding window {args.window} (N4)" if getattr(args, "window", 0) else ""),
            "q_topk": "fused into the attention prologue (N3(ii)); stage_ms.attn includes it"
                      if (getattr(args, "fused_q", False) and not getattr(args, "edges_only", False) and W.d_v == 128
                          and W.dtype == "bf16" and args.kernel in ("auto", "ot")) else "own kernel",
            "l2": f"explicit {L2_FLUSH_MB} MB write between timed steps (outside the step events); "
                  "inputs+outputs also exceed the 126 MB L2"}


L2_FLUSH_MB = 512


# --------------------------------------------------------------------------------------------
def run_bwd(args, W, rank, world, local):
    """the backward with the straight-through rule (sfa_attn_bwd) on the metric's
    workload.  Inputs: codes of generated Q/K, V, the forward's O/LSE, a generated upstream dO.  The
    step is the D prep + the dK~/dV and dQ~ tensor-core kernels (P recomputed from the codes)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2603_22300_b200 import inputs, sfa
    dev = torch.device("cuda", local)
    B, H, H_kv, n, d, d_v, k = W.B, W.H, W.H_kv, W.n, W.d, W.d_v, W.k
    seed = accounting.SEEDS[args.config]
    bf = torch.bfloat16
    Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=bf, device=dev), seed, inputs.TID_Q, offset=rank * B * H * n * d)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=bf, device=dev), seed, inputs.TID_K, offset=rank * B * H_kv * n * d)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=bf, device=dev), seed, inputs.TID_V,
                     offset=rank * B * H_kv * n * d_v)
    dO = sfa.gen_fill(torch.empty((B, H, n, d_v), dtype=bf, device=dev), seed, inputs.TID_DO,
                      offset=rank * B * H * n * d_v)
    qi, qv = sfa.topk_codes(Q, k)
    ki, kv = sfa.topk_codes(K, k)
    del Q, K
    O, LSE = sfa.attn_fwd(qi, qv, ki, kv, V, d=d, causal=W.causal)
    f32 = dict(dtype=torch.float32, device=dev)
    dq, dk, dv = (torch.empty((B, H, n, k), **f32), torch.empty((B, H_kv, n, k), **f32),
                  torch.empty((B, H_kv, n, d_v), **f32))
    desc = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=n, n_kv=n, causal=W.causal)
    L = sfa.lib()
    ws = torch.empty(max(int(L.sfa_attn_bwd_workspace_bytes(ctypes.byref(desc))), 16), dtype=torch.uint8, device=dev)
    flush = torch.empty(L2_FLUSH_MB * 2 ** 20, dtype=torch.uint8, device=dev)
    P_ = lambda t: ctypes.c_void_p(t.data_ptr())
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def step():
        r = L.sfa_attn_bwd(ctypes.byref(desc), P_(qi), P_(qv), P_(ki), P_(kv), P_(V), P_(O), P_(LSE), P_(dO), P_(dq),
                           P_(dk), P_(dv), P_(ws), ws.numel(), st())
        if r:
            raise RuntimeError(f"sfa_attn_bwd failed: {r}")

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e0, e1 in evs:
            flush.zero_()
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pk = peaks()
    pairs = B * H * accounting.causal_pairs(n, n, 0, W.causal)
    # tensor FLOPs per allowed pair: S and dP recomputed in both kernels (2 x (2d + 2d_v)), then
    # dV (2 d_v), dK~ (2 d) and dQ~ (2 d)
    flops = pairs * (8 * d + 6 * d_v)
    tf = flops / (ms / 1e3) / 1e12
    if rank == 0:
        line = {"metric": "FlashSFA backward (straight-through rule) ms & tokens/s at n=32K, d=128, k=16 (SURVEY 8(f) N1)",
                "value": B * n * world / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded generator; codes from sfa_topk_codes)",
                "config": {"workload": f"{args.config} backward: B={B} per GPU, H={H}, H_kv={H_kv}, n={n}, d={d}, "
                                       f"d_v={d_v}, k={k}, causal", "global_batch": B * world, "seq_len": n,
                           "parallelism": "weak: batch element r on rank r", "l2": f"explicit {L2_FLUSH_MB} MB write between steps"},
                "roofline": {"bound": "tensor", "kernel": "bwd_dkdv_kernel + bwd_dq_kernel",
                             "achieved": tf, "peak": pk["bf16_tflops"], "unit": "TFLOP/s", "frac": tf / pk["bf16_tflops"],
                             "traffic": None, "flops_per_pair": 8 * d + 6 * d_v,
                             "mufu_floor_ms": 2 * pairs / (N_SMS * MUFU_EX2_PER_CLK_SM * pk["sm_max_mhz"] * 1e6) * 1e3},
                "cpu_baseline": None, "e2e": None, "gpu_launches": 3 * args.steps, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def run_blocksel(args, W, rank, world, local):
    """the forward composed with NSA-style block selection (sfa_attn_fwd_blocksel): every
    query block of 128 rows attends its diagonal key block and --blocks - 1 earlier ones (spread evenly,
    deterministic), intersected with the causal mask.  The step is stage 1 (Q + K codes, one launch) +
    step 3 + the attention over the listed tiles.  Context: the full causal SFA step on the same inputs."""
    import ctypes

    import numpy as np
    import torch

    from paper_2603_22300_b200 import inputs, sfa
    dev = torch.device("cuda", local)
    B, H, H_kv, n, d, d_v, k = W.B, W.H, W.H_kv, W.n, W.d, W.d_v, W.k
    seed = accounting.SEEDS[args.config]
    bf = torch.bfloat16
    Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=bf, device=dev), seed, inputs.TID_Q)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=bf, device=dev), seed, inputs.TID_K)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=bf, device=dev), seed, inputs.TID_V)
    nqb = (n + 127) // 128
    S = max(1, args.blocks)
    sel = np.full((B, H_kv, nqb, S), -1, np.int32)
    for qb in range(nqb):  # the diagonal block + S - 1 earlier ones spread evenly over [0, qb)
        chosen = sorted(set([int(x) for x in np.linspace(0, qb - 1, S - 1)] if qb > 0 and S > 1 else []) | {qb})
        sel[:, :, qb, :len(chosen)] = chosen
    sel_t = torch.from_numpy(sel).to(dev)
    selected_pairs = 0  # allowed pairs: causal within the listed blocks
    for qb in range(nqb):
        rows = min(128, n - qb * 128)
        for t in sel[0, 0, qb]:
            if t < 0:
                continue
            if t < qb:
                selected_pairs += rows * min(128, n - t * 128)
            elif t == qb:
                selected_pairs += rows * (rows + 1) // 2
    selected_pairs *= B * H
    qi = torch.empty((B, H, n, k), dtype=torch.uint8, device=dev); qv = torch.empty((B, H, n, k), dtype=bf, device=dev)
    ki = torch.empty((B, H_kv, n, k), dtype=torch.uint8, device=dev); kv = torch.empty((B, H_kv, n, k), dtype=bf, device=dev)
    desc = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=n, n_kv=n, causal=True)
    L = sfa.lib()
    ws = torch.empty(sfa.workspace_bytes(desc), dtype=torch.uint8, device=dev)
    O = torch.empty((B, H, n, d_v), dtype=bf, device=dev); LSE = torch.empty((B, H, n), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_MB * 2 ** 20, dtype=torch.uint8, device=dev)
    P_ = lambda t: ctypes.c_void_p(t.data_ptr())
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def step(full, ev=None):
        if ev: ev[0].record()
        r1 = L.sfa_topk_codes_qk(P_(Q), B * H * n, d, P_(qi), P_(qv), P_(K), B * H_kv * n, d, P_(ki), P_(kv),
                                 desc.dtype, d, k, None, st())
        if ev: ev[1].record()
        if full:
            r2 = L.sfa_attn_fwd(ctypes.byref(desc), P_(qi), P_(qv), P_(ki), P_(kv), P_(V), P_(O), P_(LSE), P_(ws),
                                ws.numel(), st())
        else:
            r2 = L.sfa_attn_fwd_blocksel(ctypes.byref(desc), P_(qi), P_(qv), P_(ki), P_(kv), P_(V), P_(sel_t), S,
                                         P_(O), P_(LSE), P_(ws), ws.numel(), st())
        if ev: ev[2].record()
        if r1 or r2:
            raise RuntimeError(f"sfa call failed: {(r1, r2)}")

    def timed(full):
        for _ in range(args.warmup):
            flush.zero_()
            step(full)
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        with ClockSampler(local) as clk:
            for e in evs:
                flush.zero_()
                step(full, e)
            torch.cuda.synchronize()
        tot = sum(e[0].elapsed_time(e[2]) for e in evs) / args.steps
        att = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
        return tot, att, clk.summary()

    ms, att_ms, clocks = timed(False)
    full_ms, full_att_ms, _ = timed(True)
    pk = peaks()
    mufu_peak = N_SMS * MUFU_EX2_PER_CLK_SM * pk["sm_max_mhz"] * 1e6
    if rank == 0:
        line = {"metric": "FlashSFA fwd with NSA-style block selection, ms & tokens/s (SURVEY 8(f) N4)",
                "value": B * n / (ms / 1e3), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded generator on device)",
                "config": {"workload": f"{args.config}: B={B}, H={H}, H_kv={H_kv}, n={n}, d={d}, d_v={d_v}, k={k}, "
                                       f"causal, {S} key blocks of 128 per query block (diagonal + {S - 1} earlier)",
                           "global_batch": B, "seq_len": n, "l2": f"explicit {L2_FLUSH_MB} MB write between steps"},
                "stage_ms": {"topk_qk": ms - att_ms, "prepare_and_attn": att_ms},
                "selected_pairs": selected_pairs,
                "roofline": {"bound": "alu", "kernel": "attn_sm100_ot_kernel<BSEL>", "unit": "G pairs/s",
                             "achieved": selected_pairs / (att_ms / 1e3) / 1e9, "peak": mufu_peak / 1e9,
                             "frac": selected_pairs / (att_ms / 1e3) / mufu_peak},
                "context": {"full_causal_step_ms": full_ms, "full_causal_prepare_and_attn_ms": full_att_ms},
                "cpu_baseline": None, "e2e": None, "gpu_launches": 6 * args.steps, "clocks": clocks}
        print(json.dumps(line), flush=True)


def run_decode(args, W, rank, world, local):
    """a decode step -- one query row per (sequence, head) against a K/V cache of n
    tokens already coded (k-sparse key codes + bf16 V in HBM).  HBM-bound: the algorithmic traffic is
    the cache read, n * (3k + 2 d_v) bytes per (sequence, kv head)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2603_22300_b200 import inputs, sfa
    dev = torch.device("cuda", local)
    B, H, H_kv, n, d, d_v, k = args.decode_batch, W.H, W.H_kv, W.n, W.d, W.d_v, W.k
    seed = accounting.SEEDS[args.config]
    bf = torch.bfloat16
    Qn = sfa.gen_fill(torch.empty((B, H, 1, d), dtype=bf, device=dev), seed, inputs.TID_Q, offset=rank * B * H * d)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=bf, device=dev), seed, inputs.TID_K, offset=rank * B * H_kv * n * d)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=bf, device=dev), seed, inputs.TID_V,
                     offset=rank * B * H_kv * n * d_v)
    qi, qv = sfa.topk_codes(Qn, k)
    ki, kv = sfa.topk_codes(K, k)  # the cache, coded once (not part of a decode step)
    # context only: the same decode step over a DENSE bf16 K/V cache through torch SDPA (flash decode
    # backend), L2 flushed the same way -- what the k-sparse cache replaces
    dense_ctx = None
    if rank == 0 and not args.no_dense_context:
        try:
            import torch.nn.functional as F
            fl = torch.empty(L2_FLUSH_MB * 2 ** 20, dtype=torch.uint8, device=dev)
            for _ in range(3):
                F.scaled_dot_product_attention(Qn, K, V, enable_gqa=True)
            tms = []
            for _ in range(10):
                fl.zero_()
                c0 = torch.cuda.Event(enable_timing=True); c1 = torch.cuda.Event(enable_timing=True)
                c0.record()
                F.scaled_dot_product_attention(Qn, K, V, enable_gqa=True)
                c1.record()
                torch.cuda.synchronize()
                tms.append(c0.elapsed_time(c1))
            del fl
            dms = sum(tms) / len(tms)
            dense_ctx = {"dense_sdpa_ms": dms, "dense_cache_bytes": B * H_kv * n * (d + d_v) * 2,
                         "dense_sdpa_gbs": B * H_kv * n * (d + d_v) * 2 / (dms / 1e3) / 1e9,
                         "note": "torch SDPA (bf16, GQA) over the dense K/V cache of the same shape; context only"}
        except Exception as ex:
            dense_ctx = {"dense_sdpa_error": str(ex)[:200]}
    del K
    desc = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=1, n_kv=n, q_pos0=n - 1,
                         kernel=sfa.KERNEL_DECODE)
    ws = torch.empty(max(sfa.workspace_bytes(desc), 16), dtype=torch.uint8, device=dev)
    O = torch.empty((B, H, 1, d_v), dtype=bf, device=dev)
    LSE = torch.empty((B, H, 1), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_MB * 2 ** 20, dtype=torch.uint8, device=dev)
    L = sfa.lib()
    P_ = lambda t: ctypes.c_void_p(t.data_ptr())
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def step():
        r = L.sfa_attn_fwd_prepared(ctypes.byref(desc), P_(qi), P_(qv), P_(ki), P_(kv), P_(V), P_(O), P_(LSE), P_(ws),
                                    ws.numel(), st())
        if r:
            raise RuntimeError(f"sfa_attn_fwd_prepared failed: {r}")

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e0, e1 in evs:
            flush.zero_()
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    cache_bytes = B * H_kv * n * (k * 3 + d_v * 2)
    io_bytes = B * H * (k * 3 + d_v * 2 + 4)
    pk = peaks()
    gbs = (cache_bytes + io_bytes) / (ms / 1e3) / 1e9
    if rank == 0:
        line = {"metric": "FlashSFA decode step: tokens/s and HBM GB/s over a k-sparse KV cache (SURVEY 8(f) N2)",
                "value": B * world / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded generator; cache coded with sfa_topk_codes)",
                "config": {"workload": f"decode: {B} sequences x H={H} (H_kv={H_kv}) x 1 new token over a {n}-token cache, "
                                       f"d={d}, d_v={d_v}, k={k}", "global_batch": B * world, "seq_len": n,
                           "parallelism": "weak: independent sequences per rank",
                           "l2": f"explicit {L2_FLUSH_MB} MB write between steps; cache {cache_bytes / 2**20:.0f} MiB"},
                "roofline": {"bound": "hbm", "kernel": "decode_partial_kernel + decode_combine_kernel",
                             "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
                             "traffic": None, "algorithmic_bytes_per_step": cache_bytes + io_bytes,
                             "dense_kv_cache_bytes_for_comparison": B * H_kv * n * (d + d_v) * 2},
                "cpu_baseline": None, "e2e": None, "gpu_launches": 2 * args.steps, "clocks": clk.summary(),
                "context": dense_ctx}
        print(json.dumps(line), flush=True)


def measure_sharded(W, seed, rank, world, local, steps, warmup, workload_name="long"):
    """Long-context query-block sharding: one sequence of n tokens over `world`
    GPUs, zig-zag chunks (the library's sfa_dist_zigzag_chunk), one NCCL all-gather of key codes + V
    per step through sfa_dist_allgather_kv (strong scaling).  Needs an initialised process group (for
    the NCCL id broadcast).  Returns rank 0's JSON object (None elsewhere)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2603_22300_b200 import dist as sdist
    from paper_2603_22300_b200 import inputs, sfa
    dev = torch.device("cuda", local)
    B, H, H_kv, n, d, d_v, k = W.B, W.H, W.H_kv, W.n, W.d, W.d_v, W.k
    c = sdist.chunk_size(n, world)
    chunks = sdist.owned_chunks(rank, world)
    bf = torch.bfloat16

    def local_fill(hh, dd, tid):  # chunk-major [2][B][hh][c][dd] slice of the global [B][hh][n][dd] tensor
        t = torch.empty((2, B, hh, c, dd), dtype=bf, device=dev)
        for half, q in enumerate(chunks):
            for b in range(B):
                for h in range(hh):
                    sfa.gen_fill(t[half, b, h], seed, tid, offset=((b * hh + h) * n + q * c) * dd)
        return t

    Q, K, V = local_fill(H, d, inputs.TID_Q), local_fill(H_kv, d, inputs.TID_K), local_fill(H_kv, d_v, inputs.TID_V)
    sh = sdist.ShardedAttention()
    L = sfa.lib()
    P_ = lambda t: ctypes.c_void_p(t.data_ptr())
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    qi = torch.empty((2, B, H, c, k), dtype=torch.uint8, device=dev)
    qv = torch.empty((2, B, H, c, k), dtype=bf, device=dev)
    ki = torch.empty((2, B, H_kv, c, k), dtype=torch.uint8, device=dev)
    kv = torch.empty((2, B, H_kv, c, k), dtype=bf, device=dev)
    kfi = torch.empty((B, H_kv, n, k), dtype=torch.uint8, device=dev)
    kfv = torch.empty((B, H_kv, n, k), dtype=bf, device=dev)
    vf = torch.empty((B, H_kv, n, d_v), dtype=bf, device=dev)
    ldesc = sfa.make_desc(B=B, H=H_kv, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=2 * c, n_kv=2 * c)
    nst = int(L.sfa_dist_staging_bytes(ctypes.byref(ldesc), world))
    staging = torch.empty(nst, dtype=torch.uint8, device=dev)
    desc = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=c, n_kv=n, causal=W.causal)
    ws = torch.empty(max(sfa.workspace_bytes(desc), 16), dtype=torch.uint8, device=dev)
    O = torch.empty((2, B, H, c, d_v), dtype=bf, device=dev)
    LSE = torch.empty((2, B, H, c), dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_MB * 2 ** 20, dtype=torch.uint8, device=dev)

    def step(ev=None):
        if ev: ev[0].record()
        r = [L.sfa_topk_codes(P_(Q), sfa.SFA_BF16, 2 * B * H * c, d, d, k, P_(qi), P_(qv), P_(status), st()),
             L.sfa_topk_codes(P_(K), sfa.SFA_BF16, 2 * B * H_kv * c, d, d, k, P_(ki), P_(kv), P_(status), st())]
        if ev: ev[1].record()
        r.append(L.sfa_dist_allgather_kv(sh._h, ctypes.byref(ldesc), P_(ki), P_(kv), P_(V), P_(kfi), P_(kfv), P_(vf),
                                         P_(staging), nst, st()))
        if ev: ev[2].record()
        r.append(L.sfa_attn_prepare(ctypes.byref(desc), P_(kfi), P_(kfv), P_(vf), P_(ws), ws.numel(), st()))
        if ev: ev[3].record()
        for half, q in enumerate(chunks):
            desc.q_pos0 = q * c
            r.append(L.sfa_attn_fwd_prepared(ctypes.byref(desc), P_(qi[half]), P_(qv[half]), P_(kfi), P_(kfv),
                                             P_(vf), P_(O[half]), P_(LSE[half]), P_(ws), ws.numel(), st()))
        if ev: ev[4].record()
        if any(r):
            raise RuntimeError(f"sfa call failed: {r}")

    for _ in range(warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(steps):
            flush.zero_()
            step(evs[i])
        torch.cuda.synchronize()
    dist.barrier()
    per = [[e[j].elapsed_time(e[j + 1]) for j in range(4)] for e in evs]
    tot = torch.tensor([sum(sum(p) for p in per)], dtype=torch.float64, device=dev)
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = float(tot.item()) / steps
    stage = [sum(p[j] for p in per) / steps for j in range(4)]
    stage_max = torch.tensor(stage, dtype=torch.float64, device=dev)
    dist.all_reduce(stage_max, op=dist.ReduceOp.MAX)
    stage_max = [float(x) for x in stage_max.tolist()]
    pairs_rank = B * H * sdist.causal_pairs_of_rank(rank, world, n)
    pk = peaks()
    mufu_peak = N_SMS * MUFU_EX2_PER_CLK_SM * pk["sm_max_mhz"] * 1e6
    achieved = pairs_rank / (stage_max[3] / 1e3)
    ag_bytes = world * (ki.numel() + kv.numel() * 2 + V.numel() * 2)
    sh.close()
    if rank != 0:
        return None
    return {"metric": METRIC, "value": B * n / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter-based generator on device, DESIGN.md input recipe)",
            "config": {"workload": f"{workload_name}: B={B}, H={H}, H_kv={H_kv}, n={n}, d={d}, d_v={d_v}, k={k}, "
                                   f"causal, bf16 V; one sequence query-block sharded over {world} GPU(s)",
                       "global_batch": B, "seq_len": n,
                       "parallelism": f"zig-zag query blocks x{world} (chunks p, 2P-1-p of {c} tokens), "
                                      "one NCCL all-gather of key codes + V per step (sfa_dist_allgather_kv)",
                       "l2": f"explicit {L2_FLUSH_MB} MB write between timed steps"},
            "stage_ms": {"topk_qk": stage_max[0], "allgather_kv": stage_max[1], "prepare": stage_max[2],
                         "attn": stage_max[3], "note": "each stage's max over ranks"},
            "allgather_bytes_total": ag_bytes,
            "allgather_bytes_received_per_rank": ag_bytes * (world - 1) // world,
            "roofline": {"bound": "alu", "kernel": ("attn_sm100_ot_kernel" if W.d_v == 128 else "attn_sm100_kernel")
                         + " (steps 4-8), slowest rank", "achieved": achieved / 1e9, "peak": mufu_peak / 1e9,
                         "unit": "G pairs/s (1 MUFU ex2 per allowed causal pair)", "frac": achieved / mufu_peak,
                         "traffic": None, "peak_source": "148 SMs x 16 ex2/clk x max SM clock"},
            "cpu_baseline": None, "e2e": None,
            "gpu_launches": 10 * steps, "clocks": clk.summary()}


def spawn_ranks(args):
    """`--gpus N` (N > 1) without a launcher: run this same command as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1) and exit with its status."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def init_group(world, rank, local):
    """torch.distributed for the plumbing: NCCL when there are several ranks; a 1-rank gloo group when a
    single process needs a group (the NCCL id broadcast of the sharded path)."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        return
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(s.getsockname()[1])
    s.close()
    dist.init_process_group("gloo", rank=0, world_size=1)


def main():
    args = parse()
    W = accounting.CONFIGS[args.config]
    if args.k is not None:
        W = accounting.Workload(**{**W.__dict__, "k": args.k})
    if args.seq_len is not None:
        W = accounting.Workload(**{**W.__dict__, "n": args.seq_len})
    if args.impl == "reference":
        run_reference(args, W, int(os.environ.get("RANK", "0")))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but this launch has WORLD_SIZE={world} ranks")
    import torch
    import torch.distributed as dist

    from paper_2603_22300_b200 import dist as sdist
    from paper_2603_22300_b200 import inputs, sfa
    torch.cuda.set_device(local)
    if torch.cuda.device_count() < world and local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} has no GPU (only {torch.cuda.device_count()} visible)")
    if args.mode == "bwd":
        if world > 1:
            init_group(world, rank, local)
        run_bwd(args, W, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.mode == "blocksel":
        run_blocksel(args, W, rank, world, local)
        return
    if args.mode == "decode":
        if world > 1:
            init_group(world, rank, local)
        run_decode(args, W, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.shard_seq or (args.config == "long" and world > 1):
        init_group(world, rank, local)
        line = measure_sharded(W, accounting.SEEDS[args.config], rank, world, local, args.steps, args.warmup,
                               workload_name=args.config)
        if rank == 0:
            print(json.dumps(line), flush=True)
        dist.destroy_process_group()
        return
    if world > 1:
        init_group(world, rank, local)
    kernel = {"auto": sfa.KERNEL_AUTO, "simt": sfa.KERNEL_SIMT, "sm100": sfa.KERNEL_SM100,
              "ot": sfa.KERNEL_SM100_OT, "pp": sfa.KERNEL_SM100_PP, "oth": sfa.KERNEL_SM100_OTH}[args.kernel]
    dt = torch.bfloat16 if W.dtype == "bf16" else torch.float32
    seed = accounting.SEEDS[args.config]
    dev = torch.device("cuda", local)
    # The global problem: B = W.B (strong scaling, the default) or W.B * world (weak: one batch element per
    # rank).  It is split by (batch, kv head) units over the ranks (sfa_dist_head_shard): this
    # rank's units [u0, u0 + sub.B) are contiguous in every global tensor, so the rank generates exactly that
    # slice of the seeded global Q, K, V (generator offset = first element of its units) and runs the whole hot
    # path on it as the problem (B = #units, H = H/H_kv, H_kv = 1).  No data-path collective.
    B_glob = W.B * (world if args.scaling == "weak" else 1)
    full = sfa.make_desc(B=B_glob, H=W.H, H_kv=W.H_kv, d=W.d, k=W.k, d_v=W.d_v, n_q=W.n, n_kv=W.n, causal=W.causal,
                         dtype=sfa.SFA_BF16 if W.dtype == "bf16" else sfa.SFA_F32, kernel=kernel,
                         edges_only=args.edges_only, window=args.window)
    desc, u0 = sdist.head_shard(full, world, rank)
    B, H, H_kv, n, d, d_v, k = desc.B, desc.H, desc.H_kv, W.n, W.d, W.d_v, W.k
    Q = torch.empty((B, H, n, d), dtype=dt, device=dev)
    K = torch.empty((B, H_kv, n, d), dtype=dt, device=dev)
    V = torch.empty((B, H_kv, n, d_v), dtype=dt, device=dev)
    sfa.gen_fill(Q, seed, inputs.TID_Q, offset=u0 * H * n * d)
    sfa.gen_fill(K, seed, inputs.TID_K, offset=u0 * n * d)
    sfa.gen_fill(V, seed, inputs.TID_V, offset=u0 * n * d_v)
    q_idx = torch.empty((B, H, n, k), dtype=torch.uint8, device=dev)
    q_val = torch.empty((B, H, n, k), dtype=dt, device=dev)
    k_idx = torch.empty((B, H_kv, n, k), dtype=torch.uint8, device=dev)
    k_val = torch.empty((B, H_kv, n, k), dtype=dt, device=dev)
    ws = torch.empty(sfa.workspace_bytes(desc), dtype=torch.uint8, device=dev)
    O = torch.empty((B, H, n, d_v), dtype=dt, device=dev)
    LSE = torch.empty((B, H, n), dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_MB * 2 ** 20, dtype=torch.uint8, device=dev)
    L = sfa.lib()
    import ctypes
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    dcode = desc.dtype

    fused_q = (W.dtype == "bf16" and d_v == 128 and args.kernel in ("auto", "ot") and not args.edges_only
               and args.fused_q)

    # the key path (stage 1 on K, step 3) is independent of stage 1 on Q: it runs on a second stream and
    # joins before the attention with --concurrent-stages (default: one stream, the stages back to back)
    s2 = torch.cuda.Stream(device=dev)
    kev = {}

    def step(ev=None):
        # stage 1 on Q, stage 1 on K, step 3 (V prep for sm100 / buckets for simt), steps 4-8 attention
        if ev: ev[0].record()
        if not args.concurrent_stages and not fused_q and not args.separate_topk:
            # stage 1 on Q and on K in one launch (sfa_topk_codes_qk); stage slot 1 stays empty
            r1 = L.sfa_topk_codes_qk(P(Q), B * H * n, d, P(q_idx), P(q_val), P(K), B * H_kv * n, d, P(k_idx),
                                     P(k_val), dcode, d, k, P(status), st())
            r2 = 0
            if ev: ev[1].record()
            if ev: ev[2].record()
            r3 = L.sfa_attn_prepare(ctypes.byref(desc), P(k_idx), P(k_val), P(V), P(ws), ws.numel(), st())
            if ev: ev[3].record()
        elif not args.concurrent_stages:
            r1 = 0 if fused_q else L.sfa_topk_codes(P(Q), dcode, B * H * n, d, d, k, P(q_idx), P(q_val), P(status), st())
            if ev: ev[1].record()
            r2 = L.sfa_topk_codes(P(K), dcode, B * H_kv * n, d, d, k, P(k_idx), P(k_val), P(status), st())
            if ev: ev[2].record()
            r3 = L.sfa_attn_prepare(ctypes.byref(desc), P(k_idx), P(k_val), P(V), P(ws), ws.numel(), st())
            if ev: ev[3].record()
        else:
            fork = torch.cuda.Event()
            fork.record()
            s2.wait_event(fork)
            with torch.cuda.stream(s2):
                if ev: kev[id(ev)][0].record()
                r2 = L.sfa_topk_codes(P(K), dcode, B * H_kv * n, d, d, k, P(k_idx), P(k_val), P(status), st())
                if ev: kev[id(ev)][1].record()
                r3 = L.sfa_attn_prepare(ctypes.byref(desc), P(k_idx), P(k_val), P(V), P(ws), ws.numel(), st())
                if ev: kev[id(ev)][2].record()
                join = torch.cuda.Event()
                join.record()
            r1 = 0 if fused_q else L.sfa_topk_codes(P(Q), dcode, B * H * n, d, d, k, P(q_idx), P(q_val), P(status), st())
            if ev: ev[1].record()
            torch.cuda.current_stream().wait_event(join)
            if ev: ev[2].record()
            if ev: ev[3].record()
        if fused_q:  # step 1 on Q inside the attention prologue (N3(ii)); the q codes are still written out
            r4 = L.sfa_attn_fwd_fused_q(ctypes.byref(desc), P(Q), P(k_idx), P(k_val), P(V), P(O), P(LSE), P(q_idx),
                                        P(q_val), P(status), P(ws), ws.numel(), st())
        else:
            r4 = L.sfa_attn_fwd_prepared(ctypes.byref(desc), P(q_idx), P(q_val), P(k_idx), P(k_val), P(V), P(O),
                                         P(LSE), P(ws), ws.numel(), st())
        if ev: ev[4].record()
        if r1 or r2 or r3 or r4:
            raise RuntimeError(f"sfa call failed: {(r1, r2, r3, r4)}")

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for e in evs:
        kev[id(e)] = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    graph = None
    if args.graph:  # the whole step as one CUDA graph (launch gaps of the 4-6 kernels collapse)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()  # L2 flush: outside the step's events
            if graph is not None:
                evs[i][0].record()
                graph.replay()
                evs[i][4].record()
            else:
                step(evs[i])
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    if world > 1:
        dist.barrier()
    if graph is not None:  # the step from the replays; the stage split from as many eager steps
        tot_ms = sum(e[0].elapsed_time(e[4]) for e in evs)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
        for e in evs:
            kev[id(e)] = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        for i in range(args.steps):
            flush.zero_()
            step(evs[i])
        torch.cuda.synchronize()
    per = [[e[j].elapsed_time(e[j + 1]) for j in range(4)] for e in evs]  # ms per stage per step
    step_ms = [sum(p) for p in per]
    if graph is None:
        tot_ms = sum(step_ms)
    stage_ms = [sum(p[j] for p in per) / args.steps for j in range(4)]
    join_wait_ms = None
    if args.concurrent_stages:  # key path timed on its own stream; [1] + [2] of `per` are the join wait
        join_wait_ms = stage_ms[1] + stage_ms[2]
        stage_ms[1] = sum(kev[id(e)][0].elapsed_time(kev[id(e)][1]) for e in evs) / args.steps
        stage_ms[2] = sum(kev[id(e)][1].elapsed_time(kev[id(e)][2]) for e in evs) / args.steps
    if world > 1:  # the whole-job step time is the slowest rank's; stages likewise
        t = torch.tensor([tot_ms] + stage_ms, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, stage_ms = float(t[0].item()), [float(x) for x in t[1:].tolist()]
    ms_per_step = tot_ms / args.steps
    tokens_per_step = B_glob * n  # every rank's units together = the global problem
    value = tokens_per_step / (ms_per_step / 1e3)
    torch.cuda.synchronize()
    if int(status.item()) != 0:
        raise RuntimeError("non-finite inputs flagged")

    # ---- end to end through the C ABI with HOST buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        qh = Q.cpu().pin_memory(); kh = K.cpu().pin_memory(); vh = V.cpu().pin_memory()
        oh = torch.empty(O.shape, dtype=dt).pin_memory()
        lh = torch.empty(LSE.shape, dtype=torch.float32).pin_memory()
        scratch = torch.empty(sfa.scratch_bytes(desc), dtype=torch.uint8, device=dev)
        bufs = (torch.empty_like(Q), torch.empty_like(K), torch.empty_like(V), torch.empty_like(O),
                torch.empty_like(LSE))
        chunks = min(8, B * H_kv)  # pipelined: copies overlap the kernels (sfa_forward_host_pipelined)
        for _ in range(max(1, args.warmup)):
            sfa.forward_host(desc, qh, kh, vh, oh, lh, bufs, scratch, chunks=chunks)
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(e2e_steps):
            sfa.forward_host(desc, qh, kh, vh, oh, lh, bufs, scratch, chunks=chunks)
        e1.record()
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        h2d = (Q.numel() + K.numel() + V.numel()) * Q.element_size()
        d2h = O.numel() * O.element_size() + LSE.numel() * 4 + 4
        e2e = {"value": tokens_per_step / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": f"sfa_forward_host_pipelined, {chunks} chunks (pinned host q,k,v -> o,lse; H2D, kernels and "
                      "D2H of neighbouring chunks overlap; synchronised)"}
        del qh, kh, vh, oh, lh, scratch, bufs

    # context only (not a step, not a target): dense causal attention on the same shapes through torch's
    # SDPA (FlashAttention/cuDNN backend on B200), bf16 Q, K, V with GQA -- what the codes replace
    context = None
    if rank == 0 and world == 1 and W.dtype == "bf16" and not args.no_dense_context and not args.window:
        try:
            import torch.nn.functional as F
            qd, kd, vd = Q, K, V
            for _ in range(2):
                F.scaled_dot_product_attention(qd, kd, vd, is_causal=W.causal, enable_gqa=True)
            torch.cuda.synchronize()
            c0 = torch.cuda.Event(enable_timing=True); c1 = torch.cuda.Event(enable_timing=True)
            c0.record()
            for _ in range(5):
                F.scaled_dot_product_attention(qd, kd, vd, is_causal=W.causal, enable_gqa=True)
            c1.record()
            torch.cuda.synchronize()
            dense_ms = c0.elapsed_time(c1) / 5
            dpairs = B * H * accounting.causal_pairs(n, n, 0, W.causal)
            context = {"dense_sdpa_ms": dense_ms, "dense_sdpa_tflops": 2.0 * (d + d_v) * dpairs / (dense_ms / 1e3) / 1e12,
                       "sfa_attention_ms": stage_ms[3], "sfa_step_ms": ms_per_step,
                       "note": "torch.nn.functional.scaled_dot_product_attention(bf16, causal, GQA) on the dense "
                               "Q, K, V of the same step; context only, not part of the step or a target"}
        except Exception as ex:  # context is optional
            context = {"dense_sdpa_error": str(ex)[:200]}

    qk_fused = not args.concurrent_stages and not fused_q and not args.separate_topk
    # our kernels per step: stage 1 (1 fused launch, 2 separate, 1 for K when Q is fused into the attention),
    # step 3 (sm100: max|V| + fp16 V, + the decompressed K~ rows for OT/PP, + R2 bitsets; simt: buckets),
    # the attention kernel
    kern_res = args.kernel if args.kernel != "auto" else ("ot" if d_v == 128 else "sm100")
    launches_per_step = (1 if (qk_fused or fused_q) else 2) + 1
    if W.dtype == "bf16" and args.kernel != "simt":
        launches_per_step += 2 + int(kern_res in ("ot", "pp", "oth")) + int(bool(args.edges_only))
    else:
        launches_per_step += 1
    pk = peaks()
    attn_ms = stage_ms[3]
    pairs = B * H * accounting.causal_pairs(n, n, 0, W.causal, args.window)  # this rank's units
    mufu_peak = N_SMS * MUFU_EX2_PER_CLK_SM * pk["sm_max_mhz"] * 1e6  # ex2/s
    achieved = pairs / (attn_ms / 1e3)  # attn_ms: the slowest rank's (ranks hold equal work up to one unit)
    traffic = None  # dram__bytes_read + dram__bytes_write per launch of the attention kernel (ncu --set full)
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            ent = json.load(open(tp)).get(args.config, {}).get(f"attn_{args.kernel}" + ("_fusedq" if fused_q else ""))
            traffic = ent["dram_bytes_per_launch"] if ent else None
        except Exception:
            traffic = None
    s_v = 2 if W.dtype == "bf16" else 4
    topk_bytes = B * (H + H_kv) * n * (d * s_v + k * (1 + s_v))  # this rank's rows (stage times are its own)
    if fused_q:  # only the K rows go through the stand-alone top-k kernel
        topk_bytes = B * H_kv * n * (d * s_v + k * (1 + s_v))
    # exact score interactions E of the whole job (prefix counts over the codes this step computed)
    E_rank = accounting.exact_edges(q_idx, k_idx, d, causal=bool(W.causal)) if not args.window else None
    E_total = None
    if E_rank is not None:
        E_total = E_rank
        if world > 1:
            t = torch.tensor([E_rank], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            E_total = int(t.item())
    pairs_total = B_glob * W.H * accounting.causal_pairs(n, n, 0, W.causal, args.window)
    sm100 = W.dtype == "bf16" and args.kernel != "simt"
    kname = {"auto": "attn_sm100_ot_kernel" if d_v == 128 else "attn_sm100_kernel", "sm100": "attn_sm100_kernel",
             "ot": "attn_sm100_ot_kernel", "pp": "attn_sm100_pp_kernel", "oth": "attn_sm100_oth_kernel",
             "simt": "attn_simt_kernel"}[args.kernel if sm100 else "simt"]
    roofline = {"bound": "alu", "kernel": kname + (" (step 1 on Q fused + steps 4-8)" if fused_q else " (steps 4-8)"),
                "achieved": achieved / 1e9, "peak": mufu_peak / 1e9,
                "unit": "G pairs/s (1 MUFU ex2 per allowed causal pair)",
                "frac": achieved / mufu_peak, "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch (ncu --set full capture, profiles/ncu_traffic.json); "
                                f"algorithmic minimum {W.attn_min_bytes()} B",
                "peak_source": f"148 SMs x 16 ex2/clk (measured, profiles/r02_mufu_bench.txt) x {pk['sm_max_mhz']:.0f} MHz",
                "other_floors": {
                    # tensor pipe: S = Q~K~^T (2d) + P.V (2 d_v) FLOPs per allowed pair, vs the measured bf16 peak
                    "tensor_frac": (2.0 * (d + d_v) * pairs / (attn_ms / 1e3)) / (pk["bf16_tflops"] * 1e12)
                    if sm100 else None,
                    "tensor_pv_frac": (2.0 * d_v * pairs / (attn_ms / 1e3)) / (pk["bf16_tflops"] * 1e12),
                    "hbm_attn_frac": (W.attn_min_bytes() / (attn_ms / 1e3)) / (pk["hbm_gbs"] * 1e9),
                    "topk_hbm_gbs": topk_bytes / ((stage_ms[0] + stage_ms[1]) / 1e3) / 1e9,
                    "topk_hbm_frac": topk_bytes / ((stage_ms[0] + stage_ms[1]) / 1e3) / (pk["hbm_gbs"] * 1e9),
                    "peaks": pk["source"]}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        # bounded sample of ~15 s of CPU work: a 1024-row probe sizes the timed sample
        probe = oracle_sample(W, seed + 1, 1024, 2048, threads)
        n_rows = int(max(1024, min(W.H * W.n // 2, 1024 * 16.0 / max(probe["t_sample"], 1e-3))))
        r = oracle_sample(W, seed, n_rows, 2048, threads)
        cpu = {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": threads, "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": r["sample"], "sample_seconds": r["t_sample"]}
    # the north star's long-context requirement in the same line: one 128K-token sequence query-block sharded
    # over the same ranks (zig-zag + the NCCL all-gather of key codes and V), strong scaling
    long_ctx = None
    if not args.no_long and args.config != "long" and W.dtype == "bf16" and W.d_v == 128 and not args.window \
            and not args.edges_only and args.kernel in ("auto", "ot"):
        init_group(world, rank, local)
        del flush
        torch.cuda.empty_cache()
        WL = accounting.CONFIGS["long"]
        try:
            long_ctx = measure_sharded(WL, accounting.SEEDS["long"], rank, world, local,
                                       steps=max(2, min(args.steps, 5)), warmup=3)
        except Exception as ex:  # reported, never hidden
            long_ctx = {"error": str(ex)[:300]}
        if long_ctx is not None:
            long_ctx = {key: long_ctx[key] for key in ("value", "unit", "ms_per_step", "steps", "warmup", "scaling",
                                                       "config", "stage_ms", "allgather_bytes_total",
                                                       "allgather_bytes_received_per_rank", "roofline", "clocks")
                        if key in long_ctx} if "error" not in long_ctx else long_ctx
    if rank == 0:
        scaling = "weak" if args.scaling == "weak" else "strong"
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": W.dtype,
                "data": "synthetic (seeded counter-based generator on device, DESIGN.md input recipe)",
                "config": config_of(args, W, B_glob, world),
                "stage_ms": ({"topk_qk": stage_ms[0]} if qk_fused else {"topk_q": stage_ms[0], "topk_k": stage_ms[1]}) |
                            {"prepare": stage_ms[2], "attn": stage_ms[3],
                             "note": ("topk_k and prepare run on a second stream concurrently with topk_q; the step "
                                      f"waited {join_wait_ms:.4f} ms for them after topk_q")
                             if join_wait_ms is not None else "stages back to back on one stream; each stage's "
                                                              "max over ranks" +
                             ("; topk_qk = Q and K codes in one launch (sfa_topk_codes_qk)" if qk_fused else "") +
                             ("; the step timed as CUDA graph replays, the stage split from as many eager steps"
                              if args.graph else "")},
                "interactions": E_total,
                "interactions_per_s": E_total / (ms_per_step / 1e3) if E_total is not None else None,
                "interactions_note": "exact E = sum over allowed pairs of |S_i & S_j| (P:L114-120), prefix counts "
                                     "over this step's codes (accounting.exact_edges)",
                "pairs_per_s": pairs_total / (ms_per_step / 1e3),
                "wall_s_timed_region": t_wall,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clk.summary(), "context": context, "long_context": long_ctx}
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
