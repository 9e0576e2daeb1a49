"""Work and byte accounting for the bench (host logic, no GPU, no oracle).

Every number the bench divides by a measured time comes from here, so each formula
is pinned in tests/test_accounting.py against the paper's own tables.
"""
from __future__ import annotations

from dataclasses import dataclass


def causal_pairs(n_q: int, n_kv: int, q_pos0: int = 0, causal: bool = True, window: int = 0) -> int:
    """Allowed (query, key) pairs of one head: sum_i min(n_kv, q_pos0 + i + 1); with a causal sliding
    window w > 0 (N4) key j also needs j > q_pos0 + i - w."""
    if not causal:
        return n_q * n_kv
    if window > 0:
        return sum(max(0, min(n_kv - 1, q_pos0 + i) - max(0, q_pos0 + i - window + 1) + 1) for i in range(n_q))
    tot = 0
    # rows whose window is still growing: q_pos0 + i + 1 <= n_kv
    grow = max(0, min(n_q, n_kv - q_pos0))
    a, b = q_pos0 + 1, q_pos0 + grow
    tot += (a + b) * grow // 2
    tot += (n_q - grow) * n_kv
    return tot


def predicted_edges(n: int, d: int, k: int) -> float:
    """E ~ n^2 k^2 / d (Sec. 3.1 "Efficiency analysis"), non-causal, balanced supports."""
    return n * n * k * k / d


def appb_flops(BH: int, n: int, d: int, d_v: int, k: int | None) -> float:
    """The App.-B FLOP convention, as fitted in SURVEY Appendix A1.

    Per (query, key) pair, non-causal: 2k^2/d score FLOPs (2 per multiply-add over the
    expected overlap; 2d for the dense rows) + 2 d_v for P.V + 3 softmax + 2 d_v/64
    for one O rescale per 64-key tile."""
    score = 2.0 * d if k is None else 2.0 * k * k / d
    return BH * n * n * (score + 2.0 * d_v + 3.0 + 2.0 * d_v / 64.0)


@dataclass(frozen=True)
class Workload:
    B: int
    H: int
    H_kv: int
    n: int
    d: int
    d_v: int
    k: int
    causal: bool = True
    dtype: str = "bf16"

    @property
    def s_v(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    @property
    def tokens(self) -> int:
        return self.B * self.n

    @property
    def pairs(self) -> int:
        return self.B * self.H * causal_pairs(self.n, self.n, 0, self.causal)

    @property
    def pv_flops(self) -> float:
        """Dense P.V tensor FLOPs over the allowed pairs: 2 d_v per pair (Alg. 1)."""
        return 2.0 * self.d_v * self.pairs

    @property
    def expected_interactions(self) -> float:
        """Score multiply-adds for uniform random supports: k^2/d per pair."""
        return self.pairs * self.k * self.k / self.d

    def topk_bytes(self) -> int:
        """HBM bytes of stage 1+2: read d values, write k idx (u8) + k values, per row."""
        rows = self.B * (self.H + self.H_kv) * self.n
        return rows * (self.d * self.s_v + self.k * (1 + self.s_v))

    def attn_min_bytes(self) -> int:
        """Unavoidable HBM bytes of the attention forward: read q codes, k codes, V; write O, LSE."""
        q = self.B * self.H * self.n * (self.k * (1 + self.s_v) + self.d_v * self.s_v + 4)
        kv = self.B * self.H_kv * self.n * (self.k * (1 + self.s_v) + self.d_v * self.s_v)
        return q + kv


CONFIGS = {
    # BASELINE.json "configs", in order (SURVEY 8(d) for the unstated fields)
    "tiny": Workload(B=1, H=1, H_kv=1, n=256, d=64, d_v=64, k=8, dtype="f32"),
    "gpt2": Workload(B=8, H=12, H_kv=12, n=1024, d=64, d_v=64, k=8),
    "qwen3": Workload(B=1, H=32, H_kv=8, n=32768, d=128, d_v=128, k=16),
    "long": Workload(B=1, H=32, H_kv=8, n=131072, d=128, d_v=128, k=16),
    "sweep": Workload(B=1, H=32, H_kv=8, n=16384, d=128, d_v=128, k=16),
}
SEEDS = {"tiny": 1, "gpt2": 11, "qwen3": 21, "long": 31, "sweep": 41}


def exact_edges(q_idx, k_idx, d: int, q_pos0: int = 0, causal: bool = True) -> int:
    """The exact number of score interactions E = sum over allowed pairs (i, j) of |S_i & S_j|
    (P:L59), by one-hot prefix counts in O(n d) per (batch, kv head) instead of O(n^2 k):
    E = sum_i sum_{u in S_i} #{allowed j : u in S_j}.  q_idx [B,H,n_q,k], k_idx [B,H_kv,n_kv,k] uint8
    torch tensors on any device (the bench counts the codes it just computed, outside the timed region).
    Supports are index sets (zero-valued selected entries count, reading A8)."""
    import torch
    B, H, n_q, _ = q_idx.shape
    H_kv, n_kv = k_idx.shape[1], k_idx.shape[2]
    R = H // H_kv
    dev = q_idx.device
    total = 0
    last = torch.arange(n_q, device=dev, dtype=torch.int64) + q_pos0
    for b in range(B):
        for g in range(H_kv):
            onehot = torch.zeros((n_kv, d), dtype=torch.int32, device=dev)
            onehot.scatter_(1, k_idx[b, g].long(), 1)
            pref = onehot.cumsum(0, dtype=torch.int64) if causal else onehot.sum(0, keepdim=True).expand(n_kv, d)
            allowed = last.clamp(max=n_kv - 1) if causal else torch.full_like(last, n_kv - 1)
            ok = (allowed >= 0)
            rows = pref[allowed.clamp(min=0)]  # [n_q, d]: keys j <= allowed_i selecting each feature
            for r in range(R):
                cnt = rows.gather(1, q_idx[b, g * R + r].long()).sum(1)
                total += int(torch.where(ok, cnt, torch.zeros_like(cnt)).sum().item())
    return total
