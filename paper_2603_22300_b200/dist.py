"""Multi-GPU partitions of the FlashSFA forward (include/sfa.h step 9).

Host orchestration only (argument marshalling); the partition arithmetic is the C library's
(``sfa_dist_head_shard``, ``sfa_dist_zigzag_chunk``, ``sfa_dist_kv_plan``), the exchange is the
C-ABI's NCCL all-gather + unpack kernel and every compute step is a libsfa kernel.

Two partitions, both one process per GPU:

* **(batch, kv head) sharding** (no communication): the B*H_kv units -- unit
  u = b*H_kv + g, contiguous in every tensor, holding query heads [g*R, g*R+R) with R = H/H_kv --
  are split into contiguous ranges; each rank runs the whole hot path on its units as the problem
  (B = #units, H = R, H_kv = 1).  Preferred whenever B*H_kv >= P (e.g. Qwen3-32K, B=1, 8 kv heads).
* **query-block (zig-zag) sharding of one long sequence** (SURVEY 8(e)-2): the sequence of n tokens is
  cut into 2P chunks of c = n / (2P) tokens; rank p owns chunks p and 2P-1-p, so every rank has exactly
  the same causal work.  Local tensors are chunk-major ``[2][B][H][c][.]``; one NCCL all-gather of the
  key codes and V gives every rank the whole sequence, then each query chunk runs with q_pos0 = chunk
  start.  Outputs stay sharded; no LSE merge.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import sfa


# ---- zig-zag partition (the library's sfa_dist_zigzag_chunk) ----------------------------------------
def chunk_size(n: int, world: int) -> int:
    c = ctypes.c_int64()
    if world < 1 or sfa.lib().sfa_dist_zigzag_chunk(n, world, 0, 0, ctypes.byref(c), None) != 0:
        raise ValueError(f"n={n} must be a positive multiple of 2*world={2 * world}")
    return c.value


def chunk_start(n: int, world: int, rank: int, half: int) -> int:
    """Global position of the first token of `rank`'s chunk `half` (0: chunk rank, 1: chunk 2P-1-rank)."""
    q0 = ctypes.c_int64()
    sfa._check(sfa.lib().sfa_dist_zigzag_chunk(n, world, rank, half, None, ctypes.byref(q0)),
               "sfa_dist_zigzag_chunk")
    return q0.value


def owned_chunks(rank: int, world: int) -> tuple[int, int]:
    """The two chunk indices rank `rank` owns (zig-zag): chunk_start(n, world, rank, h) // c."""
    n = 2 * world
    return chunk_start(n, world, rank, 0), chunk_start(n, world, rank, 1)


def local_token_positions(rank: int, world: int, n: int) -> np.ndarray:
    """Global sequence positions of the local tokens, in local (chunk-major) order."""
    c = chunk_size(n, world)
    return np.concatenate([np.arange(chunk_start(n, world, rank, h), chunk_start(n, world, rank, h) + c)
                           for h in (0, 1)])


def causal_pairs_of_rank(rank: int, world: int, n: int) -> int:
    """Allowed (query, key) pairs of one head handled by `rank` (equal for every rank)."""
    return int(sum(int(p) + 1 for p in local_token_positions(rank, world, n)))


def kv_plan(local_desc, world: int):
    """sfa_dist_kv_plan: staging offsets / per-rank bytes / row bytes of the K/V all-gather."""
    pl = sfa.KvPlan()
    sfa._check(sfa.lib().sfa_dist_kv_plan(ctypes.byref(local_desc), world, ctypes.byref(pl)), "sfa_dist_kv_plan")
    return pl


def unpack_reference(gathered: np.ndarray, world: int, bh: int, c: int) -> np.ndarray:
    """What sfa_dist_unpack_zigzag computes, written as array indexing (host tests):
    gathered [P][2][bh][c][...] (rank-major all-gather of chunk-major locals) -> [bh][2P*c][...]."""
    g = gathered.reshape((world, 2, bh, c) + gathered.shape[4:])
    out = np.empty((bh, 2 * world, c) + gathered.shape[4:], gathered.dtype)
    for r in range(world):
        for half in range(2):
            out[:, owned_chunks(r, world)[half]] = g[r, half]
    return out.reshape((bh, 2 * world * c) + gathered.shape[4:])


# ---- (batch, kv head) partition (the library's sfa_dist_head_shard) -----------------------------------
def head_shard(desc, world: int, rank: int):
    """(sub_desc, unit0): rank's units [unit0, unit0 + sub_desc.B) of the full problem `desc`."""
    sub = sfa.AttnDesc()
    u0 = ctypes.c_int64()
    sfa._check(sfa.lib().sfa_dist_head_shard(ctypes.byref(desc), world, rank, ctypes.byref(sub), ctypes.byref(u0)),
               "sfa_dist_head_shard")
    return sub, u0.value


def unit_slices(desc, world: int, rank: int):
    """Element ranges of rank's units in the flattened Q / K / V / O / LSE tensors of `desc`:
    dict name -> (start, stop) along the flattened tensor."""
    sub, u0 = head_shard(desc, world, rank)
    R = desc.H // desc.H_kv
    per = {"q": R * desc.n_q * desc.d, "k": desc.n_kv * desc.d, "v": desc.n_kv * desc.d_v,
           "o": R * desc.n_q * desc.d_v, "lse": R * desc.n_q,
           "q_codes": R * desc.n_q * desc.k, "k_codes": desc.n_kv * desc.k}
    return sub, {name: (u0 * e, (u0 + sub.B) * e) for name, e in per.items()}


def forward_head_sharded(q, k, v, *, k_code, world: int, rank: int, causal=True, scale=None):
    """This rank's share of the (batch, kv head) partition: dense q [B,H,n,d], k [B,H_kv,n,d],
    v [B,H_kv,n,d_v] (the FULL tensors, or any tensors holding at least this rank's units at their global
    offsets) -> (o_units [nu, R, n_q, d_v], lse_units [nu, R, n_q], unit0).  No communication."""
    B, H, n_q, d = q.shape
    _, H_kv, n_kv, _ = k.shape
    d_v = v.shape[-1]
    full = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k_code, d_v=d_v, n_q=n_q, n_kv=n_kv, causal=causal,
                         scale=scale, dtype=sfa._dt(v))
    sub, u0 = head_shard(full, world, rank)
    R = H // H_kv
    qs = q.reshape(B * H_kv, R, n_q, d)[u0:u0 + sub.B]
    ks = k.reshape(B * H_kv, 1, n_kv, d)[u0:u0 + sub.B]
    vs = v.reshape(B * H_kv, 1, n_kv, d_v)[u0:u0 + sub.B]
    o, lse = sfa.forward(qs, ks, vs, k_code=k_code, causal=causal, scale=scale)
    return o, lse, u0


class ShardedAttention:
    """One NCCL communicator (owned by libsfa) + the zig-zag forward.  Collective: every rank of the
    default torch.distributed group constructs it (rank 0 creates the NCCL id, broadcast over the
    existing process group)."""

    def __init__(self):
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            sfa._check(sfa.lib().sfa_dist_unique_id(uid), "sfa_dist_unique_id")
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0)
        uid = ctypes.create_string_buffer(box[0], 128)
        self._h = ctypes.c_void_p()
        sfa._check(sfa.lib().sfa_dist_init(self.rank, self.world, uid, ctypes.byref(self._h)), "sfa_dist_init")

    def close(self):
        if self._h:
            sfa._check(sfa.lib().sfa_dist_destroy(self._h), "sfa_dist_destroy")
            self._h = ctypes.c_void_p()

    def allgather_kv(self, k_idx, k_val, v, d: int):
        """Local codes/V [2][B][H_kv][c][.] -> full [B][H_kv][2Pc][.] in sequence order."""
        two, B, H_kv, c, k = k_idx.shape
        d_v = v.shape[-1]
        if two != 2 or tuple(k_val.shape) != tuple(k_idx.shape) or tuple(v.shape[:4]) != (2, B, H_kv, c):
            raise ValueError("allgather_kv takes chunk-major [2][B][H_kv][c][.] codes and V")
        n = 2 * self.world * c
        desc = sfa.make_desc(B=B, H=H_kv, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=2 * c, n_kv=2 * c, dtype=sfa._dt(v))
        dev = v.device
        full = (torch.empty((B, H_kv, n, k), dtype=torch.uint8, device=dev),
                torch.empty((B, H_kv, n, k), dtype=k_val.dtype, device=dev),
                torch.empty((B, H_kv, n, d_v), dtype=v.dtype, device=dev))
        nb = kv_plan(desc, self.world).staging_bytes
        staging = torch.empty(nb, dtype=torch.uint8, device=dev)
        sfa._check(sfa.lib().sfa_dist_allgather_kv(self._h, ctypes.byref(desc), sfa._p(k_idx), sfa._p(k_val),
                                                    sfa._p(v), sfa._p(full[0]), sfa._p(full[1]), sfa._p(full[2]),
                                                    sfa._p(staging), nb, sfa._stream()), "sfa_dist_allgather_kv")
        return full

    def forward(self, q, k, v, *, k_code, causal=True, scale=None):
        """q [2][B][H][c][d], k [2][B][H_kv][c][d], v [2][B][H_kv][c][d_v] (this rank's two chunks)
        -> (o [2][B][H][c][d_v], lse [2][B][H][c]) for the same query rows."""
        two, B, H, c, d = q.shape
        H_kv, d_v = k.shape[2], v.shape[-1]
        if scale is None:
            scale = 1.0 / math.sqrt(d)
        qi, qv = sfa.topk_codes(q, k_code)       # stage 1 on the local queries
        ki, kv = sfa.topk_codes(k, k_code)       # stage 1 on the local keys
        k_full_idx, k_full_val, v_full = self.allgather_kv(ki, kv, v, d)   # step 9
        n = 2 * self.world * c
        desc = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k_code, d_v=d_v, n_q=c, n_kv=n, causal=causal,
                             scale=scale, dtype=sfa._dt(v))
        ws = torch.empty(max(sfa.workspace_bytes(desc), 16), dtype=torch.uint8, device=v.device)
        L = sfa.lib()
        sfa._check(L.sfa_attn_prepare(ctypes.byref(desc), sfa._p(k_full_idx), sfa._p(k_full_val), sfa._p(v_full),
                                      sfa._p(ws), ws.numel(), sfa._stream()), "sfa_attn_prepare")
        o = torch.empty((2, B, H, c, d_v), dtype=v.dtype, device=v.device)
        lse = torch.empty((2, B, H, c), dtype=torch.float32, device=v.device)
        for half in range(2):
            desc.q_pos0 = chunk_start(n, self.world, self.rank, half)
            sfa._check(L.sfa_attn_fwd_prepared(ctypes.byref(desc), sfa._p(qi[half]), sfa._p(qv[half]),
                                               sfa._p(k_full_idx), sfa._p(k_full_val), sfa._p(v_full),
                                               sfa._p(o[half]), sfa._p(lse[half]), sfa._p(ws), ws.numel(),
                                               sfa._stream()), "sfa_attn_fwd_prepared")
        return o, lse
