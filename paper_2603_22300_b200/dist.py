"""Query-block sharding of one long sequence over P GPUs (include/sfa.h step 9).

Host orchestration only (argument marshalling and the partition arithmetic); the exchange is the
C-ABI's NCCL all-gather + unpack kernel and every compute step is a libsfa kernel.

Zig-zag partition: the sequence of n tokens is cut into 2P chunks of c = n / (2P) tokens; rank p
owns chunks p and 2P-1-p, so every rank has exactly the same causal work (chunk q of a causal
sequence costs ~ q + 1/2 key tiles per query tile; q + (2P-1-q) is the same for every rank).
Local tensors are chunk-major ``[2][B][H][c][.]`` (chunk p, then chunk 2P-1-p).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import sfa


def chunk_size(n: int, world: int) -> int:
    if world < 1 or n % (2 * world):
        raise ValueError(f"n={n} must be a multiple of 2*world={2 * world}")
    return n // (2 * world)


def owned_chunks(rank: int, world: int) -> tuple[int, int]:
    """The two chunk indices rank `rank` owns (zig-zag)."""
    return rank, 2 * world - 1 - rank


def local_token_positions(rank: int, world: int, n: int) -> np.ndarray:
    """Global sequence positions of the local tokens, in local (chunk-major) order."""
    c = chunk_size(n, world)
    a, b = owned_chunks(rank, world)
    return np.concatenate([np.arange(a * c, (a + 1) * c), np.arange(b * c, (b + 1) * c)])


def causal_pairs_of_rank(rank: int, world: int, n: int) -> int:
    """Allowed (query, key) pairs of one head handled by `rank` (equal for every rank)."""
    return int(sum(int(p) + 1 for p in local_token_positions(rank, world, n)))


def unpack_reference(gathered: np.ndarray, world: int, bh: int, c: int) -> np.ndarray:
    """What sfa_dist_unpack_zigzag computes, written as array indexing (host tests):
    gathered [P][2][bh][c][...] (rank-major all-gather of chunk-major locals) -> [bh][2P*c][...]."""
    g = gathered.reshape((world, 2, bh, c) + gathered.shape[4:])
    out = np.empty((bh, 2 * world, c) + gathered.shape[4:], gathered.dtype)
    for r in range(world):
        for half in range(2):
            out[:, owned_chunks(r, world)[half]] = g[r, half]
    return out.reshape((bh, 2 * world * c) + gathered.shape[4:])


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

    def allgather_kv(self, k_idx, k_val, v):
        """Local codes/V [2][B][H_kv][c][.] -> full [B][H_kv][2Pc][.] in sequence order."""
        two, B, H_kv, c, k = k_idx.shape
        d_v = v.shape[-1]
        n = 2 * self.world * c
        desc = sfa.make_desc(B=B, H=H_kv, H_kv=H_kv, d=128, k=k, d_v=d_v, n_q=2 * c, n_kv=2 * c,
                             dtype=sfa._dt(v))
        dev = v.device
        full = (torch.empty((B, H_kv, n, k), dtype=torch.uint8, device=dev),
                torch.empty((B, H_kv, n, k), dtype=k_val.dtype, device=dev),
                torch.empty((B, H_kv, n, d_v), dtype=v.dtype, device=dev))
        nb = int(sfa.lib().sfa_dist_staging_bytes(ctypes.byref(desc), self.world))
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
        k_full_idx, k_full_val, v_full = self.allgather_kv(ki, kv, v)   # step 9
        n = 2 * self.world * c
        desc = sfa.make_desc(B=B, H=H, H_kv=H_kv, d=d, k=k_code, d_v=d_v, n_q=c, n_kv=n, causal=causal,
                             scale=scale, dtype=sfa._dt(v))
        ws = torch.empty(max(sfa.workspace_bytes(desc), 16), dtype=torch.uint8, device=v.device)
        L = sfa.lib()
        sfa._check(L.sfa_attn_prepare(ctypes.byref(desc), sfa._p(k_full_idx), sfa._p(k_full_val), sfa._p(v_full),
                                      sfa._p(ws), ws.numel(), sfa._stream()), "sfa_attn_prepare")
        o = torch.empty((2, B, H, c, d_v), dtype=v.dtype, device=v.device)
        lse = torch.empty((2, B, H, c), dtype=torch.float32, device=v.device)
        for half, chunk in enumerate(owned_chunks(self.rank, self.world)):
            desc.q_pos0 = chunk * c
            sfa._check(L.sfa_attn_fwd_prepared(ctypes.byref(desc), sfa._p(qi[half]), sfa._p(qv[half]),
                                               sfa._p(k_full_idx), sfa._p(k_full_val), sfa._p(v_full),
                                               sfa._p(o[half]), sfa._p(lse[half]), sfa._p(ws), ws.numel(),
                                               sfa._stream()), "sfa_attn_fwd_prepared")
        return o, lse
