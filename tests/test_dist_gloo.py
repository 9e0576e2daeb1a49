"""Multi-process (world_size 2, gloo, CPU) checks of the multi-GPU partitions.

The partition arithmetic is the C library's own host code (sfa_dist_zigzag_chunk, sfa_dist_kv_plan,
sfa_dist_head_shard, called through paper_2603_22300_b200/dist.py; they need no GPU).  Each rank
executes exactly the plan sfa_dist_allgather_kv executes over NCCL -- the three rank-major byte
gathers into the staging layout the library reports, then the unpack (its array-indexing reference;
the unpack kernel itself is checked against that reference on the GPU) -- with gloo as the transport
and the oracle as the compute.  The gathered keys must equal the codes of the whole sequence, and
every rank's rows must equal the single-process oracle's rows bit for bit.  The (batch, kv head)
partition is checked the same way: each rank runs the oracle on its sub-problem only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_22300_b200 import dist as sdist
from paper_2603_22300_b200 import inputs, sfa


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


B, H, H_kv, N, D, DV, K = 1, 2, 1, 256, 64, 64, 8


def _codes(x, k=K):
    idx, val = oracle.topk_codes(x.reshape(-1, x.shape[-1]), k)
    return idx.reshape(x.shape[:-1] + (k,)), val.reshape(x.shape[:-1] + (k,))


def _local(x, rank, world):
    """chunk-major local slice [2][B][h][c][.] of a global [B][h][N][.] tensor (library chunk starts)"""
    c = sdist.chunk_size(N, world)
    return np.stack([x[:, :, q0:q0 + c] for q0 in (sdist.chunk_start(N, world, rank, h) for h in (0, 1))])


def _gather_bytes(a, world):
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy())
    buf = torch.empty(world * t.numel(), dtype=torch.uint8)
    dist.all_gather_into_tensor(buf, t)
    return buf.numpy()


def _zigzag_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, kx, v = inputs.qkv(5, B, H, H_kv, N, D, DV, "f32")
        c = sdist.chunk_size(N, world)
        ql, kl, vl = _local(q, rank, world), _local(kx, rank, world), _local(v, rank, world)
        qi, qv = _codes(ql)                       # stage 1 on local tokens only
        ki, kv = _codes(kl)
        # the library's plan for this rank's local keys (what sfa_dist_allgather_kv runs over NCCL)
        ldesc = sfa.make_desc(B=B, H=H_kv, H_kv=H_kv, d=D, k=K, d_v=DV, n_q=2 * c, n_kv=2 * c, dtype=sfa.SFA_F32)
        pl = sdist.kv_plan(ldesc, world)
        assert (pl.bh, pl.chunk) == (B * H_kv, c)
        staging = np.zeros(pl.staging_bytes, np.uint8)
        full = []
        for t, (a, dt, width) in enumerate(((ki, np.uint8, K), (kv, np.float32, K), (vl, np.float32, DV))):
            assert a.nbytes == pl.bytes_per_rank[t] and pl.row_bytes[t] == width * np.dtype(dt).itemsize
            off = pl.staging_offset[t]
            assert off % 256 == 0
            staging[off:off + world * pl.bytes_per_rank[t]] = _gather_bytes(a, world)   # rank-major gather
            block = staging[off:off + world * pl.bytes_per_rank[t]].reshape(world, 2, pl.bh, pl.chunk,
                                                                            pl.row_bytes[t])
            full.append(sdist.unpack_reference(block, world, pl.bh, pl.chunk).view(dt).reshape(B, H_kv, N, width))
        assert pl.staging_bytes == sfa.lib().sfa_dist_staging_bytes(sfa.ctypes.byref(ldesc), world)
        ki_f, kv_f, v_f = full
        ki_ref, kv_ref = _codes(kx)
        assert np.array_equal(ki_f, ki_ref) and np.array_equal(kv_f, kv_ref) and np.array_equal(v_f, v)
        rows = []
        for half in range(2):
            q0 = sdist.chunk_start(N, world, rank, half)
            o, lse = oracle.attn_fwd(qi[half], qv[half], ki_f, kv_f, v_f, d=D, q_pos0=q0)
            rows.append((q0, o, lse))
        out[rank] = rows
    finally:
        dist.destroy_process_group()


def _heads_worker(rank, world, port, shape, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, h, hkv, n, d, dv, k = shape
        q, kx, v = inputs.qkv(9, b, h, hkv, n, d, dv, "f32")
        full = sfa.make_desc(B=b, H=h, H_kv=hkv, d=d, k=k, d_v=dv, n_q=n, n_kv=n, dtype=sfa.SFA_F32)
        sub, sl = sdist.unit_slices(full, world, rank)
        # this rank's inputs: only its units, cut from the flattened global tensors at the library's offsets
        qs = q.reshape(-1)[slice(*sl["q"])].reshape(sub.B, sub.H, n, d)
        ks = kx.reshape(-1)[slice(*sl["k"])].reshape(sub.B, 1, n, d)
        vs = v.reshape(-1)[slice(*sl["v"])].reshape(sub.B, 1, n, dv)
        o, lse = oracle.attn_fwd(*_codes(qs, k), *_codes(ks, k), vs, d=d)
        out[rank] = (sl["o"], o.reshape(-1), sl["lse"], lse.reshape(-1))
    finally:
        dist.destroy_process_group()


def test_partition_covers_sequence_once_and_balances_work():
    for world in (1, 2, 4, 8):
        n = 2 * world * 64
        pos = np.concatenate([sdist.local_token_positions(r, world, n) for r in range(world)])
        assert np.array_equal(np.sort(pos), np.arange(n))
        work = {sdist.causal_pairs_of_rank(r, world, n) for r in range(world)}
        assert len(work) == 1  # zig-zag: identical causal work on every rank
        assert work.pop() * world == n * (n + 1) // 2


def test_zigzag_chunk_rejects_bad_sizes():
    with pytest.raises(ValueError):
        sdist.chunk_size(100, 8)        # not a multiple of 2P
    with pytest.raises(sfa.SfaError):
        sdist.chunk_start(64, 2, 2, 0)  # rank out of range


def test_unpack_reference_roundtrip():
    world, bh, c = 4, 3, 5
    full = np.arange(bh * 2 * world * c * 2).reshape(bh, 2 * world * c, 2)
    locs = np.stack([np.stack([full[:, q * c:(q + 1) * c] for q in sdist.owned_chunks(r, world)])
                     for r in range(world)])  # [P][2][bh][c][2]
    assert np.array_equal(sdist.unpack_reference(locs, world, bh, c), full)


@pytest.mark.parametrize("B_,Hkv,world", [(1, 8, 8), (1, 8, 3), (2, 3, 4), (3, 1, 2), (1, 2, 2)])
def test_head_shard_ranges_cover_units_once(B_, Hkv, world):
    desc = sfa.make_desc(B=B_, H=4 * Hkv, H_kv=Hkv, d=128, k=16, d_v=128, n_q=64, n_kv=64)
    seen, sizes = [], []
    for r in range(world):
        sub, u0 = sdist.head_shard(desc, world, r)
        assert (sub.H, sub.H_kv, sub.n_q, sub.k) == (4, 1, 64, 16)
        seen.extend(range(u0, u0 + sub.B))
        sizes.append(sub.B)
    assert seen == list(range(B_ * Hkv))          # contiguous, in order, each unit once
    assert max(sizes) - min(sizes) <= 1


def test_head_shard_rejects_more_ranks_than_units():
    desc = sfa.make_desc(B=1, H=8, H_kv=2, d=128, k=16, d_v=128, n_q=64, n_kv=64)
    with pytest.raises(sfa.SfaError):
        sdist.head_shard(desc, 4, 0)


def test_two_rank_zigzag_equals_single_process():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_zigzag_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    q, kx, v = inputs.qkv(5, B, H, H_kv, N, D, DV, "f32")
    o_ref, l_ref = oracle.attn_fwd(*_codes(q), *_codes(kx), v, d=D)
    c = sdist.chunk_size(N, world)
    seen = set()
    for rank in range(world):
        for q0, o, lse in out[rank]:
            assert np.array_equal(o, o_ref[:, :, q0:q0 + c])
            assert np.array_equal(lse, l_ref[:, :, q0:q0 + c])
            seen.add(q0 // c)
    assert seen == set(range(2 * world))


@pytest.mark.parametrize("shape", [(1, 4, 2, 96, 64, 64, 8), (3, 2, 1, 64, 64, 64, 4)])
def test_two_rank_head_shard_equals_single_process(shape):
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_heads_worker, args=(world, _free_port(), shape, out), nprocs=world, join=True)
    b, h, hkv, n, d, dv, k = shape
    q, kx, v = inputs.qkv(9, b, h, hkv, n, d, dv, "f32")
    o_ref, l_ref = oracle.attn_fwd(*_codes(q, k), *_codes(kx, k), v, d=d)
    o_all = np.full(o_ref.size, np.nan)
    l_all = np.full(l_ref.size, np.nan)
    for rank in range(world):
        (o0, o1), o, (l0, l1), lse = out[rank]
        o_all[o0:o1] = o
        l_all[l0:l1] = lse
    assert np.array_equal(o_all, o_ref.reshape(-1)) and np.array_equal(l_all, l_ref.reshape(-1))
