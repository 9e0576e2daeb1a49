"""Multi-process (world_size 2, gloo, CPU) checks of the sharded path's host logic
(paper_2603_22300_b200/dist.py).

Each rank builds its zig-zag chunks of a seeded global input, codes them with the oracle,
all-gathers the chunk-major key codes and V over gloo exactly as sfa_dist_allgather_kv does over
NCCL, unpacks them with the reference of the unpack kernel, and runs the oracle attention for its
two query chunks at q_pos0 = chunk start.  The gathered keys must equal the codes of the whole
sequence, and each rank's rows must equal the single-process oracle's rows bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_22300_b200 import dist as sdist
from paper_2603_22300_b200 import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


B, H, H_kv, N, D, DV, K = 1, 2, 1, 256, 64, 64, 8


def _codes(x):
    idx, val = oracle.topk_codes(x.reshape(-1, x.shape[-1]), K)
    return idx.reshape(x.shape[:-1] + (K,)), val.reshape(x.shape[:-1] + (K,))


def _local(x, rank, world):
    """chunk-major local slice [2][B][h][c][.] of a global [B][h][N][.] tensor"""
    c = sdist.chunk_size(N, world)
    return np.stack([x[:, :, q * c:(q + 1) * c] for q in sdist.owned_chunks(rank, world)])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, kx, v = inputs.qkv(5, B, H, H_kv, N, D, DV, "f32")
        c = sdist.chunk_size(N, world)
        ql, kl, vl = _local(q, rank, world), _local(kx, rank, world), _local(v, rank, world)
        qi, qv = _codes(ql)                       # stage 1 on local tokens only
        ki, kv = _codes(kl)
        gathered = []
        for a in (ki, kv, vl):                    # the all-gather (rank-major)
            t = torch.from_numpy(np.ascontiguousarray(a))
            buf = torch.empty((world * t.shape[0],) + t.shape[1:], dtype=t.dtype)
            dist.all_gather_into_tensor(buf, t)
            gathered.append(sdist.unpack_reference(buf.numpy(), world, B * H_kv, c).reshape(B, H_kv, N, -1))
        ki_f, kv_f, v_f = gathered
        ki_ref, kv_ref = _codes(kx)
        assert np.array_equal(ki_f, ki_ref) and np.array_equal(kv_f, kv_ref) and np.array_equal(v_f, v)
        rows = []
        for half, chunk in enumerate(sdist.owned_chunks(rank, world)):
            o, lse = oracle.attn_fwd(qi[half], qv[half], ki_f, kv_f, v_f, d=D, q_pos0=chunk * c)
            rows.append((chunk, o, lse))
        out[rank] = rows
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


def test_unpack_reference_roundtrip():
    world, bh, c = 4, 3, 5
    full = np.arange(bh * 2 * world * c * 2).reshape(bh, 2 * world * c, 2)
    locs = np.stack([np.stack([full[:, q * c:(q + 1) * c] for q in sdist.owned_chunks(r, world)])
                     for r in range(world)])  # [P][2][bh][c][2]
    assert np.array_equal(sdist.unpack_reference(locs, world, bh, c), full)


def test_two_rank_sharded_oracle_equals_single_process():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    q, kx, v = inputs.qkv(5, B, H, H_kv, N, D, DV, "f32")
    o_ref, l_ref = oracle.attn_fwd(*_codes(q), *_codes(kx), v, d=D)
    c = sdist.chunk_size(N, world)
    seen = set()
    for rank in range(world):
        for chunk, o, lse in out[rank]:
            assert np.array_equal(o, o_ref[:, :, chunk * c:(chunk + 1) * c])
            assert np.array_equal(lse, l_ref[:, :, chunk * c:(chunk + 1) * c])
            seen.add(chunk)
    assert seen == set(range(2 * world))
