"""GPU checks of the two multi-GPU partitions (paper_2603_22300_b200/dist.py).

* (batch, kv head) sharding: every rank's share computed through the library's sfa_dist_head_shard
  plan must equal the matching slice of the single-call forward bit for bit.  The ranks of a P-way
  split are run one after the other on one GPU (the partition has no communication).
* zig-zag query-block sharding with P ranks on ONE GPU: each rank's local stage 1, the rank-major
  all-gather NCCL would produce (the ranks' blocks concatenated in rank order into the staging layout
  of sfa_dist_kv_plan), the library's unpack kernel, then each rank's two query chunks -- bitwise equal
  to the single-call forward.
* the real thing where the box has the GPUs: P processes, one NCCL communicator (ShardedAttention,
  sfa_dist_allgather_kv), P = 2, 4, 8; skipped when fewer GPUs are visible.
"""
import os
import socket

import numpy as np
import pytest

from paper_2603_22300_b200 import dist as sdist
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu


def _qkv(sfa, B, H, H_kv, n, d, d_v, seed=3):
    import torch
    bf = torch.bfloat16
    Q = sfa.gen_fill(torch.empty((B, H, n, d), dtype=bf, device="cuda"), seed, inputs.TID_Q)
    K = sfa.gen_fill(torch.empty((B, H_kv, n, d), dtype=bf, device="cuda"), seed, inputs.TID_K)
    V = sfa.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=bf, device="cuda"), seed, inputs.TID_V)
    return Q, K, V


@pytest.mark.parametrize("shape,world", [((1, 32, 8, 1024, 128, 128, 16), 8), ((1, 32, 8, 700, 128, 128, 16), 3),
                                         ((2, 12, 12, 512, 64, 64, 8), 5), ((3, 8, 2, 300, 128, 128, 16), 4)])
def test_head_shard_equals_full_forward(lib, shape, world):
    import torch
    B, H, H_kv, n, d, d_v, k = shape
    Q, K, V = _qkv(lib, B, H, H_kv, n, d, d_v)
    o_full, l_full = lib.forward(Q, K, V, k_code=k)
    R = H // H_kv
    of = o_full.reshape(B * H_kv, R, n, d_v)
    lf = l_full.reshape(B * H_kv, R, n)
    covered = 0
    for rank in range(world):
        o, lse, u0 = sdist.forward_head_sharded(Q, K, V, k_code=k, world=world, rank=rank)
        torch.cuda.synchronize()
        nu = o.shape[0]
        assert torch.equal(o, of[u0:u0 + nu]) and torch.equal(lse, lf[u0:u0 + nu])
        covered += nu
    assert covered == B * H_kv


@pytest.mark.parametrize("world,n", [(2, 1024), (4, 2048), (8, 4096), (3, 1536)])
def test_zigzag_all_ranks_on_one_gpu_equal_full_forward(lib, world, n):
    """Every piece of the sharded path except NCCL itself, at P > 1, on one GPU."""
    import ctypes

    import torch
    B, H, H_kv, d, d_v, k = 1, 8, 2, 128, 128, 16
    Q, K, V = _qkv(lib, B, H, H_kv, n, d, d_v, seed=5)
    o_full, l_full = lib.forward(Q, K, V, k_code=k)
    c = sdist.chunk_size(n, world)
    starts = [[sdist.chunk_start(n, world, r, h) for h in (0, 1)] for r in range(world)]
    loc = lambda x, r: torch.stack([x[:, :, s:s + c] for s in starts[r]]).contiguous()
    # stage 1 on every rank's own tokens
    codes = [(lib.topk_codes(loc(Q, r), k), lib.topk_codes(loc(K, r), k), loc(V, r)) for r in range(world)]
    ldesc = lib.make_desc(B=B, H=H_kv, H_kv=H_kv, d=d, k=k, d_v=d_v, n_q=2 * c, n_kv=2 * c)
    pl = sdist.kv_plan(ldesc, world)
    staging = torch.zeros(pl.staging_bytes, dtype=torch.uint8, device="cuda")
    full = (torch.empty((B, H_kv, n, k), dtype=torch.uint8, device="cuda"),
            torch.empty((B, H_kv, n, k), dtype=torch.bfloat16, device="cuda"),
            torch.empty((B, H_kv, n, d_v), dtype=torch.bfloat16, device="cuda"))
    for t in range(3):
        # what ncclAllGather leaves in the staging: the ranks' local blocks, rank-major
        blocks = [(codes[r][1][0], codes[r][1][1], codes[r][2])[t].reshape(-1).view(torch.uint8) for r in range(world)]
        off = pl.staging_offset[t]
        staging[off:off + world * pl.bytes_per_rank[t]] = torch.cat(blocks)
        lib._check(lib.lib().sfa_dist_unpack_zigzag(ctypes.c_void_p(staging.data_ptr() + off),
                                                    lib._p(full[t]), world, pl.bh, pl.chunk, pl.row_bytes[t],
                                                    lib._stream()), "sfa_dist_unpack_zigzag")
    ki_ref, kv_ref = lib.topk_codes(K, k)
    torch.cuda.synchronize()
    assert torch.equal(full[0], ki_ref) and torch.equal(full[1], kv_ref) and torch.equal(full[2], V)
    for r in range(world):
        qi, qv = codes[r][0]
        for half in range(2):
            s = starts[r][half]
            o, lse = lib.attn_fwd(qi[half], qv[half], full[0], full[1], full[2], d=d, q_pos0=s)
            torch.cuda.synchronize()
            assert torch.equal(o, o_full[:, :, s:s + c]) and torch.equal(lse, l_full[:, :, s:s + c])


def _nccl_worker(rank, world, port, n, errq):
    import torch
    import torch.distributed as dist

    from paper_2603_22300_b200 import sfa
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        B, H, H_kv, d, d_v, k = 1, 8, 2, 128, 128, 16
        Q, K, V = _qkv(sfa, B, H, H_kv, n, d, d_v, seed=7)
        o_full, l_full = sfa.forward(Q, K, V, k_code=k)           # every rank: the 1-GPU reference
        c = sdist.chunk_size(n, world)
        starts = [sdist.chunk_start(n, world, rank, h) for h in (0, 1)]
        loc = lambda x: torch.stack([x[:, :, s:s + c] for s in starts]).contiguous()
        sh = sdist.ShardedAttention()
        o, lse = sh.forward(loc(Q), loc(K), loc(V), k_code=k)
        torch.cuda.synchronize()
        sh.close()
        for half, s in enumerate(starts):
            assert torch.equal(o[half], o_full[:, :, s:s + c]), f"rank {rank} half {half}: O differs"
            assert torch.equal(lse[half], l_full[:, :, s:s + c]), f"rank {rank} half {half}: LSE differs"
        o2, l2, u0 = sdist.forward_head_sharded(Q, K, V, k_code=k, world=world, rank=rank) if B * H_kv >= world \
            else (None, None, None)
        if o2 is not None:
            R = H // H_kv
            assert torch.equal(o2, o_full.reshape(B * H_kv, R, n, d_v)[u0:u0 + o2.shape[0]])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # surfaced by the parent
        errq.put(f"rank {rank}: {ex!r}")
        raise


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_world_n_sharded_forward_equals_one_gpu(lib, world):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    mp.start_processes(_nccl_worker, args=(world, port, 2048 * world, errq), nprocs=world, join=True,
                       start_method="spawn")
    assert errq.empty(), errq.get()
