"""GPU checks of the sharded path (include/sfa.h step 9) on one B200.

- sfa_dist_unpack_zigzag against its array-indexing reference (dist.unpack_reference), for rows
  moved as 16-byte words and as bytes.
- The whole sharded forward through a real NCCL communicator with world = 1 (the only size one GPU
  allows): chunks 0 and 1 at q_pos0 = 0 and c must reproduce the single-call forward bit for bit.
  Multi-rank orchestration is covered on CPU by tests/test_dist_gloo.py.
"""
import os
import socket

import numpy as np
import pytest

from paper_2603_22300_b200 import dist as sdist
from paper_2603_22300_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,bh,c,row", [(2, 3, 5, 16), (4, 2, 7, 48), (3, 2, 4, 24), (8, 1, 3, 1)])
def test_unpack_kernel_matches_reference(lib, world, bh, c, row):
    import torch
    rng = np.random.default_rng(world * 100 + row)
    host = rng.integers(0, 256, size=(world, 2, bh, c, row), dtype=np.uint8)
    src = torch.from_numpy(host).cuda()
    dst = torch.zeros(bh * 2 * world * c * row, dtype=torch.uint8, device="cuda")
    lib._check(lib.lib().sfa_dist_unpack_zigzag(lib._p(src), lib._p(dst), world, bh, c, row, lib._stream()),
               "sfa_dist_unpack_zigzag")
    torch.cuda.synchronize()
    ref = sdist.unpack_reference(host, world, bh, c)
    assert np.array_equal(dst.cpu().numpy().reshape(ref.shape), ref)


def test_single_rank_nccl_sharded_forward_equals_full(lib):
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sh = sdist.ShardedAttention()
        B, H, H_kv, n, d, d_v, k = 1, 4, 2, 512, 128, 128, 16
        Q = lib.gen_fill(torch.empty((B, H, n, d), dtype=torch.bfloat16, device="cuda"), 3, inputs.TID_Q)
        K = lib.gen_fill(torch.empty((B, H_kv, n, d), dtype=torch.bfloat16, device="cuda"), 3, inputs.TID_K)
        V = lib.gen_fill(torch.empty((B, H_kv, n, d_v), dtype=torch.bfloat16, device="cuda"), 3, inputs.TID_V)
        o_full, l_full = lib.forward(Q, K, V, k_code=k)
        c = sdist.chunk_size(n, 1)
        loc = lambda x: torch.stack([x[:, :, q * c:(q + 1) * c] for q in sdist.owned_chunks(0, 1)]).contiguous()
        o, lse = sh.forward(loc(Q), loc(K), loc(V), k_code=k)
        torch.cuda.synchronize()
        sh.close()
        for half, q in enumerate(sdist.owned_chunks(0, 1)):
            assert torch.equal(o[half], o_full[:, :, q * c:(q + 1) * c])
            assert torch.equal(lse[half], l_full[:, :, q * c:(q + 1) * c])
    finally:
        dist.destroy_process_group()
