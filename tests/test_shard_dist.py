"""Multi-rank path on CPU (gloo, world_size 2): row sharding + the single
mod-2^32 reduce.  The per-rank partial answers come from the
oracle here (no GPU in this container); on GPUs the same shard.row_range /
shard.reduce_partial_shares drive dpf_eval_batch_wire + NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2301_10904_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, N, D, B, q):
    from oracle import oracle as orc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        T = synth.table(N, D, 77)
        seeds = synth.gen_seeds(B, 77)
        al = synth.alphas(B, N, 77)
        keys = [orc.gen(n, int(a), 1, s)[b % 2] for b, (a, s) in enumerate(zip(al, seeds))]
        r0, rows = shard.row_range(N, world, rank)
        part = orc.answer_batch(keys, T[r0:r0 + rows], row_begin=r0)
        t = torch.from_numpy(part.view(np.int32).copy())
        shard.reduce_partial_shares(t, dst=0)
        # wrap check: every rank contributes 0x7FFFFFFF
        w = torch.full((4,), 0x7FFFFFFF, dtype=torch.int32)
        shard.reduce_partial_shares(w, dst=0)
        if rank == 0:
            whole = orc.answer_batch(keys, T)
            q.put((bool(np.array_equal(t.numpy().view(np.uint32), whole)),
                   int(w[0].item()) & 0xFFFFFFFF == (world * 0x7FFFFFFF) & 0xFFFFFFFF))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 1 << 11), (2, 3000), (3, 2500)])
def test_row_sharded_reduce_equals_whole(world, N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 12, N, 8, 6, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    same, wrapped = q.get(timeout=10)
    assert same and wrapped


def test_row_range_partitions():
    for N, G in ((1 << 20, 8), (12345, 7), (16, 16)):
        ranges = [shard.row_range(N, G, r) for r in range(G)]
        assert ranges[0][0] == 0
        assert sum(c for _, c in ranges) == N
        for (a, c), (b, _) in zip(ranges, ranges[1:]):
            assert a + c == b
    with pytest.raises(ValueError):
        shard.row_range(4, 8, 0)
