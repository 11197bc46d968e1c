"""The product's row-sharded path under a process group: every
rank evaluates its row shard with dpf_eval_batch_wire / _packed on the GPU
(this pool has one GPU, so all ranks share cuda:0), the int32 partial
answers are summed by shard.reduce_partial_shares (gloo here; NCCL in
bench.py on a multi-GPU node), and rank 0 compares the sum with the oracle
over the whole table, bit-exactly.  An all-0xFFFFFFFF table makes every
partial wrap int32, so the reduce must be the wrapping Z_2^32 sum."""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, N, D, B, packed, ones, q):
    import torch.distributed as dist
    from oracle import oracle as orc
    from paper_2301_10904_b200 import dpfpir, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        T = np.full((N, D), 0xFFFFFFFF, np.uint32) if ones else synth.table(N, D, 91)
        al = synth.alphas(B, N, 91)
        pairs = [dpfpir.gen(n, int(a), 1, s) for a, s in zip(al, synth.gen_seeds(B, 91))]
        keys = [p[b % 2] for b, p in enumerate(pairs)]
        r0, rows = shard.row_range(N, world, rank)
        Tsh = torch.from_numpy(T[r0:r0 + rows].view(np.int32)).cuda()
        wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
        if packed:
            part = dpfpir.eval_batch_wire_packed(wire, n, dpfpir.table_pack(Tsh, r0))
        else:
            part = dpfpir.eval_batch_wire(wire, n, Tsh, r0)
        torch.cuda.synchronize()
        host = part.cpu()
        shard.reduce_partial_shares(host, dst=0)
        if rank == 0:
            want = orc.answer_batch([orc.key_from_wire(dpfpir.key_serialize(k)) for k in keys], T, threads=4)
            q.put(bool(np.array_equal(host.numpy().view(np.uint32), want)))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_10904_b200 import build as pbuild
    pbuild.build()


@pytest.mark.parametrize("world,n,N,D,B,packed,ones", [
    (2, 14, 1 << 14, 64, 40, False, False),
    (3, 13, 7000, 128, 33, True, False),
    (2, 12, 4096, 32, 17, False, True),
])
def test_product_shards_reduce_to_whole(built, world, n, N, D, B, packed, ones):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, N, D, B, packed, ones, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=10)
