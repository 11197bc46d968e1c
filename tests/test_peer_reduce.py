"""Fused cross-GPU reduction: every rank's fused
kernel red.adds its row shard's partial answers straight into the egress
rank's buffer through a CUDA IPC mapping (DPF_EVAL_ACCUMULATE), instead of a
separate NCCL reduce.  The pool has one GPU, so the ranks here are processes
sharing cuda:0: the IPC mapping, the accumulate launches and the two barriers
are the multi-GPU code path; only the NVLink hop is absent.  The sum must equal
the CPU oracle on the whole table bit-exactly."""
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


def _worker(rank, world, port, case, outdir, mode="p2p"):
    import torch.distributed as dist
    from paper_2301_10904_b200 import dpfpir, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    n, N, D, B, prf, packed = case
    r0, rows = shard.row_range(N, world, rank)
    T = synth.table_rows(N, D, 77, r0, r0 + rows)
    Td = torch.from_numpy(T.view(np.int32)).cuda()
    tbl = dpfpir.table_pack(Td, r0) if packed else Td
    al = synth.alphas(B, N, 78)
    keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[i % 2] for i, (a, s) in enumerate(zip(al, synth.gen_seeds(B, 79)))]
    wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
    ws = torch.empty(dpfpir.eval_workspace_bytes(B, n, rows, D), dtype=torch.uint8, device="cuda")
    out = torch.full((B, D), -1, dtype=torch.int32, device="cuda")  # garbage until the owner zeroes it
    if mode == "reduce":
        # the product's shard evaluation under a process group, answers summed
        # by shard.reduce_partial_shares (the bench's NCCL path; gloo on host
        # tensors here because the ranks share one GPU)
        for _ in range(2):
            part = dpfpir.eval_batch_wire_packed(wire, n, tbl, out=out, workspace=ws, prf=prf) if packed else \
                dpfpir.eval_batch_wire(wire, n, tbl, r0, out=out, workspace=ws, prf=prf)
            host = part.cpu()
            shard.reduce_partial_shares(host, dst=0)
        if rank == 0:
            np.save(os.path.join(outdir, "sum.npy"), host.numpy().view(np.uint32))
            np.save(os.path.join(outdir, "keys.npy"), dpfpir.keys_to_wire(keys))
        dist.barrier()
        dist.destroy_process_group()
        return
    red = shard.PeerShareReducer(out, dst=0)
    for _ in range(3):  # repeated steps: zero, accumulate, complete
        red.begin()
        dpfpir.eval_batch_wire_ex(wire, n, tbl, r0, rows, D, red.ptr, dpfpir.DPF_EVAL_ACCUMULATE, ws, prf=prf,
                                  packed=packed)
        red.finish()
    if rank == 0:
        np.save(os.path.join(outdir, "sum.npy"), dpfpir.as_u32(out))
        np.save(os.path.join(outdir, "keys.npy"), dpfpir.keys_to_wire(keys))
    dist.barrier()
    red.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (12, 4096, 64, 40, 1, False)),      # IMAD kernel
    (3, (12, 4000, 256, 70, 1, True)),      # tcgen05 CTA pairs, unequal shards
    (2, (14, 10000, 128, 33, 3, True)),     # early termination, tcgen05
])
@pytest.mark.parametrize("mode", ["p2p", "reduce"])
def test_peer_accumulate_equals_oracle(oracle, tmp_path, world, case, mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_2301_10904_b200 import build as pbuild
    pbuild.build()
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path), mode), nprocs=world, join=True)
    n, N, D, B, prf, packed = case
    got = np.load(tmp_path / "sum.npy")
    wire = np.load(tmp_path / "keys.npy")
    okeys = [oracle.key_from_wire(bytes(wire[i])) for i in range(B)]
    want = oracle.answer_batch(okeys, synth.table(N, D, 77), threads=16)
    np.testing.assert_array_equal(got, want)
