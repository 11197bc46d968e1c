"""Row sharding across GPUs and the one exchange step ("each of
the N GPUs evaluate the DPF on a subset of the table indices, then summing
the result across GPUs at the end").

Rank r of G owns table rows [floor(r N / G), floor((r+1) N / G)) and calls
dpf_eval_batch_shard / dpf_eval_batch_wire with that row range (the kernel
descends the root path to its range, then expands only its subtrees).  The B x
D partial answers are summed mod 2^32 at the egress rank, either by ONE NCCL
reduce over NVLink (int32 SUM is two's-complement wrapping addition, i.e.
exactly Z_2^32 addition; gloo in the CPU tests), or inside the fused kernels
themselves (PeerShareReducer): every rank's epilogue red.global.adds its
partial answers straight into the egress rank's buffer, mapped over NVLink
with CUDA IPC, so the exchange overlaps the evaluation and no collective runs
on the data path.
"""
from __future__ import annotations


def row_range(N: int, world: int, rank: int) -> tuple[int, int]:
    """(row_begin, row_count) of `rank`'s shard."""
    if not (0 <= rank < world) or N < world:
        raise ValueError("need 0 <= rank < world <= N")
    r0 = N * rank // world
    r1 = N * (rank + 1) // world
    return r0, r1 - r0


def reduce_partial_shares(partial, dst: int = 0, group=None):
    """Sum the ranks' int32 [B, D] partial answers into `partial` on rank
    `dst` (mod 2^32).  The only collective on the data path."""
    import torch
    import torch.distributed as dist
    if partial.dtype != torch.int32:
        raise TypeError("partial shares travel as int32 (uint32 bit patterns)")
    dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return partial


class PeerShareReducer:
    """Fused cross-GPU reduction: all ranks accumulate (DPF_EVAL_ACCUMULATE)
    into the egress rank's answer buffer through a CUDA IPC mapping.

    Per step: the egress rank zeroes its buffer, a barrier orders that before
    any rank's kernel, every rank launches its shard's evaluation into the
    shared buffer, and a second barrier (after each rank's stream drained)
    makes the sum complete at the egress rank.  Handles travel once, at set-up,
    over the process group (64 bytes)."""

    def __init__(self, out, dst: int = 0, group=None):
        import torch
        import torch.distributed as dist
        from . import dpfpir
        self.dist, self.group, self.dst = dist, group, dst
        self.rank = dist.get_rank(group)
        self.out = out  # the egress rank's [B, D] int32 answer buffer (same shape on every rank)
        h = torch.zeros(dpfpir.IPC_HANDLE_BYTES + 8, dtype=torch.uint8)  # handle | u64 offset
        if self.rank == dst:
            handle, off = dpfpir.ipc_export(out)
            h.copy_(torch.frombuffer(bytearray(handle + off.to_bytes(8, "little")), dtype=torch.uint8))
        hb = h.to(out.device) if dist.get_backend(group) == "nccl" else h
        dist.broadcast(hb, src=dst, group=group)
        raw = bytes(hb.cpu().numpy().tobytes())
        self._mapped = None
        if self.rank == dst:
            self.ptr = out.data_ptr()
        else:
            self._mapped = dpfpir.ipc_open(raw[:dpfpir.IPC_HANDLE_BYTES])
            self.ptr = self._mapped + int.from_bytes(raw[dpfpir.IPC_HANDLE_BYTES:], "little")

    def begin(self, stream=None):
        """Egress rank zeroes the buffer; no rank adds before that completes."""
        import torch
        if self.rank == self.dst:
            self.out.zero_()
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        self.dist.barrier(group=self.group)

    def finish(self, stream=None):
        """After every rank's accumulate launch: the sum is complete at dst."""
        import torch
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        self.dist.barrier(group=self.group)

    def close(self):
        from . import dpfpir
        if self._mapped is not None:
            dpfpir.ipc_close(self._mapped)
            self._mapped = None
