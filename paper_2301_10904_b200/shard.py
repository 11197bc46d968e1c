"""Row sharding across GPUs and the one exchange step ("each of
the N GPUs evaluate the DPF on a subset of the table indices, then summing
the result across GPUs at the end").

Rank r of G owns table rows [floor(r N / G), floor((r+1) N / G)) and calls
dpf_eval_batch_shard / dpf_eval_batch_wire with that row range (the kernel
descends the root path to its range, then expands only its subtrees).  The B x
D partial answers are summed mod 2^32 by ONE reduce to the egress rank: NCCL
over NVLink on GPUs (int32 SUM is two's-complement wrapping addition, i.e.
exactly Z_2^32 addition), gloo in the CPU tests.
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
