"""Synthetic workload generators (see synth/__init__.py and DESIGN.md).

All streams come from numpy's PCG64 seeded with (config seed, stream id), so
every process (oracle, CUDA path, every rank) regenerates identical inputs.
Distributions follow the paper's workloads: embedding tables of L rows with
D int32 words per row ("2048-bit entries"), stored as uint32 bit
patterns uniform over all 2^32 values; query indices uniform over the rows
(one queried index per DPF key); beta = 1 for PIR unless a test
asks for a random beta.
"""
from __future__ import annotations

import dataclasses

import numpy as np

__all__ = ["Workload", "CONFIGS", "CODESIGN_LOG2_ROWS", "CODESIGN_D", "codesign_frequency", "codesign_needed", "table", "table_rows", "alphas", "betas", "gen_seeds", "rng"]

_STREAM_TABLE, _STREAM_ALPHA, _STREAM_BETA, _STREAM_GEN = 1, 2, 3, 4


def rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, stream]))


TABLE_BLOCK_ROWS = 1 << 16


def table_rows(N: int, D: int, seed: int, r0: int, r1: int) -> np.ndarray:
    """Rows [r0, r1) of the int32 embedding table T[N][D] (uint32 bit patterns,
    uniform).  Generated in blocks of 2^16 rows, each from its own PCG64
    stream, so a rank can build just its row shard."""
    assert 0 <= r0 <= r1 <= N
    out = np.empty((r1 - r0, D), np.uint32)
    blk = r0 // TABLE_BLOCK_ROWS
    while blk * TABLE_BLOCK_ROWS < r1:
        b0 = blk * TABLE_BLOCK_ROWS
        b1 = min(b0 + TABLE_BLOCK_ROWS, N)
        g = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, _STREAM_TABLE, blk]))
        rows = g.integers(0, 1 << 32, size=(b1 - b0, D), dtype=np.uint32)
        lo, hi = max(b0, r0), min(b1, r1)
        out[lo - r0:hi - r0] = rows[lo - b0:hi - b0]
        blk += 1
    return out


def table(N: int, D: int, seed: int) -> np.ndarray:
    """The whole int32 embedding table T[N][D] (see table_rows)."""
    return table_rows(N, D, seed, 0, N)


def alphas(B: int, N: int, seed: int) -> np.ndarray:
    """Queried row per key, uniform over [0, N)."""
    return rng(seed, _STREAM_ALPHA).integers(0, N, size=B, dtype=np.uint64)


def betas(B: int, seed: int, random: bool = False) -> np.ndarray:
    if not random:
        return np.ones(B, np.uint32)
    return rng(seed, _STREAM_BETA).integers(0, 1 << 32, size=B, dtype=np.uint32)


def gen_seeds(B: int, seed: int) -> list[bytes]:
    """32-byte DRBG seed per key (the randomness Gen draws)."""
    raw = rng(seed, _STREAM_GEN).integers(0, 256, size=(B, 32), dtype=np.uint8)
    return [bytes(r) for r in raw]


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    log_n: int      # tree depth n; domain 2^n
    N: int          # table rows (<= 2^n)
    D: int          # int32 words per row
    B: int          # keys per batch
    seed: int
    note: str = ""


# BASELINE.json "configs" (c1..c4); c5 is the grouped co-design workload (NEXT).
CONFIGS = {
    "c1": Workload("c1", 10, 1 << 10, 16, 1, 0x7AB1E001, "2^10 x 16, B=1, both servers in-process"),
    "c2": Workload("c2", 16, 1 << 16, 64, 64, 0x7AB1E002, "2^16 x 64, B=64, 1 GPU"),
    "c3": Workload("c3", 20, 1 << 20, 256, 256, 0x7AB1E003, "2^20 x 256 int32 (1 GiB), B=256, 1 GPU"),
    "c4": Workload("c4", 24, 1 << 24, 64, 512, 0x7AB1E004, "2^24 x 64, B=512, row-sharded over G GPUs"),
    "t5": Workload("t5", 20, 1 << 20, 64, 512, 0x7AB1E005, "Table 5 shape: 2^20 x 64, B=512 (context)"),
}


# Config c5 (BASELINE.json): 26 recommendation tables of mixed sizes, D = 32.
# log2 row counts [12..22, 12..22, 12..15]; accesses Zipf(1.0)
# per table (embedding accesses are heavily skewed).
CODESIGN_LOG2_ROWS = list(range(12, 23)) + list(range(12, 23)) + list(range(12, 16))
CODESIGN_D = 32


def codesign_frequency(table_id: int, n_rows: int, seed: int = 0xC0DE5) -> np.ndarray:
    """Zipf(1.0) access frequency of each row, over a random row permutation."""
    g = rng(seed + table_id, 11)
    perm = g.permutation(n_rows)
    freq = np.empty(n_rows, np.float64)
    freq[perm] = 1.0 / np.arange(1, n_rows + 1)
    return freq


def codesign_needed(table_id: int, n_rows: int, n_inferences: int, per_inference: int,
                    seed: int = 0xC0DE5) -> np.ndarray:
    """Rows each inference needs from one table: `per_inference` draws from
    the table's Zipf(1.0) access distribution.  int64 [n_inferences, per_inference]."""
    freq = codesign_frequency(table_id, n_rows, seed)
    p = freq / freq.sum()
    g = rng(seed + table_id, 12)
    return g.choice(n_rows, size=(n_inferences, per_inference), p=p)
