"""Client-side batch-PIR / ML co-design planner (row f2; §4).

The server side of the co-design workload is dpf_eval_grouped (one launch over
every table's hot and full batches); this module is the client half:

* hot-table split: each embedding table is split into a small
  "hot" table holding its most frequently accessed rows and the full table;
  the client keeps the hot-row index map;
* fixed query budget: every inference issues exactly Q_hot keys to
  each hot table and Q_full keys to each full table, padding with dummy
  queries, so the servers learn nothing from the number of keys; rows beyond
  the budget are dropped (the client tolerates dropped queries);
* partial batch retrieval (PBR, reading R21): the table is
  segmented into bins of I = 2^log_i rows and the client sends one key per
  bin, so one full-table PRF cost retrieves up to n_bins rows; a bin's second
  and later wanted rows are dropped, empty bins get dummy keys;
* reconstruction: the two servers' answers are added mod 2^32.

Pure host logic (numpy); the DPF keys come from libdpfpir's dpf_gen.
"""
from __future__ import annotations

import dataclasses
from typing import Sequence

import numpy as np


@dataclasses.dataclass
class HotSplit:
    """Hot rows of one table: the `n_hot` most frequent ("hot table")."""
    hot_rows: np.ndarray  # table row of hot entry h (sorted by decreasing frequency)
    n_rows: int

    @classmethod
    def from_frequency(cls, freq: np.ndarray, hot_fraction: float) -> "HotSplit":
        n_hot = max(1, int(round(len(freq) * hot_fraction)))
        order = np.argsort(-np.asarray(freq, dtype=np.float64), kind="stable")
        return cls(hot_rows=order[:n_hot].astype(np.int64), n_rows=len(freq))

    @property
    def n_hot(self) -> int:
        return len(self.hot_rows)

    def hot_table(self, table: np.ndarray) -> np.ndarray:
        """The server-side hot table (built offline, like the table itself)."""
        return np.ascontiguousarray(table[self.hot_rows])

    def hot_index(self) -> dict:
        """Client-side map: table row -> hot-table index."""
        return {int(r): h for h, r in enumerate(self.hot_rows)}


@dataclasses.dataclass
class TablePlan:
    """One inference's queries to one table: exactly q_hot hot and q_full full."""
    hot_idx: np.ndarray    # indices into the hot table (dummies included)
    hot_real: np.ndarray   # bool: real query (else dummy)
    hot_rows: np.ndarray   # table row each real hot query retrieves (-1 for dummies)
    full_idx: np.ndarray   # indices into the full table
    full_real: np.ndarray
    dropped: int           # needed rows that did not fit the budget


def plan_table(needed_rows: Sequence[int], split: HotSplit, hot_map: dict, q_hot: int, q_full: int,
               rng: np.random.Generator) -> TablePlan:
    """Route each needed row to the hot table if present there, else to the full
    table; pad both to the fixed budgets with uniformly random dummy indices."""
    needed = list(dict.fromkeys(int(r) for r in needed_rows))  # dedupe, keep order
    hot_q, full_q, dropped = [], [], 0
    for r in needed:
        if r in hot_map and len(hot_q) < q_hot:
            hot_q.append((hot_map[r], r))
        elif len(full_q) < q_full:
            full_q.append(r)
        else:
            dropped += 1
    hot_idx = np.empty(q_hot, np.int64)
    hot_real = np.zeros(q_hot, bool)
    hot_rows = np.full(q_hot, -1, np.int64)
    for i in range(q_hot):
        if i < len(hot_q):
            hot_idx[i], hot_rows[i], hot_real[i] = hot_q[i][0], hot_q[i][1], True
        else:
            hot_idx[i] = rng.integers(0, split.n_hot)
    full_idx = np.empty(q_full, np.int64)
    full_real = np.zeros(q_full, bool)
    for i in range(q_full):
        if i < len(full_q):
            full_idx[i], full_real[i] = full_q[i], True
        else:
            full_idx[i] = rng.integers(0, split.n_rows)
    return TablePlan(hot_idx, hot_real, hot_rows, full_idx, full_real, dropped)


def log2_domain(rows: int) -> int:
    """Tree depth for a table of `rows` rows (rows >= 2^n absent, reading R12)."""
    return max(1, int(rows - 1).bit_length())


@dataclasses.dataclass
class PbrPlan:
    """One client's PBR query to one table: one key per bin."""
    log_i: int
    index: np.ndarray    # in-bin index each bin's key targets (dummies included)
    real: np.ndarray     # bool per bin: a wanted row (else a dummy)
    rows: np.ndarray     # table row retrieved per bin (-1 for dummies)
    dropped: np.ndarray  # wanted rows lost to bin collisions (request order)

    @property
    def n_bins(self) -> int:
        return len(self.index)


def pbr_n_bins(n_rows: int, log_i: int) -> int:
    """ceil(L / I): the last bin is ragged when I does not divide L."""
    return -(-n_rows >> log_i)


def plan_pbr(needed_rows: Sequence[int], n_rows: int, log_i: int, rng: np.random.Generator) -> PbrPlan:
    """Bin each wanted row (bin = row >> log_i); per bin keep the first wanted
    row in request order (repeats of a row count once), drop the others; bins
    with no wanted row get a uniformly random dummy index."""
    rows = np.asarray(needed_rows, dtype=np.int64).ravel()
    nb = pbr_n_bins(n_rows, log_i)
    _, first = np.unique(rows, return_index=True)
    uniq = rows[np.sort(first)]                       # distinct rows, request order
    bins = uniq >> log_i
    _, keep_at = np.unique(bins, return_index=True)   # first wanted row of each hit bin
    keep = np.zeros(len(uniq), bool)
    keep[keep_at] = True
    index = rng.integers(0, 1 << log_i, size=nb, dtype=np.int64)
    real = np.zeros(nb, bool)
    out_rows = np.full(nb, -1, np.int64)
    kb = bins[keep]
    index[kb] = uniq[keep] - (kb << log_i)
    real[kb] = True
    out_rows[kb] = uniq[keep]
    return PbrPlan(log_i, index, real, out_rows, uniq[~keep])
