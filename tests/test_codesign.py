"""Co-design planner (row f2): hot-table split, fixed per-table
query budgets with dummy padding, dropped-query accounting, and (with the
oracle as the two servers) reconstruction of every real query's row."""
import numpy as np

import synth
from paper_2301_10904_b200 import codesign


def test_hot_split_takes_most_frequent_rows():
    freq = synth.codesign_frequency(3, 4096)
    sp = codesign.HotSplit.from_frequency(freq, 0.1)
    assert sp.n_hot == 410
    assert freq[sp.hot_rows].min() >= np.delete(freq, sp.hot_rows).max()
    T = synth.table(4096, 8, 1)
    np.testing.assert_array_equal(sp.hot_table(T)[5], T[sp.hot_rows[5]])


def test_plan_fixed_budget_and_drops():
    rng = np.random.default_rng(0)
    freq = synth.codesign_frequency(0, 1 << 12)
    sp = codesign.HotSplit.from_frequency(freq, 0.1)
    hm = sp.hot_index()
    needed = synth.codesign_needed(0, 1 << 12, 200, 6)
    total_drop = 0
    for row in needed:
        tp = codesign.plan_table(row, sp, hm, q_hot=3, q_full=2, rng=rng)
        assert len(tp.hot_idx) == 3 and len(tp.full_idx) == 2          # fixed shape: nothing leaks
        assert tp.hot_idx.min() >= 0 and tp.hot_idx.max() < sp.n_hot
        assert tp.full_idx.min() >= 0 and tp.full_idx.max() < sp.n_rows
        real = set(sp.hot_rows[tp.hot_idx[tp.hot_real]]) | set(tp.full_idx[tp.full_real])
        distinct = set(int(r) for r in row)
        assert real <= distinct
        assert len(real) + tp.dropped == len(distinct)
        np.testing.assert_array_equal(sp.hot_rows[tp.hot_idx[tp.hot_real]], tp.hot_rows[tp.hot_real])
        total_drop += tp.dropped
    assert total_drop > 0  # the budget is binding for some inferences


def test_end_to_end_reconstruction_with_oracle_servers(oracle):
    """Two servers (the oracle) answer the hot and full batches of 3 tables;
    the client adds the answers and gets the rows of every real query."""
    rng = np.random.default_rng(1)
    seeds = iter(synth.gen_seeds(1000, 77))
    for t, lg in enumerate((12, 13, 12)):
        N = 1 << lg
        T = synth.table(N, 4, 100 + t)
        sp = codesign.HotSplit.from_frequency(synth.codesign_frequency(t, N), 0.1)
        H = sp.hot_table(T)
        needed = synth.codesign_needed(t, N, 4, 5)
        for row in needed:
            tp = codesign.plan_table(row, sp, sp.hot_index(), q_hot=2, q_full=1, rng=rng)
            for idx, real, tbl, dom_rows, rows_of in ((tp.hot_idx, tp.hot_real, H, sp.n_hot, tp.hot_rows),
                                                     (tp.full_idx, tp.full_real, T, N, tp.full_idx)):
                n = codesign.log2_domain(dom_rows)
                pairs = [oracle.gen(n, int(i), 1, next(seeds)) for i in idx]
                a0 = oracle.answer_batch([p[0] for p in pairs], tbl)
                a1 = oracle.answer_batch([p[1] for p in pairs], tbl)
                got = oracle.reconstruct(a0, a1)
                for q in np.nonzero(real)[0]:
                    np.testing.assert_array_equal(got[q], T[rows_of[q]])


def test_pbr_planner_matches_oracle_rule(oracle):
    """The product's client PBR planner (vectorised) keeps and drops exactly
    the rows the oracle's loop (R21) does."""
    rng = np.random.default_rng(3)
    for N, log_i, need in ((1 << 12, 8, 30), (1 << 12, 10, 6), (5000, 9, 40), (1 << 10, 10, 3)):
        for row in synth.codesign_needed(1, N, 20, need):
            pp = codesign.plan_pbr(row, N, log_i, rng)
            index, dropped = oracle.pbr_plan(row, N, log_i)
            assert pp.n_bins == len(index) == codesign.pbr_n_bins(N, log_i)
            np.testing.assert_array_equal(pp.real, np.array(index) >= 0)
            np.testing.assert_array_equal(pp.index[pp.real], np.array(index)[pp.real])
            np.testing.assert_array_equal(pp.dropped, dropped)
            assert pp.index.min() >= 0 and pp.index.max() < (1 << log_i)
            np.testing.assert_array_equal(pp.rows[pp.real], (np.nonzero(pp.real)[0] << log_i) + pp.index[pp.real])
