"""Pins of the PBR oracle (partial batch retrieval, §4.1, P:598-602;
reading R21): the bin split, the one-query-per-bin rule with drops, and the
server answers, each checked against something other than the oracle itself:
brute-force reconstruction of the table rows, closed-form drop counts and
block counts, and the I = N special case (one bin = plain DPF-PIR)."""
import numpy as np
import pytest

import synth


def _pbr_keys(oracle, index, log_i, I, seeds, rng):
    """Both parties' keys for every bin: the kept in-bin index, or a dummy."""
    k0, k1 = [], []
    for b, idx in enumerate(index):
        a = idx if idx >= 0 else int(rng.integers(0, I))
        p = oracle.gen(log_i, a, 1, next(seeds))
        k0.append([p[0]])
        k1.append([p[1]])
    return k0, k1


@pytest.mark.parametrize("N,log_i,need", [(1 << 10, 6, 12), (1 << 10, 8, 9), (1000, 7, 20), (1 << 9, 9, 5)])
def test_pbr_reconstructs_kept_rows_and_counts_drops(oracle, N, log_i, need):
    """Every kept row reconstructs to T[r] (brute force from the table);
    drops = distinct needed rows - distinct bins they hit (closed form)."""
    I = 1 << log_i
    T = synth.table(N, 8, 31 + N + log_i)
    rng = np.random.default_rng(N + log_i)
    seeds = iter(synth.gen_seeds(4096, N + log_i))
    for trial in range(4):
        needed = rng.integers(0, N, size=need)
        index, dropped = oracle.pbr_plan(needed, N, log_i)
        distinct = list(dict.fromkeys(int(r) for r in needed))
        assert len(index) == -(-N // I)
        assert len(dropped) == len(distinct) - len({r // I for r in distinct})
        kept = {b * I + i for b, i in enumerate(index) if i >= 0}
        assert kept | set(dropped) == set(distinct) and not (kept & set(dropped))
        for r in dropped:  # a dropped row's bin kept an earlier request
            b = r // I
            assert index[b] >= 0 and distinct.index(b * I + index[b]) < distinct.index(r)
        k0, k1 = _pbr_keys(oracle, index, log_i, I, seeds, rng)
        a0 = oracle.pbr_answer(k0, T, log_i)
        a1 = oracle.pbr_answer(k1, T, log_i)
        got = (a0.astype(np.uint64) + a1) & 0xFFFFFFFF
        for b, i in enumerate(index):
            if i >= 0:
                np.testing.assert_array_equal(got[b, 0], T[b * I + i])


def test_pbr_single_bin_is_plain_pir(oracle):
    """I = N: one bin, PBR reduces to one DPF-PIR query over the whole table."""
    n = 9
    N = 1 << n
    T = synth.table(N, 4, 5)
    al = synth.alphas(6, N, 5)
    keys = [oracle.gen(n, int(a), 1, s)[0] for a, s in zip(al, synth.gen_seeds(6, 5))]
    np.testing.assert_array_equal(oracle.pbr_answer([keys], T, n)[0], oracle.answer_batch(keys, T))


def test_pbr_work_law(oracle):
    """L/I bins x (I - 1) blocks per client (P:600 'saves computation by a
    factor of L/I' against L/I separate full-table queries)."""
    N, log_i = 1 << 10, 6
    I = 1 << log_i
    blocks = 0
    for b in range(oracle.pbr_n_bins(N, log_i)):
        k = oracle.gen(log_i, b % I, 1, synth.gen_seeds(1, b)[0])[0]
        blocks += oracle.eval_full(k, count_blocks=True)[1]
    assert blocks == (N // I) * (I - 1)


def test_pbr_ragged_last_bin_and_duplicates(oracle):
    """N not a multiple of I: the last bin holds N mod I rows; a row asked for
    twice is one query, not a drop."""
    N, log_i = 300, 7  # bins of 128: [0,128), [128,256), [256,300)
    assert oracle.pbr_n_bins(N, log_i) == 3
    index, dropped = oracle.pbr_plan([299, 5, 299, 7, 260], N, log_i)
    assert index == [5, -1, 43] and dropped == [7, 260]
    T = synth.table(N, 4, 9)
    k = oracle.gen(log_i, 43, 1, synth.gen_seeds(1, 9)[0])
    s = [oracle.answer_batch([k[x]], T[256:300]) for x in (0, 1)]
    np.testing.assert_array_equal((s[0].astype(np.uint64) + s[1]) & 0xFFFFFFFF, T[299:300])
