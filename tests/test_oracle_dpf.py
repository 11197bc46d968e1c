"""Pins for oracle O2-O8 (tree step, Eval, Gen, contraction, reconstruct,
naive PIR) against what the paper and the mathematics fix:

* the DPF contract Eval(k_a, j) + Eval(k_b, j) = beta [j = alpha],
  exhaustively over every alpha for small n and for config c1 (n = 10, BJ:7);
* Eq. 1-3 evaluated recursively with the *library* ChaCha20 on a tiny tree;
* eval_point == eval_full, path parity;
* PRF block counts: n per point, N-1 per full eval (one block per
  internal node, reading R9), 2n per Gen;
* key payload = 64 log2 L bytes = Table 4;
* contraction == numpy uint32 matmul (wraps mod 2^32), naive PIR,
  reconstruction = beta T[alpha], shard linearity.
"""
import numpy as np
import pytest
from conftest import read_golden

import synth


def _seed(i):
    return bytes((i * 131 + k * 7) & 0xFF for k in range(32))


def _contract_check(oracle, n, alpha, beta, seed):
    k0, k1 = oracle.gen(n, alpha, beta, seed)
    y0, y1 = oracle.eval_full(k0), oracle.eval_full(k1)
    want = np.zeros(1 << n, np.uint32)
    want[alpha] = beta & 0xFFFFFFFF
    np.testing.assert_array_equal(y0 + y1, want)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_contract_exhaustive_small(oracle, n):
    r = np.random.default_rng(n)
    for alpha in range(1 << n):
        beta = int(r.integers(0, 1 << 32))
        _contract_check(oracle, n, alpha, beta, _seed(alpha + 100 * n))


def test_contract_exhaustive_c1(oracle):
    # config c1 (BJ:7): 2^10-entry domain, every alpha, beta = 1
    for alpha in range(1 << 10):
        _contract_check(oracle, 10, alpha, 1, _seed(alpha))


@pytest.mark.parametrize("n", [12, 16, 18])
def test_contract_random_alpha(oracle, n):
    r = np.random.default_rng(n)
    for t in range(3):
        alpha = int(r.integers(0, 1 << n))
        _contract_check(oracle, n, alpha, int(r.integers(0, 1 << 32)), _seed(1000 + t))


def test_beta_zero_and_max(oracle):
    _contract_check(oracle, 8, 77, 0, _seed(5))
    _contract_check(oracle, 8, 0, 0xFFFFFFFF, _seed(6))
    _contract_check(oracle, 8, 255, 0x80000000, _seed(7))


def test_eq3_recursion_with_library_prf(oracle):
    """Eq. 3 evaluated literally, recursively, with the
    `cryptography` ChaCha20 as PRF, on every leaf of a depth-3 tree."""
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

    def prf(s, c):
        enc = Cipher(algorithms.ChaCha20(s + bytes(16), bytes(16)), mode=None).encryptor()
        return enc.update(bytes(32))[16 * c:16 * c + 16]

    import ctypes
    n = 3
    k0, k1 = oracle.gen(n, 5, 1, _seed(9))
    for k in (k0, k1):
        cw = bytes(ctypes.string_at(ctypes.addressof(k.cw), 32 * 64))

        def C(t, c, d):  # C_t[c, d], stored cw[d-1][t][c]
            off = ((d - 1) * 4 + t * 2 + c) * 16
            return cw[off:off + 16]

        def P(d, j):
            if d == 0:
                return bytes(k.root)
            par = P(d - 1, j // 2)
            return bytes(a ^ b for a, b in zip(prf(par, j % 2), C(par[0] & 1, j % 2, d)))

        for j in range(1 << n):
            s = P(n, j)
            v = (int.from_bytes(s[4:8], "little") + (s[0] & 1) * k.cw_out) & 0xFFFFFFFF
            if k.party:
                v = (-v) & 0xFFFFFFFF
            assert oracle.eval_point(k, j) == v


def test_eval_point_equals_full_and_counts(oracle):
    for n in (1, 5, 11):
        k0, k1, gblocks = oracle.gen(n, (1 << n) - 1, 3, _seed(n), count_blocks=True)
        assert gblocks == 2 * n
        for k in (k0, k1):
            y, fblocks = oracle.eval_full(k, count_blocks=True)
            assert fblocks == (1 << n) - 1          # N-1: one block per internal node
            for j in list(range(min(1 << n, 64))) + [(1 << n) - 1]:
                v, pblocks = oracle.eval_point(k, j, count_blocks=True)
                assert pblocks == n
                assert v == y[j]


def test_path_parity_and_shared_codewords(oracle):
    n, alpha = 9, 300
    k0, k1 = oracle.gen(n, alpha, 1, _seed(42))
    assert bytes(k0.cw) == bytes(k1.cw)                # R4: codewords shared
    assert k0.root[0] & 1 == 0 and k1.root[0] & 1 == 1  # lsb(root) = party
    assert k0.cw_out == k1.cw_out
    s0, s1 = oracle.eval_full_seeds(k0), oracle.eval_full_seeds(k1)
    same = np.all(s0 == s1, axis=1)
    assert not same[alpha] and same.sum() == (1 << n) - 1
    assert (s0[alpha, 0] & 1) != (s1[alpha, 0] & 1)


def test_key_sizes_table4(oracle):
    for entries, log_n, key_bytes in read_golden("table4_key_bytes.txt"):
        assert 1 << int(log_n) == int(entries)
        assert oracle.key_wire_size(int(log_n)) - 32 == int(key_bytes)
    k0, k1 = oracle.gen(20, 12345, 1, _seed(1))
    w = oracle.key_to_wire(k0)
    assert len(w) == 32 + 1280
    k0b = oracle.key_from_wire(w)
    assert oracle.key_to_wire(k0b) == w
    assert len(oracle.key_to_wire(oracle.gen(20, 7, 1, _seed(2))[1])) == len(w)  # shape leakage


def test_gen_rejects_bad_args(oracle):
    with pytest.raises(ValueError):
        oracle.gen(4, 16, 1, _seed(0))
    with pytest.raises(ValueError):
        oracle.gen(0, 0, 1, _seed(0))
    with pytest.raises(ValueError):
        oracle.gen(33, 0, 1, _seed(0))


def test_contraction_is_uint32_matmul(oracle):
    r = np.random.default_rng(3)
    for rows, D in ((1, 4), (37, 16), (4096, 12)):
        y = r.integers(0, 1 << 32, rows, dtype=np.uint32)
        T = r.integers(0, 1 << 32, (rows, D), dtype=np.uint32)
        np.testing.assert_array_equal(oracle.contract(y, T), y @ T)
        # exact wrap check with Python integers on the first column
        assert int(oracle.contract(y, T)[0]) == sum(int(a) * int(b) for a, b in zip(y, T[:, 0])) % (1 << 32)
    y = np.full(1000, 0xFFFFFFFF, np.uint32)
    T = np.full((1000, 4), 0xFFFFFFFF, np.uint32)
    np.testing.assert_array_equal(oracle.contract(y, T), np.full(4, 1000, np.uint32))  # (-1)(-1) = 1


def test_naive_pir(oracle):
    N, D = 512, 8
    T = synth.table(N, D, 11)
    r0 = np.random.default_rng(4).integers(0, 1 << 32, N, dtype=np.uint32)
    for alpha, beta in ((0, 1), (511, 1), (200, 0xDEADBEEF)):
        r1 = oracle.naive_pir_shares(N, alpha, beta, r0)
        ans = oracle.reconstruct(oracle.contract(r0, T), oracle.contract(r1, T))
        np.testing.assert_array_equal(ans, (np.uint64(beta) * T[alpha].astype(np.uint64) % (1 << 32)).astype(np.uint32))


def test_pir_reconstructs_row_batched(oracle):
    w = synth.CONFIGS["c1"]
    T = synth.table(w.N, w.D, w.seed)
    al = synth.alphas(8, w.N, w.seed)
    seeds = synth.gen_seeds(8, w.seed)
    pairs = [oracle.gen(w.log_n, int(a), 1, s) for a, s in zip(al, seeds)]
    sh0 = oracle.answer_batch([p[0] for p in pairs], T, threads=2)
    sh1 = oracle.answer_batch([p[1] for p in pairs], T, threads=3)
    np.testing.assert_array_equal(oracle.reconstruct(sh0, sh1), T[al.astype(np.int64)])


def test_shard_linearity_and_ragged_rows(oracle):
    n, D = 11, 12
    N = (1 << n) - 37  # non-power-of-two table: rows >= N are absent (R12)
    T = synth.table(N, D, 5)
    keys = [oracle.gen(n, a, 1, _seed(a))[p] for a, p in ((3, 0), (2000, 1), (1500, 0))]
    whole = oracle.answer_batch(keys, T)
    for cuts in ([0, 1024, N], [0, 1, 700, 1999, N], [0, N]):
        acc = np.zeros_like(whole)
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            acc += oracle.answer_batch(keys, T[lo:hi], row_begin=lo)
        np.testing.assert_array_equal(acc, whole)
    for i, k in enumerate(keys):
        np.testing.assert_array_equal(whole[i], oracle.eval_full(k)[:N] @ T)
