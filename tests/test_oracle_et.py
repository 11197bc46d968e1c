"""Pins for the oracle's early-termination scheme (SURVEY 8(f) row f4,
DESIGN.md reading R20, prf id 3): the GGM tree of Eq. 1-3 stops 4
levels early (depth h = log_n - 4) and every final node s yields its 16
leaves from one ChaCha20 block, Convert(s) (counter 1), corrected by the
16-word leaf codeword CWL.

Pinned against what the mathematics and independent code fix:

* Convert == the `cryptography` library's ChaCha20 keystream block 1 under
  key s || 0^128, nonce 0;
* the DPF contract Eval(k0, j) + Eval(k1, j) = beta [j = alpha],
  exhaustively over every alpha at n = 5, 6, 7 and n = 10 (config c1's
  domain), random alpha up to n = 20;
* Eq. 3 evaluated literally and recursively with the library ChaCha20 for the
  tree AND for Convert, on every leaf of a small domain;
* eval_point == eval_full; block counts 2^(h+1) - 1 per full evaluation
  (2^h - 1 internal nodes + 2^h conversions), h + 1 per point, 2h + 2 per Gen;
* the tree part is the standard scheme: roots and codeword columns 1..h equal
  those of a depth-h ChaCha20 key for alpha >> 4 drawn from the same DRBG seed;
* key wire size 32 + 64 (log_n - 3) and codec round trip;
* reconstruction = T[alpha], shard linearity, numpy uint32 matmul.
"""
import ctypes

import numpy as np
import pytest

import synth

cryptography = pytest.importorskip("cryptography")
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms  # noqa: E402

ET = 3


def _seed(i):
    return bytes((i * 37 + k * 11 + 5) & 0xFF for k in range(32))


def _lib_block(s: bytes, counter: int) -> bytes:
    enc = Cipher(algorithms.ChaCha20(s + bytes(16), counter.to_bytes(4, "little") + bytes(12)), mode=None).encryptor()
    return enc.update(bytes(64))


def _contract(oracle, n, alpha, beta, seed):
    k0, k1 = oracle.gen(n, alpha, beta, seed, prf=ET)
    y = oracle.eval_full(k0) + oracle.eval_full(k1)
    want = np.zeros(1 << n, np.uint32)
    want[alpha] = beta & 0xFFFFFFFF
    np.testing.assert_array_equal(y, want)


def test_convert_is_library_block1(oracle):
    r = np.random.default_rng(20)
    for _ in range(200):
        s = bytes(r.integers(0, 256, 16, dtype=np.uint8))
        want = np.frombuffer(_lib_block(s, 1), "<u4")
        np.testing.assert_array_equal(oracle.convert(s), want)
        # block 0 of the same keystream is the tree PRF: conversion differs from expansion
        assert _lib_block(s, 0)[:32] == oracle.prf(s, 0) + oracle.prf(s, 1)


@pytest.mark.parametrize("n", [5, 6, 7])
def test_contract_exhaustive_small(oracle, n):
    r = np.random.default_rng(n + 50)
    for alpha in range(1 << n):
        _contract(oracle, n, alpha, int(r.integers(0, 1 << 32)), _seed(alpha + 1000 * n))


def test_contract_exhaustive_n10(oracle):
    for alpha in range(1 << 10):
        _contract(oracle, 10, alpha, 1, _seed(alpha))


@pytest.mark.parametrize("n", [12, 16, 20])
def test_contract_random_alpha(oracle, n):
    r = np.random.default_rng(n)
    for t in range(2):
        _contract(oracle, n, int(r.integers(0, 1 << n)), int(r.integers(0, 1 << 32)), _seed(77 + t))


def test_literal_recursion_with_library(oracle):
    """Eq. 3 down to depth h, then Convert, both with the library ChaCha20."""
    n = 7
    h = n - 4
    k0, k1 = oracle.gen(n, 93, 0xCAFEBABE, _seed(3), prf=ET)
    for k in (k0, k1):
        cw = bytes(ctypes.string_at(ctypes.addressof(k.cw), 32 * 64))
        cwl = list(k.cw_leaf)

        def C(t, c, d):
            off = ((d - 1) * 4 + t * 2 + c) * 16
            return cw[off:off + 16]

        def P(d, i):
            if d == 0:
                return bytes(k.root)
            par = P(d - 1, i // 2)
            ks = _lib_block(par, 0)[16 * (i % 2):16 * (i % 2) + 16]
            return bytes(a ^ b for a, b in zip(ks, C(par[0] & 1, i % 2, d)))

        for j in range(1 << n):
            s = P(h, j >> 4)
            w = int.from_bytes(_lib_block(s, 1)[4 * (j & 15):4 * (j & 15) + 4], "little")
            v = (w + (s[0] & 1) * cwl[j & 15]) & 0xFFFFFFFF
            if k.party:
                v = (-v) & 0xFFFFFFFF
            assert oracle.eval_point(k, j) == v


def test_eval_point_equals_full_and_counts(oracle):
    for n in (5, 9, 13):
        h = n - 4
        k0, k1, gblocks = oracle.gen(n, (1 << n) - 3, 5, _seed(n), count_blocks=True, prf=ET)
        assert gblocks == 2 * h + 2
        for k in (k0, k1):
            y, fblocks = oracle.eval_full(k, count_blocks=True)
            assert fblocks == (1 << (h + 1)) - 1
            for j in list(range(min(40, 1 << n))) + [(1 << n) - 1, (1 << n) - 3]:
                v, pblocks = oracle.eval_point(k, j, count_blocks=True)
                assert pblocks == h + 1
                assert v == y[j]


def test_tree_part_is_the_standard_scheme(oracle):
    n, alpha = 12, 2901
    h = n - 4
    e0, e1 = oracle.gen(n, alpha, 1, _seed(8), prf=ET)
    s0, s1 = oracle.gen(h, alpha >> 4, 1, _seed(8), prf=1)
    for e, s in ((e0, s0), (e1, s1)):
        assert bytes(e.root) == bytes(s.root)
        assert bytes(e.cw)[:64 * h] == bytes(s.cw)[:64 * h]
        assert e.cw_out == 0
    assert list(e0.cw_leaf) == list(e1.cw_leaf)
    assert e0.root[0] & 1 == 0 and e1.root[0] & 1 == 1


def test_key_size_and_codec(oracle):
    for n in (5, 10, 20, 24, 32):
        assert oracle.key_wire_size(n, ET) == 32 + 64 * (n - 3)
    k0, k1 = oracle.gen(20, 54321, 1, _seed(1), prf=ET)
    w = oracle.key_to_wire(k0)
    assert len(w) == 32 + 64 * 17 and w[5] == ET
    k0b = oracle.key_from_wire(w)
    assert oracle.key_to_wire(k0b) == w
    assert list(k0b.cw_leaf) == list(k0.cw_leaf)
    with pytest.raises(ValueError):
        oracle.key_from_wire(w[:-4])
    with pytest.raises(ValueError):
        oracle.gen(4, 3, 1, _seed(0), prf=ET)  # needs at least one tree level


def test_contraction_and_reconstruction(oracle):
    n, D = 11, 12
    N = (1 << n) - 21  # ragged: the last final node is partial
    T = synth.table(N, D, 9)
    al = [0, 15, 16, N - 1, 1000]
    pairs = [oracle.gen(n, a, 1, _seed(a), prf=ET) for a in al]
    sh0 = oracle.answer_batch([p[0] for p in pairs], T, threads=2)
    sh1 = oracle.answer_batch([p[1] for p in pairs], T)
    np.testing.assert_array_equal(oracle.reconstruct(sh0, sh1), T[al])
    for i, (k0, _) in enumerate(pairs):
        np.testing.assert_array_equal(sh0[i], oracle.eval_full(k0)[:N] @ T)
    acc = np.zeros_like(sh0)
    for lo, hi in ((0, 7), (7, 1031), (1031, N)):  # cuts inside final nodes
        acc += oracle.answer_batch([p[0] for p in pairs], T[lo:hi], row_begin=lo)
    np.testing.assert_array_equal(acc, sh0)
