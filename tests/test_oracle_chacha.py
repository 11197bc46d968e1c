"""Pins for oracle O1 (ChaCha20 block, RFC 8439 2.3) and the tree PRF layout
(reading R8: key = s || 0^128, counter 0, nonce 0, child c = bytes [16c, 16c+16)).

Pinned against (a) vectors printed in RFC 8439 (tests/golden), (b) the
independent `cryptography` library implementation of ChaCha20.
"""
import os

import numpy as np
import pytest
from conftest import read_golden

cryptography = pytest.importorskip("cryptography")
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms  # noqa: E402


def lib_keystream(key: bytes, counter: int, nonce: bytes, n: int = 64) -> bytes:
    # cryptography's ChaCha20 takes a 16-byte nonce = LE32 counter || 96-bit nonce
    enc = Cipher(algorithms.ChaCha20(key, counter.to_bytes(4, "little") + nonce), mode=None).encryptor()
    return enc.update(b"\0" * n)


def test_rfc8439_printed_vectors(oracle):
    rows = read_golden("rfc8439_chacha20_block.txt")
    assert len(rows) == 6
    for src, key, ctr, nonce, block in rows:
        got = oracle.chacha20_block(bytes.fromhex(key), int(ctr), bytes.fromhex(nonce))
        assert got.hex() == block, src


def test_block_matches_library_random(oracle):
    r = np.random.default_rng(1)
    for _ in range(300):
        key = bytes(r.integers(0, 256, 32, dtype=np.uint8))
        nonce = bytes(r.integers(0, 256, 12, dtype=np.uint8))
        ctr = int(r.integers(0, 1 << 32))
        assert oracle.chacha20_block(key, ctr, nonce) == lib_keystream(key, ctr, nonce)


def test_prf_zero_seed_is_rfc_tv1(oracle):
    # PRF(0^128, c) = RFC 8439 A.1 TV#1 keystream bytes [16c, 16c+16)
    tv1 = bytes.fromhex([r for r in read_golden("rfc8439_chacha20_block.txt") if r[0] == "RFC8439-A.1#1"][0][4])
    assert oracle.prf(bytes(16), 0) == tv1[0:16]
    assert oracle.prf(bytes(16), 1) == tv1[16:32]
    assert tv1[0:16].hex() == "76b8e0ada0f13d90405d6ae55386bd28"


def test_prf_layout_matches_library(oracle):
    r = np.random.default_rng(2)
    for _ in range(300):
        s = bytes(r.integers(0, 256, 16, dtype=np.uint8))
        ks = lib_keystream(s + bytes(16), 0, bytes(12), 32)
        assert oracle.prf(s, 0) == ks[:16]
        assert oracle.prf(s, 1) == ks[16:32]
        assert oracle.prf(s, 0) != oracle.prf(s, 1)  # S:41 distinct children
