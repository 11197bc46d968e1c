"""Pins for the oracle's AES-128 PRF (row f1; FIPS-197, the paper's baseline
PRF P:530 / Table 4): printed vectors (FIPS-197 C.1, GCM TC1), S-box entries
printed in FIPS-197 5.1.1 / Fig. 7, the `cryptography` library on random keys,
and the DPF contract with AES as the tree PRF."""
import numpy as np
import pytest
from conftest import read_golden

from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes


def lib_aes(key: bytes, block: bytes) -> bytes:
    enc = Cipher(algorithms.AES(key), modes.ECB()).encryptor()
    return enc.update(block) + enc.finalize()


def test_printed_vectors(oracle):
    rows = read_golden("fips197_aes128.txt")
    assert len(rows) == 3
    for src, key, pt, ct in rows:
        assert oracle.aes128_encrypt(bytes.fromhex(key), bytes.fromhex(pt)).hex() == ct, src


def test_sbox_printed_entries(oracle):
    # FIPS-197 5.1.1: S(0x53) = 0xed; Fig. 7 corners
    assert oracle.aes_sbox(0x53) == 0xED
    assert oracle.aes_sbox(0x00) == 0x63 and oracle.aes_sbox(0xFF) == 0x16 and oracle.aes_sbox(0x01) == 0x7C
    assert sorted(oracle.aes_sbox(x) for x in range(256)) == list(range(256))  # a permutation


def test_matches_library_random(oracle):
    r = np.random.default_rng(5)
    for _ in range(200):
        key = bytes(r.integers(0, 256, 16, dtype=np.uint8))
        blk = bytes(r.integers(0, 256, 16, dtype=np.uint8))
        assert oracle.aes128_encrypt(key, blk) == lib_aes(key, blk)


def test_prf_aes_layout(oracle):
    r = np.random.default_rng(6)
    for _ in range(100):
        s = bytes(r.integers(0, 256, 16, dtype=np.uint8))
        assert oracle.prf_aes(s, 0) == lib_aes(s, bytes(16))
        assert oracle.prf_aes(s, 1) == lib_aes(s, bytes(15) + b"\x01")


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_contract_aes_exhaustive(oracle, n):
    r = np.random.default_rng(n)
    for alpha in range(1 << n):
        beta = int(r.integers(0, 1 << 32))
        seed = bytes((alpha * 29 + k * 3 + n) & 0xFF for k in range(32))
        k0, k1, blocks = oracle.gen(n, alpha, beta, seed, count_blocks=True, prf=oracle.PRF_AES128)
        assert blocks == 2 * n and k0.prf == k1.prf == oracle.PRF_AES128
        y0, fb = oracle.eval_full(k0, count_blocks=True)
        assert fb == (1 << n) - 1
        want = np.zeros(1 << n, np.uint32)
        want[alpha] = beta
        np.testing.assert_array_equal(y0 + oracle.eval_full(k1), want)
        assert oracle.eval_point(k0, alpha) == y0[alpha]


def test_aes_key_wire_roundtrip(oracle):
    k0, _ = oracle.gen(12, 77, 1, bytes(32), prf=oracle.PRF_AES128)
    w = oracle.key_to_wire(k0)
    assert w[5] == 2 and len(w) == 32 + 64 * 12
    assert oracle.key_to_wire(oracle.key_from_wire(w)) == w
