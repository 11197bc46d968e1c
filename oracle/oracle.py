"""ctypes loader for the CPU oracle (oracle/dpf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package ``paper_2301_10904_b200``.  Shares no code with the CUDA path.

Every function here is argument marshalling around the plain C oracle; the
citations for what each computes are in dpf_oracle.c.  The exception is the
PBR section at the end (partial batch retrieval): plain Python
loops over bins, each bin answered by the C oracle's answer_batch.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dpf_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
MAX_LOG_N = 32


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C99, -O2, pthreads)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC,
                               "-lpthread"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class OracleKey(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("party", ctypes.c_uint32), ("cw_out", ctypes.c_uint32),
                ("prf", ctypes.c_uint32), ("root", ctypes.c_uint8 * 16), ("cw", ctypes.c_uint8 * (MAX_LOG_N * 2 * 2 * 16)),
                ("cw_leaf", ctypes.c_uint32 * 16)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u8p = ctypes.POINTER(ctypes.c_uint8)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        kp = ctypes.POINTER(OracleKey)
        L.oracle_chacha20_block.argtypes = [u8p, ctypes.c_uint32, u8p, u8p]
        L.oracle_prf.argtypes = [u8p, ctypes.c_uint32, u8p]
        L.oracle_key_struct_size.restype = ctypes.c_size_t
        L.oracle_gen.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, u8p, kp, kp, u64p]
        L.oracle_gen_prf.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, u8p, kp, kp,
                                     u64p]
        L.oracle_aes128_encrypt.argtypes = [u8p, u8p, u8p]
        L.oracle_aes_sbox.argtypes = [ctypes.c_uint8]
        L.oracle_aes_sbox.restype = ctypes.c_uint8
        L.oracle_prf_aes.argtypes = [u8p, ctypes.c_uint32, u8p]
        L.oracle_eval_point.argtypes = [kp, ctypes.c_uint64, u64p]
        L.oracle_eval_point.restype = ctypes.c_uint32
        L.oracle_eval_full.argtypes = [kp, u32p, u64p]
        L.oracle_eval_full_seeds.argtypes = [kp, u8p, u64p]
        L.oracle_contract.argtypes = [u32p, ctypes.c_uint64, u32p, ctypes.c_uint32, u32p]
        L.oracle_answer_rows.argtypes = [kp, u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, u32p, u64p]
        L.oracle_answer_batch.argtypes = [kp, ctypes.c_uint32, u32p, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_uint32, u32p, ctypes.c_uint32]
        L.oracle_reconstruct.argtypes = [u32p, u32p, ctypes.c_uint64, u32p]
        L.oracle_naive_pir_shares.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, u32p, u32p]
        L.oracle_key_wire_size.argtypes = [ctypes.c_uint32]
        L.oracle_key_wire_size.restype = ctypes.c_size_t
        L.oracle_key_wire_size_prf.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.oracle_key_wire_size_prf.restype = ctypes.c_size_t
        L.oracle_convert.argtypes = [u8p, u32p]
        L.oracle_key_to_wire.argtypes = [kp, u8p, ctypes.c_size_t]
        L.oracle_key_from_wire.argtypes = [u8p, ctypes.c_size_t, kp]
        assert L.oracle_key_struct_size() == ctypes.sizeof(OracleKey)
        _lib = L
    return _lib


def _u8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _u32(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _bytes_in(b) -> np.ndarray:
    return np.frombuffer(bytes(b), dtype=np.uint8).copy()


# ---------------------------------------------------------------- primitives

def chacha20_block(key: bytes, counter: int, nonce: bytes) -> bytes:
    out = np.zeros(64, np.uint8)
    lib().oracle_chacha20_block(_u8(_bytes_in(key)), counter, _u8(_bytes_in(nonce)), _u8(out))
    return out.tobytes()


PRF_CHACHA20, PRF_AES128 = 1, 2
# R20 / SURVEY 8(f) f4: ChaCha20 tree with early-terminated leaves (16 per final node)
PRF_CHACHA20_ET = 3
ET_BITS = 4


def convert(seed: bytes) -> np.ndarray:
    """R20 Convert(s): the 16 LE words of ChaCha20(key = s || 0^128, counter 1, nonce 0)."""
    w = np.zeros(16, np.uint32)
    lib().oracle_convert(_u8(_bytes_in(seed)), _u32(w))
    return w


def aes128_encrypt(key: bytes, block: bytes) -> bytes:
    out = np.zeros(16, np.uint8)
    lib().oracle_aes128_encrypt(_u8(_bytes_in(key)), _u8(_bytes_in(block)), _u8(out))
    return out.tobytes()


def aes_sbox(x: int) -> int:
    return lib().oracle_aes_sbox(x)


def prf_aes(seed: bytes, c: int) -> bytes:
    out = np.zeros(16, np.uint8)
    lib().oracle_prf_aes(_u8(_bytes_in(seed)), c, _u8(out))
    return out.tobytes()


def prf(seed: bytes, c: int) -> bytes:
    out = np.zeros(16, np.uint8)
    lib().oracle_prf(_u8(_bytes_in(seed)), c, _u8(out))
    return out.tobytes()


# ---------------------------------------------------------------- DPF

def gen(log_n: int, alpha: int, beta: int, rng_seed: bytes, count_blocks: bool = False, prf: int = PRF_CHACHA20):
    k0, k1 = OracleKey(), OracleKey()
    blocks = ctypes.c_uint64(0)
    rc = lib().oracle_gen_prf(log_n, alpha, beta & 0xFFFFFFFF, prf, _u8(_bytes_in(rng_seed)), ctypes.byref(k0),
                              ctypes.byref(k1), ctypes.byref(blocks))
    if rc:
        raise ValueError("oracle_gen rejected arguments (rc=%d)" % rc)
    return (k0, k1, blocks.value) if count_blocks else (k0, k1)


def eval_point(k: OracleKey, j: int, count_blocks: bool = False):
    blocks = ctypes.c_uint64(0)
    y = lib().oracle_eval_point(ctypes.byref(k), j, ctypes.byref(blocks))
    return (y, blocks.value) if count_blocks else y


def eval_full(k: OracleKey, count_blocks: bool = False):
    y = np.zeros(1 << k.log_n, np.uint32)
    blocks = ctypes.c_uint64(0)
    rc = lib().oracle_eval_full(ctypes.byref(k), _u32(y), ctypes.byref(blocks))
    if rc:
        raise RuntimeError("oracle_eval_full rc=%d" % rc)
    return (y, blocks.value) if count_blocks else y


def eval_full_seeds(k: OracleKey) -> np.ndarray:
    s = np.zeros((1 << k.log_n, 16), np.uint8)
    rc = lib().oracle_eval_full_seeds(ctypes.byref(k), _u8(s), None)
    if rc:
        raise RuntimeError("oracle_eval_full_seeds rc=%d" % rc)
    return s


def contract(y: np.ndarray, T: np.ndarray) -> np.ndarray:
    y = np.ascontiguousarray(y, np.uint32)
    T = np.ascontiguousarray(T, np.uint32)
    rows, D = T.shape
    assert y.shape[0] >= rows
    out = np.zeros(D, np.uint32)
    lib().oracle_contract(_u32(y), rows, _u32(T), D, _u32(out))
    return out


def answer_batch(keys, T: np.ndarray, row_begin: int = 0, threads: int = 1) -> np.ndarray:
    """shares[b][d] = sum_{j in shard} Eval(keys[b], row_begin + j) T[j][d] mod 2^32."""
    T = np.ascontiguousarray(T, np.uint32)
    rows, D = T.shape
    B = len(keys)
    arr = (OracleKey * B)(*keys)
    out = np.zeros((B, D), np.uint32)
    rc = lib().oracle_answer_batch(arr, B, _u32(T), row_begin, rows, D, _u32(out), threads)
    if rc:
        raise RuntimeError("oracle_answer_batch rc=%d" % rc)
    return out


def reconstruct(s0: np.ndarray, s1: np.ndarray) -> np.ndarray:
    s0 = np.ascontiguousarray(s0, np.uint32)
    s1 = np.ascontiguousarray(s1, np.uint32)
    out = np.zeros_like(s0)
    lib().oracle_reconstruct(_u32(s0), _u32(s1), s0.size, _u32(out))
    return out


def naive_pir_shares(N: int, alpha: int, beta: int, r0: np.ndarray) -> np.ndarray:
    r0 = np.ascontiguousarray(r0, np.uint32)
    r1 = np.zeros(N, np.uint32)
    lib().oracle_naive_pir_shares(N, alpha, beta & 0xFFFFFFFF, _u32(r0), _u32(r1))
    return r1


def key_wire_size(log_n: int, prf: int = PRF_CHACHA20) -> int:
    return lib().oracle_key_wire_size_prf(log_n, prf)


def key_to_wire(k: OracleKey) -> bytes:
    out = np.zeros(key_wire_size(k.log_n, k.prf), np.uint8)
    n = lib().oracle_key_to_wire(ctypes.byref(k), _u8(out), out.size)
    assert n == out.size
    return out.tobytes()


def key_from_wire(b: bytes) -> OracleKey:
    k = OracleKey()
    arr = _bytes_in(b)
    rc = lib().oracle_key_from_wire(_u8(arr), arr.size, ctypes.byref(k))
    if rc:
        raise ValueError("bad key wire bytes (rc=%d)" % rc)
    return k


# ---------------------------------------------------------------- PBR (row f2)
# Partial batch retrieval (§4.1): "segmenting table T into
# L/I bins of size I, and issuing individual DPF-PIR queries to each bin ...
# a single PBR can fetch only one query from each bin.  If more than one query
# index fall into the same bin, the rest of the queries except for the one
# must be dropped."  Reading R21: I = 2^log_i; bin b holds rows
# [bI, min(bI + I, N)) (the last bin is ragged: its rows >= N are absent, R12);
# the kept query of a bin is the first of its rows in the client's request
# order; a bin with no needed row gets a dummy query (its index is the
# caller's choice: P:656-659 pads with dummies so the count leaks nothing).


def pbr_n_bins(N: int, log_i: int) -> int:
    """L/I bins (rounded up: the last bin is ragged when I does not divide N)."""
    return (N + (1 << log_i) - 1) >> log_i


def pbr_plan(needed_rows, N: int, log_i: int):
    """Client side of PBR, written as the loop the text describes.
    Returns (index, dropped): index[b] = the in-bin index queried in bin b, or
    -1 where bin b gets a dummy; dropped = the needed rows that were not kept,
    in request order.  Duplicate requests of one row count once."""
    I = 1 << log_i
    index = [-1] * pbr_n_bins(N, log_i)
    dropped = []
    seen = set()
    for r in needed_rows:
        r = int(r)
        if r in seen:
            continue
        seen.add(r)
        b = r // I
        if index[b] < 0:
            index[b] = r - b * I
        else:
            dropped.append(r)
    return index, dropped


def pbr_answer(bin_keys, T: np.ndarray, log_i: int, threads: int = 1) -> np.ndarray:
    """Server side of PBR: bin b's keys (each over the I-row domain
    of the bin) answered against the bin's rows T[bI : bI + I] exactly as a
    plain PIR query on that small table (answer_batch).  Returns
    shares[n_bins][B][D] (every bin carries the same B keys per client batch)."""
    T = np.ascontiguousarray(T, np.uint32)
    N, D = T.shape
    I = 1 << log_i
    nb = pbr_n_bins(N, log_i)
    assert len(bin_keys) == nb
    B = len(bin_keys[0])
    out = np.zeros((nb, B, D), np.uint32)
    for b in range(nb):
        assert len(bin_keys[b]) == B and all(k.log_n == log_i for k in bin_keys[b])
        out[b] = answer_batch(bin_keys[b], T[b * I:(b + 1) * I], 0, threads)
    return out
