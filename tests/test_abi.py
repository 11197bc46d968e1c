"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/dpfpir.h declares, its Gen equals the oracle's Gen
bit-exactly from the same DRBG seed (two independent implementations), the key
codec matches Table 4 and the oracle's wire bytes, error codes follow the
header, and reconstruct adds mod 2^32."""
import ctypes
import os
import re

import numpy as np
import pytest
from conftest import ROOT, read_golden

from paper_2301_10904_b200 import build as pbuild
from paper_2301_10904_b200 import dpfpir


@pytest.fixture(scope="module")
def lib():
    pbuild.build()
    return dpfpir.lib()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "dpfpir.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char \*|void)\s*\*?\s*(dpf_\w+)\s*\(", hdr, re.M))
    assert {"dpf_gen", "dpf_eval_batch", "dpf_eval_batch_shard", "dpf_reconstruct"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    assert set(dpfpir.EXPORTED_SYMBOLS) == declared
    assert b"sm_100a" in lib.dpf_version()


def test_sm100a_cubin_embedded():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dpfpir.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_gen_equals_oracle_gen(lib, oracle):
    r = np.random.default_rng(0)
    for n in (1, 2, 7, 16, 20, 24):
        for _ in range(4):
            alpha = int(r.integers(0, 1 << n))
            beta = int(r.integers(0, 1 << 32))
            seed = bytes(r.integers(0, 256, 32, dtype=np.uint8))
            k0, k1 = dpfpir.gen(n, alpha, beta, seed)
            o0, o1 = oracle.gen(n, alpha, beta, seed)
            assert dpfpir.key_serialize(k0) == oracle.key_to_wire(o0)
            assert dpfpir.key_serialize(k1) == oracle.key_to_wire(o1)


def test_gen_aes_equals_oracle_gen(lib, oracle):
    r = np.random.default_rng(9)
    for n in (1, 5, 14, 20):
        alpha = int(r.integers(0, 1 << n))
        seed = bytes(r.integers(0, 256, 32, dtype=np.uint8))
        k0, k1 = dpfpir.gen(n, alpha, 12345, seed, prf=dpfpir.DPF_PRF_AES128)
        o0, o1 = oracle.gen(n, alpha, 12345, seed, prf=oracle.PRF_AES128)
        assert dpfpir.key_serialize(k0) == oracle.key_to_wire(o0)
        assert dpfpir.key_serialize(k1) == oracle.key_to_wire(o1)


def test_gen_keys_satisfy_contract_under_oracle_eval(lib, oracle):
    for alpha in (0, 5, 63):
        k0, k1 = dpfpir.gen(6, alpha, 1, bytes(32))
        y = oracle.eval_full(oracle.key_from_wire(dpfpir.key_serialize(k0))) + \
            oracle.eval_full(oracle.key_from_wire(dpfpir.key_serialize(k1)))
        want = np.zeros(64, np.uint32)
        want[alpha] = 1
        np.testing.assert_array_equal(y, want)


def test_gen_entropy_seed_differs(lib):
    a = dpfpir.key_serialize(dpfpir.gen(10, 3)[0])
    b = dpfpir.key_serialize(dpfpir.gen(10, 3)[0])
    assert a != b and len(a) == len(b) == 32 + 640


def test_key_codec_and_table4(lib):
    for entries, log_n, key_bytes in read_golden("table4_key_bytes.txt"):
        assert dpfpir.key_wire_size(int(log_n)) == 32 + int(key_bytes)
    assert dpfpir.key_wire_size(0) == 0 and dpfpir.key_wire_size(33) == 0
    k0, k1 = dpfpir.gen(14, 1000, 1, bytes(range(32)))
    w = dpfpir.key_serialize(k1)
    assert len(w) == 32 + 896
    assert w[:4] == b"DPFK" and w[6] == 1 and w[7] == 14
    assert dpfpir.key_serialize(dpfpir.key_deserialize(w)) == w
    bad = bytearray(w)
    bad[0] ^= 1
    with pytest.raises(dpfpir.DpfError) as e:
        dpfpir.key_deserialize(bytes(bad))
    assert e.value.code == dpfpir.DPF_EKEY
    with pytest.raises(dpfpir.DpfError):
        dpfpir.key_deserialize(w[:-1])
    bad = bytearray(w)
    bad[16] ^= 1  # lsb(root) != party
    with pytest.raises(dpfpir.DpfError):
        dpfpir.key_deserialize(bytes(bad))


def test_gen_errors(lib):
    with pytest.raises(dpfpir.DpfError) as e:
        dpfpir.gen(4, 16)
    assert e.value.code == dpfpir.DPF_EINVAL
    with pytest.raises(dpfpir.DpfError):
        dpfpir.gen(0, 0)
    with pytest.raises(dpfpir.DpfError) as e:
        dpfpir.gen(4, 1, prf=7)
    assert e.value.code == dpfpir.DPF_EUNSUPPORTED


def test_reconstruct(lib):
    r = np.random.default_rng(1)
    a = r.integers(0, 1 << 32, 1000, dtype=np.uint32)
    b = r.integers(0, 1 << 32, 1000, dtype=np.uint32)
    np.testing.assert_array_equal(dpfpir.reconstruct(a, b), a + b)


def test_workspace_bytes(lib):
    assert dpfpir.eval_workspace_bytes(0, 20, 1 << 20, 256) == 0
    assert dpfpir.eval_workspace_bytes(256, 20, 1 << 20, 255) == 0   # D % 4
    assert dpfpir.eval_workspace_bytes(256, 20, 1 << 20, 2048) == 0  # D > 1024
    ws = dpfpir.eval_workspace_bytes(256, 20, 1 << 20, 256)
    # sized for every PRF: the AES T-tables take 64 KB of SMEM from the DFS
    # stack, so its plan keeps a one-level-deeper frontier (f = 13 at c3)
    assert 256 * (32 + 64 * 20) < ws < 96 << 20


def test_eval_rejects_bad_args_without_gpu(lib):
    """Argument validation happens before any CUDA call."""
    k0, _ = dpfpir.gen(8, 1, 1, bytes(32))
    kb = dpfpir.KeyBatch.from_keys([k0])
    L = lib
    ws = ctypes.create_string_buffer(1 << 16)
    wsp = (ctypes.addressof(ws) + 255) // 256 * 256
    tbl = ctypes.create_string_buffer(4096 + 16)
    tp = (ctypes.addressof(tbl) + 15) // 16 * 16
    out = ctypes.create_string_buffer(4096)
    assert L.dpf_eval_batch(kb.ptr, 1, tp, 257, 4, out, wsp, 60000, None) == dpfpir.DPF_EINVAL  # N > 2^n
    assert L.dpf_eval_batch(kb.ptr, 1, tp, 16, 6, out, wsp, 60000, None) == dpfpir.DPF_EINVAL   # D % 4
    assert L.dpf_eval_batch(kb.ptr, 0, tp, 16, 4, out, wsp, 60000, None) == dpfpir.DPF_EINVAL   # B = 0
    assert L.dpf_eval_batch(kb.ptr, 1, tp + 4, 16, 4, out, wsp, 60000, None) == dpfpir.DPF_EINVAL  # align
    assert L.dpf_eval_batch(kb.ptr, 1, tp, 16, 4, out, wsp, 16, None) == dpfpir.DPF_ENOMEM
    k_other, _ = dpfpir.gen(9, 1, 1, bytes(32))
    mixed = dpfpir.KeyBatch.from_keys([k0, k_other])
    assert L.dpf_eval_batch(mixed.ptr, 2, tp, 16, 4, out, wsp, 60000, None) == dpfpir.DPF_EKEY


def test_planner_accepts_every_valid_shape(lib):
    """The host planner (tile choice, subtree depth, SMEM budget) must find a
    launch plan for every argument combination the header allows."""
    bad = []
    for D in range(4, 1025, 4):
        for B in (1, 3, 17, 64, 100, 1000):
            for n, rows in ((1, 2), (3, 5), (10, 1000), (20, 1 << 20), (24, 1 << 24)):
                if dpfpir.eval_workspace_bytes(B, n, rows, D) == 0:
                    bad.append((D, B, n, rows))
    assert not bad, bad[:10]


# ---------------------------------------------------------------- early termination (row f4, R20)

def test_gen_et_equals_oracle_gen(lib, oracle):
    r = np.random.default_rng(44)
    for n in (5, 6, 10, 17, 20, 32):
        alpha = int(r.integers(0, 1 << n))
        beta = int(r.integers(0, 1 << 32))
        seed = bytes(r.integers(0, 256, 32, dtype=np.uint8))
        k0, k1 = dpfpir.gen(n, alpha, beta, seed, prf=dpfpir.DPF_PRF_CHACHA20_ET)
        o0, o1 = oracle.gen(n, alpha, beta, seed, prf=oracle.PRF_CHACHA20_ET)
        assert dpfpir.key_serialize(k0) == oracle.key_to_wire(o0)
        assert dpfpir.key_serialize(k1) == oracle.key_to_wire(o1)


def test_et_key_codec_and_errors(lib):
    ET = dpfpir.DPF_PRF_CHACHA20_ET
    assert dpfpir.key_wire_size(20, ET) == 32 + 64 * 17
    assert dpfpir.key_wire_size(4, ET) == 0 and dpfpir.key_wire_size(33, ET) == 0
    assert dpfpir.key_wire_size(20, 9) == 0
    k0, k1 = dpfpir.gen(20, 777, 1, bytes(range(32)), prf=ET)
    w = dpfpir.key_serialize(k1)
    assert len(w) == 32 + 64 * 17 and w[5] == ET
    assert dpfpir.key_serialize(dpfpir.key_deserialize(w)) == w
    with pytest.raises(dpfpir.DpfError):
        dpfpir.key_deserialize(w + bytes(64))  # a standard-length payload is not an ET key
    bad = bytearray(w)
    bad[8] = 1  # ET keys carry cw_out = 0
    with pytest.raises(dpfpir.DpfError) as e:
        dpfpir.key_deserialize(bytes(bad))
    assert e.value.code == dpfpir.DPF_EKEY
    with pytest.raises(dpfpir.DpfError) as e:
        dpfpir.gen(4, 3, prf=ET)  # needs h = log_n - 4 >= 1
    assert e.value.code == dpfpir.DPF_EINVAL


def test_et_gen_keys_satisfy_contract(lib, oracle):
    for alpha in (0, 17, 255, 200):
        k0, k1 = dpfpir.gen(8, alpha, 9, bytes(32), prf=dpfpir.DPF_PRF_CHACHA20_ET)
        y = oracle.eval_full(oracle.key_from_wire(dpfpir.key_serialize(k0))) + \
            oracle.eval_full(oracle.key_from_wire(dpfpir.key_serialize(k1)))
        want = np.zeros(256, np.uint32)
        want[alpha] = 9
        np.testing.assert_array_equal(y, want)


def test_planner_all_schemes_and_paths(lib):
    """dpf_eval_plan (host only) finds a plan for every shape each path
    accepts, and its block count is the closed form: N - 1 per key (R9) or
    N/8 - 1 with early termination (R20) over a full power-of-two domain."""
    ET = dpfpir.DPF_PRF_CHACHA20_ET
    bad = []
    for prf in (1, 2, ET):
        for packed in (False, True):
            Ds = range(4, 1025, 28)
            for D in Ds:
                for B in (1, 17, 64, 256, 1000):
                    for n, r0, rows in ((5, 0, 32), (6, 3, 50), (10, 0, 1000), (20, 0, 1 << 20), (24, 5, 1 << 23),
                                        (32, (1 << 32) - 4096, 4096)):
                        if packed and n < 3:
                            continue
                        try:
                            dpfpir.eval_plan(B, n, rows, D, prf, r0, packed)
                        except dpfpir.DpfError:
                            bad.append((prf, packed, D, B, n, rows))
    assert not bad, bad[:10]
    for prf, per in ((1, (1 << 20) - 1), (ET, (1 << 17) - 1)):
        for packed in (False, True):
            assert dpfpir.eval_plan(256, 20, 1 << 20, 256, prf, 0, packed)["prf_blocks"] == 256 * per


def test_new_entry_points_reject_bad_args_without_gpu(lib):
    """dpf_eval_batch_wire_ex, the IPC helpers and the packed grouped planner
    validate their arguments before any CUDA call."""
    L = lib
    keys = ctypes.create_string_buffer(4096 + 16)
    kp = (ctypes.addressof(keys) + 15) // 16 * 16
    ws = ctypes.create_string_buffer(1 << 16)
    wsp = (ctypes.addressof(ws) + 255) // 256 * 256
    out = ctypes.create_string_buffer(4096)
    # unknown flag bits, null keys, misaligned keys
    assert L.dpf_eval_batch_wire_ex(kp, 1, 8, 1, kp, 0, 0, 16, 4, out, 2, wsp, 60000, None) == dpfpir.DPF_EINVAL
    assert L.dpf_eval_batch_wire_ex(None, 1, 8, 1, kp, 0, 0, 16, 4, out, 1, wsp, 60000, None) == dpfpir.DPF_EINVAL
    assert L.dpf_eval_batch_wire_ex(kp + 4, 1, 8, 1, kp, 0, 0, 16, 4, out, 1, wsp, 60000, None) == dpfpir.DPF_EINVAL
    # unknown scheme
    assert L.dpf_eval_batch_wire_ex(kp, 1, 8, 9, kp, 0, 0, 16, 4, out, 0, wsp, 60000, None) == dpfpir.DPF_EUNSUPPORTED
    h = (ctypes.c_uint8 * dpfpir.IPC_HANDLE_BYTES)()
    off = ctypes.c_uint64()
    p = ctypes.c_void_p()
    assert L.dpf_ipc_export(None, h, ctypes.byref(off)) == dpfpir.DPF_EINVAL
    assert L.dpf_ipc_open(None, ctypes.byref(p)) == dpfpir.DPF_EINVAL
    assert L.dpf_ipc_close(None) == dpfpir.DPF_EINVAL
    # grouped planners: an empty group list and a bad D plan nothing
    assert L.dpf_eval_grouped_workspace_bytes(None, 0, 32, 1) == 0
    assert L.dpf_eval_grouped_packed_workspace_bytes(None, 0, 32, 1) == 0
    g = dpfpir.DpfEvalGroup()
    g.keys_wire, g.B, g.log_n, g.table, g.row_begin, g.row_count, g.shares = kp, 3, 10, kp, 0, 1000, kp
    arr = (dpfpir.DpfEvalGroup * 1)(g)
    assert L.dpf_eval_grouped_packed_workspace_bytes(arr, 1, 32, 1) > 0
    assert L.dpf_eval_grouped_packed_workspace_bytes(arr, 1, 30, 1) == 0   # D % 4
    assert L.dpf_eval_grouped_packed_workspace_bytes(arr, 1, 32, 3) > 0    # early termination
    g.log_n = 2                                                             # below the packed minimum depth
    arr = (dpfpir.DpfEvalGroup * 1)(g)
    assert L.dpf_eval_grouped_packed_workspace_bytes(arr, 1, 32, 1) == 0
