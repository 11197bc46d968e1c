"""Thin Python binding of libdpfpir (include/dpfpir.h): argument marshalling only.

Every step of the evaluation runs in the CUDA library; this module only turns
numpy arrays / torch tensors into pointers and sizes.  PyTorch supplies device
memory (tables, shares, workspace) and streams.  There is no CPU fallback: if
libdpfpir.so is missing or no CUDA device is present, the device entry points
raise.

Names follow the C ABI: gen, key_serialize, key_deserialize, reconstruct,
eval_workspace_bytes, eval_batch, eval_batch_shard, eval_batch_wire,
serve_batch, eval_leaves, last_eval_stats.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# DPFPIR_LIB overrides the in-tree library (A/B builds during tuning)
LIB_PATH = os.environ.get("DPFPIR_LIB") or os.path.join(_PKG, "libdpfpir.so")

DPF_MAX_LOG_N = 32
DPF_PRF_CHACHA20 = 1
DPF_PRF_AES128 = 2
DPF_PRF_CHACHA20_ET = 3  # early-terminated leaves (R20), log_n >= 5
DPF_ET_BITS = 4
DPF_OK, DPF_EINVAL, DPF_EKEY, DPF_ENOMEM, DPF_ECUDA, DPF_EUNSUPPORTED, DPF_EBUSY = 0, -1, -2, -3, -4, -6, -7


class DpfError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__("%s: %s (%d)" % (what, strerror(code), code))
        self.code = code


class DpfKey(ctypes.Structure):
    """dpf_key (include/dpfpir.h), 2080 bytes, POD."""
    _fields_ = [("magic", ctypes.c_uint32), ("version", ctypes.c_uint8), ("prf", ctypes.c_uint8),
                ("party", ctypes.c_uint8), ("log_n", ctypes.c_uint8), ("cw_out", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("root", ctypes.c_uint8 * 16),
                ("cw", ctypes.c_uint8 * (DPF_MAX_LOG_N * 2 * 2 * 16))]


class DpfEvalStats(ctypes.Structure):
    _fields_ = [("prf_blocks", ctypes.c_uint64), ("kernels", ctypes.c_uint32), ("frontier_depth", ctypes.c_uint32),
                ("keys_per_tile", ctypes.c_uint32), ("nodes_per_tile", ctypes.c_uint32),
                ("work_items", ctypes.c_uint32), ("grid", ctypes.c_uint32), ("kernel_id", ctypes.c_uint32)]


class DpfEvalGroup(ctypes.Structure):
    """dpf_eval_group (include/dpfpir.h)."""
    _fields_ = [("keys_wire", ctypes.c_void_p), ("B", ctypes.c_uint32), ("log_n", ctypes.c_uint32),
                ("table", ctypes.c_void_p), ("row_begin", ctypes.c_uint64), ("row_count", ctypes.c_uint64),
                ("shares", ctypes.c_void_p)]


KEY_BYTES = ctypes.sizeof(DpfKey)
_lib = None


def lib() -> ctypes.CDLL:
    """Load libdpfpir.so (built by __graft_entry__.build() / `python -m
    paper_2301_10904_b200.build`).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libdpfpir.so not built (%s); run `python -m paper_2301_10904_b200.build`" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, u32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64
    L.dpf_gen.argtypes = [u32, u64, u32, u32, vp, vp, vp]
    L.dpf_key_wire_size.argtypes = [u32]
    L.dpf_key_wire_size.restype = sz
    L.dpf_key_wire_size_prf.argtypes = [u32, u32]
    L.dpf_key_wire_size_prf.restype = sz
    L.dpf_key_serialize.argtypes = [vp, vp, sz, ctypes.POINTER(sz)]
    L.dpf_key_deserialize.argtypes = [vp, sz, vp]
    L.dpf_reconstruct.argtypes = [vp, vp, sz, vp]
    L.dpf_eval_workspace_bytes.argtypes = [u32, u32, u64, u32]
    L.dpf_eval_workspace_bytes.restype = sz
    L.dpf_eval_batch.argtypes = [vp, u32, vp, u64, u32, vp, vp, sz, vp]
    L.dpf_eval_batch_shard.argtypes = [vp, u32, vp, u64, u64, u32, vp, vp, sz, vp]
    L.dpf_eval_batch_wire.argtypes = [vp, u32, u32, u32, vp, u64, u64, u32, vp, vp, sz, vp]
    L.dpf_serve_batch.argtypes = [vp, u32, vp, u64, u64, u32, vp, vp, sz, vp]
    L.dpf_eval_batch_wire_ex.argtypes = [vp, u32, u32, u32, vp, ctypes.c_int, u64, u64, u32, vp, u32, vp, sz, vp]
    L.dpf_ipc_export.argtypes = [vp, vp, ctypes.POINTER(u64)]
    L.dpf_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
    L.dpf_ipc_close.argtypes = [vp]
    L.dpf_server_workspace_bytes.argtypes = [u32, u32, u32, u64, u32]
    L.dpf_server_workspace_bytes.restype = sz
    L.dpf_server_create.argtypes = [u32, u32, u32, vp, ctypes.c_int, u64, u64, u32, vp, sz, vp, ctypes.POINTER(vp)]
    L.dpf_server_run.argtypes = [vp, vp, vp]
    L.dpf_server_pipeline_workspace_bytes.argtypes = [u32, u32, u32, u64, u32, u32]
    L.dpf_server_pipeline_workspace_bytes.restype = sz
    L.dpf_server_pipeline_create.argtypes = [u32, u32, u32, vp, ctypes.c_int, u64, u64, u32, u32, vp, sz, vp,
                                             ctypes.POINTER(vp)]
    L.dpf_server_submit.argtypes = [vp, vp]
    L.dpf_server_collect.argtypes = [vp, vp]
    L.dpf_server_destroy.argtypes = [vp]
    L.dpf_server_destroy.restype = None
    L.dpf_eval_leaves.argtypes = [vp, u32, vp, vp, sz, vp]
    L.dpf_table_packed_bytes.argtypes = [u64, u64, u32]
    L.dpf_table_packed_bytes.restype = sz
    L.dpf_table_pack.argtypes = [vp, u64, u64, u32, vp, vp]
    L.dpf_eval_batch_packed.argtypes = [vp, u32, vp, u64, u64, u32, vp, vp, sz, vp]
    L.dpf_eval_batch_wire_packed.argtypes = [vp, u32, u32, u32, vp, u64, u64, u32, vp, vp, sz, vp]
    L.dpf_eval_grouped_workspace_bytes.argtypes = [vp, u32, u32, u32]
    L.dpf_eval_grouped_workspace_bytes.restype = sz
    L.dpf_eval_grouped.argtypes = [vp, u32, u32, u32, vp, sz, vp]
    L.dpf_eval_grouped_packed_workspace_bytes.argtypes = [vp, u32, u32, u32]
    L.dpf_eval_grouped_packed_workspace_bytes.restype = sz
    L.dpf_eval_grouped_packed.argtypes = [vp, u32, u32, u32, vp, sz, vp]
    L.dpf_eval_pbr_workspace_bytes.argtypes = [u32, u32, u64, u32, u32, ctypes.c_int]
    L.dpf_eval_pbr_workspace_bytes.restype = sz
    L.dpf_eval_pbr.argtypes = [vp, u32, u32, u32, vp, ctypes.c_int, u64, u32, vp, vp, sz, vp]
    L.dpf_last_eval_stats.argtypes = [vp]
    L.dpf_eval_plan.argtypes = [u32, u32, u32, u64, u64, u32, ctypes.c_int, vp]
    L.dpf_kernel_timer_begin.argtypes = [u32]
    L.dpf_kernel_timer_read.argtypes = [vp, u32, vp]
    L.dpf_strerror.argtypes = [ctypes.c_int]
    L.dpf_strerror.restype = ctypes.c_char_p
    L.dpf_version.restype = ctypes.c_char_p
    assert KEY_BYTES == 2080
    _lib = L
    return L


EXPORTED_SYMBOLS = ("dpf_gen", "dpf_key_wire_size", "dpf_key_wire_size_prf", "dpf_key_serialize", "dpf_key_deserialize", "dpf_reconstruct",
                    "dpf_eval_workspace_bytes", "dpf_eval_batch", "dpf_eval_batch_shard", "dpf_eval_batch_wire",
                    "dpf_serve_batch", "dpf_eval_leaves", "dpf_last_eval_stats", "dpf_eval_plan", "dpf_kernel_timer_begin",
                    "dpf_table_packed_bytes", "dpf_table_pack", "dpf_eval_batch_packed", "dpf_eval_batch_wire_packed",
                    "dpf_eval_grouped_workspace_bytes", "dpf_eval_grouped",
                    "dpf_eval_grouped_packed_workspace_bytes", "dpf_eval_grouped_packed",
                    "dpf_eval_pbr_workspace_bytes", "dpf_eval_pbr",
                    "dpf_eval_batch_wire_ex", "dpf_ipc_export", "dpf_ipc_open", "dpf_ipc_close",
                    "dpf_server_workspace_bytes", "dpf_server_create", "dpf_server_run", "dpf_server_destroy",
                    "dpf_server_pipeline_workspace_bytes", "dpf_server_pipeline_create", "dpf_server_submit",
                    "dpf_server_collect",
                    "dpf_kernel_timer_read", "dpf_strerror", "dpf_version")


def strerror(code: int) -> str:
    try:
        return lib().dpf_strerror(code).decode()
    except RuntimeError:
        return "status %d" % code


def _check(rc: int, what: str) -> None:
    if rc != DPF_OK:
        raise DpfError(rc, what)


# ------------------------------------------------------------------ keys (host)

class KeyBatch:
    """B dpf_key records in one contiguous host buffer (numpy uint8 [B, 2080])."""

    def __init__(self, raw: np.ndarray):
        assert raw.dtype == np.uint8 and raw.ndim == 2 and raw.shape[1] == KEY_BYTES
        self.raw = np.ascontiguousarray(raw)

    @classmethod
    def from_keys(cls, keys: Iterable[DpfKey]) -> "KeyBatch":
        keys = list(keys)
        raw = np.zeros((len(keys), KEY_BYTES), np.uint8)
        for i, k in enumerate(keys):
            ctypes.memmove(raw[i].ctypes.data, ctypes.addressof(k), KEY_BYTES)
        return cls(raw)

    def __len__(self) -> int:
        return self.raw.shape[0]

    def __getitem__(self, i: int) -> DpfKey:
        return DpfKey.from_buffer_copy(self.raw[i].tobytes())

    @property
    def ptr(self) -> int:
        return self.raw.ctypes.data

    @property
    def log_n(self) -> int:
        return int(self.raw[0, 7])

    @property
    def prf(self) -> int:
        return int(self.raw[0, 5])


def _as_batch(keys) -> KeyBatch:
    if isinstance(keys, KeyBatch):
        return keys
    if isinstance(keys, DpfKey):
        return KeyBatch.from_keys([keys])
    return KeyBatch.from_keys(keys)


def gen(log_n: int, alpha: int, beta: int = 1, rng_seed: Optional[bytes] = None,
        prf: int = DPF_PRF_CHACHA20) -> tuple[DpfKey, DpfKey]:
    """dpf_gen: (k0, k1) with Eval(k0,j)+Eval(k1,j) = beta [j == alpha] mod 2^32."""
    k0, k1 = DpfKey(), DpfKey()
    seed = None
    if rng_seed is not None:
        assert len(rng_seed) == 32
        seed = ctypes.create_string_buffer(bytes(rng_seed), 32)
    _check(lib().dpf_gen(log_n, alpha, beta & 0xFFFFFFFF, prf, seed, ctypes.byref(k0), ctypes.byref(k1)), "dpf_gen")
    return k0, k1


def key_wire_size(log_n: int, prf: int = DPF_PRF_CHACHA20) -> int:
    return lib().dpf_key_wire_size_prf(log_n, prf)


def key_serialize(k: DpfKey) -> bytes:
    n = key_wire_size(k.log_n, k.prf)
    buf = ctypes.create_string_buffer(max(n, 1))
    written = ctypes.c_size_t(0)
    _check(lib().dpf_key_serialize(ctypes.byref(k), buf, n, ctypes.byref(written)), "dpf_key_serialize")
    return buf.raw[:written.value]


def key_deserialize(b: bytes) -> DpfKey:
    k = DpfKey()
    buf = ctypes.create_string_buffer(bytes(b), max(len(b), 1))
    _check(lib().dpf_key_deserialize(buf, len(b), ctypes.byref(k)), "dpf_key_deserialize")
    return k


def reconstruct(share0: np.ndarray, share1: np.ndarray) -> np.ndarray:
    s0 = np.ascontiguousarray(share0, dtype=np.uint32)
    s1 = np.ascontiguousarray(share1, dtype=np.uint32)
    assert s0.shape == s1.shape
    out = np.empty_like(s0)
    _check(lib().dpf_reconstruct(s0.ctypes.data, s1.ctypes.data, s0.size, out.ctypes.data), "dpf_reconstruct")
    return out


# ------------------------------------------------------------------ device

def eval_workspace_bytes(B: int, log_n: int, rows: int, D: int) -> int:
    return lib().dpf_eval_workspace_bytes(B, log_n, rows, D)


_ws_cache: dict = {}


def _workspace(nbytes: int, device, stream=None):
    """Scratch workspace for calls that pass none: one buffer per (device,
    stream), so calls ordered on one stream never overlap on it; a call on
    another stream gets another buffer.  Long-lived users (Server) own theirs."""
    import torch
    key = (str(device), _stream_ptr(stream))
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _check_table(table):
    import torch
    if not table.is_cuda:
        raise ValueError("table must be a CUDA tensor (server state lives in HBM)")
    if table.dtype not in (torch.int32, torch.uint32) or table.dim() != 2 or not table.is_contiguous():
        raise ValueError("table must be a contiguous 2-D int32/uint32 CUDA tensor")


def eval_batch_shard(keys, table_shard, row_begin: int = 0, out=None, workspace=None, stream=None):
    """dpf_eval_batch_shard: partial[b][d] = sum_j Eval(k_b, row_begin+j) * table_shard[j][d] mod 2^32.
    Returns an int32 CUDA tensor [B, D] (uint32 bit patterns)."""
    import torch
    kb = _as_batch(keys)
    _check_table(table_shard)
    rows, D = table_shard.shape
    B = len(kb)
    if out is None:
        out = torch.empty((B, D), dtype=torch.int32, device=table_shard.device)
    need = eval_workspace_bytes(B, kb.log_n, rows, D)
    if need == 0:
        raise DpfError(DPF_EINVAL, "dpf_eval_workspace_bytes")
    ws = workspace if workspace is not None else _workspace(need, table_shard.device, stream)
    _check(lib().dpf_eval_batch_shard(kb.ptr, B, table_shard.data_ptr(), row_begin, rows, D, out.data_ptr(),
                                      ws.data_ptr(), ws.numel() * ws.element_size(), _stream_ptr(stream)),
           "dpf_eval_batch_shard")
    return out


def eval_batch(keys, table, out=None, workspace=None, stream=None):
    """dpf_eval_batch: shares[b][d] = sum_{j<N} Eval(k_b, j) * table[j][d] mod 2^32."""
    return eval_batch_shard(keys, table, 0, out, workspace, stream)


def keys_to_wire(keys) -> np.ndarray:
    """Serialize a key batch into consecutive wire records (uint8 [B, key_wire_size(n, prf)])."""
    kb = _as_batch(keys)
    w = key_wire_size(kb.log_n, kb.prf)
    out = np.zeros((len(kb), w), np.uint8)
    written = ctypes.c_size_t(0)
    for i in range(len(kb)):
        _check(lib().dpf_key_serialize(kb.ptr + i * KEY_BYTES, out[i].ctypes.data, w, ctypes.byref(written)),
               "dpf_key_serialize")
    return out


DPF_EVAL_ACCUMULATE = 1
IPC_HANDLE_BYTES = 64


def eval_batch_wire_ex(keys_wire_dev, log_n: int, table, row_begin: int, row_count: int, D: int, shares_ptr: int,
                       flags: int, workspace, stream=None, prf: int = DPF_PRF_CHACHA20, packed: bool = False):
    """dpf_eval_batch_wire_ex: `table` is a row-major CUDA shard or a PackedTable;
    `shares_ptr` a device address (possibly a peer rank's buffer from ipc_open)."""
    tptr = table.data.data_ptr() if packed else table.data_ptr()
    _check(lib().dpf_eval_batch_wire_ex(keys_wire_dev.data_ptr(), keys_wire_dev.shape[0], log_n, prf, tptr,
                                        int(packed), row_begin, row_count, D, shares_ptr, flags,
                                        workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                        _stream_ptr(stream)), "dpf_eval_batch_wire_ex")


def ipc_export(tensor) -> tuple[bytes, int]:
    """dpf_ipc_export: (64-byte CUDA IPC handle of the allocation holding a CUDA
    tensor, the tensor's byte offset inside it)."""
    h = (ctypes.c_uint8 * IPC_HANDLE_BYTES)()
    off = ctypes.c_uint64()
    _check(lib().dpf_ipc_export(tensor.data_ptr(), h, ctypes.byref(off)), "dpf_ipc_export")
    return bytes(h), int(off.value)


def ipc_open(handle: bytes) -> int:
    """dpf_ipc_open: map another process's allocation; returns its base device address."""
    if len(handle) != IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be %d bytes" % IPC_HANDLE_BYTES)
    p = ctypes.c_void_p()
    _check(lib().dpf_ipc_open((ctypes.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(handle), ctypes.byref(p)),
           "dpf_ipc_open")
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(lib().dpf_ipc_close(ptr), "dpf_ipc_close")


class Server:
    """dpf_server_*: one serving step of a fixed shape captured as a CUDA graph
    (`depth` > 1: dpf_server_pipeline_create, that many batches in flight).
    run(keys_wire_host uint8 [B, w], out int32 [B, D] host) -> out;
    submit(keys_wire_host) / collect(out) for the pipelined form."""

    def __init__(self, B: int, log_n: int, table, row_begin: int = 0, prf: int = DPF_PRF_CHACHA20, stream=None,
                 depth: int = 1):
        import torch
        packed = isinstance(table, PackedTable)
        rows, D = (table.row_count, table.D) if packed else table.shape
        dev = table.data.device if packed else table.device
        need = lib().dpf_server_pipeline_workspace_bytes(B, log_n, prf, rows, D, depth)
        if need == 0:
            raise DpfError(DPF_EINVAL, "dpf_server_pipeline_workspace_bytes")
        # private workspace: the captured graph replays on the server's own
        # stream for the object's lifetime, so no other call may share it
        self.ws = torch.empty(need, dtype=torch.uint8, device=dev)
        self.table = table  # keep alive
        self.B, self.D, self.wire = B, D, key_wire_size(log_n, prf)
        h = ctypes.c_void_p()
        tptr = table.data.data_ptr() if packed else table.data_ptr()
        _check(lib().dpf_server_pipeline_create(B, log_n, prf, tptr, int(packed), row_begin, rows, D, depth,
                                                self.ws.data_ptr(), self.ws.numel() * self.ws.element_size(),
                                                _stream_ptr(stream), ctypes.byref(h)),
               "dpf_server_pipeline_create")
        self.h = h
        self.depth = depth

    def run(self, keys_wire_host: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        kw = np.ascontiguousarray(keys_wire_host, dtype=np.uint8)
        if kw.size != self.B * self.wire:
            raise ValueError("expected %d keys of %d wire bytes" % (self.B, self.wire))
        if out is None:
            out = np.empty((self.B, self.D), dtype=np.uint32)
        _check(lib().dpf_server_run(self.h, kw.ctypes.data, out.ctypes.data), "dpf_server_run")
        return out

    def submit(self, keys_wire_host: np.ndarray) -> None:
        """dpf_server_submit: launch one batch without waiting (the keys are
        copied into the slot's pinned staging before this returns)."""
        kw = np.ascontiguousarray(keys_wire_host, dtype=np.uint8)
        if kw.size != self.B * self.wire:
            raise ValueError("expected %d keys of %d wire bytes" % (self.B, self.wire))
        _check(lib().dpf_server_submit(self.h, kw.ctypes.data), "dpf_server_submit")

    def collect(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """dpf_server_collect: wait for the oldest batch in flight, its answers."""
        if out is None:
            out = np.empty((self.B, self.D), dtype=np.uint32)
        _check(lib().dpf_server_collect(self.h, out.ctypes.data), "dpf_server_collect")
        return out

    def close(self):
        if self.h is not None and self.h.value:
            lib().dpf_server_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eval_batch_wire(keys_wire_dev, log_n: int, table_shard, row_begin: int = 0, out=None, workspace=None,
                    stream=None, prf: int = DPF_PRF_CHACHA20):
    """dpf_eval_batch_wire: keys already in HBM as wire records (uint8 CUDA tensor [B, 32+64n])."""
    import torch
    _check_table(table_shard)
    rows, D = table_shard.shape
    B = keys_wire_dev.shape[0]
    if out is None:
        out = torch.empty((B, D), dtype=torch.int32, device=table_shard.device)
    need = eval_workspace_bytes(B, log_n, rows, D)
    ws = workspace if workspace is not None else _workspace(need, table_shard.device, stream)
    _check(lib().dpf_eval_batch_wire(keys_wire_dev.data_ptr(), B, log_n, prf, table_shard.data_ptr(), row_begin, rows, D,
                                     out.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(),
                                     _stream_ptr(stream)), "dpf_eval_batch_wire")
    return out


class PackedTable:
    """A device table shard re-laid-out by dpf_table_pack for the tcgen05 path."""

    def __init__(self, data, row_begin: int, row_count: int, D: int):
        self.data, self.row_begin, self.row_count, self.D = data, row_begin, row_count, D

    @property
    def shape(self):
        return (self.row_count, self.D)


def table_packed_bytes(row_begin: int, row_count: int, D: int) -> int:
    return lib().dpf_table_packed_bytes(row_begin, row_count, D)


def table_pack(table_shard, row_begin: int = 0, stream=None) -> PackedTable:
    """dpf_table_pack: limb-packed copy of a row-major CUDA table shard."""
    import torch
    _check_table(table_shard)
    rows, D = table_shard.shape
    nbytes = table_packed_bytes(row_begin, rows, D)
    if nbytes == 0:
        raise DpfError(DPF_EINVAL, "dpf_table_packed_bytes")
    buf = torch.empty(nbytes, dtype=torch.uint8, device=table_shard.device)
    _check(lib().dpf_table_pack(table_shard.data_ptr(), row_begin, rows, D, buf.data_ptr(), _stream_ptr(stream)),
           "dpf_table_pack")
    return PackedTable(buf, row_begin, rows, D)


def eval_batch_packed(keys, packed: PackedTable, out=None, workspace=None, stream=None):
    """dpf_eval_batch_packed: the tcgen05 contraction path on a packed table shard."""
    import torch
    kb = _as_batch(keys)
    B, D = len(kb), packed.D
    if out is None:
        out = torch.empty((B, D), dtype=torch.int32, device=packed.data.device)
    need = eval_workspace_bytes(B, kb.log_n, packed.row_count, D)
    ws = workspace if workspace is not None else _workspace(need, packed.data.device, stream)
    _check(lib().dpf_eval_batch_packed(kb.ptr, B, packed.data.data_ptr(), packed.row_begin, packed.row_count, D,
                                       out.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(),
                                       _stream_ptr(stream)), "dpf_eval_batch_packed")
    return out


def eval_batch_wire_packed(keys_wire_dev, log_n: int, packed: PackedTable, out=None, workspace=None, stream=None,
                           prf: int = DPF_PRF_CHACHA20):
    """dpf_eval_batch_wire_packed: device-resident wire keys, packed table."""
    import torch
    B, D = keys_wire_dev.shape[0], packed.D
    if out is None:
        out = torch.empty((B, D), dtype=torch.int32, device=packed.data.device)
    need = eval_workspace_bytes(B, log_n, packed.row_count, D)
    ws = workspace if workspace is not None else _workspace(need, packed.data.device, stream)
    _check(lib().dpf_eval_batch_wire_packed(keys_wire_dev.data_ptr(), B, log_n, prf, packed.data.data_ptr(),
                                            packed.row_begin, packed.row_count, D, out.data_ptr(), ws.data_ptr(),
                                            ws.numel() * ws.element_size(), _stream_ptr(stream)),
           "dpf_eval_batch_wire_packed")
    return out


def _group_array(groups):
    """groups: (keys_wire, log_n, table, row_begin, shares); `table` a row-major
    CUDA shard or a PackedTable (dpf_eval_grouped_packed)."""
    arr = (DpfEvalGroup * len(groups))()
    for i, g in enumerate(groups):
        keys_wire, log_n, table, row_begin, shares = g
        arr[i].keys_wire = keys_wire.data_ptr()
        arr[i].B = keys_wire.shape[0]
        arr[i].log_n = log_n
        if isinstance(table, PackedTable):
            arr[i].table = table.data.data_ptr()
            arr[i].row_count = table.row_count
            if table.row_begin != row_begin:
                raise ValueError("packed table row_begin differs from the group's")
        else:
            arr[i].table = table.data_ptr()
            arr[i].row_count = table.shape[0]
        arr[i].row_begin = row_begin
        arr[i].shares = shares.data_ptr()
    return arr


def eval_grouped_workspace_bytes(groups, D: int, prf: int = DPF_PRF_CHACHA20) -> int:
    return lib().dpf_eval_grouped_workspace_bytes(_group_array(groups), len(groups), D, prf)


def eval_grouped(groups, D: int, prf: int = DPF_PRF_CHACHA20, workspace=None, stream=None):
    """dpf_eval_grouped.  groups: list of (keys_wire_dev uint8 [B, 32+64n], log_n,
    table_shard int32 [rows, D], row_begin, shares int32 [B, D]); all CUDA tensors."""
    arr = _group_array(groups)
    need = lib().dpf_eval_grouped_workspace_bytes(arr, len(groups), D, prf)
    if need == 0:
        raise DpfError(DPF_EINVAL, "dpf_eval_grouped_workspace_bytes")
    dev = groups[0][2].device
    ws = workspace if workspace is not None else _workspace(need, dev, stream)
    _check(lib().dpf_eval_grouped(arr, len(groups), D, prf, ws.data_ptr(), ws.numel() * ws.element_size(),
                                  _stream_ptr(stream)), "dpf_eval_grouped")
    return [g[4] for g in groups]


def eval_grouped_packed_workspace_bytes(groups, D: int, prf: int = DPF_PRF_CHACHA20) -> int:
    return lib().dpf_eval_grouped_packed_workspace_bytes(_group_array(groups), len(groups), D, prf)


def eval_grouped_packed(groups, D: int, prf: int = DPF_PRF_CHACHA20, workspace=None, stream=None):
    """dpf_eval_grouped_packed: as eval_grouped with every group's table a
    PackedTable (table_pack of that group's shard), tcgen05 contraction."""
    arr = _group_array(groups)
    need = lib().dpf_eval_grouped_packed_workspace_bytes(arr, len(groups), D, prf)
    if need == 0:
        raise DpfError(DPF_EINVAL, "dpf_eval_grouped_packed_workspace_bytes")
    dev = groups[0][4].device
    ws = workspace if workspace is not None else _workspace(need, dev, stream)
    _check(lib().dpf_eval_grouped_packed(arr, len(groups), D, prf, ws.data_ptr(), ws.numel() * ws.element_size(),
                                         _stream_ptr(stream)), "dpf_eval_grouped_packed")
    return [g[4] for g in groups]


def eval_pbr_workspace_bytes(B: int, log_i: int, N: int, D: int, prf: int = DPF_PRF_CHACHA20,
                             packed: bool = False) -> int:
    return lib().dpf_eval_pbr_workspace_bytes(B, log_i, N, D, prf, int(packed))


def eval_pbr(keys_wire_dev, B: int, log_i: int, table, out=None, workspace=None, stream=None,
             prf: int = DPF_PRF_CHACHA20):
    """dpf_eval_pbr (partial batch retrieval): keys_wire_dev uint8
    [n_bins * B, wire bytes] bin-major (client c's key for bin b at row b*B + c),
    `table` the whole row-major CUDA table [N, D] or its PackedTable (row_begin 0).
    Returns shares int32 [n_bins, B, D]."""
    import torch
    packed = isinstance(table, PackedTable)
    if packed:
        if table.row_begin != 0:
            raise ValueError("PBR needs the packed copy of the whole table (row_begin 0)")
        N, D, ptr, dev = table.row_count, table.D, table.data.data_ptr(), table.data.device
    else:
        _check_table(table)
        (N, D), ptr, dev = table.shape, table.data_ptr(), table.device
    nb = (N + (1 << log_i) - 1) >> log_i
    if keys_wire_dev.shape[0] != nb * B:
        raise ValueError("expected %d bin-major keys, got %d" % (nb * B, keys_wire_dev.shape[0]))
    if out is None:
        out = torch.empty((nb, B, D), dtype=torch.int32, device=dev)
    need = eval_pbr_workspace_bytes(B, log_i, N, D, prf, packed)
    if need == 0:
        raise DpfError(DPF_EINVAL, "dpf_eval_pbr_workspace_bytes")
    ws = workspace if workspace is not None else _workspace(need, dev, stream)
    _check(lib().dpf_eval_pbr(keys_wire_dev.data_ptr(), B, log_i, prf, ptr, int(packed), N, D, out.data_ptr(),
                              ws.data_ptr(), ws.numel() * ws.element_size(), _stream_ptr(stream)), "dpf_eval_pbr")
    return out


def serve_workspace_bytes(B: int, log_n: int, rows: int, D: int) -> int:
    return eval_workspace_bytes(B, log_n, rows, D) + (B * D * 4 + 255) // 256 * 256


def serve_batch(keys, table_shard, shares_host, row_begin: int = 0, workspace=None, stream=None):
    """dpf_serve_batch: host keys in, host answers out (synchronous)."""
    kb = _as_batch(keys)
    _check_table(table_shard)
    rows, D = table_shard.shape
    B = len(kb)
    need = serve_workspace_bytes(B, kb.log_n, rows, D)
    ws = workspace if workspace is not None else _workspace(need, table_shard.device, stream)
    if isinstance(shares_host, np.ndarray):
        assert shares_host.dtype in (np.uint32, np.int32) and shares_host.size >= B * D
        hptr = shares_host.ctypes.data
    else:
        assert not shares_host.is_cuda and shares_host.numel() >= B * D
        hptr = shares_host.data_ptr()
    _check(lib().dpf_serve_batch(kb.ptr, B, table_shard.data_ptr(), row_begin, rows, D, hptr, ws.data_ptr(),
                                 ws.numel() * ws.element_size(), _stream_ptr(stream)), "dpf_serve_batch")
    return shares_host


def eval_leaves(keys, device="cuda", stream=None):
    """dpf_eval_leaves (test/debug): leaves[b][j] = Eval(k_b, j), log_n <= 20."""
    import torch
    kb = _as_batch(keys)
    B, n = len(kb), kb.log_n
    out = torch.empty((B, 1 << n), dtype=torch.int32, device=device)
    ws = _workspace(B * key_wire_size(n, kb.prf) + 256, out.device, stream)
    _check(lib().dpf_eval_leaves(kb.ptr, B, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
           "dpf_eval_leaves")
    return out


def last_eval_stats() -> dict:
    s = DpfEvalStats()
    _check(lib().dpf_last_eval_stats(ctypes.byref(s)), "dpf_last_eval_stats")
    return {f: getattr(s, f) for f, _ in DpfEvalStats._fields_}


def kernel_name(kernel_id: int) -> str:
    """The fused-kernel template a plan launches (dpf_eval_stats.kernel_id), in
    the form ncu prints it (namespaces dropped)."""
    prf = {DPF_PRF_CHACHA20: "PrfChacha", DPF_PRF_AES128: "PrfAesTt", DPF_PRF_CHACHA20_ET: "PrfChachaEt"}.get(
        (kernel_id >> 8) & 0xF, "?")
    np_ = (kernel_id >> 12) & 0x3F
    if kernel_id & 1:
        return "fused_eval_tc_kernel<%s, %d, %d, 4, %d, %d, %d>" % (
            prf, np_, (kernel_id >> 4) & 0xF, (kernel_id >> 1) & 1, (kernel_id >> 2) & 1, (kernel_id >> 3) & 1)
    return "fused_eval_kernel<%s, %d, 4, %d, %d>" % (prf, np_, (kernel_id >> 18) & 0x3F, kernel_id >> 24)


def eval_plan(B: int, log_n: int, rows: int, D: int, prf: int = DPF_PRF_CHACHA20, row_begin: int = 0,
              packed: bool = False) -> dict:
    """dpf_eval_plan: the launch plan (host only, no device calls)."""
    s = DpfEvalStats()
    _check(lib().dpf_eval_plan(B, log_n, prf, row_begin, rows, D, int(packed), ctypes.byref(s)), "dpf_eval_plan")
    return {f: getattr(s, f) for f, _ in DpfEvalStats._fields_}


def kernel_timer_begin(capacity: int) -> None:
    _check(lib().dpf_kernel_timer_begin(capacity), "dpf_kernel_timer_begin")


def kernel_timer_read(capacity: int) -> list:
    ms = (ctypes.c_float * max(capacity, 1))()
    cnt = ctypes.c_uint32(0)
    _check(lib().dpf_kernel_timer_read(ms, capacity, ctypes.byref(cnt)), "dpf_kernel_timer_read")
    return [ms[i] for i in range(cnt.value)]


def as_u32(t) -> np.ndarray:
    """CUDA/CPU int32 tensor -> numpy uint32 (bit patterns)."""
    return t.detach().cpu().numpy().view(np.uint32)
