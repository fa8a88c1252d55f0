"""ctypes binding of libkvc.so (the C ABI declared in include/kvc.h).

There is no fallback: if the library is missing or no CUDA device is
present, every device entry point raises.  The product path is the CUDA
library; the CPU oracle under oracle/ is test infrastructure only.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVC_LIB_PATH") or os.path.join(_HERE, "libkvc.so")  # (override: experiments)

KVC_FREE_TILE = 1024

# kvc_status codes (include/kvc.h)
OK = 0
ERR_INVALID = -1
ERR_UNSUPPORTED = -2
ERR_CUDA = -3
DEV_PREEMPTION = 1
DEV_ALLOCATION_ORDER = 2
DEV_EMPTY_CONTEXT = 3
DEV_NUMERIC = 4
DEV_SCHEDULE_CORRUPTION = 5
DEV_CACHE_CORRUPTION = 6
DEV_CAPACITY = 7

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f32 = ctypes.c_float


class KvcPool(ctypes.Structure):
    _fields_ = [
        ("k_cache", _p), ("v_cache", _p), ("metric", _p), ("logical", _p), ("protected_", _p), ("fresh", _p),
        ("free_flag", _p), ("free_tile", _p), ("tables", _p), ("nblocks", _p), ("ctx", _p),
        ("status", _p), ("scratch", _p), ("scratch_bytes", _i64), ("num_blocks", _i64),
        ("block_size", _i32), ("head_dim", _i32), ("num_layers", _i32), ("num_kv_heads", _i32),
        ("max_seqs", _i32), ("max_blocks", _i32),
    ]


class DecodeArgs(ctypes.Structure):
    _fields_ = [
        ("seq_rows", _p), ("batch", _i32), ("layer", _i32), ("num_query_heads", _i32),
        ("q", _p), ("k_new", _p), ("v_new", _p), ("out", _p), ("out_f32", _i32),
        ("rows_out", _p), ("rows_stride", _i64), ("metric_mode", _i32), ("append_fresh", _i32),
        ("max_ctx", _i32), ("splits", _i32), ("queue", _p), ("metric_stream", _p), ("early_pull", _i32),
    ]


class WindowArgs(ctypes.Structure):
    _fields_ = [
        ("seq_row", _i32), ("layer", _i32), ("num_query_heads", _i32), ("L", _i32),
        ("q_win", _p), ("k", _p), ("window", _i32), ("pool", _i32), ("aggregation", _i32),
        ("protect_window", _i32), ("metrics_out", _p), ("n_layers", _i32), ("q_layer_stride", _i64),
        ("k_layer_stride", _i64), ("out_layer_stride", _i64), ("write_k", _i32),
    ]


class FullArgs(ctypes.Structure):
    _fields_ = [
        ("num_query_heads", _i32), ("L", _i32), ("q", _p), ("k", _p), ("excluded", _i32), ("aggregation", _i32),
        ("metrics_out", _p),
    ]


class DenseArgs(ctypes.Structure):
    _fields_ = [
        ("num_query_heads", _i32), ("L", _i32), ("q", _p), ("k", _p), ("v", _p), ("out", _p), ("attn", _p),
    ]


class AttnMetricArgs(ctypes.Structure):
    _fields_ = [
        ("num_query_heads", _i32), ("L", _i32), ("attn", _p), ("mode", _i32), ("window", _i32), ("pool", _i32),
        ("excluded", _i32), ("aggregation", _i32), ("metrics_out", _p),
    ]


class EvictArgs(ctypes.Structure):
    _fields_ = [
        ("seq_rows", _p), ("budgets", _p), ("n_seqs", _i32), ("max_slots_per_head", _i64),
        ("clamped", _p), ("evict", _p), ("evicted_kvs", _p), ("freed", _p), ("moves", _p),
        ("moves_capacity", _i64), ("move_offsets", _p), ("move_counts", _p), ("totals", _p),
        ("src_pos", _p),
    ]


_SIGS = {
    "kvc_abi_version": ([], _i32),
    "kvc_status_name": ([_i32], ctypes.c_char_p),
    "kvc_pool_init": ([_p, _p], _i32),
    "kvc_scratch_bytes": ([_p, _i64, _i64, _i32], _i64),
    "kvc_alloc_prefill": ([_p, _i32, _i32, _p], _i32),
    "kvc_alloc_heads": ([_p, _i32, _p, _i64, _p], _i32),
    "kvc_alloc_decode": ([_p, _p, _i32, _p, _p], _i32),
    "kvc_free_trailing": ([_p, _p, _p, _i32, _p], _i32),
    "kvc_free_sequence": ([_p, _i32, _p], _i32),
    "kvc_append_kv": ([_p, _p, _p, _p, _i32, _i32, _p], _i32),
    "kvc_write_prefill_kv": ([_p, _i32, _i32, _p, _p, _i32, _p], _i32),
    "kvc_write_prefill_kv_layers": ([_p, _i32, _i32, _i32, _p, _p, _i32, _p], _i32),
    "kvc_write_prefill_v_layers": ([_p, _i32, _i32, _i32, _p, _p, _i32, _p], _i32),
    "kvc_write_prompt_pass": ([_p, _i32, _i32, _p, _i64, _p, _i32, _p], _i32),
    "kvc_paged_decode": ([_p, _p, _p], _i32),
    "kvc_decode_scratch_bytes": ([_p, _i32, _i32, _i32], _i64),
    "kvc_accumulate_rows": ([_p, _i32, _i32, _p, _i32, _i64, _i32, _p], _i32),
    "kvc_clear_fresh": ([_p, _p, _i32, _p], _i32),
    "kvc_window_metric": ([_p, _p, _p], _i32),
    "kvc_schedule_evictions": ([_p, _p, _p], _i32),
    "kvc_execute_moves": ([_p, _p, _p], _i32),
    "kvc_compress": ([_p, _p, _p], _i32),
    "kvc_full_metric": ([_p, _p, _p], _i32),
    "kvc_prefill_compress": ([_p, _p, _p, _p, _i32, _p], _i32),
    "kvc_gqa_attention": ([_p, _p, _p], _i32),
    "kvc_attn_metrics": ([_p, _p, _p], _i32),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libkvc.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int, what: str = "") -> None:
    """Map an immediate launch status onto an exception."""
    if rc == OK:
        return
    name = lib().kvc_status_name(rc).decode()
    if rc == ERR_INVALID:
        raise ValueError(f"{what}: {name}")
    if rc == ERR_UNSUPPORTED:
        raise E.ConfigError(what or "shape", name)
    raise RuntimeError(f"{what}: {name} ({rc})")


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda(device) -> torch.device:
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device() if torch.cuda.is_available() else 0)
    if device.type != "cuda" or not torch.cuda.is_available():
        raise RuntimeError("paper_2410_00161_b200 requires a CUDA device (no CPU fallback)")
    load()
    return device


class DeviceContext:
    """Per-device shared state: status word and a growable workspace."""

    _by_device: dict = {}

    def __init__(self, device: torch.device):
        self.device = device
        self.status = torch.zeros(4, dtype=torch.int32, device=device)
        self._scratch = torch.empty(1 << 22, dtype=torch.uint8, device=device)
        self._queues: dict = {}

    @classmethod
    def get(cls, device) -> "DeviceContext":
        device = torch.device(device)
        key = (device.type, device.index if device.index is not None else torch.cuda.current_device())
        if key not in cls._by_device:
            cls._by_device[key] = cls(torch.device("cuda", key[1]))
        return cls._by_device[key]

    def decode_queue(self, n: int, stream: int) -> torch.Tensor:
        """Zeroed int32 work-queue counters for kvc_paged_decode on `stream`
        (the call leaves them zero, so they are allocated once per stream,
        not cleared per call)."""
        qt = self._queues.get(stream)
        if qt is None or qt.numel() < n:
            qt = self._queues[stream] = torch.zeros(max(n, 1024), dtype=torch.int32, device=self.device)
        return qt

    def scratch(self, nbytes: int) -> torch.Tensor:
        if self._scratch.numel() < nbytes:
            self._scratch = torch.empty(int(nbytes * 1.25) + (1 << 20), dtype=torch.uint8, device=self.device)
        return self._scratch

    def raise_status(self) -> None:
        """Synchronise on the status word and raise the mapped exception."""
        st = self.status.tolist()
        if st[0] == 0:
            return
        self.status.zero_()
        code, a, b = st[0], st[1], st[2]
        if code == DEV_PREEMPTION:
            raise E.PreemptionNeeded(a)
        if code == DEV_ALLOCATION_ORDER:
            raise E.AllocationOrderError(f"no block allocated for position {b} (head {a})")
        if code == DEV_EMPTY_CONTEXT:
            raise E.EmptyContextError(f"head {a} has no live KVs")
        if code == DEV_NUMERIC:
            raise E.NumericError("non-finite values in attention inputs")
        if code == DEV_SCHEDULE_CORRUPTION:
            raise E.ScheduleCorruptionError(f"compaction contract violated (head {a}, {b})")
        if code == DEV_CACHE_CORRUPTION:
            raise E.CacheCorruptionError(f"head {a}: context {b} exceeds allocated slots")
        if code == DEV_CAPACITY:
            raise E.DeviceCapacityError(f"head {a} needs {b} table entries")
        raise RuntimeError(f"device status {st}")


def is_host_array(x) -> bool:
    """True for a caller-side (non-torch) array: the reference-signature entry
    points then return NumPy arrays like the reference does (computed on the
    GPU, copied back); device tensors in give device tensors out."""
    return not torch.is_tensor(x)


def to_host(t: torch.Tensor):
    """A device result as the reference's NumPy type (floats as float64)."""
    t = t.detach()
    if t.is_floating_point():
        t = t.to(torch.float64)
    return t.cpu().numpy()

