"""ctypes binding of libkvmig.so (include/kvmig.h).

This is the only way the package reaches the GPU.  If the library is absent
the import of any data-path object fails loudly (NativeLibraryMissing); there
is no eager-PyTorch or CPU fallback for the copy or the re-prefill.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import (ConfigError, KvmCudaError, KvmUnsupported, NativeLibraryMissing, NoCategory, NotPlaced,
                     RequestTooLarge)

HERE = os.path.dirname(os.path.abspath(__file__))
# KVM_LIB_PATH: load another build of the library (A/B experiments with kernel variants)
LIB_PATH = os.environ.get("KVM_LIB_PATH") or os.path.join(HERE, "_lib", "libkvmig.so")

KVM_OK = 0
ABI_VERSION = 2   # include/kvmig.h KVM_ABI_VERSION
KVM_ERR_INVALID = -1
KVM_ERR_CONFIG = -2
KVM_ERR_CUDA = -3
KVM_ERR_NOT_FOUND = -4
KVM_ERR_UNSUPPORTED = -5
KVM_ERR_KEY = -6
KVM_ERR_TOO_LARGE = -7
KVM_ERR_NO_CATEGORY = -8
KVM_ERR_ASSERT = -9
KVM_NONE = -(2 ** 63)

KVM_F_BLOCKS_ON_HOST = 0x1
KVM_F_ENGINE_BULK = 0x2
KVM_F_L2_EVICT_FIRST = 0x4
KVM_F_SYS_SCOPE = 0x8
KVM_MAX_MOVES = 96
KVM_REPREFILL_SINGLE_CTA = 0x1
KVM_REPREFILL_ROPE = 0x2
KVM_REPREFILL_X_PER_LAYER = 0x4


def KVM_F_CTAS_PER_SM(n: int) -> int:
    return (n & 0xFF) << 8


def KVM_F_MAX_SMS(n: int) -> int:
    return (n & 0xFF) << 16


def KVM_REPREFILL_MAX_SMS(n: int) -> int:
    return (n & 0xFF) << 8

# Every symbol include/kvmig.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "kvm_version", "kvm_last_error", "kvm_device_count", "kvm_init", "kvm_can_access_peer",
    "kvm_pool_register", "kvm_pool_register_strided", "kvm_pool_unregister", "kvm_pool_piece_bytes", "kvm_pool_bytes",
    "kvm_ipc_export", "kvm_ipc_import", "kvm_ipc_close",
    "kvm_migrate", "kvm_compact", "kvm_wait_flag", "kvm_reprefill", "kvm_paged_decode",
    "kvm_plan_hybrid", "kvm_wait_flag_timeout", "kvm_split_migrate", "kvm_launch_count",
    "kvm_cluster_create", "kvm_cluster_destroy", "kvm_cluster_op", "kvm_cluster_terminate_idle",
    "kvm_cluster_snapshot", "kvm_cluster_verify", "kvm_sched_create", "kvm_sched_destroy",
    "kvm_sched_set_batching", "kvm_sched_step_epoch", "kvm_sched_op", "kvm_sched_class_of",
    "kvm_sched_priority", "kvm_read_back",
)
KVM_DECODE_BF16 = 0x1
KVM_DECODE_CUDA_CORES = 0x2
KVM_DECODE_WAIT_LAYERS = 0x4


class PoolDesc(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int32), ("kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("block_tokens", ctypes.c_int32),
                ("num_blocks", ctypes.c_int32), ("elem_bytes", ctypes.c_int32)]


class Move(ctypes.Structure):
    _fields_ = [("src_pool", ctypes.c_int32), ("dst_pool", ctypes.c_int32),
                ("n_blocks", ctypes.c_int32), ("done_value", ctypes.c_uint32),
                ("src_blocks", ctypes.c_void_p), ("dst_blocks", ctypes.c_void_p),
                ("dst_table_row", ctypes.c_void_p), ("done_flag", ctypes.c_void_p),
                ("layer_flags", ctypes.c_void_p)]


class ReprefillArgs(ctypes.Structure):
    _fields_ = [("dst_pool", ctypes.c_int32), ("rows", ctypes.c_int32),
                ("d_model", ctypes.c_int32), ("q_cols", ctypes.c_int32),
                ("tok0", ctypes.c_int32), ("n_dst_blocks", ctypes.c_int32),
                ("x", ctypes.c_void_p), ("w", ctypes.c_void_p), ("q_out", ctypes.c_void_p),
                ("dst_blocks", ctypes.c_void_p), ("done_flag", ctypes.c_void_p),
                ("done_value", ctypes.c_uint32), ("flags", ctypes.c_int32), ("rope_theta", ctypes.c_float)]


class SplitArgs(ctypes.Structure):
    _fields_ = [("src_pool", ctypes.c_int32), ("dst_pool", ctypes.c_int32), ("tokens", ctypes.c_int32),
                ("prefix_blocks", ctypes.c_int32), ("d_model", ctypes.c_int32), ("q_cols", ctypes.c_int32),
                ("src_blocks", ctypes.c_void_p), ("dst_blocks", ctypes.c_void_p), ("x", ctypes.c_void_p),
                ("w", ctypes.c_void_p), ("q_out", ctypes.c_void_p), ("dst_table_row", ctypes.c_void_p),
                ("done_flag", ctypes.c_void_p), ("done_value", ctypes.c_uint32), ("flags", ctypes.c_int32),
                ("rope_theta", ctypes.c_float)]


class DecodeArgs(ctypes.Structure):
    _fields_ = [("pool", ctypes.c_int32), ("layer0", ctypes.c_int32), ("n_layers", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("q_heads", ctypes.c_int32), ("max_blocks", ctypes.c_int32),
                ("max_seq_len", ctypes.c_int32), ("flags", ctypes.c_int32), ("scale", ctypes.c_float),
                ("q", ctypes.c_void_p), ("block_tables", ctypes.c_void_p), ("seq_lens", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("layer_flags", ctypes.c_void_p), ("layer_value", ctypes.c_uint32),
                ("_pad", ctypes.c_uint32), ("timeout_ns", ctypes.c_uint64), ("err_word", ctypes.c_void_p)]


class Pending(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("item", "src", "dst", "kv_bytes", "tokens", "defer_count")]


class PlanParams(ctypes.Structure):
    _fields_ = [("gpus_per_machine", ctypes.c_int32), ("max_defer", ctypes.c_int32),
                ("intra_bandwidth", ctypes.c_double), ("inter_bandwidth", ctypes.c_double),
                ("prefill_tokens_per_s", ctypes.c_double), ("comp_budget", ctypes.c_double),
                ("intra_comm_budget", ctypes.c_double), ("inter_comm_budget", ctypes.c_double),
                ("n_overrides", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("override_link", ctypes.c_void_p), ("override_budget", ctypes.c_void_p)]


class Planned(ctypes.Structure):
    _fields_ = [("index", ctypes.c_int32), ("mode", ctypes.c_int32), ("latency_s", ctypes.c_double)]


class PlanLedgers(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int32), ("n_links", ctypes.c_int32), ("n_dests", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("link_key", ctypes.c_void_p), ("link_used", ctypes.c_void_p),
                ("dest_key", ctypes.c_void_p), ("dest_used", ctypes.c_void_p)]


class SchedParams(ctypes.Structure):
    _fields_ = [("weight_free_mem", ctypes.c_double), ("weight_request_count", ctypes.c_double),
                ("weight_same_machine", ctypes.c_double), ("batching", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


_lib = None
_lock = threading.Lock()


def _declare(L: ctypes.CDLL) -> None:
    I, P, I64 = ctypes.c_int, ctypes.c_void_p, ctypes.c_int64
    sig = {
        "kvm_version": ([], I),
        "kvm_last_error": ([], ctypes.c_char_p),
        "kvm_device_count": ([ctypes.POINTER(I)], I),
        "kvm_init": ([I], I),
        "kvm_can_access_peer": ([I, I, ctypes.POINTER(I)], I),
        "kvm_pool_register": ([I, P, ctypes.POINTER(PoolDesc)], I),
        "kvm_pool_register_strided": ([I, ctypes.POINTER(PoolDesc), ctypes.POINTER(P), I64, I64], I),
        "kvm_pool_unregister": ([I], I),
        "kvm_pool_piece_bytes": ([I, ctypes.POINTER(I64)], I),
        "kvm_pool_bytes": ([ctypes.POINTER(PoolDesc), ctypes.POINTER(I64)], I),
        "kvm_ipc_export": ([P, P, ctypes.POINTER(I64)], I),
        "kvm_ipc_import": ([I, P, I64, ctypes.POINTER(P)], I),
        "kvm_ipc_close": ([P, I64], I),
        "kvm_migrate": ([ctypes.POINTER(Move), I, I, P], I),
        "kvm_compact": ([I, P, P, I, P, I, P], I),
        "kvm_wait_flag": ([P, ctypes.c_uint32, P], I),
        "kvm_wait_flag_timeout": ([P, ctypes.c_uint32, ctypes.c_uint64, P, P], I),
        "kvm_reprefill": ([ctypes.POINTER(ReprefillArgs), P], I),
        "kvm_paged_decode": ([ctypes.POINTER(DecodeArgs), P], I),
        "kvm_split_migrate": ([ctypes.POINTER(SplitArgs), P], I),
        "kvm_plan_hybrid": ([ctypes.POINTER(Pending), I, ctypes.POINTER(PlanParams), ctypes.POINTER(Planned),
                             ctypes.POINTER(PlanLedgers)], I),
        "kvm_launch_count": ([], I64),
        "kvm_cluster_create": ([I64, I64, ctypes.POINTER(P)], I),
        "kvm_cluster_destroy": ([P], None),
        "kvm_cluster_op": ([P, I, I64, I64, ctypes.POINTER(I64)], I),
        "kvm_cluster_terminate_idle": ([P, ctypes.POINTER(P), ctypes.POINTER(I64)], I),
        "kvm_cluster_snapshot": ([P, ctypes.POINTER(P), ctypes.POINTER(I64)], I),
        "kvm_cluster_verify": ([P, P, I64, ctypes.POINTER(P), ctypes.POINTER(I64)], I),
        "kvm_sched_create": ([P, ctypes.POINTER(SchedParams), ctypes.POINTER(P)], I),
        "kvm_sched_destroy": ([P], None),
        "kvm_sched_set_batching": ([P, I], I),
        "kvm_sched_step_epoch": ([P, P, I64, P, I64, P, I64, ctypes.POINTER(P), ctypes.POINTER(I64)], I),
        "kvm_sched_op": ([P, I, P, I64, I64, ctypes.POINTER(P), ctypes.POINTER(I64)], I),
        "kvm_sched_class_of": ([P, I64, ctypes.POINTER(ctypes.c_int32)], I),
        "kvm_sched_priority": ([P, I64, I64, ctypes.POINTER(ctypes.c_double)], I),
        "kvm_read_back": ([P, P, I64, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> ctypes.CDLL:
    """Load libkvmig.so once; raise NativeLibraryMissing if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (there is no CPU fallback for the KV data path)")
            L = ctypes.CDLL(LIB_PATH)
            _declare(L)
            if L.kvm_version() != ABI_VERSION:   # struct layouts below must match the build
                raise NativeLibraryMissing(
                    f"{LIB_PATH} has ABI {L.kvm_version()}, this package needs {ABI_VERSION}: rebuild it")
            _lib = L
    return _lib


def check(rc: int, what: str = "") -> int:
    """Map a KVM_ERR_* return code onto the reference's exception classes."""
    if rc >= 0:
        return rc
    msg = lib().kvm_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == KVM_ERR_INVALID:
        raise ValueError(text)
    if rc == KVM_ERR_CONFIG:
        raise ConfigError(text)
    if rc == KVM_ERR_NOT_FOUND:
        raise NotPlaced(text)
    if rc == KVM_ERR_UNSUPPORTED:
        raise KvmUnsupported(text)
    if rc == KVM_ERR_KEY:
        raise KeyError(text)
    if rc == KVM_ERR_TOO_LARGE:
        raise RequestTooLarge(text)
    if rc == KVM_ERR_NO_CATEGORY:
        raise NoCategory(text)
    if rc == KVM_ERR_ASSERT:
        raise AssertionError(text)
    raise KvmCudaError(text)


def records(ptr: ctypes.c_void_p, n: ctypes.c_int64, width: int = 5) -> list:
    """Copy a library-owned int64 record buffer (n records of `width` words)."""
    count = int(n.value) * width
    if count == 0:
        return []
    return ctypes.cast(ptr, ctypes.POINTER(ctypes.c_int64))[:count]


def launch_count() -> int:
    return int(lib().kvm_launch_count())
