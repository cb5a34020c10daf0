"""ORACLE — TEST INFRASTRUCTURE ONLY: ctypes wrapper over liboracle_kvmig.so.

Operates on numpy arrays (host memory).  See kvmig_oracle.c for what is
restated from the reference and what is frozen by this repo.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_kvmig.so")


class PoolDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("layers", "kv_heads", "head_dim", "block_tokens", "num_blocks", "elem_bytes")]


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.oracle_migrate.argtypes = [P, ctypes.POINTER(PoolDesc), P, ctypes.POINTER(PoolDesc), P, P,
                                     ctypes.c_int, P, ctypes.c_int]
        L.oracle_migrate.restype = ctypes.c_int
        L.oracle_alloc_ascending.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
        L.oracle_alloc_ascending.restype = ctypes.c_int
        L.oracle_piece_offset.argtypes = [ctypes.POINTER(PoolDesc), ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int]
        L.oracle_piece_offset.restype = ctypes.c_int64
        L.oracle_reprefill.argtypes = [ctypes.POINTER(PoolDesc), P, P, ctypes.c_int, P, P,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.oracle_reprefill.restype = ctypes.c_int
        _lib = L
    return _lib


def desc(layers, kv_heads, head_dim, block_tokens, num_blocks, elem_bytes=2) -> PoolDesc:
    return PoolDesc(layers, kv_heads, head_dim, block_tokens, num_blocks, elem_bytes)


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def migrate(src: np.ndarray, sd: PoolDesc, dst: np.ndarray, dd: PoolDesc,
            src_blocks, dst_blocks, threads: int = 1) -> np.ndarray:
    """In-place on `dst`; returns the rewritten dst block-table row."""
    sb = np.ascontiguousarray(src_blocks, dtype=np.int32)
    db = np.ascontiguousarray(dst_blocks, dtype=np.int32)
    row = np.full(len(sb), -1, dtype=np.int32)
    rc = lib().oracle_migrate(_ptr(src), ctypes.byref(sd), _ptr(dst), ctypes.byref(dd), _ptr(sb),
                              _ptr(db), len(sb), _ptr(row), threads)
    if rc != 0:
        raise ValueError("oracle_migrate rejected its arguments")
    return row


def alloc_ascending(free_mask: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    rc = lib().oracle_alloc_ascending(_ptr(free_mask), len(free_mask), n, _ptr(out))
    if rc != 0:
        raise MemoryError("not enough free blocks")
    return out


def reprefill(dd: PoolDesc, dst: np.ndarray, dst_blocks, x: np.ndarray, w: np.ndarray, rows: int,
              d_model: int, q_cols: int, tok0: int, q_out=None) -> None:
    """x, w, q_out are uint16 arrays holding bf16 bits."""
    db = np.ascontiguousarray(dst_blocks, dtype=np.int32)
    rc = lib().oracle_reprefill(ctypes.byref(dd), _ptr(dst), _ptr(db), len(db), _ptr(x), _ptr(w),
                                rows, d_model, q_cols, tok0,
                                None if q_out is None else _ptr(q_out))
    if rc != 0:
        raise ValueError("oracle_reprefill rejected its arguments")
