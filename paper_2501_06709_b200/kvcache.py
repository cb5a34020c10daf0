"""Paged KV pools, block allocation and block tables (the objects the
reference only models as byte counts).

The reference tracks a request's KV cache as one integer,
`kv_size_at = (prompt + generated) * kv_bytes_per_token` (model.py:58-69),
and a GPU as `capacity_bytes` (model.py:122-131).  Here those numbers become
memory: a per-GPU paged pool in HBM and a per-request block table.

Frozen layout (vLLM-style, layer-major):

    pool[layers][2 (K,V)][num_blocks][block_tokens][kv_heads][head_dim]

so one (layer, K|V, block) piece is a contiguous
block_tokens*kv_heads*head_dim*elem_bytes run (128 KiB for Llama-2-7B) and a
token's K row is a contiguous kv_heads*head_dim run inside it.
Allocation is deterministic: the n lowest free block ids, ascending.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Dict, Iterable, Optional

import numpy as np

from . import _native
from .errors import ConfigError, NotPlaced, RequestTooLarge


@dataclass(frozen=True)
class ModelShape:
    """KV geometry of one model family (fp16/bf16, 16-token blocks)."""

    name: str
    layers: int
    kv_heads: int
    head_dim: int
    q_heads: int
    d_model: int
    block_tokens: int = 16
    elem_bytes: int = 2

    @property
    def kv_bytes_per_token(self) -> int:
        """The reference's `kv_bytes_per_token` (config.py:92) for this shape."""
        return self.layers * 2 * self.kv_heads * self.head_dim * self.elem_bytes

    @property
    def piece_bytes(self) -> int:
        return self.block_tokens * self.kv_heads * self.head_dim * self.elem_bytes

    @property
    def token_row_bytes(self) -> int:
        return self.kv_heads * self.head_dim * self.elem_bytes

    @property
    def kv_cols(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def q_cols(self) -> int:
        return self.q_heads * self.head_dim

    def blocks_for(self, tokens: int) -> int:
        return -(-tokens // self.block_tokens)

    def pool_bytes(self, num_blocks: int) -> int:
        return self.layers * 2 * num_blocks * self.piece_bytes

    def desc(self, num_blocks: int) -> _native.PoolDesc:
        return _native.PoolDesc(self.layers, self.kv_heads, self.head_dim, self.block_tokens,
                                num_blocks, self.elem_bytes)


LLAMA2_7B = ModelShape("llama2-7b", layers=32, kv_heads=32, head_dim=128, q_heads=32, d_model=4096)
LLAMA2_13B = ModelShape("llama2-13b", layers=40, kv_heads=40, head_dim=128, q_heads=40, d_model=5120)
LLAMA3_70B = ModelShape("llama3-70b-gqa", layers=80, kv_heads=8, head_dim=128, q_heads=64,
                        d_model=8192)
SHAPES = {s.name: s for s in (LLAMA2_7B, LLAMA2_13B, LLAMA3_70B)}


class BlockAllocator:
    """Free-block bookkeeping of one pool; `alloc(n)` returns the n lowest free
    ids in ascending order (the frozen, reproducible allocation order)."""

    def __init__(self, num_blocks: int):
        if num_blocks <= 0:
            raise ConfigError("num_blocks must be > 0")
        self.num_blocks = num_blocks
        self._free = np.ones(num_blocks, dtype=bool)
        self._n_free = num_blocks
        self._lo = 0    # every id below _lo is in use (lower bound of the lowest free id)

    @property
    def n_free(self) -> int:
        return self._n_free

    def alloc(self, n: int) -> np.ndarray:
        if n < 0:
            raise ValueError("n must be >= 0")
        if n == 0:
            return np.zeros(0, dtype=np.int32)
        if n == 1:   # decode growth: one block at a time (argmax finds the first free id in a window)
            i = self._lo
            while i < self.num_blocks:
                w = self._free[i:i + 512]
                j = int(w.argmax())
                if w[j]:
                    b = i + j
                    self._free[b] = False
                    self._n_free -= 1
                    self._lo = b + 1
                    return np.array([b], dtype=np.int32)
                i += len(w)
            raise RequestTooLarge(f"pool has {self.n_free} free blocks, 1 requested")
        parts, got, i = [], 0, self._lo
        while got < n and i < self.num_blocks:   # scan windows upward from the lowest possibly-free id
            w = self._free[i:i + max(1024, 2 * (n - got))]
            ids = np.flatnonzero(w)[:n - got] + i
            parts.append(ids)
            got += len(ids)
            i += len(w)
        if got < n:
            raise RequestTooLarge(f"pool has {self.n_free} free blocks, {n} requested")
        ids = np.concatenate(parts) if len(parts) > 1 else parts[0]
        self._free[ids] = False
        self._n_free -= len(ids)
        self._lo = int(ids[-1]) + 1
        return ids.astype(np.int32)

    def take(self, blocks: Iterable[int]) -> None:
        """Mark specific blocks used (pre-occupation / imported state)."""
        b = np.asarray(list(blocks) if not isinstance(blocks, np.ndarray) else blocks, dtype=np.int64)
        if b.size and (b.min() < 0 or b.max() >= self.num_blocks):
            raise ValueError("block id out of range")
        if not self._free[b].all():
            raise ValueError("block already in use")
        self._free[b] = False
        self._n_free -= int(np.unique(b).size) if b.size > 1 else int(b.size)

    def free(self, blocks: Iterable[int]) -> None:
        b = np.asarray(list(blocks) if not isinstance(blocks, np.ndarray) else blocks, dtype=np.int64)
        if b.size and (b.min() < 0 or b.max() >= self.num_blocks):
            raise ValueError("block id out of range")
        if self._free[b].any():
            raise ValueError("double free")
        self._free[b] = True
        self._n_free += int(np.unique(b).size) if b.size > 1 else int(b.size)
        if b.size:
            self._lo = min(self._lo, int(b.min()))

    def free_mask(self) -> np.ndarray:
        return self._free.copy()


class KVPool:
    """One GPU's paged KV cache, registered with libkvmig.

    `device` is the CUDA ordinal whose HBM backs the pool (for an IPC-imported
    peer pool: the local device that maps it).  The storage is a torch
    tensor owned by this object unless `tensor` is supplied by the caller.
    """

    def __init__(self, shape: ModelShape, num_blocks: int, device: int = 0, dtype=None,
                 tensor=None, *, allocator: bool = True, _base_ptr: Optional[int] = None):
        import torch

        self.shape = shape
        self.num_blocks = num_blocks
        self.device = device
        self.dtype = dtype or torch.float16
        self._mapped = None
        if _base_ptr is not None:
            self.tensor = None
            base = _base_ptr
        else:
            if tensor is None:
                tensor = torch.empty(self.view_shape, dtype=self.dtype, device=f"cuda:{device}")
            if tuple(tensor.shape) != self.view_shape or not tensor.is_contiguous():
                raise ConfigError(f"pool tensor must be contiguous {self.view_shape}")
            if tensor.element_size() != shape.elem_bytes:
                raise ConfigError("pool dtype size does not match shape.elem_bytes")
            self.tensor = tensor
            base = tensor.data_ptr()
        self.base_ptr = base
        self._desc = shape.desc(num_blocks)
        self.pool_id = _native.check(
            _native.lib().kvm_pool_register(device, ctypes.c_void_p(base), ctypes.byref(self._desc)),
            "kvm_pool_register")
        self.allocator = BlockAllocator(num_blocks) if allocator else None

    @property
    def view_shape(self):
        s = self.shape
        return (s.layers, 2, self.num_blocks, s.block_tokens, s.kv_heads, s.head_dim)

    @property
    def nbytes(self) -> int:
        return self.shape.pool_bytes(self.num_blocks)

    def close(self) -> None:
        if getattr(self, "pool_id", None) is not None and self.pool_id >= 0:
            _native.lib().kvm_pool_unregister(self.pool_id)
            self.pool_id = -1
        if self._mapped is not None:
            ptr, off = self._mapped
            _native.lib().kvm_ipc_close(ctypes.c_void_p(ptr), off)
            self._mapped = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library may already be gone
            pass

    # -- cross-process (one process per GPU) ---------------------------------
    def ipc_handle(self) -> tuple:
        """(64-byte handle, offset) a peer process can map with from_ipc()."""
        h = (ctypes.c_ubyte * 64)()
        off = ctypes.c_int64()
        _native.check(_native.lib().kvm_ipc_export(ctypes.c_void_p(self.base_ptr), h, ctypes.byref(off)),
                      "kvm_ipc_export")
        return bytes(h), off.value

    @classmethod
    def from_ipc(cls, shape: ModelShape, num_blocks: int, local_device: int, handle: bytes,
                 offset: int, dtype=None) -> "KVPool":
        """Map a peer process's pool; kernels launched on `local_device` then
        store into it over NVLink/NVSwitch."""
        if len(handle) != 64:
            raise ValueError("IPC handle must be 64 bytes")
        buf = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
        ptr = ctypes.c_void_p()
        _native.check(_native.lib().kvm_ipc_import(local_device, buf, offset, ctypes.byref(ptr)),
                      "kvm_ipc_import")
        pool = cls(shape, num_blocks, device=local_device, dtype=dtype, allocator=False,
                   _base_ptr=ptr.value)
        pool._mapped = (ptr.value, offset)
        return pool


class BlockTable:
    """Per-request block tables of one GPU: host mirror + device rows.

    The device tensor `rows[slot, :]` is what a paged-attention kernel on this
    GPU reads; the migration kernel rewrites a row in place (fused, after the
    KV bytes land) through `row_ptr(slot)`.  Unused entries are -1.
    """

    def __init__(self, max_requests: int, max_blocks: int, device: int = 0):
        import torch

        self.device = device
        self.max_blocks = max_blocks
        self._rows = torch.full((max_requests, max_blocks), -1, dtype=torch.int32,
                                device=f"cuda:{device}")
        self._slot_of: Dict[int, int] = {}
        self._free_slots = list(range(max_requests - 1, -1, -1))
        self._dirty: set = set()   # freed slots whose row still holds the old request's blocks
        self.host: Dict[int, np.ndarray] = {}
        # host-side row updates (admission, decode growth) awaiting one batched write
        self._staged: Dict[int, tuple] = {}    # slot -> (first entry to write, blocks)
        self._bufs: list = [None, None]        # pinned (index, value) staging, double-buffered
        self._buf_ev: list = [None, None]
        self._flip = 0

    @property
    def rows(self):
        """The device rows [max_requests][max_blocks].  Row updates staged by
        the host (stage()) are flushed first — one H2D copy + one scatter on
        the current stream for all of them — so every reader sees them."""
        if self._staged:
            self.flush()
        return self._rows

    def slot(self, rid: int) -> int:
        if rid not in self._slot_of:
            if not self._free_slots:
                raise ConfigError("block table full")
            s = self._free_slots.pop()
            if s in self._dirty:   # cleared on reuse, not on release (keeps drop() off the pause path)
                self._dirty.discard(s)
                self._rows[s].fill_(-1)
            self._slot_of[rid] = s
        return self._slot_of[rid]

    def stage(self, rid: int, blocks: np.ndarray, start: int = 0) -> None:
        """Host mirror := blocks; device entries [start, len(blocks)) are
        written at the next flush() (any read of `rows` / `row_ptr` flushes)."""
        if len(blocks) > self.max_blocks:
            raise RequestTooLarge(f"{len(blocks)} blocks > table width {self.max_blocks}")
        s = self.slot(rid)
        b = np.asarray(blocks, dtype=np.int32)
        self.host[rid] = b
        prev = self._staged.get(s)
        self._staged[s] = (min(start, prev[0]) if prev is not None else start, b)

    def flush(self) -> None:
        """Write every staged row update to the device: one pinned H2D copy of
        (flat index, block id) pairs and one index_copy_ into the rows, on the
        current stream."""
        import torch

        staged, self._staged = self._staged, {}
        parts = [(s, st, b) for s, (st, b) in staged.items() if st < len(b)]
        if not parts:
            return
        W = self.max_blocks
        idx = np.concatenate([s * W + np.arange(st, len(b), dtype=np.int64) for s, st, b in parts])
        val = np.concatenate([b[st:].astype(np.int64) for s, st, b in parts])
        n = len(idx)
        k = self._flip
        self._flip ^= 1
        buf = self._bufs[k]
        if buf is None or buf.shape[1] < n:
            buf = torch.empty((2, max(n, 1024, 0 if buf is None else 2 * buf.shape[1])), dtype=torch.int64,
                              pin_memory=True)
            self._bufs[k] = buf
        elif self._buf_ev[k] is not None:
            self._buf_ev[k].synchronize()   # the copy that last read this staging buffer is done
        bn = buf.numpy()
        bn[0, :n] = idx
        bn[1, :n] = val
        dev = buf[:, :n].to(self._rows.device, non_blocking=True)
        self._rows.view(-1).index_copy_(0, dev[0], dev[1].to(torch.int32))
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self._rows.device))
        self._buf_ev[k] = ev

    def has(self, rid: int) -> bool:
        return rid in self._slot_of

    @property
    def free_slots(self) -> int:
        return len(self._free_slots)

    def row_ptr(self, rid: int) -> int:
        return self.rows.data_ptr() + self.slot(rid) * self.max_blocks * 4   # (flushes staged updates)

    def set_host(self, rid: int, blocks: np.ndarray) -> None:
        if len(blocks) > self.max_blocks:
            raise RequestTooLarge(f"{len(blocks)} blocks > table width {self.max_blocks}")
        self.slot(rid)
        self.host[rid] = np.asarray(blocks, dtype=np.int32)

    def drop(self, rid: int) -> None:
        self.host.pop(rid, None)
        s = self._slot_of.pop(rid, None)
        if s is not None:   # nobody reads a released row; it is reset to -1 when the slot is reused
            self._staged.pop(s, None)
            self._dirty.add(s)
            self._free_slots.append(s)

    def blocks(self, rid: int) -> np.ndarray:
        try:
            return self.host[rid]
        except KeyError:
            raise NotPlaced(f"request {rid} has no block table on GPU {self.device}") from None


def blocks_for_bytes(kv_bytes: int, shape: ModelShape) -> int:
    """Blocks needed for `kv_bytes` of KV (kv_bytes is tokens * bpt exactly,
    sim.py:214-217, so this is ceil(tokens / block_tokens))."""
    tokens, rem = divmod(kv_bytes, shape.kv_bytes_per_token)
    if rem:
        raise ValueError("kv_bytes is not a whole number of tokens for this shape")
    return math.ceil(tokens / shape.block_tokens)
