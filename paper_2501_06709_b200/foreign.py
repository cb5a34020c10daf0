"""KV caches laid out by another engine, registered for kvm_migrate/kvm_compact.

The paper's prototype serves through vLLM, whose paged KV
cache is one tensor per layer.  `StridedKVPool` registers such caches as they
are (kvm_pool_register_strided: one base pointer per layer, a K|V stride and a
block stride), so a request can be migrated straight out of, or into, a vLLM
instance's cache — or between a vLLM cache and a native `KVPool` — without a
staging copy.  Pieces (16 tokens x kv_heads x head_dim of one layer, K or V) are
copied as opaque bytes, so any two layouts whose piece bytes are ordered the
same way interoperate; paged decode, re-prefill and fused split moves
address a strided pool in place too (pieces ordered [16][H][D], as in both
vLLM layouts).

Layouts (vLLM 0.22, `get_kv_cache_shape(num_blocks, block_size, kv_heads, head_size)`):
  "flash_attn"  [2][num_blocks][16][H][D] per layer  (FlashAttentionBackend)
  "flashinfer"  [num_blocks][2][16][H][D] per layer  (FlashInferBackend)
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

from . import _native
from .errors import ConfigError
from .kvcache import BlockAllocator, ModelShape

LAYOUTS = ("flash_attn", "flashinfer")


def vllm_cache_shape(layout: str, num_blocks: int, block_tokens: int, kv_heads: int, head_dim: int):
    """The per-layer tensor shape vLLM's backend allocates for `layout`."""
    if layout == "flash_attn":
        return (2, num_blocks, block_tokens, kv_heads, head_dim)
    if layout == "flashinfer":
        return (num_blocks, 2, block_tokens, kv_heads, head_dim)
    raise ConfigError(f"layout must be one of {LAYOUTS}")


class StridedKVPool:
    """A borrowed, per-layer paged KV cache (see module docstring).

    layer_tensors: one tensor per layer, all on `device`, same dtype; the piece
    of (layer l, kv, block b) starts at layer_tensors[l].data_ptr() +
    kv * kv_stride + b * block_stride (bytes).  The tensors must stay alive
    while the pool is registered.
    """

    def __init__(self, shape: ModelShape, num_blocks: int, layer_tensors: Optional[Sequence], kv_stride: int,
                 block_stride: int, *, allocator: bool = True, layout: str = "strided",
                 _layer_ptrs: Optional[Sequence[int]] = None, _device: int = 0, _dtype=None):
        self._mapped = []
        if layer_tensors is not None:
            if len(layer_tensors) != shape.layers:
                raise ConfigError(f"need {shape.layers} layer tensors, got {len(layer_tensors)}")
            t0 = layer_tensors[0]
            if any(t.device != t0.device or t.dtype != t0.dtype for t in layer_tensors):
                raise ConfigError("layer tensors must share device and dtype")
            if t0.element_size() != shape.elem_bytes:
                raise ConfigError("layer tensor dtype size does not match shape.elem_bytes")
            self.device, self.dtype = t0.device.index, t0.dtype
            self.layers = list(layer_tensors)
            self.layer_ptrs = [t.data_ptr() for t in layer_tensors]
        else:   # peer-mapped (from_ipc): raw pointers, no tensors
            self.device, self.dtype = _device, _dtype
            self.layers = None
            self.layer_ptrs = list(_layer_ptrs)
        self.shape = shape
        self.num_blocks = num_blocks
        self.layout = layout
        self.kv_stride, self.block_stride = kv_stride, block_stride
        self._desc = shape.desc(num_blocks)
        ptrs = (ctypes.c_void_p * shape.layers)(*self.layer_ptrs)
        self.pool_id = _native.check(
            _native.lib().kvm_pool_register_strided(self.device, ctypes.byref(self._desc), ptrs,
                                                    ctypes.c_int64(kv_stride), ctypes.c_int64(block_stride)),
            "kvm_pool_register_strided")
        self.allocator = BlockAllocator(num_blocks) if allocator else None

    @classmethod
    def from_vllm(cls, kv_caches: Sequence, layout: str = "flash_attn", *, name: str = "vllm",
                  q_heads: Optional[int] = None, allocator: bool = True) -> "StridedKVPool":
        """Wrap vLLM's per-layer caches (`kv_caches[l]` of vllm_cache_shape(layout, ...))."""
        t = kv_caches[0]
        if t.dim() != 5 or not t.is_contiguous():
            raise ConfigError("vLLM KV caches are contiguous 5-D tensors")
        if layout == "flash_attn":
            two, nb, bt, h, d = t.shape
        elif layout == "flashinfer":
            nb, two, bt, h, d = t.shape
        else:
            raise ConfigError(f"layout must be one of {LAYOUTS}")
        if two != 2:
            raise ConfigError(f"not a {layout} cache: K|V axis has size {two}")
        if any(tuple(c.shape) != tuple(t.shape) or not c.is_contiguous() for c in kv_caches):
            raise ConfigError("all layers must have the same contiguous shape")
        shape = ModelShape(name, layers=len(kv_caches), kv_heads=h, head_dim=d, q_heads=q_heads or h,
                           d_model=(q_heads or h) * d, block_tokens=bt, elem_bytes=t.element_size())
        piece = shape.piece_bytes
        kv_stride, block_stride = (nb * piece, piece) if layout == "flash_attn" else (piece, 2 * piece)
        return cls(shape, nb, kv_caches, kv_stride, block_stride, allocator=allocator, layout=layout)

    # -- cross-process (one process per GPU, e.g. one vLLM instance per GPU) ----
    def ipc_handles(self) -> list:
        """(64-byte handle, offset) per layer, for from_ipc() in a peer process."""
        out = []
        for ptr in self.layer_ptrs:
            h = (ctypes.c_ubyte * 64)()
            off = ctypes.c_int64()
            _native.check(_native.lib().kvm_ipc_export(ctypes.c_void_p(ptr), h, ctypes.byref(off)),
                          "kvm_ipc_export")
            out.append((bytes(h), off.value))
        return out

    @classmethod
    def from_ipc(cls, shape: ModelShape, num_blocks: int, local_device: int, handles: Sequence, kv_stride: int,
                 block_stride: int, dtype=None, layout: str = "strided") -> "StridedKVPool":
        """Map a peer process's strided cache (handles from ipc_handles()); each
        distinct allocation is mapped once (vLLM carves every layer out of one)."""
        import torch

        bases = {}
        for h, _ in handles:
            if h not in bases:
                ptr = ctypes.c_void_p()
                _native.check(_native.lib().kvm_ipc_import(local_device, (ctypes.c_ubyte * 64).from_buffer_copy(h),
                                                           0, ctypes.byref(ptr)), "kvm_ipc_import")
                bases[h] = ptr.value
        pool = cls(shape, num_blocks, None, kv_stride, block_stride, allocator=False, layout=layout,
                   _layer_ptrs=[bases[h] + off for h, off in handles], _device=local_device,
                   _dtype=dtype or torch.float16)
        pool._mapped = list(bases.values())
        return pool

    def piece(self, layer: int, kv: int, block: int):
        """View of one piece, [block_tokens][kv_heads][head_dim] (for tests and tools)."""
        if self.layers is None:
            raise ValueError("a peer-mapped pool has no local tensors")
        t = self.layers[layer]
        off = (kv * self.kv_stride + block * self.block_stride) // t.element_size()
        s = self.shape
        return t.view(-1)[off:off + s.block_tokens * s.kv_heads * s.head_dim].view(
            s.block_tokens, s.kv_heads, s.head_dim)

    def close(self) -> None:
        if getattr(self, "pool_id", None) is not None and self.pool_id >= 0:
            _native.lib().kvm_pool_unregister(self.pool_id)
            self.pool_id = -1
        for ptr in getattr(self, "_mapped", []):
            _native.lib().kvm_ipc_close(ctypes.c_void_p(ptr), 0)
        self._mapped = []

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library may already be gone
            pass
