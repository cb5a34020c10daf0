"""Paged-attention decode over a KV pool (csrc/attention.cu, kvm_paged_decode).

The consumer of a migrated cache: run on the destination with the block-table
row the migration kernel rewrote, it must produce exactly what the source
produced before the move.
"""
from __future__ import annotations

import ctypes
import math

from . import _native
from .errors import ConfigError
from .kvcache import KVPool


def paged_decode(pool: KVPool, q, block_tables, seq_lens, out=None, *, layer0: int = 0,
                 n_layers: int = None, max_seq_len: int = None, scale: float = None, stream=None,
                 cuda_cores: bool = False, layer_flags=None, layer_value: int = 1, timeout_ns: int = 0,
                 err_word=None):
    """q: [n_layers][batch][q_heads][128] in the pool dtype; block_tables:
    int32 [batch][max_blocks] (device); seq_lens: int32 [batch] (device).
    Runs on tensor cores (mma.sync, cp.async-staged tiles) for up to 8 query
    heads per kv head, unless cuda_cores=True.  Returns out (same shape as q).

    layer_flags: int32 tensor [layers] (device or pinned host) -- the per-layer
    flags an incoming kvm_migrate publishes: layer l is decoded as soon as
    layer_flags[l] >= layer_value (KVM_DECODE_WAIT_LAYERS), overlapping the
    copy of later layers.  block_tables must already name the destination
    blocks.  timeout_ns bounds the wait (err_word: int32 tensor set to 1)."""
    import torch

    n_layers = n_layers if n_layers is not None else q.shape[0]
    if q.dim() != 4 or q.shape[0] != n_layers or q.shape[3] != pool.shape.head_dim:
        raise ConfigError("q must be [n_layers][batch][q_heads][head_dim]")
    if q.dtype != pool.dtype:
        raise ConfigError("q must have the pool's dtype")
    if block_tables.dtype != torch.int32 or seq_lens.dtype != torch.int32:
        raise ValueError("block_tables and seq_lens must be int32")
    if not (q.is_contiguous() and block_tables.is_contiguous()):
        raise ValueError("q and block_tables must be contiguous")
    batch, q_heads = q.shape[1], q.shape[2]
    if out is None:
        out = torch.empty_like(q)
    if max_seq_len is None:
        max_seq_len = int(seq_lens.max().item())
    a = _native.DecodeArgs()
    a.pool, a.layer0, a.n_layers, a.batch, a.q_heads = pool.pool_id, layer0, n_layers, batch, q_heads
    a.max_blocks, a.max_seq_len = block_tables.shape[1], max(1, max_seq_len)
    a.flags = (_native.KVM_DECODE_BF16 if pool.dtype == torch.bfloat16 else 0) | (
        _native.KVM_DECODE_CUDA_CORES if cuda_cores else 0) | (
        _native.KVM_DECODE_WAIT_LAYERS if layer_flags is not None else 0)
    if layer_flags is not None:
        a.layer_flags = layer_flags if isinstance(layer_flags, int) else layer_flags.data_ptr()
        a.layer_value, a.timeout_ns = layer_value, timeout_ns
        a.err_word = None if err_word is None else (err_word if isinstance(err_word, int) else err_word.data_ptr())
    a.scale = scale if scale is not None else 1.0 / math.sqrt(pool.shape.head_dim)
    a.q, a.block_tables, a.seq_lens, a.out = q.data_ptr(), block_tables.data_ptr(), seq_lens.data_ptr(), out.data_ptr()
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    _native.check(_native.lib().kvm_paged_decode(ctypes.byref(a), ctypes.c_void_p(s.cuda_stream)),
                  "kvm_paged_decode")
    return out
