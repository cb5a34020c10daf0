"""Adaptive split migration (BASELINE configs[2]; extension of the reference).

The reference decides per move, all or nothing: KV transfer if the link budget
fits, else re-prefill if the destination's compute budget fits
(migration.py:155-169).  A split move does both at once: the first n - s
tokens' blocks travel over the link (K1, launched on the source GPU) while the
destination re-prefills the last s tokens (K3, launched on the destination
GPU), with s from `reprefill.split_point` so the two finish together.

Completion is tracked with two flag words on the destination (one per part),
so the destination stream can wait for both without a host round trip.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigError
from .kvcache import KVPool
from .reprefill import reprefill


@dataclass
class SplitPlan:
    tokens: int          # n
    suffix: int          # s (re-prefilled)
    prefix_blocks: int   # blocks transferred
    total_blocks: int

    @property
    def prefix_tokens(self) -> int:
        return self.tokens - self.suffix


def make_split(tokens: int, suffix: int, block_tokens: int = 16) -> SplitPlan:
    if not 0 <= suffix <= tokens:
        raise ValueError("suffix must be in [0, tokens]")
    if (tokens - suffix) % block_tokens:
        raise ValueError("the transferred prefix must be whole blocks")
    return SplitPlan(tokens, suffix, (tokens - suffix) // block_tokens, -(-tokens // block_tokens))


def split_migrate(src: KVPool, dst: KVPool, src_blocks: np.ndarray, dst_blocks, plan: SplitPlan,
                  x_suffix, w, *, xfer_stream, rp_stream, flags_dev, seq: int = 1,
                  table_row: int = 0, engine_flags: int = _native.KVM_F_ENGINE_BULK,
                  rp_first: bool = True) -> None:
    """Launch both halves of a split move; returns immediately.

    src_blocks: host int32 [total_blocks] (source block table of the request);
    dst_blocks: device int32 tensor [total_blocks] on dst's device (already
    allocated); x_suffix: bf16 [s][d_model] hidden states of the suffix tokens;
    w: bf16 [layers][n_out][d_model] on dst's device; flags_dev: int32 device
    tensor with >= 2 words on dst's device: word 0 <- seq when the prefix has
    landed, word 1 <- seq when the suffix is recomputed.
    rp_first launches the persistent GEMM first so that, when both halves share
    one GPU, the copy (capped CTAs/SM) fills the SM slots the GEMM leaves.
    """
    if src.shape != dst.shape:
        raise ConfigError("split migration needs identical KV shapes")
    sb = np.ascontiguousarray(src_blocks[:plan.prefix_blocks], dtype=np.int32)
    db_host = dst_blocks[:plan.prefix_blocks].cpu().numpy().astype(np.int32) if plan.prefix_blocks else sb

    def launch_xfer():
        if plan.prefix_blocks == 0:
            return
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, plan.prefix_blocks, seq
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db_host.ctypes.data
        m.dst_table_row = table_row or None
        m.done_flag = flags_dev.data_ptr()
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | engine_flags,
                                                ctypes.c_void_p(xfer_stream.cuda_stream)), "kvm_migrate")

    def launch_rp():
        if plan.suffix == 0:
            return
        reprefill(dst, x_suffix, w, dst_blocks, tok0=plan.prefix_tokens, stream=rp_stream,
                  done_flag=flags_dev.data_ptr() + 4, done_value=seq)

    if rp_first:
        launch_rp()
        launch_xfer()
    else:
        launch_xfer()
        launch_rp()


def wait_split(flags_dev, plan: SplitPlan, seq: int, stream) -> None:
    """Make `stream` (on the destination) wait for both halves."""
    lib = _native.lib()
    if plan.prefix_blocks:
        _native.check(lib.kvm_wait_flag(ctypes.c_void_p(flags_dev.data_ptr()), seq,
                                        ctypes.c_void_p(stream.cuda_stream)))
    if plan.suffix:
        _native.check(lib.kvm_wait_flag(ctypes.c_void_p(flags_dev.data_ptr() + 4), seq,
                                        ctypes.c_void_p(stream.cuda_stream)))


def flops_per_token(shape, with_q: bool = True) -> int:
    n_out = (shape.q_cols if with_q else 0) + 2 * shape.kv_cols
    return 2 * shape.d_model * n_out * shape.layers


def split_migrate_fused(src: KVPool, dst: KVPool, src_blocks_dev, dst_blocks_dev, plan: SplitPlan, x_suffix, w,
                        *, stream=None, table_row: int = 0, done_flag: int = 0, done_value: int = 1,
                        single_cta: bool = False, rope_theta: float = 0.0, max_sms: int = 0) -> None:
    """One-launch split migration on the destination (kvm_split_migrate): warps
    idle in the re-prefill GEMM copy the prefix while the tensor cores
    recompute the suffix.  src must be registered on dst's device (same GPU, or
    an IPC-imported peer pool: the prefix is then pulled over NVLink).
    max_sms > 0: at most that many SMs (KVM_REPREFILL_MAX_SMS)."""
    import torch

    per_layer = x_suffix is not None and x_suffix.dim() == 3   # [layers][suffix][d_model]
    if plan.suffix and (x_suffix is None or x_suffix.shape[-2] != plan.suffix
                        or (per_layer and x_suffix.shape[0] != dst.shape.layers)):
        raise ValueError("x_suffix must be [suffix][d_model] or [layers][suffix][d_model]")
    q_cols = w.shape[1] - 2 * dst.shape.kv_cols
    a = _native.SplitArgs()
    a.src_pool, a.dst_pool, a.tokens, a.prefix_blocks = src.pool_id, dst.pool_id, plan.tokens, plan.prefix_blocks
    a.d_model, a.q_cols = w.shape[2], q_cols
    a.src_blocks, a.dst_blocks = src_blocks_dev.data_ptr(), dst_blocks_dev.data_ptr()
    a.x = x_suffix.data_ptr() if plan.suffix else None
    a.w = w.data_ptr()
    a.q_out = None
    a.dst_table_row, a.done_flag, a.done_value = table_row or None, done_flag or None, done_value
    a.flags = (_native.KVM_REPREFILL_SINGLE_CTA if single_cta else 0) | (   # GEMM engine (default: CTA pair)
        _native.KVM_REPREFILL_ROPE if rope_theta else 0) | (_native.KVM_REPREFILL_X_PER_LAYER if per_layer else 0) | \
        _native.KVM_REPREFILL_MAX_SMS(max_sms)
    a.rope_theta = float(rope_theta or 0.0)
    s = stream if stream is not None else torch.cuda.current_stream(dst.device)
    _native.check(_native.lib().kvm_split_migrate(ctypes.byref(a), ctypes.c_void_p(s.cuda_stream)),
                  "kvm_split_migrate")
