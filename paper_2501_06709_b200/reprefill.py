"""Re-prefill (token_transfer) on the destination GPU, through kvm_reprefill.

The reference prices a token_transfer as `tokens / prefill_tokens_per_s`
(migration.py:159-163) and computes nothing.  Here the dense core of that
recompute — each layer's QKV projection of the tokens' hidden states — runs
on tcgen05 tensor cores and its epilogue writes K/V straight into the
destination pool blocks (csrc/reprefill.cu).

Proxy, stated: true recompute of layer l needs layer l-1's
hidden states (attention over the prefix); the proxy feeds the same X to every
layer, and K is stored pre-RoPE.  The FLOPs, bytes and the pool writes are
those of the real projection: 2 * s * d_model * (q_cols + 2 * kv_cols) per layer.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _native
from .errors import ConfigError
from .kvcache import KVPool, ModelShape


def synthetic_weights(shape: ModelShape, device: int, with_q: bool = True, seed: int = 3):
    """W[l] ~ N(0, d_model^-1/2), bf16, layout [layers][n_out][d_model] (nn.Linear)."""
    import torch

    n_out = (shape.q_cols if with_q else 0) + 2 * shape.kv_cols
    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed)
    w = torch.empty(shape.layers, n_out, shape.d_model, dtype=torch.bfloat16, device=f"cuda:{device}")
    for l in range(shape.layers):  # per layer keeps the fp32 temporary small
        w[l] = (torch.randn(n_out, shape.d_model, generator=g, device=w.device) *
                shape.d_model ** -0.5).to(torch.bfloat16)
    return w


def synthetic_hidden(shape: ModelShape, rows: int, device: int, seed: int = 2):
    """X ~ N(0, 1), bf16 [rows][d_model]."""
    import torch

    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed)
    return torch.randn(rows, shape.d_model, generator=g, device=f"cuda:{device}").to(torch.bfloat16)


def reprefill(pool: KVPool, x, w, dst_blocks, tok0: int = 0, q_out=None, stream=None,
              done_flag: int = 0, done_value: int = 1, single_cta: bool = False,
              rope_theta: Optional[float] = None, max_sms: int = 0) -> None:
    """Launch kvm_reprefill: K/V of tokens [tok0, tok0 + rows) into `dst_blocks`.

    x: bf16 [rows][d_model] (device) fed to every layer, or [layers][rows][d_model]
    per-layer hidden states (KVM_REPREFILL_X_PER_LAYER), w: bf16 [layers][n_out][d_model] with
    n_out = q_cols + 2 * kv_cols, dst_blocks: int32 device tensor covering the
    token range, q_out: optional bf16 [layers][rows][q_cols].  single_cta
    selects the single-CTA kernel instead of the default CTA-pair one.
    rope_theta: apply rotary position embedding (HF rotate_half, positions
    tok0 + t) to Q and K in the epilogue, so the pool holds post-RoPE K as a
    Llama KV cache does (head_dim 128).  max_sms > 0: run on at most that many
    SMs (KVM_REPREFILL_MAX_SMS), leaving the rest of the GPU to decode.
    """
    import torch

    shape = pool.shape
    if not 0 <= max_sms <= 255:
        raise ValueError("max_sms must be in [0, 255] (0 = every SM)")
    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise ConfigError("re-prefill operands must be bf16")
    if pool.dtype != torch.bfloat16:
        raise ConfigError("re-prefill writes bf16 K/V: pool dtype must be bfloat16")
    if not (x.is_contiguous() and w.is_contiguous()):
        raise ValueError("x and w must be contiguous")
    per_layer = x.dim() == 3
    if per_layer and x.shape[0] != shape.layers:
        raise ConfigError(f"per-layer x must be [layers={shape.layers}][rows][d_model]")
    rows, d_model = x.shape[-2:]
    if w.shape[0] != shape.layers or w.shape[2] != d_model:
        raise ConfigError(f"w must be [layers={shape.layers}][n_out][d_model={d_model}]")
    q_cols = w.shape[1] - 2 * shape.kv_cols
    if q_cols < 0:
        raise ConfigError("w has fewer than 2 * kv_cols output rows")
    if q_out is not None and tuple(q_out.shape) != (shape.layers, rows, q_cols):
        raise ConfigError("q_out must be [layers][rows][q_cols]")
    if dst_blocks.dtype != torch.int32 or not dst_blocks.is_cuda:
        raise ValueError("dst_blocks must be an int32 CUDA tensor")
    a = _native.ReprefillArgs()
    a.dst_pool, a.rows, a.d_model, a.q_cols = pool.pool_id, rows, d_model, q_cols
    a.tok0, a.n_dst_blocks = tok0, dst_blocks.numel()
    a.x, a.w = x.data_ptr(), w.data_ptr()
    a.q_out = q_out.data_ptr() if q_out is not None else None
    a.dst_blocks = dst_blocks.data_ptr()
    a.done_flag, a.done_value = done_flag or None, done_value
    a.flags = (_native.KVM_REPREFILL_SINGLE_CTA if single_cta else 0) | (
        _native.KVM_REPREFILL_ROPE if rope_theta else 0) | (_native.KVM_REPREFILL_X_PER_LAYER if per_layer else 0) | \
        _native.KVM_REPREFILL_MAX_SMS(max_sms)
    a.rope_theta = float(rope_theta or 0.0)
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    _native.check(_native.lib().kvm_reprefill(ctypes.byref(a), ctypes.c_void_p(s.cuda_stream)),
                  "kvm_reprefill")


class ReprefillEngine:
    """Executor plug-in for token_transfer moves: recompute a request's KV on
    the destination from its (synthetic, seeded) hidden states.  One set of
    synthetic weights per (device, model shape).

    max_sms: the destination's compute budget as an SM share (0 = every SM):
    each re-prefill runs on at most that many SMs, so decode steps of the
    destination's resident requests keep the others (see
    tools/bench_interference.py)."""

    def __init__(self, shapes, devices, with_q: bool = False, seed: int = 3, rope_theta: Optional[float] = None,
                 max_sms: int = 0):
        shapes = [shapes] if isinstance(shapes, ModelShape) else list(shapes)
        self.shapes = {s.name: s for s in shapes}
        self.with_q = with_q
        self.rope_theta = rope_theta   # post-RoPE K in the pool (KVM_REPREFILL_ROPE)
        self.max_sms = max_sms
        self.weights = {(d, s.name): synthetic_weights(s, d, with_q=with_q, seed=seed)
                        for d in set(devices) for s in shapes}

    def validate(self, pool: KVPool) -> None:
        """Raise before anything is reserved or launched if this engine cannot
        write into `pool` (the executor calls it in its validation phase)."""
        import torch

        if pool.dtype != torch.bfloat16:
            raise ConfigError("re-prefill writes bf16 K/V: pool dtype must be bfloat16")
        if pool.shape.name not in self.shapes:
            raise ConfigError(f"re-prefill engine has no weights for model {pool.shape.name!r}")

    def hidden(self, shape: ModelShape, rid: int, tokens: int, device: int):
        return synthetic_hidden(shape, tokens, device, seed=10_000 + rid)

    def __call__(self, executor, rid: int, dst_gpu: int, dst_blocks: np.ndarray, tokens: int, stream):
        import torch

        pool = executor.pool(dst_gpu, executor.loc[rid].model)
        dev = pool.device
        with torch.cuda.stream(stream):
            x = self.hidden(pool.shape, rid, tokens, dev)
            blocks = torch.from_numpy(np.ascontiguousarray(dst_blocks, dtype=np.int32)).to(f"cuda:{dev}",
                                                                                          non_blocking=False)
            reprefill(pool, x, self.weights[(dev, pool.shape.name)], blocks, tok0=0, stream=stream,
                      rope_theta=self.rope_theta, max_sms=self.max_sms)
            # keep the temporaries alive until the stream has consumed them
            x.record_stream(stream)
            blocks.record_stream(stream)


def sm_budget(fraction: float, sm_count: int) -> int:
    """The destination's compute budget as an SM share: the reference gives
    re-prefill `budget_fraction` of the destination's prefill capacity per
    epoch (Boundaries.comp_budget = prefill rate x epoch x fraction,
    migration.py:77-91); a re-prefill confined to that fraction of the SMs
    (KVM_REPREFILL_MAX_SMS) runs at about that fraction of the full rate while
    decode keeps the rest of the GPU.  Returns the cap for
    ReprefillEngine(max_sms=...) (0 = every SM, for fraction >= 1), at least 2
    (one CTA pair)."""
    if not fraction > 0:
        raise ValueError("fraction must be > 0")
    if fraction >= 1:
        return 0
    return max(2, min(255, int(round(fraction * sm_count))))


def split_point(tokens: int, bytes_per_token: int, link_bytes_per_s: float,
                flops_per_token: float, tensor_flops_per_s: float, block_tokens: int = 16) -> int:
    """Extension of the binary kv/token choice (migration.py:155-169): transfer
    the first n - s tokens, re-prefill the last s, minimising
    max((n - s) * bpt / BW, s * flops_per_token / F) with the reference's own
    linear cost terms.  s is rounded to whole blocks so the transferred prefix
    is block-aligned (the suffix may end mid-block)."""
    if tokens <= 0:
        return 0
    t_xfer = bytes_per_token / link_bytes_per_s
    t_comp = flops_per_token / tensor_flops_per_s
    s = tokens * t_xfer / (t_xfer + t_comp)
    prefix = tokens - s
    prefix_blocks = int(round(prefix / block_tokens))
    prefix_tok = min(tokens, max(0, prefix_blocks * block_tokens))
    return tokens - prefix_tok


def reprefill_flops(shape: ModelShape, rows: int, with_q: bool = True) -> int:
    n_out = (shape.q_cols if with_q else 0) + 2 * shape.kv_cols
    return 2 * rows * shape.d_model * n_out * shape.layers
