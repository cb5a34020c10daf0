"""GPU: argument validation of the C ABI maps onto the reference's exception
classes, and nothing is launched for rejected calls."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2501_06709_b200 import ConfigError, KvmUnsupported, NotPlaced, _native
from paper_2501_06709_b200.attention import paged_decode
from paper_2501_06709_b200.kvcache import KVPool, ModelShape
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights

pytestmark = pytest.mark.gpu
S = ModelShape("e", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=128)


def test_reprefill_argument_errors():
    pool = KVPool(S, 8, dtype=torch.bfloat16)
    x = synthetic_hidden(S, 20, 0)
    w = synthetic_weights(S, 0)
    blocks = torch.arange(2, dtype=torch.int32, device="cuda")
    n0 = _native.launch_count()
    with pytest.raises(ValueError):          # 2 blocks do not cover tokens [30, 50)
        reprefill(pool, x, w, blocks, tok0=30)
    with pytest.raises(ConfigError):         # fp16 pool
        reprefill(KVPool(S, 8), x, w, blocks)
    odd = ModelShape("odd", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=96)
    with pytest.raises(ConfigError):         # d_model not a multiple of 64
        reprefill(KVPool(odd, 8, dtype=torch.bfloat16), synthetic_hidden(odd, 20, 0), synthetic_weights(odd, 0), blocks)
    with pytest.raises(ConfigError):         # w has the wrong layer count
        reprefill(pool, x, w[:1].contiguous(), blocks)
    assert _native.launch_count() == n0
    reprefill(pool, x[:0].contiguous(), w, blocks)   # zero rows: no-op
    assert _native.launch_count() == n0


def test_decode_argument_errors():
    pool = KVPool(S, 8)                     # head_dim 64: unsupported by the decode kernel
    q = torch.zeros(1, 1, 2, 64, dtype=torch.float16, device="cuda")
    t = torch.zeros(1, 1, dtype=torch.int32, device="cuda")
    lens = torch.ones(1, dtype=torch.int32, device="cuda")
    with pytest.raises((KvmUnsupported, ConfigError)):
        paged_decode(pool, q, t, lens)
    s128 = ModelShape("d", layers=2, kv_heads=2, head_dim=128, q_heads=2, d_model=128)
    p128 = KVPool(s128, 8)
    q = torch.zeros(1, 1, 2, 128, dtype=torch.float16, device="cuda")
    with pytest.raises(ValueError):         # max_seq_len beyond the table width
        paged_decode(p128, q, t, lens, max_seq_len=17)
    with pytest.raises(ValueError):         # layer range out of the pool
        paged_decode(p128, torch.zeros(3, 1, 2, 128, dtype=torch.float16, device="cuda"), t, lens)


def test_migrate_flag_and_pool_errors():
    pool = KVPool(S, 8)
    sb = np.array([0], dtype=np.int32)
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks = pool.pool_id, pool.pool_id, 1
    m.src_blocks, m.dst_blocks = sb.ctypes.data, sb.ctypes.data
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    with pytest.raises(ValueError):         # unknown flag bit
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, 0x80, stream))
    pool.close()
    with pytest.raises(NotPlaced):          # unregistered pool
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST, stream))
