"""Paged-attention decode (the consumer of a migrated cache, §8f row 3):
matches an fp32 torch reference within fp16/bf16 tolerance, and decoding on
the destination after a migration is bit-identical to decoding on the source
before it."""
import ctypes

import pytest
import torch

from paper_2501_06709_b200 import _native
from oracle.attention_ref import reference_decode
from paper_2501_06709_b200.attention import paged_decode
from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape

pytestmark = pytest.mark.gpu


def _fill_normal(pool, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    pool.tensor.copy_(torch.randn(pool.view_shape, generator=g, device="cuda").to(pool.dtype))


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("kv_heads,q_heads,seqs", [(4, 4, [1, 17, 300]), (2, 4, [256, 5]), (2, 16, [700]),
                                                   (1, 8, [4096, 1, 33]), (4, 12, [15, 16, 17, 500]),
                                                   (2, 8, [0, 40, 0])])
def test_decode_matches_reference(dtype, kv_heads, q_heads, seqs):
    shape = ModelShape("dec", layers=2, kv_heads=kv_heads, head_dim=128, q_heads=q_heads, d_model=256)
    nb = sum((s + 15) // 16 for s in seqs) + 8
    pool = KVPool(shape, nb, dtype=dtype)
    _fill_normal(pool, 1)
    maxb = max((s + 15) // 16 for s in seqs)
    perm = torch.randperm(nb, generator=torch.Generator().manual_seed(2))
    tables = torch.full((len(seqs), maxb), -1, dtype=torch.int32)
    off = 0
    for b, s in enumerate(seqs):
        k = (s + 15) // 16
        tables[b, :k] = perm[off:off + k].to(torch.int32)
        off += k
    tables = tables.cuda()
    lens = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    q = torch.randn(2, len(seqs), q_heads, 128, device="cuda").to(dtype)
    out = paged_decode(pool, q, tables, lens)
    ref = reference_decode(pool, q, tables, lens)
    ref[:, lens.cpu() == 0] = 0.0  # an empty request attends to nothing: defined as 0
    torch.testing.assert_close(out.float(), ref, atol=2e-2, rtol=2e-2)
    if q_heads // kv_heads in (1, 2, 4, 8):  # tensor-core (default) and CUDA-core paths both match
        out_cc = paged_decode(pool, q, tables, lens, cuda_cores=True)
        torch.testing.assert_close(out_cc.float(), ref, atol=2e-2, rtol=2e-2)


def test_decode_after_migration_is_bit_identical():
    shape = ModelShape("dec", layers=3, kv_heads=8, head_dim=128, q_heads=8, d_model=256)
    nb = 96
    src, dst = KVPool(shape, nb), KVPool(shape, nb)
    _fill_normal(src, 3)
    _fill_normal(dst, 4)
    seq = 700
    n = (seq + 15) // 16
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(5))[:n].to(torch.int32).numpy()
    db = dst.allocator.alloc(n)
    table = BlockTable(2, n)
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, 1
    m.src_blocks, m.dst_blocks, m.dst_table_row = sb.ctypes.data, db.ctypes.data, table.row_ptr(0)
    _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    q = torch.randn(3, 1, 8, 128, device="cuda").half()
    lens = torch.tensor([seq], dtype=torch.int32, device="cuda")
    before = paged_decode(src, q, torch.from_numpy(sb)[None].cuda(), lens)
    after = paged_decode(dst, q, table.rows[table.slot(0)][None].contiguous(), lens)   # the rewritten row
    torch.cuda.synchronize()
    assert torch.equal(before.view(torch.int16), after.view(torch.int16))


def test_decode_concurrent_streams_have_private_workspaces():
    """Split-K decode on several streams of one GPU at once (each call's
    partials in its own per-stream workspace): every stream's outputs equal the
    same calls run one at a time, bit for bit."""
    shape = ModelShape("dws", layers=4, kv_heads=2, head_dim=128, q_heads=8, d_model=256)
    seq = 6000   # long enough for many splits
    nb = 4 * ((seq + 15) // 16) + 8
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    _fill_normal(pool, 5)
    maxb = (seq + 15) // 16
    perm = torch.randperm(nb, generator=torch.Generator().manual_seed(6))[:4 * maxb].to(torch.int32)
    tables = perm.view(4, maxb).contiguous().cuda()
    lens = torch.tensor([seq, seq - 100, 4000, seq], dtype=torch.int32, device="cuda")
    qs = [torch.randn(4, 4, 8, 128, generator=torch.Generator(device="cuda").manual_seed(10 + i),
                      device="cuda").to(torch.bfloat16) for i in range(4)]
    expect = [paged_decode(pool, q, tables, lens, max_seq_len=seq) for q in qs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in qs]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    outs = [torch.empty_like(q) for q in qs]
    for rep in range(20):
        for s, q, o in zip(streams, qs, outs):
            paged_decode(pool, q, tables, lens, out=o, max_seq_len=seq, stream=s)
    for s in streams:
        s.synchronize()
    for o, e in zip(outs, expect):
        assert torch.equal(o.view(torch.int16), e.view(torch.int16))


def _wait_setup(layers=4, seq=3000, seed=21):
    shape = ModelShape("dw", layers=layers, kv_heads=2, head_dim=128, q_heads=8, d_model=1024)
    k = (seq + 15) // 16
    nb = 2 * k + 8
    src, dst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    _fill_normal(src, seed)
    dst.tensor.zero_()
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(seed))[:k].to(torch.int32)
    db = torch.randperm(nb, generator=torch.Generator().manual_seed(seed + 1))[:k].to(torch.int32)
    q = torch.randn(layers, 1, 8, 128, generator=torch.Generator(device="cuda").manual_seed(seed),
                    device="cuda").to(torch.bfloat16)
    lens = torch.tensor([seq], dtype=torch.int32, device="cuda")
    return shape, src, dst, sb, db, q, lens


def test_decode_waits_on_layer_flags_written_by_the_host():
    """KVM_DECODE_WAIT_LAYERS with flags in pinned host memory, released by the
    host one layer at a time after the kernel is queued: the decode waits, then
    equals an unconditional decode bit for bit; no timeout fired."""
    import threading
    import time

    shape, src, dst, sb, db, q, lens = _wait_setup()
    ref = paged_decode(src, q, sb[None].contiguous().cuda(), lens)
    flags = torch.zeros(shape.layers, dtype=torch.int32).pin_memory()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()

    def release():
        for l in range(shape.layers):
            time.sleep(0.005)
            flags[l] = 7
    th = threading.Thread(target=release)
    t0 = time.perf_counter()
    out = paged_decode(src, q, sb[None].contiguous().cuda(), lens, stream=s, layer_flags=flags, layer_value=7,
                       timeout_ns=10_000_000_000, err_word=err)
    th.start()
    s.synchronize()
    waited = time.perf_counter() - t0
    th.join()
    assert err.item() == 0
    assert waited >= 0.015   # the kernel could not finish before the last layer was released
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def test_decode_layer_wait_times_out_instead_of_hanging():
    shape, src, dst, sb, db, q, lens = _wait_setup(layers=2, seq=200)
    flags = torch.zeros(shape.layers, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    paged_decode(src, q, sb[None].contiguous().cuda(), lens, layer_flags=flags, timeout_ns=2_000_000, err_word=err)
    torch.cuda.synchronize()
    assert err.item() == 1
    # a bounded wait whose expiry nobody could observe is refused up front
    with pytest.raises(ValueError):
        paged_decode(src, q, sb[None].contiguous().cuda(), lens, layer_flags=flags, timeout_ns=2_000_000)


def test_decode_pipelined_behind_an_incoming_migration():
    """Layer-wise pipelining on one GPU: kvm_migrate (per-layer flags) on one
    stream, the destination decode (waiting on those flags, destination block
    table known up front) on another; the result equals decoding the source."""
    import ctypes

    from paper_2501_06709_b200 import _native

    shape, src, dst, sb, db, q, lens = _wait_setup(layers=8, seq=6000, seed=33)
    ref = paged_decode(src, q, sb[None].contiguous().cuda(), lens)
    flags = torch.zeros(shape.layers, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    copy_s, dec_s = torch.cuda.Stream(), torch.cuda.Stream()
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, len(sb), 1
    sbn, dbn = sb.numpy(), db.numpy()
    m.src_blocks, m.dst_blocks, m.layer_flags = sbn.ctypes.data, dbn.ctypes.data, flags.data_ptr()
    _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                            ctypes.c_void_p(copy_s.cuda_stream)))
    out = paged_decode(dst, q, db[None].contiguous().cuda(), lens, stream=dec_s, layer_flags=flags, layer_value=1,
                       timeout_ns=5_000_000_000, err_word=err)
    torch.cuda.synchronize()
    assert err.item() == 0
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVM_FUZZ_SEEDS", "100"))))
def test_decode_randomized(seed):
    """Random GQA ratio (1..8 query heads per kv head), batch, ragged lengths
    (incl. empty requests), layer window, dtype and block scatter: within the
    stated tolerance of the fp32 reference (tensor-core path; CUDA cores too
    when the ratio is a power of two)."""
    import numpy as np

    rng = np.random.default_rng(9000 + seed)
    kv_heads = int(rng.integers(1, 5))
    G = int(rng.integers(1, 9))
    layers = int(rng.integers(1, 4))
    dtype = torch.float16 if rng.integers(2) else torch.bfloat16
    batch = int(rng.integers(1, 5))
    seqs = [int(rng.choice([0, 1, 15, 16, 17])) if rng.random() < 0.3 else int(rng.integers(1, 3000))
            for _ in range(batch)]
    if max(seqs) == 0:
        seqs[0] = 5
    shape = ModelShape(f"dz{seed}", layers=layers, kv_heads=kv_heads, head_dim=128, q_heads=kv_heads * G,
                       d_model=128 * kv_heads * G)
    maxb = max((s + 15) // 16 for s in seqs)
    nb = sum((s + 15) // 16 for s in seqs) + int(rng.integers(1, 6))
    pool = KVPool(shape, nb, dtype=dtype)
    _fill_normal(pool, seed)
    perm = rng.permutation(nb)
    tables = torch.full((batch, maxb), -1, dtype=torch.int32)
    off = 0
    for b, s in enumerate(seqs):
        k = (s + 15) // 16
        tables[b, :k] = torch.from_numpy(perm[off:off + k].astype(np.int32))
        off += k
    tables = tables.cuda()
    lens = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    l0 = int(rng.integers(0, layers))
    nl = int(rng.integers(1, layers - l0 + 1))
    q = torch.randn(nl, batch, kv_heads * G, 128, generator=torch.Generator(device="cuda").manual_seed(seed),
                    device="cuda").to(dtype)
    out = paged_decode(pool, q, tables, lens, layer0=l0, n_layers=nl)
    ref = reference_decode(pool, q, tables, lens, layer0=l0)
    ref[:, lens.cpu() == 0] = 0.0
    torch.testing.assert_close(out.float(), ref, atol=2e-2, rtol=2e-2)
    if G in (1, 2, 4, 8):
        out_cc = paged_decode(pool, q, tables, lens, layer0=l0, n_layers=nl, cuda_cores=True)
        torch.testing.assert_close(out_cc.float(), ref, atol=2e-2, rtol=2e-2)
