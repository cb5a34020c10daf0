"""Strided (foreign-layout) pools: vLLM per-layer KV caches registered as they
are and migrated to/from native pools and each other (kvm_pool_register_strided).

Copy is identity, so the oracle is the piece-for-piece equality of the int16
views: every destination piece (l, kv, dst_blocks[i]) equals the source piece
(l, kv, src_blocks[i]), the destination table row lists dst_blocks, and no
other destination byte changes.
"""
import ctypes

import numpy as np
import pytest
import torch

from paper_2501_06709_b200 import _native
from paper_2501_06709_b200.foreign import StridedKVPool, vllm_cache_shape
from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape

pytestmark = pytest.mark.gpu
SHAPE = ModelShape("fx", layers=3, kv_heads=4, head_dim=64, q_heads=4, d_model=256)   # 8 KiB pieces
ENGINES = {"ldg": 0, "bulk": _native.KVM_F_ENGINE_BULK}


def _vllm(layout, nb, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    caches = [torch.randint(-2 ** 15, 2 ** 15, vllm_cache_shape(layout, nb, 16, SHAPE.kv_heads, SHAPE.head_dim),
                            generator=g, device="cuda", dtype=torch.int16).view(torch.float16)
              for _ in range(SHAPE.layers)]
    return StridedKVPool.from_vllm(caches, layout, name="fx"), caches


def _native_pool(nb, seed):
    p = KVPool(SHAPE, nb)
    g = torch.Generator(device="cuda").manual_seed(seed)
    p.tensor.view(torch.int16).copy_(torch.randint(-2 ** 15, 2 ** 15, p.view_shape, generator=g, device="cuda",
                                                   dtype=torch.int16))
    return p


def _piece(pool, l, kv, b):
    if isinstance(pool, StridedKVPool):
        return pool.piece(l, kv, b)
    return pool.tensor[l, kv, b]


def _snapshot(pool):
    nb = pool.num_blocks
    return torch.stack([torch.stack([torch.stack([_piece(pool, l, kv, b).view(torch.int16) for b in range(nb)])
                                     for kv in range(2)]) for l in range(SHAPE.layers)]).cpu()


def _make(kind, nb, seed):
    if kind == "native":
        return _native_pool(nb, seed), None
    return _vllm(kind, nb, seed)


@pytest.mark.parametrize("engine", ["bulk", "ldg"])
@pytest.mark.parametrize("src_kind,dst_kind", [("flash_attn", "native"), ("native", "flashinfer"),
                                               ("flash_attn", "flashinfer"), ("flashinfer", "flash_attn"),
                                               ("flash_attn", "flash_attn")])
@pytest.mark.parametrize("n", [1, 37, 200])
def test_migrate_between_layouts(engine, src_kind, dst_kind, n):
    nb = 2 * n + 11
    src, _keep_s = _make(src_kind, nb, 1)
    dst, _keep_d = _make(dst_kind, nb, 2)
    rng = np.random.default_rng(n)
    sb = rng.permutation(nb)[:n].astype(np.int32)
    dst.allocator.take(rng.permutation(nb)[:5])
    db = dst.allocator.alloc(n).astype(np.int32)
    before_src, before_dst = _snapshot(src), _snapshot(dst)
    table = BlockTable(2, n + 3)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, 3
    m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
    m.dst_table_row, m.done_flag = table.row_ptr(1), flag.data_ptr()
    _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine],
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    exp = before_dst.clone()
    exp[:, :, torch.from_numpy(db).long()] = before_src[:, :, torch.from_numpy(sb).long()]
    assert torch.equal(_snapshot(dst), exp)
    assert torch.equal(_snapshot(src), before_src)
    assert np.array_equal(table.rows[table.slot(1), :n].cpu().numpy(), db)
    assert flag.item() == 3


def test_compact_inside_a_vllm_cache_and_batch_of_moves():
    """kvm_compact on a strided pool, and one batched launch mixing native and
    strided pools (96+ moves, split internally)."""
    src, _k1 = _vllm("flashinfer", 300, 5)
    before = _snapshot(src)
    sb = np.arange(0, 40, dtype=np.int32)
    db = np.arange(200, 240, dtype=np.int32)
    _native.check(_native.lib().kvm_compact(src.pool_id, sb.ctypes.data, db.ctypes.data, 40, None,
                                            _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    exp = before.clone()
    exp[:, :, 200:240] = before[:, :, 0:40]
    assert torch.equal(_snapshot(src), exp)
    natives = [_native_pool(8, 10 + i) for i in range(2)]
    fa, _k2 = _vllm("flash_attn", 400, 7)
    snap = [_snapshot(p) for p in natives]
    moves, keep = [], []
    for i in range(130):
        p = natives[i % 2]
        s_ = np.array([i % 8], dtype=np.int32)
        d_ = np.array([i + 3], dtype=np.int32)
        keep += [s_, d_]
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = p.pool_id, fa.pool_id, 1, 1
        m.src_blocks, m.dst_blocks = s_.ctypes.data, d_.ctypes.data
        moves.append(m)
    arr = (_native.Move * len(moves))(*moves)
    _native.check(_native.lib().kvm_migrate(arr, len(moves), _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    got = _snapshot(fa)
    for i in range(130):
        assert torch.equal(got[:, :, i + 3], snap[i % 2][:, :, i % 8])


def test_strided_pool_rejections():
    fa, caches = _vllm("flash_attn", 16, 3)
    desc = SHAPE.desc(16)
    ptrs = (ctypes.c_void_p * SHAPE.layers)(*[c.data_ptr() for c in caches])
    piece = SHAPE.piece_bytes
    lib = _native.lib()
    with pytest.raises(ValueError):   # block stride smaller than a piece
        _native.check(lib.kvm_pool_register_strided(0, ctypes.byref(desc), ptrs, 16 * piece, piece // 2))
    with pytest.raises(ValueError):   # K|V planes overlap
        _native.check(lib.kvm_pool_register_strided(0, ctypes.byref(desc), ptrs, 8 * piece, piece))
    with pytest.raises(ValueError):   # misaligned stride
        _native.check(lib.kvm_pool_register_strided(0, ctypes.byref(desc), ptrs, 16 * piece + 8, piece))


@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer"])
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_decode_over_vllm_cache_equals_native(layout, dtype):
    """kvm_paged_decode reads a strided pool through its per-layer pointers:
    a request migrated out of a vLLM cache into a native pool decodes
    bit-identically from either copy (GQA tensor-core path and CUDA cores)."""
    from paper_2501_06709_b200.attention import paged_decode

    shape = ModelShape("dv", layers=2, kv_heads=2, head_dim=128, q_heads=8, d_model=1024)
    nb, n_tok = 96, 1000
    g = torch.Generator(device="cuda").manual_seed(3)
    caches = [torch.randn(vllm_cache_shape(layout, nb, 16, 2, 128), generator=g, device="cuda").to(dtype)
              for _ in range(shape.layers)]
    src = StridedKVPool.from_vllm(caches, layout, name="dv", q_heads=8)
    dst = KVPool(shape, nb, dtype=dtype)
    k = (n_tok + 15) // 16
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(4))[:k].to(torch.int32)
    db = torch.randperm(nb, generator=torch.Generator().manual_seed(5))[:k].to(torch.int32)
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, k, 1
    sbn, dbn = sb.numpy(), db.numpy()
    m.src_blocks, m.dst_blocks = sbn.ctypes.data, dbn.ctypes.data
    _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    q = torch.randn(shape.layers, 1, 8, 128, generator=g, device="cuda").to(dtype)
    lens = torch.tensor([n_tok], dtype=torch.int32, device="cuda")
    for cc in (False, True):
        a = paged_decode(src, q, sb[None].contiguous().cuda(), lens, cuda_cores=cc)
        b = paged_decode(dst, q, db[None].contiguous().cuda(), lens, cuda_cores=cc)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def _bf16_pair(layout, nb, shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    caches = [torch.randint(-2 ** 15, 2 ** 15, vllm_cache_shape(layout, nb, 16, shape.kv_heads, shape.head_dim),
                            generator=g, device="cuda", dtype=torch.int16).view(torch.bfloat16)
              for _ in range(shape.layers)]
    return StridedKVPool.from_vllm(caches, layout, name=shape.name, q_heads=shape.q_heads), caches


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer"])
def test_reprefill_into_vllm_cache_equals_native(layout, single_cta):
    """Re-prefill writes a strided pool's pieces in place: every recomputed
    token slot equals the same re-prefill into a native pool, bit for bit
    (RoPE on), and nothing else in the vLLM cache changes."""
    from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights

    shape = ModelShape("rv", layers=2, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
    nb, rows, tok0 = 40, 300, 21
    fx, _caches = _bf16_pair(layout, nb, shape, 8)
    nat = KVPool(shape, nb, dtype=torch.bfloat16)
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(9))[:(tok0 + rows + 15) // 16]
    blocks = blocks.to(torch.int32).cuda()
    x = synthetic_hidden(shape, rows, 0, seed=10)
    w = synthetic_weights(shape, 0, with_q=True, seed=11)
    before = [[[fx.piece(l, kv, b).clone() for b in range(nb)] for kv in range(2)] for l in range(2)]
    reprefill(fx, x, w, blocks, tok0=tok0, single_cta=single_cta, rope_theta=10000.0)
    reprefill(nat, x, w, blocks, tok0=tok0, single_cta=single_cta, rope_theta=10000.0)
    torch.cuda.synchronize()
    written = set()
    for t in range(tok0, tok0 + rows):
        written.add((int(blocks[t // 16]), t % 16))
    for l in range(2):
        for kv in range(2):
            for b in range(nb):
                got = fx.piece(l, kv, b).view(torch.int16)
                for slot in range(16):
                    if (b, slot) in written:
                        assert torch.equal(got[slot], nat.tensor[l, kv, b, slot].view(torch.int16))
                    else:
                        assert torch.equal(got[slot], before[l][kv][b][slot].view(torch.int16))


@pytest.mark.parametrize("src_kind,dst_kind", [("flash_attn", "native"), ("native", "flashinfer"),
                                               ("flashinfer", "flash_attn")])
def test_fused_split_between_layouts(src_kind, dst_kind):
    """kvm_split_migrate with strided pools on either side: the prefix arrives
    bit-exact, the recomputed suffix equals the same split into native pools."""
    from paper_2501_06709_b200.reprefill import synthetic_hidden, synthetic_weights
    from paper_2501_06709_b200.split import make_split, split_migrate_fused

    shape = ModelShape("sv", layers=2, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
    tokens, suffix = 700, 188
    plan = make_split(tokens, suffix)
    nb = plan.total_blocks + 6

    def mk(kind, seed):
        if kind == "native":
            p = KVPool(shape, nb, dtype=torch.bfloat16)
            p.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1,
                                              generator=torch.Generator(device="cuda").manual_seed(seed))
            return p
        return _bf16_pair(kind, nb, shape, seed)[0]

    def piece(pool, l, kv, b):
        return pool.piece(l, kv, b) if isinstance(pool, StridedKVPool) else pool.tensor[l, kv, b]

    src, dst = mk(src_kind, 1), mk(dst_kind, 2)
    nsrc, ndst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    for l in range(2):
        for kv in range(2):
            for b in range(nb):
                nsrc.tensor[l, kv, b] = piece(src, l, kv, b)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(3))[:plan.total_blocks].to(torch.int32).cuda()
    db = torch.randperm(nb, generator=torch.Generator().manual_seed(4))[:plan.total_blocks].to(torch.int32).cuda()
    x = synthetic_hidden(shape, suffix, 0, seed=5)
    w = synthetic_weights(shape, 0, with_q=True, seed=6)
    split_migrate_fused(src, dst, sb, db, plan, x, w, rope_theta=10000.0)
    split_migrate_fused(nsrc, ndst, sb, db, plan, x, w, rope_theta=10000.0)
    torch.cuda.synchronize()
    for l in range(2):
        for kv in range(2):
            for i in range(plan.total_blocks):
                b = int(db[i])
                got, exp = piece(dst, l, kv, b).view(torch.int16), ndst.tensor[l, kv, b].view(torch.int16)
                n_valid = min(16, tokens - 16 * i)
                assert torch.equal(got[:n_valid], exp[:n_valid])


def test_executor_and_live_migration_on_vllm_caches():
    """The executor and live migration take strided pools like native ones:
    a plan moves requests from a FlashAttention-layout cache (logical GPU 0)
    to a FlashInfer-layout cache (logical GPU 1), then live migration brings
    one back, with the block tables rewritten by the kernels."""
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.live import LiveMigration
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    p0, _c0 = _vllm("flash_attn", 64, 1)
    p1, _c1 = _vllm("flashinfer", 64, 2)
    tables = {0: BlockTable(4, 16), 1: BlockTable(4, 16)}
    ex = MigrationExecutor({0: p0, 1: p1}, tables)
    ex.admit(1, 0, 70)
    ex.admit(2, 0, 40)
    src = {r: [[[p0.piece(l, kv, int(b)).clone() for b in ex.where(r).blocks] for kv in range(2)]
               for l in range(SHAPE.layers)] for r in (1, 2)}
    bpt = SHAPE.kv_bytes_per_token
    ex.execute([PlannedMove(PendingMove(1, 0, 1, 70 * bpt, 70), KV_TRANSFER),
                PlannedMove(PendingMove(2, 0, 1, 40 * bpt, 40), KV_TRANSFER)])
    for r in (1, 2):
        res = ex.where(r)
        assert res.gpu == 1
        assert np.array_equal(tables[1].rows[tables[1].slot(r), :len(res.blocks)].cpu().numpy(), res.blocks)
        for l in range(SHAPE.layers):
            for kv in range(2):
                for i, b in enumerate(res.blocks):
                    assert torch.equal(p1.piece(l, kv, int(b)).view(torch.int16), src[r][l][kv][i].view(torch.int16))
    lm = LiveMigration(ex, 1, 0)
    lm.precopy()
    lm.drain()
    lm.finish()
    res = ex.where(1)
    assert res.gpu == 0
    for l in range(SHAPE.layers):
        for kv in range(2):
            for i, b in enumerate(res.blocks):
                assert torch.equal(p0.piece(l, kv, int(b)).view(torch.int16), src[1][l][kv][i].view(torch.int16))


@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer"])
def test_fp8_vllm_cache_migrates_bit_exact(layout):
    """vLLM's fp8 (e4m3) KV caches: one byte per element, pieces of 16 x H x D
    bytes, moved into a native fp8 pool and back, bit-exact."""
    shape = ModelShape("f8", layers=2, kv_heads=8, head_dim=128, q_heads=8, d_model=1024, elem_bytes=1)
    nb = 24
    g = torch.Generator(device="cuda").manual_seed(12)
    caches = [torch.randint(0, 256, vllm_cache_shape(layout, nb, 16, 8, 128), generator=g, device="cuda",
                            dtype=torch.uint8).view(torch.float8_e4m3fn) for _ in range(2)]
    fx = StridedKVPool.from_vllm(caches, layout, name="f8")
    nat = KVPool(shape, nb, dtype=torch.float8_e4m3fn)
    nat.tensor.view(torch.uint8).zero_()
    sb = np.array([3, 17, 0, 9], dtype=np.int32)
    db = np.array([1, 2, 20, 23], dtype=np.int32)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for s_pool, d_pool, s_b, d_b in ((fx, nat, sb, db), (nat, fx, db, np.array([4, 5, 6, 7], dtype=np.int32))):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = s_pool.pool_id, d_pool.pool_id, 4, 1
        m.src_blocks, m.dst_blocks = s_b.ctypes.data, d_b.ctypes.data
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST |
                                                _native.KVM_F_ENGINE_BULK, stream))
    torch.cuda.synchronize()
    for l in range(2):
        for kv in range(2):
            for i in range(4):
                orig = fx.piece(l, kv, int(sb[i])).view(torch.uint8)
                assert torch.equal(nat.tensor[l, kv, int(db[i])].view(torch.uint8), orig)
                assert torch.equal(fx.piece(l, kv, 4 + i).view(torch.uint8), orig)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVM_FUZZ_SEEDS", "100"))))
def test_foreign_layouts_randomized(seed):
    """Random layouts on both sides (native / FlashAttention / FlashInfer),
    random geometry, one to three moves per launch, host or device lists,
    either engine: every destination piece equals its source piece and nothing
    else changes."""
    rng = np.random.default_rng(11000 + seed)
    shape = ModelShape(f"fr{seed}", layers=int(rng.integers(1, 4)), kv_heads=int(rng.integers(1, 6)),
                       head_dim=int(rng.choice([8, 64, 128])), q_heads=1, d_model=64)
    kinds = ["native", "flash_attn", "flashinfer"]

    def make(kind, nb, sd):
        if kind == "native":
            p = KVPool(shape, nb)
            p.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1,
                                              generator=torch.Generator(device="cuda").manual_seed(sd))
            return p, None
        g = torch.Generator(device="cuda").manual_seed(sd)
        caches = [torch.randint(-2 ** 15, 2 ** 15, vllm_cache_shape(kind, nb, 16, shape.kv_heads, shape.head_dim),
                                generator=g, device="cuda", dtype=torch.int16).view(torch.float16)
                  for _ in range(shape.layers)]
        return StridedKVPool.from_vllm(caches, kind, name=shape.name), caches

    def snap(pool):
        return torch.stack([torch.stack([torch.stack([_piece(pool, l, kv, b).reshape(-1).view(torch.int16)
                                                      for b in range(pool.num_blocks)]) for kv in range(2)])
                            for l in range(shape.layers)]).cpu()

    nb = int(rng.integers(8, 40))
    src, _k1 = make(kinds[int(rng.integers(3))], nb, seed)
    dst, _k2 = make(kinds[int(rng.integers(3))], nb, seed + 1)
    bs, bd = snap(src), snap(dst)
    exp = bd.clone()
    free = list(rng.permutation(nb))
    moves, keep = [], []
    host = bool(rng.integers(2))
    for _ in range(int(rng.integers(1, 4))):
        n = int(rng.integers(0, min(6, len(free)) + 1))
        sbn = rng.permutation(nb)[:n].astype(np.int32)
        dbn = np.array([free.pop() for _ in range(n)], dtype=np.int32)
        exp[:, :, torch.from_numpy(dbn).long()] = bs[:, :, torch.from_numpy(sbn).long()]
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, 1
        if host:
            keep += [sbn, dbn]
            m.src_blocks, m.dst_blocks = sbn.ctypes.data, dbn.ctypes.data
        else:
            ts, td = torch.from_numpy(sbn).cuda(), torch.from_numpy(dbn).cuda()
            keep += [ts, td]
            m.src_blocks, m.dst_blocks = ts.data_ptr(), td.data_ptr()
        moves.append(m)
    arr = (_native.Move * len(moves))(*moves)
    flags = (_native.KVM_F_BLOCKS_ON_HOST if host else 0) | (_native.KVM_F_ENGINE_BULK if rng.integers(2) else 0)
    _native.check(_native.lib().kvm_migrate(arr, len(moves), flags,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(snap(dst), exp)
    assert torch.equal(snap(src), bs)
