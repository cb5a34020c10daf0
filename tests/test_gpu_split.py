"""configs[2] split migration on one B200: the transferred prefix is bit-exact
and the re-prefilled suffix is within the stated bf16 tolerance, with the two
halves running concurrently on two streams (GEMM first, copy in the SM slots
it leaves)."""
import numpy as np
import pytest
import torch

from paper_2501_06709_b200 import _native
from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape
from paper_2501_06709_b200.reprefill import split_point, synthetic_hidden, synthetic_weights
from paper_2501_06709_b200.split import flops_per_token, make_split, split_migrate, wait_split

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tokens,suffix", [(1024, 240), (1000, 232), (512, 0), (512, 512), (16 * 40, None)])
def test_split_migration(tokens, suffix):
    shape = ModelShape("sp", layers=6, kv_heads=4, head_dim=128, q_heads=8, d_model=512)
    if suffix is None:
        suffix = split_point(tokens, shape.kv_bytes_per_token, 770e9, flops_per_token(shape), 1.2e15)
    plan = make_split(tokens, suffix)
    nb = plan.total_blocks + 20
    src, dst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    src.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    dst.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(3))[:plan.total_blocks].to(torch.int32).numpy()
    db = torch.from_numpy(dst.allocator.alloc(plan.total_blocks)).cuda()
    x = synthetic_hidden(shape, max(suffix, 1), 0, seed=4)[:suffix].contiguous()
    w = synthetic_weights(shape, 0, with_q=True, seed=5)
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    table = BlockTable(1, plan.total_blocks)
    sa, sb_ = torch.cuda.Stream(), torch.cuda.Stream()
    sa.wait_stream(torch.cuda.current_stream())   # inputs were produced on the default stream
    sb_.wait_stream(torch.cuda.current_stream())
    split_migrate(src, dst, sb, db, plan, x, w, xfer_stream=sa, rp_stream=sb_, flags_dev=flags, seq=7,
                  table_row=table.row_ptr(0), engine_flags=_native.KVM_F_CTAS_PER_SM(3))
    wait_split(flags, plan, 7, sb_)
    sb_.synchronize()
    sa.synchronize()
    pre = plan.prefix_blocks
    assert torch.equal(dst.tensor[:, :, db[:pre].long()].view(torch.int16),
                       src.tensor[:, :, torch.from_numpy(sb[:pre]).long().cuda()].view(torch.int16))
    assert np.array_equal(table.rows[0, :pre].cpu().numpy(), db[:pre].cpu().numpy())
    if suffix:
        kvd, qc = shape.kv_cols, shape.q_cols
        toks = torch.arange(plan.prefix_tokens, tokens, device="cuda")
        blk, slot = db.long()[toks // 16], toks % 16
        for l in range(shape.layers):
            ref = x.float() @ w[l].float().t()
            torch.testing.assert_close(dst.tensor[l, 0, blk, slot].reshape(suffix, kvd).float(),
                                       ref[:, qc:qc + kvd], atol=1e-2, rtol=1.6e-2)
            torch.testing.assert_close(dst.tensor[l, 1, blk, slot].reshape(suffix, kvd).float(),
                                       ref[:, qc + kvd:], atol=1e-2, rtol=1.6e-2)
    assert flags.cpu().tolist() == [7 if pre else 0, 7 if suffix else 0]


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("tokens,suffix", [(1024, 240), (1000, 232), (512, 0), (512, 512), (16 * 40, None),
                                           (4096, 1024)])
def test_fused_split_migration(tokens, suffix, single_cta):
    """kvm_split_migrate: one launch; prefix copied by the GEMM's idle warps."""
    from paper_2501_06709_b200.split import split_migrate_fused

    shape = ModelShape("spf", layers=6, kv_heads=4, head_dim=128, q_heads=8, d_model=512)
    if suffix is None:
        suffix = split_point(tokens, shape.kv_bytes_per_token, 770e9, flops_per_token(shape), 1.2e15)
    plan = make_split(tokens, suffix)
    nb = plan.total_blocks + 20
    src, dst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    src.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    dst.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = dst.tensor.view(torch.int16).clone()
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(3))[:plan.total_blocks].to(torch.int32).cuda()
    db = torch.from_numpy(dst.allocator.alloc(plan.total_blocks)).cuda()
    x = synthetic_hidden(shape, max(suffix, 1), 0, seed=4)[:suffix].contiguous()
    w = synthetic_weights(shape, 0, with_q=True, seed=5)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    table = BlockTable(1, plan.total_blocks)
    split_migrate_fused(src, dst, sb, db, plan, x, w, table_row=table.row_ptr(0), done_flag=flag.data_ptr(),
                        done_value=9, single_cta=single_cta)
    torch.cuda.synchronize()
    pre = plan.prefix_blocks
    assert torch.equal(dst.tensor[:, :, db[:pre].long()].view(torch.int16),
                       src.tensor[:, :, sb[:pre].long()].view(torch.int16))
    if suffix:
        kvd, qc = shape.kv_cols, shape.q_cols
        toks = torch.arange(plan.prefix_tokens, tokens, device="cuda")
        blk, slot = db.long()[toks // 16], toks % 16
        for l in range(shape.layers):
            ref = x.float() @ w[l].float().t()
            torch.testing.assert_close(dst.tensor[l, 0, blk, slot].reshape(suffix, kvd).float(),
                                       ref[:, qc:qc + kvd], atol=1e-2, rtol=1.6e-2)
            torch.testing.assert_close(dst.tensor[l, 1, blk, slot].reshape(suffix, kvd).float(),
                                       ref[:, qc + kvd:], atol=1e-2, rtol=1.6e-2)
    # nothing outside the request's destination slots changed
    mask = torch.ones(nb, 16, dtype=torch.bool, device="cuda")
    mask[db[:pre].long()] = False
    if suffix:
        mask[blk, slot] = False
    assert torch.equal(dst.tensor.view(torch.int16)[:, :, mask], before[:, :, mask])
    assert np.array_equal(table.rows[0].cpu().numpy(), db.cpu().numpy())
    assert flag.item() == 9


def test_executor_split_move():
    """MigrationExecutor.split_move: the fused split through the host API."""
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.reprefill import ReprefillEngine

    shape = ModelShape("spx", layers=4, kv_heads=4, head_dim=128, q_heads=4, d_model=512)
    pools = {0: KVPool(shape, 64, dtype=torch.bfloat16), 1: KVPool(shape, 64, dtype=torch.bfloat16)}
    tables = {0: BlockTable(4, 64), 1: BlockTable(4, 64)}
    ex = MigrationExecutor(pools, tables, reprefill=ReprefillEngine(shape, [0], with_q=False))
    pools[0].tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    ex.admit(3, 0, 600)
    sb = ex.where(3).blocks.copy()
    rec = ex.split_move(3, 1, suffix=200)
    r = ex.where(3)
    assert r.gpu == 1 and rec.tokens_recomputed == 200 + (600 - 200) % 16
    pre = (600 - rec.tokens_recomputed) // 16
    assert torch.equal(pools[1].tensor[:, :, torch.from_numpy(r.blocks[:pre]).long().cuda()].view(torch.int16),
                       pools[0].tensor[:, :, torch.from_numpy(sb[:pre]).long().cuda()].view(torch.int16))
    assert np.array_equal(tables[1].rows[tables[1].slot(3), :len(r.blocks)].cpu().numpy(), r.blocks)
    assert pools[0].allocator.n_free == 64


@pytest.mark.parametrize("single_cta", [False, True])
def test_fused_split_with_rope(single_cta):
    """The fused split migration with RoPE in the re-prefill epilogue: prefix
    bit-exact, suffix K post-RoPE at positions prefix_tokens + t."""
    from paper_2501_06709_b200.split import split_migrate_fused
    from test_gpu_reprefill import _rope_ref

    shape = ModelShape("spr", layers=3, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
    tokens, suffix = 1000, 232
    plan = make_split(tokens, suffix)
    nb = plan.total_blocks + 10
    src, dst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    src.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(5))[:plan.total_blocks].to(torch.int32).cuda()
    db = torch.from_numpy(dst.allocator.alloc(plan.total_blocks)).cuda()
    x = synthetic_hidden(shape, suffix, 0, seed=6)
    w = synthetic_weights(shape, 0, with_q=True, seed=7)
    split_migrate_fused(src, dst, sb, db, plan, x, w, single_cta=single_cta, rope_theta=500000.0)
    torch.cuda.synchronize()
    pre = plan.prefix_blocks
    assert torch.equal(dst.tensor[:, :, db[:pre].long()].view(torch.int16),
                       src.tensor[:, :, sb[:pre].long()].view(torch.int16))
    toks = torch.arange(plan.prefix_tokens, tokens, device="cuda")
    ref = _rope_ref(torch.einsum("tk,lnk->ltn", x.float(), w.float()), toks, 500000.0, shape.q_cols, shape.kv_cols)
    blk, slot = db.long()[toks // 16], toks % 16
    kvd, qc = shape.kv_cols, shape.q_cols
    for l in range(shape.layers):
        torch.testing.assert_close(dst.tensor[l, 0, blk, slot].reshape(suffix, kvd).float(), ref[l, :, qc:qc + kvd],
                                   atol=1e-2, rtol=1.6e-2)
        torch.testing.assert_close(dst.tensor[l, 1, blk, slot].reshape(suffix, kvd).float(), ref[l, :, qc + kvd:],
                                   atol=1e-2, rtol=1.6e-2)


@pytest.mark.parametrize("per_layer", [False, True])
@pytest.mark.parametrize("single_cta", [False, True])
def test_split_migrated_cache_decodes_like_the_original(single_cta, per_layer):
    """End to end through the consumer: the source cache is prefilled by the same
    projection (+RoPE) for all n tokens; a split migration copies the prefix and
    recomputes the suffix on the destination; paged decode over the migrated
    cache must equal decode over the source.  The recomputed rows are the same
    GEMM on the same inputs with the same per-element accumulation order, so
    the migrated cache is BIT-IDENTICAL to the original (and so is decode).
    per_layer: every layer has its own hidden states (KVM_REPREFILL_X_PER_LAYER)."""
    from paper_2501_06709_b200.attention import paged_decode
    from paper_2501_06709_b200.reprefill import reprefill
    from paper_2501_06709_b200.split import split_migrate_fused

    shape = ModelShape("e2e", layers=2, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
    n, suffix = 1000, 232
    plan = make_split(n, suffix)
    nb = plan.total_blocks + 8
    src, dst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    dst.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(11))[:plan.total_blocks].to(torch.int32).cuda()
    db = torch.from_numpy(dst.allocator.alloc(plan.total_blocks)).cuda()
    if per_layer:
        g = torch.Generator(device="cuda").manual_seed(12)
        x = torch.randn(shape.layers, n, shape.d_model, generator=g, device="cuda").to(torch.bfloat16)
    else:
        x = synthetic_hidden(shape, n, 0, seed=12)
    w = synthetic_weights(shape, 0, with_q=False, seed=13)
    reprefill(src, x, w, sb, tok0=0, rope_theta=10000.0, single_cta=single_cta)   # the original prefill
    xs = x[..., plan.prefix_tokens:, :].contiguous()
    split_migrate_fused(src, dst, sb, db, plan, xs, w, single_cta=single_cta, rope_theta=10000.0)
    torch.cuda.synchronize()
    q = torch.randn(shape.layers, 1, shape.q_heads, 128, device="cuda").to(torch.bfloat16)
    lens = torch.tensor([n], dtype=torch.int32, device="cuda")
    a = paged_decode(src, q, sb[None].contiguous(), lens)
    b = paged_decode(dst, q, db[None].contiguous(), lens)
    torch.cuda.synchronize()
    toks = torch.arange(n, device="cuda")   # every token slot of the request (the last block is partial)
    got = dst.tensor[:, :, db.long()[toks // 16], toks % 16].view(torch.int16)
    exp = src.tensor[:, :, sb.long()[toks // 16], toks % 16].view(torch.int16)
    assert torch.equal(got, exp)
    assert torch.equal(b.view(torch.int16), a.view(torch.int16))


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVM_FUZZ_SEEDS", "50"))))
def test_fused_split_randomized(seed):
    """Random geometry, request length, split point (incl. all-transfer and
    all-recompute), RoPE, GEMM engine, SM budget and block scatter for kvm_split_migrate:
    prefix blocks bit-exact, suffix token slots within tolerance, the table
    row rewritten, nothing else in the destination pool written."""
    from paper_2501_06709_b200.split import split_migrate_fused
    from test_gpu_reprefill import ATOL, RTOL, _rope_ref

    rng = np.random.default_rng(7000 + seed)
    head_dim = int(rng.choice([64, 128]))
    kv_heads = int(rng.integers(1, 4))
    shape = ModelShape(f"sz{seed}", layers=int(rng.integers(1, 4)), kv_heads=kv_heads, head_dim=head_dim,
                       q_heads=kv_heads * int(rng.choice([1, 2])), d_model=64 * int(rng.integers(1, 7)))
    tokens = int(rng.integers(1, 1200))
    prefix_blocks = int(rng.integers(0, tokens // 16 + 1))
    plan = make_split(tokens, tokens - 16 * prefix_blocks)
    rope = head_dim == 128 and bool(rng.integers(2))
    nb = plan.total_blocks + int(rng.integers(1, 12))
    src, dst = KVPool(shape, nb, dtype=torch.bfloat16), KVPool(shape, nb, dtype=torch.bfloat16)
    src.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    dst.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = dst.tensor.view(torch.int16).clone()
    sb = torch.from_numpy(rng.permutation(nb)[:plan.total_blocks].astype(np.int32)).cuda()
    db = torch.from_numpy(rng.permutation(nb)[:plan.total_blocks].astype(np.int32)).cuda()
    x = synthetic_hidden(shape, max(plan.suffix, 1), 0, seed=seed)[:plan.suffix].contiguous()
    w = synthetic_weights(shape, 0, with_q=True, seed=seed + 1)
    table = BlockTable(1, plan.total_blocks + 1)
    single_cta = bool(rng.integers(2))
    split_migrate_fused(src, dst, sb, db, plan, x if plan.suffix else None, w, table_row=table.row_ptr(0),
                        single_cta=single_cta, rope_theta=10000.0 if rope else 0.0,
                        max_sms=int(rng.choice([0, 0, 2, 9, 64])))   # SM budget (KVM_REPREFILL_MAX_SMS)
    torch.cuda.synchronize()
    got = dst.tensor.view(torch.int16)
    pre = plan.prefix_blocks
    if pre:
        assert torch.equal(got[:, :, db[:pre].long()], src.tensor.view(torch.int16)[:, :, sb[:pre].long()])
    assert np.array_equal(table.rows[0, :plan.total_blocks].cpu().numpy(), db.cpu().numpy())
    mask = torch.ones(nb, 16, dtype=torch.bool, device="cuda")
    mask[db[:pre].long()] = False
    if plan.suffix:
        toks = torch.arange(plan.prefix_tokens, tokens, device="cuda")
        blk, slot = db.long()[toks // 16], toks % 16
        mask[blk, slot] = False
        ref = torch.einsum("tk,lnk->ltn", x.float(), w.float())
        if rope:
            ref = _rope_ref(ref, toks, 10000.0, shape.q_cols, shape.kv_cols)
        kvd, qc = shape.kv_cols, shape.q_cols
        for l in range(shape.layers):
            torch.testing.assert_close(dst.tensor[l, 0, blk, slot].reshape(plan.suffix, kvd).float(),
                                       ref[l, :, qc:qc + kvd], atol=ATOL, rtol=RTOL)
            torch.testing.assert_close(dst.tensor[l, 1, blk, slot].reshape(plan.suffix, kvd).float(),
                                       ref[l, :, qc + kvd:], atol=ATOL, rtol=RTOL)
    assert torch.equal(got[:, :, mask], before[:, :, mask])


@pytest.mark.parametrize("force_two", [False, True])
def test_bench_split_tool_paths(force_two):
    """tools/bench_split.run_split_bench (the bench line's configs[2] extra):
    the same-device path and the two-device path (peer alias of the source
    pool, done-flag waits, two kernels overlapped) forced onto one GPU, at a
    reduced 2k-token size: prefix bit-exact, suffix within tolerance."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from bench_split import run_split_bench

    r = run_split_bench(tokens=2048, iters=2, warmup=1, src_dev=0, dst_dev=0, force_two=force_two)
    assert r["prefix_bit_exact"] is True and r["suffix_within_tolerance"] is True, r
    assert r["suffix_reprefilled"] > 0 and r["prefix_blocks"] > 0
    assert (r["ms"]["split_two_kernels"] is not None) == force_two
