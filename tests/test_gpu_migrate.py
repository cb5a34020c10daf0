"""GPU parity of the migration kernels (through the C ABI) against the oracle.

Small seeded cases are compared with the C oracle byte-for-byte over the WHOLE
destination pool (so any stray write outside the target blocks fails);
full-size configs use size-independent properties (gathered src == gathered
dst, everything else unchanged, via per-piece checksums on the device).
"""
import ctypes
import os

import numpy as np
import pytest
import torch

from oracle import kvmig_oracle as orc
from paper_2501_06709_b200 import ConfigError, NotPlaced, RequestTooLarge, _native
from paper_2501_06709_b200.kvcache import (LLAMA2_7B, LLAMA2_13B, LLAMA3_70B, BlockTable, KVPool,
                                           ModelShape)

pytestmark = pytest.mark.gpu
ENGINES = {"ldg": 0, "bulk": _native.KVM_F_ENGINE_BULK}


def _fill(pool, seed):
    g = torch.Generator(device=f"cuda:{pool.device}").manual_seed(seed)
    t = pool.tensor.view(torch.int16)
    t.copy_(torch.randint(-2 ** 15, 2 ** 15, t.shape, generator=g, device=t.device, dtype=torch.int16))


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _move(src, dst, sb, db, row=0, flag=0, layer_flags=0, value=1, n=None):
    m = _native.Move()
    n = len(sb) if n is None else n
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, value
    m.src_blocks, m.dst_blocks = sb.ctypes.data if isinstance(sb, np.ndarray) else sb, \
        db.ctypes.data if isinstance(db, np.ndarray) else db
    m.dst_table_row, m.done_flag, m.layer_flags = row, flag, layer_flags
    return m


def _run(moves, flags):
    arr = (_native.Move * len(moves))(*moves)
    _native.check(_native.lib().kvm_migrate(arr, len(moves), flags, _stream()))
    torch.cuda.synchronize()


def _desc(pool):
    s = pool.shape
    return orc.desc(s.layers, s.kv_heads, s.head_dim, s.block_tokens, pool.num_blocks, s.elem_bytes)


SMALL = ModelShape("t", layers=3, kv_heads=4, head_dim=64, q_heads=4, d_model=256)   # 8 KiB pieces
ODD = ModelShape("odd", layers=2, kv_heads=5, head_dim=40, q_heads=5, d_model=200)   # 6400 B pieces
BIG = ModelShape("b", layers=2, kv_heads=40, head_dim=128, q_heads=40, d_model=5120)  # 160 KiB pieces


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
@pytest.mark.parametrize("shape", [SMALL, ODD, BIG], ids=lambda s: s.name)
@pytest.mark.parametrize("host_blocks", [True, False])
def test_migrate_bit_exact_vs_oracle(engine, shape, host_blocks):
    nb = 48
    src, dst = KVPool(shape, nb), KVPool(shape, nb)
    _fill(src, 1)
    _fill(dst, 2)
    rng = np.random.default_rng(7)
    sb = rng.permutation(nb)[:17].astype(np.int32)
    dst.allocator.take(rng.permutation(nb)[:20])
    db = dst.allocator.alloc(17)
    exp = dst.tensor.view(torch.int16).cpu().numpy()
    row_exp = orc.migrate(src.tensor.view(torch.int16).cpu().numpy(), _desc(src), exp, _desc(dst), sb, db)
    table = BlockTable(2, 32)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    if host_blocks:
        m = _move(src, dst, sb, db, table.row_ptr(5), flag.data_ptr(), value=9)
        _run([m], _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine])
    else:
        sbd = torch.from_numpy(sb).cuda()
        dbd = torch.from_numpy(db).cuda()
        m = _move(src, dst, sbd.data_ptr(), dbd.data_ptr(), table.row_ptr(5), flag.data_ptr(), value=9,
                  n=17)
        _run([m], ENGINES[engine])
    assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)
    assert np.array_equal(table.rows[table.slot(5), :17].cpu().numpy(), row_exp)
    assert (table.rows[table.slot(5), 17:] == -1).all()
    assert flag.item() == 9


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_batch_of_many_moves_and_layer_flags(engine):
    """130 moves (> KVM_MAX_MOVES, so the batch is split) with ragged sizes,
    including empty moves, every one with layer flags and a done flag."""
    nb = 400
    src, dst = KVPool(SMALL, nb), KVPool(SMALL, nb)
    _fill(src, 3)
    _fill(dst, 4)
    rng = np.random.default_rng(11)
    perm = rng.permutation(nb).astype(np.int32)
    sizes = [int(rng.integers(0, 6)) for _ in range(130)]
    sizes[0] = 0
    moves, keep, exp_rows = [], [], []
    flags = torch.zeros(130, dtype=torch.int32, device="cuda")
    lflags = torch.zeros(130, SMALL.layers, dtype=torch.int32, device="cuda")
    table = BlockTable(130, 8)
    exp = dst.tensor.view(torch.int16).cpu().numpy()
    src_np = src.tensor.view(torch.int16).cpu().numpy()
    off = 0
    for i, n in enumerate(sizes):
        sb = perm[off:off + n].copy()
        off += n
        db = dst.allocator.alloc(n)
        keep += [sb, db]
        exp_rows.append(orc.migrate(src_np, _desc(src), exp, _desc(dst), sb, db))
        moves.append(_move(src, dst, sb, db, table.row_ptr(i), flags[i:].data_ptr(),
                           lflags[i].data_ptr(), value=100 + i))
    _run(moves, _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine])
    assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)
    assert flags.cpu().tolist() == [100 + i for i in range(130)]
    assert (lflags.cpu() == torch.arange(100, 230, dtype=torch.int32)[:, None]).all()
    for i, n in enumerate(sizes):
        assert np.array_equal(table.rows[table.slot(i), :n].cpu().numpy(), exp_rows[i])


def test_compaction_and_overlap_rejected():
    nb = 64
    pool = KVPool(SMALL, nb)
    _fill(pool, 5)
    before = pool.tensor.view(torch.int16).cpu().numpy()
    sb = np.array([60, 3, 41, 17], dtype=np.int32)
    pool.allocator.take(sb)
    db = pool.allocator.alloc(4)
    exp = before.copy()
    orc.migrate(before, _desc(pool), exp, _desc(pool), sb, db)
    table = BlockTable(1, 8)
    _native.check(_native.lib().kvm_compact(pool.pool_id, sb.ctypes.data, db.ctypes.data, 4,
                                            ctypes.c_void_p(table.row_ptr(0)),
                                            _native.KVM_F_BLOCKS_ON_HOST, _stream()))
    torch.cuda.synchronize()
    assert np.array_equal(pool.tensor.view(torch.int16).cpu().numpy(), exp)
    bad = np.array([3, 5, 6, 7], dtype=np.int32)
    with pytest.raises(ValueError):
        _native.check(_native.lib().kvm_compact(pool.pool_id, sb.ctypes.data, bad.ctypes.data, 4,
                                                None, _native.KVM_F_BLOCKS_ON_HOST, _stream()))


def test_errors_map_to_reference_exceptions():
    pool = KVPool(SMALL, 8)
    other = KVPool(ODD, 8)
    sb = np.array([0], dtype=np.int32)
    db = np.array([9], dtype=np.int32)
    with pytest.raises(ValueError):  # dst block out of range
        _run([_move(pool, pool, sb, db)], _native.KVM_F_BLOCKS_ON_HOST)
    with pytest.raises(ConfigError):  # shape mismatch
        _run([_move(pool, other, sb, sb)], _native.KVM_F_BLOCKS_ON_HOST)
    m = _move(pool, pool, sb, sb)
    m.dst_pool = 10 ** 6
    with pytest.raises(NotPlaced):
        _run([m], _native.KVM_F_BLOCKS_ON_HOST)


@pytest.mark.parametrize("shape,tokens", [(LLAMA2_7B, 4096), (LLAMA2_13B, 8192), (LLAMA3_70B, 16384)],
                         ids=["7b-4k", "13b-8k", "70b-16k"])
@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_full_size_property(shape, tokens, engine):
    """BASELINE configs 2-4 at full size: moved pieces identical, nothing else
    touched (checksums of all pieces before/after), table row exact."""
    n = tokens // 16
    nb = 2 * n + 64
    pool_src, pool_dst = KVPool(shape, nb), KVPool(shape, nb)
    _fill(pool_src, 1)
    _fill(pool_dst, 2)
    g = torch.Generator().manual_seed(1)
    sb = torch.randperm(nb, generator=g)[:n].to(torch.int32).numpy()
    occ = torch.randperm(nb, generator=torch.Generator().manual_seed(2))[: nb // 2].numpy()
    pool_dst.allocator.take(occ)
    db = pool_dst.allocator.alloc(n)

    def piece_sums(pool):  # [L, 2, nb] int64 position-weighted checksum per piece
        t = pool.tensor.view(torch.int16).view(shape.layers, 2, nb, -1)
        w = torch.arange(1, t.shape[-1] + 1, device=t.device, dtype=torch.int64)
        return torch.stack([(t[l].to(torch.int64) * w).sum(-1) for l in range(shape.layers)])

    src_sums = piece_sums(pool_src)
    before = piece_sums(pool_dst)
    table = BlockTable(1, n)
    _run([_move(pool_src, pool_dst, sb, db, table.row_ptr(0))],
         _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine])
    after = piece_sums(pool_dst)
    sbt, dbt = torch.from_numpy(sb).long().cuda(), torch.from_numpy(db).long().cuda()
    assert torch.equal(after[:, :, dbt], src_sums[:, :, sbt])
    mask = torch.ones(nb, dtype=torch.bool, device="cuda")
    mask[dbt] = False
    assert torch.equal(after[:, :, mask], before[:, :, mask])
    # exact bytes on a sample of pieces (first/last layer, K and V)
    for l in (0, shape.layers - 1):
        for kv in (0, 1):
            assert torch.equal(pool_dst.tensor[l, kv, dbt[:8]].view(torch.int16),
                               pool_src.tensor[l, kv, sbt[:8]].view(torch.int16))
    assert np.array_equal(table.rows[0].cpu().numpy(), db)


def test_wait_flag_kernel():
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    pool = KVPool(SMALL, 8)
    sb = np.array([1, 2], dtype=np.int32)
    db = np.array([5, 6], dtype=np.int32)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        _native.check(_native.lib().kvm_wait_flag(ctypes.c_void_p(flag.data_ptr()), 3,
                                                  ctypes.c_void_p(side.cuda_stream)))
    m = _move(pool, pool, sb, db, flag=flag.data_ptr(), value=3)
    _run([m], _native.KVM_F_BLOCKS_ON_HOST)
    side.synchronize()
    assert flag.item() == 3


def test_executor_plan_roundtrip():
    """Planner -> executor on two logical GPUs of one device; bytes follow."""
    from paper_2501_06709_b200 import PendingMove, Topology, load_boundaries, plan_hybrid
    from paper_2501_06709_b200.executor import MigrationExecutor

    pools = {0: KVPool(SMALL, 64), 1: KVPool(SMALL, 64)}
    tables = {0: BlockTable(8, 16), 1: BlockTable(8, 16)}
    ex = MigrationExecutor(pools, tables, timing=True)
    _fill(pools[0], 8)
    ex.admit(10, 0, 50)
    ex.admit(11, 0, 17)
    b10, b11 = ex.where(10).blocks.copy(), ex.where(11).blocks.copy()
    src_np = pools[0].tensor.view(torch.int16).cpu().numpy()
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9)
    bounds = load_boundaries(topo, 1.0, 1.0)
    bpt = SMALL.kv_bytes_per_token
    plan = plan_hybrid([PendingMove(10, 0, 1, 50 * bpt, 50), PendingMove(11, 0, 1, 17 * bpt, 17)],
                       bounds, topo)
    rep = ex.execute(plan)
    assert rep.bytes_moved == (4 + 2) * 16 * bpt
    assert set(rep.device_ms) == {0} and rep.device_ms[0] > 0 and rep.copy_GBps > 0
    dst_np = pools[1].tensor.view(torch.int16).cpu().numpy()
    for rid, sb in ((10, b10), (11, b11)):
        r = ex.where(rid)
        assert r.gpu == 1
        assert np.array_equal(dst_np[:, :, r.blocks], src_np[:, :, sb])
        assert np.array_equal(tables[1].rows[tables[1].slot(rid), :len(sb)].cpu().numpy(), r.blocks)
    assert pools[0].allocator.n_free == 64
    rec = ex.compact(10)
    assert rec.bytes_moved == 4 * 16 * bpt


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVM_FUZZ_SEEDS", "100"))))
def test_randomized_batches_vs_oracle(seed):
    """Random shapes (piece sizes from 1 KiB to 160 KiB, odd head counts), random
    pools and block lists, several moves of DIFFERENT shapes in one kvm_migrate
    batch (one launch), random engine / block-list placement / flags."""
    rng = np.random.default_rng(1000 + seed)
    shapes = []
    for k in range(int(rng.integers(1, 4))):
        shapes.append(ModelShape(f"r{seed}_{k}", layers=int(rng.integers(1, 5)), kv_heads=int(rng.integers(1, 9)),
                                 head_dim=int(rng.choice([8, 64, 128])), q_heads=1, d_model=64))
    pools = []
    for sh in shapes:
        nb = int(rng.integers(8, 40))
        src, dst = KVPool(sh, nb), KVPool(sh, nb)
        _fill(src, int(rng.integers(1 << 30)))
        _fill(dst, int(rng.integers(1 << 30)))
        pools.append((src, dst))
    engine = int(rng.choice([0, _native.KVM_F_ENGINE_BULK]))
    host = bool(rng.integers(2))
    moves, keep, checks = [], [], []
    flags = torch.zeros(16, dtype=torch.int32, device="cuda")
    for i in range(int(rng.integers(1, 9))):
        src, dst = pools[int(rng.integers(len(pools)))]
        free = np.flatnonzero(dst.allocator.free_mask())
        n = int(rng.integers(0, min(len(free), src.num_blocks) + 1))
        sb = rng.permutation(src.num_blocks)[:n].astype(np.int32)
        db = dst.allocator.alloc(n)
        if host:
            keep += [sb, db]
            m = _move(src, dst, sb, db, flag=flags[i:].data_ptr(), value=i + 1)
        else:
            sbd, dbd = torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()
            keep += [sbd, dbd]
            m = _move(src, dst, sbd.data_ptr(), dbd.data_ptr(), flag=flags[i:].data_ptr(), value=i + 1, n=n)
        moves.append(m)
        checks.append((src, dst, sb, db))
    expect = {}
    for src, dst, sb, db in checks:  # oracle applies the moves in order on host copies
        key = id(dst)
        if key not in expect:
            expect[key] = (dst, dst.tensor.view(torch.int16).cpu().numpy())
        orc.migrate(src.tensor.view(torch.int16).cpu().numpy(), _desc(src), expect[key][1], _desc(dst), sb, db)
    cap = int(rng.choice([0, 0, 0, 1, 5, 37]))   # copy SM budget (KVM_F_MAX_SMS), drawn last
    _run(moves, engine | (_native.KVM_F_BLOCKS_ON_HOST if host else 0) | _native.KVM_F_MAX_SMS(cap))
    for dst, exp in expect.values():
        assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)
    assert flags[:len(moves)].cpu().tolist() == list(range(1, len(moves) + 1))


def test_wait_flag_timeout_reports_instead_of_hanging():
    flag = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    _native.check(_native.lib().kvm_wait_flag_timeout(ctypes.c_void_p(flag.data_ptr()), 5, 20_000_000,
                                                      ctypes.c_void_p(flag.data_ptr() + 4),
                                                      ctypes.c_void_p(s.cuda_stream)))
    s.synchronize()   # returns after ~20 ms although the flag never reaches 5
    assert flag.cpu().tolist() == [0, 1]


def test_compact_stream_ordered_back_to_back():
    """compact(stream_ordered=True) returns before the copy finishes, with the
    residency already updated; back-to-back calls stay correct because every
    launch on the pool is queued on the executor's ordered stream, and each
    call's rewritten table row is read back (kvm_read_back) in stream order."""
    from paper_2501_06709_b200.executor import MigrationExecutor

    pool = KVPool(SMALL, 96)
    table = BlockTable(2, 16)
    ex = MigrationExecutor({0: pool}, {0: table})
    _fill(pool, 3)
    pool.allocator.take(range(0, 96, 3))     # scatter the free blocks
    ex.admit(5, 0, 200)
    orig_blocks = ex.where(5).blocks.copy()
    orig = pool.tensor.view(torch.int16)[:, :, torch.from_numpy(orig_blocks).long().cuda()].clone()
    rows = [torch.empty(16, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    recs, expect = [], []
    for i in range(6):
        recs.append(ex.compact(5, row_out=rows[i & 1], stream_ordered=True))
        expect.append(ex.where(5).blocks.copy())
        if i >= 1:
            recs[i - 1].done.synchronize()
            assert np.array_equal(rows[(i - 1) & 1].numpy()[:len(expect[i - 1])], expect[i - 1])
    recs[-1].done.synchronize()
    assert np.array_equal(rows[1].numpy()[:len(expect[-1])], expect[-1])
    now = pool.tensor.view(torch.int16)[:, :, torch.from_numpy(ex.where(5).blocks).long().cuda()]
    assert torch.equal(now, orig)


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
@pytest.mark.parametrize("n", [1, 127, 128, 129, 255, 256, 257, 300])
@pytest.mark.parametrize("consumers", ["none", "device", "host_flag", "sys_scope"])
def test_single_move_launch_class(engine, n, consumers):
    """One-move launches use the small parameter block: host lists of <= 256
    blocks ride inline (no staging copy), larger ones are staged; moves with no
    table row / flags skip completion accounting; completion stores are .gpu
    scope when every written pointer is this GPU's memory, .sys for a flag in
    pinned host memory or with KVM_F_SYS_SCOPE.  Bytes, row and flags exact."""
    nb = 2 * n + 8
    src, dst = KVPool(SMALL, nb), KVPool(SMALL, nb)
    _fill(src, n)
    _fill(dst, n + 1)
    rng = np.random.default_rng(n)
    sb = rng.permutation(nb)[:n].astype(np.int32)
    dst.allocator.take(rng.permutation(nb)[:3])
    db = dst.allocator.alloc(n)
    exp = dst.tensor.view(torch.int16).cpu().numpy()
    row_exp = orc.migrate(src.tensor.view(torch.int16).cpu().numpy(), _desc(src), exp, _desc(dst), sb, db)
    table = BlockTable(2, n + 4)
    lflags = torch.zeros(SMALL.layers, dtype=torch.int32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    flags = _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine]
    if consumers == "none":
        m = _move(src, dst, sb, db)
    elif consumers == "host_flag":
        flag = torch.zeros(1, dtype=torch.int32).pin_memory()
        m = _move(src, dst, sb, db, table.row_ptr(1), flag.data_ptr(), lflags.data_ptr(), value=7)
    else:
        m = _move(src, dst, sb, db, table.row_ptr(1), flag.data_ptr(), lflags.data_ptr(), value=7)
        if consumers == "sys_scope":
            flags |= _native.KVM_F_SYS_SCOPE
    _run([m], flags)
    assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)
    if consumers != "none":
        assert np.array_equal(table.rows[table.slot(1), :n].cpu().numpy(), row_exp)
        assert flag.item() == 7
        assert lflags.cpu().tolist() == [7] * SMALL.layers
    # back to back on one stream, alternating inline / staged: no slot reuse hazard
    for k in range(40):
        _native.check(_native.lib().kvm_migrate(ctypes.byref(_move(src, dst, sb, db)), 1, flags, _stream()))
    torch.cuda.synchronize()
    assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)


def test_executor_stream_ordered_chain():
    """execute(stream_ordered=True): no host wait; residencies switch at issue,
    so the same request can be moved again at once (0 -> 1 -> 2); a consumer
    stream that waits on `report.done` sees the final bytes and table row."""
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    pools = {g: KVPool(SMALL, 64) for g in range(3)}
    tables = {g: BlockTable(8, 16) for g in range(3)}
    ex = MigrationExecutor(pools, tables)
    _fill(pools[0], 21)
    ex.admit(5, 0, 70)
    ex.admit(6, 0, 33)
    src_np = pools[0].tensor.view(torch.int16).cpu().numpy()
    b5, b6 = ex.where(5).blocks.copy(), ex.where(6).blocks.copy()
    bpt = SMALL.kv_bytes_per_token
    r1 = ex.execute([PlannedMove(PendingMove(5, 0, 1, 70 * bpt, 70), KV_TRANSFER),
                     PlannedMove(PendingMove(6, 0, 2, 33 * bpt, 33), KV_TRANSFER)], stream_ordered=True)
    assert ex.where(5).gpu == 1 and ex.where(6).gpu == 2
    assert set(r1.src_done) == {0} and set(r1.done) == {0}   # all logical GPUs share cuda:0
    assert r1.records[0].done is r1.done[0]
    # the freed source blocks are reused at once by a new request, written on the executor's stream
    ex.admit(7, 0, 16 * 7)
    with torch.cuda.stream(ex.stream(0)):
        pools[0].tensor[:, :, ex.where(7).blocks.tolist()] = 0
    r2 = ex.execute([PlannedMove(PendingMove(5, 1, 2, 70 * bpt, 70), KV_TRANSFER)], stream_ordered=True)
    consumer = torch.cuda.Stream()
    consumer.wait_event(r2.done[0])
    with torch.cuda.stream(consumer):
        got5 = pools[2].tensor[:, :, ex.where(5).blocks.tolist()].clone()
        got6 = pools[2].tensor[:, :, ex.where(6).blocks.tolist()].clone()
        row5 = tables[2].rows[tables[2].slot(5), :len(b5)].clone()
    consumer.synchronize()
    assert np.array_equal(got5.view(torch.int16).cpu().numpy(), src_np[:, :, b5])
    assert np.array_equal(got6.view(torch.int16).cpu().numpy(), src_np[:, :, b6])
    assert np.array_equal(row5.cpu().numpy(), ex.where(5).blocks)
    assert pools[1].allocator.n_free == 64


def test_batch_write_write_and_read_write_conflicts_rejected():
    """Host block lists: a launch may not write one destination block twice, nor
    read a block another move of the same launch writes; rejected before any
    byte moves (ValueError), legal batches still run."""
    nb = 32
    a, b = KVPool(SMALL, nb), KVPool(SMALL, nb)
    _fill(a, 1)
    _fill(b, 2)
    before = (a.tensor.view(torch.int16).clone(), b.tensor.view(torch.int16).clone())
    flags = _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK
    arrs = lambda *xs: [np.array(x, dtype=np.int32) for x in xs]  # noqa: E731
    s1, d1, s2, d2 = arrs([1, 2], [5, 6], [3, 4], [6, 7])          # dst 6 written twice
    with pytest.raises(ValueError, match="written twice"):
        _run([_move(a, b, s1, d1), _move(a, b, s2, d2)], flags)
    s1, d1, s2, d2 = arrs([1, 2], [5, 6], [6, 9], [10, 11])        # move 2 reads b:6 that move 1 writes
    with pytest.raises(ValueError, match="read and written"):
        _run([_move(a, b, s1, d1), _move(b, a, s2, d2)], flags)
    s1, d1 = arrs([1, 2, 3], [9, 2, 8])                            # compaction-style self overlap
    with pytest.raises(ValueError, match="read and written"):
        _run([_move(a, a, s1, d1)], flags)
    assert torch.equal(a.tensor.view(torch.int16), before[0]) and torch.equal(b.tensor.view(torch.int16), before[1])
    s1, d1, s2, d2 = arrs([1, 2], [5, 6], [1, 2], [7, 8])          # the same source read twice is fine
    _run([_move(a, b, s1, d1), _move(a, b, s2, d2)], flags)
    got = b.tensor.view(torch.int16)
    assert torch.equal(got[:, :, [5, 6]], before[0][:, :, [1, 2]]) and torch.equal(got[:, :, [7, 8]],
                                                                                    before[0][:, :, [1, 2]])


def test_executor_layer_flags_feed_a_pipelined_decode():
    """execute(stream_ordered=True, layer_flags=True): the destination decode
    starts right away, layer by layer behind the copy, and equals decoding the
    request where it was."""
    from paper_2501_06709_b200.attention import paged_decode
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    shape = ModelShape("lf", layers=6, kv_heads=2, head_dim=128, q_heads=8, d_model=1024)
    pools = {0: KVPool(shape, 200, dtype=torch.bfloat16), 1: KVPool(shape, 200, dtype=torch.bfloat16)}
    g = torch.Generator(device="cuda").manual_seed(4)
    pools[0].tensor.copy_(torch.randn(pools[0].view_shape, generator=g, device="cuda").to(torch.bfloat16))
    ex = MigrationExecutor(pools)
    ex.admit(9, 0, 2500)
    q = torch.randn(shape.layers, 1, 8, 128, generator=g, device="cuda").to(torch.bfloat16)
    lens = torch.tensor([2500], dtype=torch.int32, device="cuda")
    ref = paged_decode(pools[0], q, torch.from_numpy(ex.where(9).blocks)[None].contiguous().cuda(), lens)
    torch.cuda.synchronize()
    rep = ex.execute([PlannedMove(PendingMove(9, 0, 1, 2500 * shape.kv_bytes_per_token, 2500), KV_TRANSFER)],
                     stream_ordered=True, layer_flags=True)
    rec = rep.records[0]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    dec = torch.cuda.Stream()
    out = paged_decode(pools[1], q, torch.from_numpy(ex.where(9).blocks)[None].contiguous().cuda(), lens,
                       stream=dec, layer_flags=rec.layer_flags[9], timeout_ns=5_000_000_000, err_word=err)
    torch.cuda.synchronize()
    assert err.item() == 0 and rec.layer_flags[9].cpu().tolist() == [1] * shape.layers
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def test_block_table_released_rows_reset_on_reuse():
    t = BlockTable(2, 8)
    t.set_host(1, np.arange(6, dtype=np.int32))
    t.rows[t.slot(1), :6] = torch.arange(6, dtype=torch.int32, device="cuda")
    s = t.slot(1)
    t.drop(1)                                   # no device work in the release
    assert t.rows[s, :6].tolist() == list(range(6))
    t.set_host(2, np.array([9, 8], dtype=np.int32))
    t.set_host(3, np.array([7], dtype=np.int32))
    assert {t.slot(2), t.slot(3)} == {0, 1}
    assert t.rows[s].tolist() == [-1] * 8       # the reused slot was reset first


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_batches_of_empty_moves_without_consumers(engine):
    """Found by the foreign-layout fuzz: a launch whose moves are all empty and
    have no table row / flags needs no staging slot at all (it used to
    dereference the missing slot)."""
    a, b = KVPool(SMALL, 8), KVPool(SMALL, 8)
    e = np.zeros(0, dtype=np.int32)
    for n in (1, 2, 5):
        _run([_move(a, b, e, e) for _ in range(n)], _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine])
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _run([_move(a, b, e, e), _move(a, b, e, e, flag=flag.data_ptr(), value=3)],
         _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine])
    assert flag.item() == 3


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVM_FUZZ_SEEDS", "100"))))
def test_same_pool_batches_randomized(seed):
    """Random same-pool batches (compaction-like): a batch with a write-write or
    read-write block conflict is rejected with nothing moved; a conflict-free
    batch equals the oracle."""
    rng = np.random.default_rng(3000 + seed)
    nb = int(rng.integers(6, 30))
    pool = KVPool(SMALL, nb)
    _fill(pool, seed)
    before = pool.tensor.view(torch.int16).cpu().numpy()
    moves, keep, writes, reads = [], [], [], []
    for _ in range(int(rng.integers(1, 5))):
        n = int(rng.integers(0, 5))
        sb = rng.integers(0, nb, n).astype(np.int32)
        db = rng.integers(0, nb, n).astype(np.int32)
        keep += [sb, db]
        reads += sb.tolist()
        writes += db.tolist()
        moves.append(_move(pool, pool, sb, db))
    conflict = len(set(writes)) != len(writes) or bool(set(writes) & set(reads))
    flags = _native.KVM_F_BLOCKS_ON_HOST | (_native.KVM_F_ENGINE_BULK if rng.integers(2) else 0)
    if conflict:
        with pytest.raises(ValueError):
            _run(moves, flags)
        assert np.array_equal(pool.tensor.view(torch.int16).cpu().numpy(), before)
    else:
        exp = before.copy()
        for k in range(0, len(keep), 2):
            orc.migrate(before, _desc(pool), exp, _desc(pool), keep[k], keep[k + 1])
        _run(moves, flags)
        assert np.array_equal(pool.tensor.view(torch.int16).cpu().numpy(), exp)


def test_executor_validation_leaves_pools_tables_untouched():
    """a plan whose token_transfer targets an fp16 pool (the re-prefill
    engine writes bf16) or whose request is wider than the destination block
    table fails before anything is reserved, launched or given a table row."""
    from paper_2501_06709_b200 import PendingMove
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.planner import KV_TRANSFER, TOKEN_TRANSFER, PlannedMove
    from paper_2501_06709_b200.reprefill import ReprefillEngine

    pools = {0: KVPool(SMALL, 64), 1: KVPool(SMALL, 64)}          # fp16 pools
    tables = {0: BlockTable(8, 16), 1: BlockTable(8, 4)}          # GPU 1 rows hold 4 blocks
    ex = MigrationExecutor(pools, tables, reprefill=ReprefillEngine(SMALL, [0]))
    _fill(pools[0], 3)
    ex.admit(1, 0, 40)      # 3 blocks
    ex.admit(2, 0, 40)
    ex.admit(3, 0, 100)     # 7 blocks > 4
    before = pools[1].tensor.view(torch.int16).clone()
    launches = _native.launch_count()
    free = [p.allocator.n_free for p in pools.values()]
    for plan in ([PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER),
                  PlannedMove(PendingMove(2, 0, 1, 0, 40), TOKEN_TRANSFER)],
                 [PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER),
                  PlannedMove(PendingMove(3, 0, 1, 0, 100), KV_TRANSFER)]):
        with pytest.raises((ConfigError, RequestTooLarge)):
            ex.execute(plan)
        torch.cuda.synchronize()
        assert [p.allocator.n_free for p in pools.values()] == free
        assert _native.launch_count() == launches and torch.equal(pools[1].tensor.view(torch.int16), before)
        assert not tables[1].has(1) and not tables[1].has(2) and not tables[1].has(3)
        assert {ex.where(r).gpu for r in (1, 2, 3)} == {0}
    rep = ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER)])
    assert rep.records[0].requests == [1] and ex.where(1).gpu == 1 and tables[1].has(1)


@pytest.mark.parametrize("tracked", [True, False])
def test_tile_queue_across_slot_reuse(tracked):
    """The bulk engine's guided tile queue (>= 8 tiles per CTA) counts on one of two words of a staging
    slot and zeroes the other for the slot's next launch.  40 back-to-back launches of varying size
    (queue and static partitions mixed, every staging slot reused) on one stream: each launch copies
    the request to fresh blocks, and the final blocks hold the original bytes, the table row and the
    done flag are the last launch's."""
    shape = ModelShape("q7b", layers=8, kv_heads=32, head_dim=128, q_heads=32, d_model=4096)   # 128 KiB pieces
    nb = 400
    pool = KVPool(shape, nb)
    _fill(pool, 17)
    table = BlockTable(2, 64)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(3)
    sizes = [40, 3, 64, 19, 1, 33, 64, 7] * 5          # 4 tiles x 16 planes per block: 64 .. 4096 tiles
    cur = np.sort(rng.permutation(nb)[:max(sizes)]).astype(np.int32)   # the request: 64 blocks
    orig = pool.tensor.view(torch.int16)[:, :, torch.from_numpy(cur).long().cuda()].clone()
    keep = [orig]
    for i, n in enumerate(sizes):
        # move the first n blocks of the request to n fresh blocks (the rest stays), other blocks untouched
        used = set(cur.tolist())
        free = np.array([b for b in rng.permutation(nb) if b not in used][:n], dtype=np.int32)
        src = cur[:n].copy()
        m = _move(pool, pool, src, free, table.row_ptr(1) if tracked else 0, flag.data_ptr() if tracked else 0,
                  value=i + 1)
        keep += [src, free]
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1,
                                                _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                                _stream()))
        cur = np.concatenate([free, cur[n:]]).astype(np.int32)
    torch.cuda.synchronize()
    now = pool.tensor.view(torch.int16)[:, :, torch.from_numpy(cur).long().cuda()]
    assert torch.equal(now, orig)
    if tracked:
        assert int(flag.item()) == len(sizes)
        assert np.array_equal(table.rows[table.slot(1), :sizes[-1]].cpu().numpy(), keep[-1])


@pytest.mark.parametrize("seed", range(max(1, int(os.environ.get("KVM_FUZZ_SEEDS", "100")) // 5)))
def test_randomized_queue_sized_batches_vs_oracle(seed):
    """Random batches large enough for the bulk engine's guided tile queue (>= 8 tiles per CTA, i.e.
    >= 2 * 148 * 4 tiles) and around its threshold: 32-160 KiB pieces, 1-6 moves of mixed pools in one
    launch, random block-list placement, per-move table row / done flag / layer flags or none; whole
    destination pools byte-exact against the C oracle, flags and rows exact."""
    rng = np.random.default_rng(5000 + seed)
    sh = ModelShape(f"q{seed}", layers=int(rng.integers(2, 9)), kv_heads=int(rng.choice([8, 16, 32, 40])),
                    head_dim=128, q_heads=8, d_model=1024)
    tpb = 2 * sh.layers * ((sh.piece_bytes + 32767) // 32768)            # tiles per block
    nb = int(min(480, max(64, (2 * 1184 // tpb) + 16)))
    pools = [(KVPool(sh, nb), KVPool(sh, nb)) for _ in range(int(rng.integers(1, 3)))]
    for s, d in pools:
        _fill(s, int(rng.integers(1 << 30)))
        _fill(d, int(rng.integers(1 << 30)))
    host = bool(rng.integers(2))
    table = BlockTable(8, nb)
    ctrl = torch.zeros(8 + 8 * sh.layers, dtype=torch.int32, device="cuda")
    moves, keep, checks, rows = [], [], [], []
    for i in range(int(rng.integers(1, 7))):
        src, dst = pools[int(rng.integers(len(pools)))]
        free = np.flatnonzero(dst.allocator.free_mask())
        n = int(rng.integers(0, min(len(free), nb) + 1))
        sb = rng.permutation(nb)[:n].astype(np.int32)
        db = dst.allocator.alloc(n)
        kind = int(rng.integers(3))    # 0 untracked, 1 row + flag, 2 row + flag + layer flags
        row = table.row_ptr(i) if kind else 0
        flag = ctrl[i:].data_ptr() if kind else 0
        lf = ctrl[8 + i * sh.layers:].data_ptr() if kind == 2 else 0
        if host:
            keep += [sb, db]
            m = _move(src, dst, sb, db, row, flag, lf, value=i + 1)
        else:
            sbd, dbd = torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()
            keep += [sbd, dbd]
            m = _move(src, dst, sbd.data_ptr(), dbd.data_ptr(), row, flag, lf, value=i + 1, n=n)
        moves.append(m)
        checks.append((src, dst, sb, db))
        rows.append((i, kind, db))
    expect = {}
    for src, dst, sb, db in checks:
        if id(dst) not in expect:
            expect[id(dst)] = (dst, dst.tensor.view(torch.int16).cpu().numpy())
        orc.migrate(src.tensor.view(torch.int16).cpu().numpy(), _desc(src), expect[id(dst)][1], _desc(dst), sb, db)
    cap = int(rng.choice([0, 0, 2, 16, 64]))     # copy SM budget (KVM_F_MAX_SMS), drawn last
    _run(moves, _native.KVM_F_ENGINE_BULK | (_native.KVM_F_BLOCKS_ON_HOST if host else 0) | _native.KVM_F_MAX_SMS(cap))
    for dst, exp in expect.values():
        assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)
    c = ctrl.cpu().numpy()
    for i, kind, db in rows:
        if kind:
            assert c[i] == i + 1
            assert np.array_equal(table.rows[table.slot(i), :len(db)].cpu().numpy(), db)
        if kind == 2:
            assert (c[8 + i * sh.layers: 8 + (i + 1) * sh.layers] == i + 1).all()   # layer flags carry the value


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
@pytest.mark.parametrize("max_sms", [1, 3, 16, 148, 255])
def test_copy_sm_budget_bit_exact(engine, max_sms):
    """KVM_F_MAX_SMS(n): the copy on at most n SMs' worth of CTAs (down to one CTA, where the bulk
    engine's tile queue takes over from the second chunk) is byte-exact against the oracle over the
    whole destination pool, table row and flag included; the executor's copy_sms applies it."""
    shape = ModelShape("cap", layers=4, kv_heads=8, head_dim=128, q_heads=8, d_model=1024)   # 32 KiB pieces
    nb = 160
    src, dst = KVPool(shape, nb), KVPool(shape, nb)
    _fill(src, 21)
    _fill(dst, 22)
    rng = np.random.default_rng(max_sms)
    sb = rng.permutation(nb)[:120].astype(np.int32)
    dst.allocator.take(rng.permutation(nb)[:30])
    db = dst.allocator.alloc(120)
    exp = dst.tensor.view(torch.int16).cpu().numpy()
    orc.migrate(src.tensor.view(torch.int16).cpu().numpy(), _desc(src), exp, _desc(dst), sb, db)
    table = BlockTable(2, 128)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    m = _move(src, dst, sb, db, table.row_ptr(3), flag.data_ptr(), value=7)
    _run([m], _native.KVM_F_BLOCKS_ON_HOST | ENGINES[engine] | _native.KVM_F_MAX_SMS(max_sms))
    assert np.array_equal(dst.tensor.view(torch.int16).cpu().numpy(), exp)
    assert int(flag.item()) == 7
    assert np.array_equal(table.rows[table.slot(3), :120].cpu().numpy(), db)


def test_executor_copy_sms():
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    pools = {0: KVPool(SMALL, 64), 1: KVPool(SMALL, 64)}
    for i, p in pools.items():
        _fill(p, 30 + i)
    ex = MigrationExecutor(pools, {0: BlockTable(4, 32), 1: BlockTable(4, 32)}, copy_sms=2)
    ex.admit(9, 0, 300)
    before = pools[0].tensor.view(torch.int16)[:, :, torch.from_numpy(ex.where(9).blocks).long().cuda()].clone()
    ex.execute([PlannedMove(PendingMove(9, 0, 1, 0, 300), KV_TRANSFER)])
    after = pools[1].tensor.view(torch.int16)[:, :, torch.from_numpy(ex.where(9).blocks).long().cuda()]
    assert ex.where(9).gpu == 1 and torch.equal(before, after)
    with pytest.raises(ConfigError):
        MigrationExecutor(pools, copy_sms=256)


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")   # nothing was captured: the point of the test
def test_graph_capture_is_rejected_not_corrupted():
    """kvm_migrate (and the re-prefill entry points) refuse a stream under CUDA-graph capture with
    KVM_ERR_UNSUPPORTED instead of baking per-launch staging / queue state into a graph whose replays
    would race the host's bookkeeping; the same move runs normally afterwards."""
    from paper_2501_06709_b200.errors import KvmUnsupported
    from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights

    src, dst = KVPool(SMALL, 16), KVPool(SMALL, 16)
    _fill(src, 1)
    sb, db = np.arange(4, dtype=np.int32), np.arange(8, 12, dtype=np.int32)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(KvmUnsupported):
        with torch.cuda.graph(g, stream=s):
            m = _move(src, dst, sb, db)
            _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST,
                                                    ctypes.c_void_p(s.cuda_stream)))
    shape = ModelShape("g", layers=1, kv_heads=1, head_dim=128, q_heads=1, d_model=64)
    pool = KVPool(shape, 4, dtype=torch.bfloat16)
    x, w = synthetic_hidden(shape, 16, 0, seed=1), synthetic_weights(shape, 0, with_q=False, seed=2)
    blocks = torch.arange(1, dtype=torch.int32, device="cuda")
    g2 = torch.cuda.CUDAGraph()
    with pytest.raises(KvmUnsupported):
        with torch.cuda.graph(g2, stream=s):
            reprefill(pool, x, w, blocks, stream=s)
    torch.cuda.synchronize()
    _run([_move(src, dst, sb, db)], _native.KVM_F_BLOCKS_ON_HOST)
    assert torch.equal(dst.tensor[:, :, 8:12].view(torch.int16), src.tensor[:, :, 0:4].view(torch.int16))
