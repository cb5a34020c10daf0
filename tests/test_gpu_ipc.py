"""One process per GPU, exercised on ONE B200: two ranks (gloo for the control
plane) each own a pool; rank 0 maps rank 1's pool, block table and flag
words through CUDA IPC and pushes a request into it with the migration
kernel.  This is the exact multi-GPU code path (peer-mapped stores, fused
table rewrite, system-scope flags, kvm_wait_flag on the receiver) minus the
NVLink hop, which needs a second GPU."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, engine_flag, result_q):
    import ctypes
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import kvmig_oracle as orc
    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.dist import exchange_objects
    from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        torch.cuda.set_device(0)
        shape = ModelShape("ipc", layers=3, kv_heads=8, head_dim=64, q_heads=8, d_model=512)
        nb = 40
        pool = KVPool(shape, nb, device=0)
        g = torch.Generator(device="cuda:0").manual_seed(100 + rank)
        pool.tensor.view(torch.int16).copy_(torch.randint(-2 ** 15, 2 ** 15, pool.view_shape, generator=g,
                                                          device="cuda:0", dtype=torch.int16))
        table = BlockTable(2, 16, device=0)
        words = torch.zeros(8, dtype=torch.int32, device="cuda:0")  # [0]=done, [1..3]=layer flags
        lib = _native.lib()

        def export(ptr):
            h = (ctypes.c_ubyte * 64)()
            off = ctypes.c_int64()
            _native.check(lib.kvm_ipc_export(ctypes.c_void_p(ptr), h, ctypes.byref(off)))
            return bytes(h), off.value

        rng = np.random.default_rng(5)
        sb = rng.permutation(nb)[:9].astype(np.int32)
        pool.allocator.take(rng.permutation(nb)[:15])
        db = pool.allocator.alloc(9)
        before = pool.tensor.view(torch.int16).cpu().numpy()
        info = exchange_objects((pool.ipc_handle(), export(table.rows.data_ptr()), export(words.data_ptr()),
                                 db.tolist(), before if rank == 0 else None))
        torch.cuda.synchronize()
        if rank == 0:
            (ph, po), (th, to), (wh, wo), peer_db, _ = info[1]
            peer = KVPool.from_ipc(shape, nb, 0, ph, po)
            tptr, wptr = ctypes.c_void_p(), ctypes.c_void_p()
            _native.check(lib.kvm_ipc_import(0, (ctypes.c_ubyte * 64).from_buffer_copy(th), to, ctypes.byref(tptr)))
            _native.check(lib.kvm_ipc_import(0, (ctypes.c_ubyte * 64).from_buffer_copy(wh), wo, ctypes.byref(wptr)))
            pdb = np.asarray(peer_db, dtype=np.int32)
            m = _native.Move()
            m.src_pool, m.dst_pool, m.n_blocks, m.done_value = pool.pool_id, peer.pool_id, 9, 5
            m.src_blocks, m.dst_blocks = sb.ctypes.data, pdb.ctypes.data
            m.dst_table_row = tptr.value  # rank 1's table row 0
            m.done_flag = wptr.value
            m.layer_flags = wptr.value + 4
            s = torch.cuda.Stream()
            _native.check(lib.kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | engine_flag,
                                          ctypes.c_void_p(s.cuda_stream)))
            s.synchronize()
            dist.barrier()
            ok = True
        else:
            s = torch.cuda.Stream()
            _native.check(lib.kvm_wait_flag(ctypes.c_void_p(words.data_ptr()), 5, ctypes.c_void_p(s.cuda_stream)))
            s.synchronize()   # returns only once rank 0's kernel published the flag
            dist.barrier()
            src0 = info[0][4]
            exp = before.copy()
            d = orc.desc(3, 8, 64, 16, nb)
            sb0 = np.random.default_rng(5).permutation(nb)[:9].astype(np.int32)
            row = orc.migrate(src0, d, exp, d, sb0, db)
            got = pool.tensor.view(torch.int16).cpu().numpy()
            ok = bool(np.array_equal(got, exp)) and bool(np.array_equal(table.rows[0, :9].cpu().numpy(), row)) \
                and words[:4].cpu().tolist() == [5, 5, 5, 5]
        result_q.put((rank, ok, ""))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        result_q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_two_process_ipc_push(engine):
    import torch.multiprocessing as mp

    from paper_2501_06709_b200 import _native

    flag = {"ldg": 0, "bulk": _native.KVM_F_ENGINE_BULK}[engine]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, flag, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank} failed:\n{err}"


def _split_worker(rank, world, port, result_q):
    """Rank 0 owns the source pool; rank 1 imports it through CUDA IPC and runs the
    fused split migration on its own GPU: the prefix is PULLED from the peer
    pool by the re-prefill GEMM's idle warps, the suffix recomputed locally."""
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2501_06709_b200.dist import exchange_objects
    from paper_2501_06709_b200.kvcache import KVPool, ModelShape
    from paper_2501_06709_b200.reprefill import synthetic_hidden, synthetic_weights
    from paper_2501_06709_b200.split import make_split, split_migrate_fused

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        shape = ModelShape("ipcs", layers=3, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
        plan = make_split(600, 88)
        nb = plan.total_blocks + 6
        pool = KVPool(shape, nb, device=0, dtype=torch.bfloat16)
        pool.tensor.view(torch.int16).copy_(torch.randint(-2 ** 15, 2 ** 15, pool.view_shape, device="cuda:0",
                                                          dtype=torch.int16,
                                                          generator=torch.Generator(device="cuda:0")
                                                          .manual_seed(50 + rank)))
        torch.cuda.synchronize()
        sb = torch.randperm(nb, generator=torch.Generator().manual_seed(3))[:plan.total_blocks].to(torch.int32)
        info = exchange_objects((pool.ipc_handle(), pool.tensor.view(torch.int16).cpu() if rank == 0 else None))
        ok = True
        if rank == 1:
            src = KVPool.from_ipc(shape, nb, 0, *info[0][0], dtype=torch.bfloat16)
            db = torch.from_numpy(pool.allocator.alloc(plan.total_blocks)).cuda()
            x = synthetic_hidden(shape, plan.suffix, 0, seed=8)
            w = synthetic_weights(shape, 0, with_q=False, seed=9)
            split_migrate_fused(src, pool, sb.cuda(), db, plan, x, w)
            torch.cuda.synchronize()
            pre = plan.prefix_blocks
            got = pool.tensor.view(torch.int16)[:, :, db[:pre].long()].cpu()
            ok = bool(torch.equal(got, info[0][1][:, :, sb[:pre].long()]))
            toks = torch.arange(plan.prefix_tokens, 600, device="cuda")
            ref = torch.einsum("tk,lnk->ltn", x.float(), w.float())
            k = pool.tensor[:, 0, db.long()[toks // 16], toks % 16].reshape(shape.layers, plan.suffix, -1).float()
            ok = ok and bool(torch.allclose(k, ref[:, :, :shape.kv_cols], atol=1e-2, rtol=1.6e-2))
        dist.barrier()   # rank 0 keeps its pool alive until rank 1 has pulled
        result_q.put((rank, ok, ""))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        result_q.put((rank, False, traceback.format_exc()))


def test_two_process_split_pull():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank} failed:\n{err}"


def _vllm_worker(rank, world, port, result_q):
    """Rank 1 plays a vLLM instance: its FlashAttention-layout per-layer caches
    are views into ONE allocation (as vLLM carves them).  Rank 0 maps them with
    StridedKVPool.from_ipc (one mapping for all layers) and pushes a request
    from its native pool straight into the peer's vLLM cache."""
    import ctypes
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.dist import exchange_objects
    from paper_2501_06709_b200.foreign import StridedKVPool, vllm_cache_shape
    from paper_2501_06709_b200.kvcache import KVPool, ModelShape

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        shape = ModelShape("vipc", layers=3, kv_heads=4, head_dim=64, q_heads=4, d_model=256)
        nb, n = 30, 7
        g = torch.Generator(device="cuda:0").manual_seed(7)
        if rank == 0:
            pool = KVPool(shape, nb)
            pool.tensor.view(torch.int16).copy_(torch.randint(-2 ** 15, 2 ** 15, pool.view_shape, generator=g,
                                                              device="cuda:0", dtype=torch.int16))
            torch.cuda.synchronize()
            info = exchange_objects(None)
            handles, kv_stride, block_stride, dst_blocks = info[1]
            peer = StridedKVPool.from_ipc(shape, nb, 0, handles, kv_stride, block_stride, dtype=torch.float16,
                                          layout="flash_attn")
            assert len(peer._mapped) == 1
            sb = np.arange(3, 3 + n, dtype=np.int32)
            db = np.asarray(dst_blocks, dtype=np.int32)
            m = _native.Move()
            m.src_pool, m.dst_pool, m.n_blocks, m.done_value = pool.pool_id, peer.pool_id, n, 1
            m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
            _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1,
                                                    _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK,
                                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
            torch.cuda.synchronize()
            exchange_objects(pool.tensor[:, :, torch.from_numpy(sb).long()].view(torch.int16).cpu().numpy())
            peer.close()
            ok = True
        else:
            per = vllm_cache_shape("flash_attn", nb, 16, shape.kv_heads, shape.head_dim)
            numel = int(np.prod(per))
            raw = torch.zeros(shape.layers * numel, dtype=torch.float16, device="cuda:0")
            caches = [raw[l * numel:(l + 1) * numel].view(per) for l in range(shape.layers)]
            mine = StridedKVPool.from_vllm(caches, "flash_attn", name="vipc")
            dst_blocks = [29, 0, 11, 5, 17, 2, 23]
            torch.cuda.synchronize()
            exchange_objects((mine.ipc_handles(), mine.kv_stride, mine.block_stride, dst_blocks))
            sent = exchange_objects(None)[0]
            got = np.stack([np.stack([np.stack([mine.piece(l, kv, b).view(torch.int16).cpu().numpy()
                                                for b in dst_blocks]) for kv in range(2)])
                            for l in range(shape.layers)])
            ok = bool(np.array_equal(got, sent))
        result_q.put((rank, ok, ""))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        result_q.put((rank, False, traceback.format_exc()))


def test_two_process_push_into_peer_vllm_cache():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vllm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank} failed:\n{err}"
