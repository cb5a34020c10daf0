"""CPU-only multi-process tests (gloo, world_size 2) of the host side of the
one-process-per-GPU path: rank bookkeeping, the ring pattern, the control-
plane exchange of (IPC handle, offset) and destination block lists, and the
max-over-ranks timing reduction."""
import os
import socket


from paper_2501_06709_b200.dist import RankInfo, ring_pairs


def test_ring_pairs_and_rank_info():
    assert ring_pairs(1) == []
    assert ring_pairs(2) == [(0, 1), (1, 0)]
    assert ring_pairs(8)[-1] == (7, 0)
    r = RankInfo(rank=3, world=4, local_rank=3)
    assert (r.send_to, r.recv_from) == (0, 2)
    # every GPU sends exactly one and receives exactly one request
    for n in (2, 4, 8):
        srcs = [s for s, _ in ring_pairs(n)]
        dsts = [d for _, d in ring_pairs(n)]
        assert sorted(srcs) == sorted(dsts) == list(range(n))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2501_06709_b200.dist import allreduce_max, exchange_handles, exchange_objects, RankInfo

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        ri = RankInfo(rank, world, rank)
        fake_handle = bytes([rank]) * 64
        hs = exchange_handles(fake_handle, 4096 * rank)
        ok = [h == bytes([r]) * 64 and o == 4096 * r for r, (h, o) in enumerate(hs)]
        # the destination allocates its blocks and the source learns them
        my_dst_blocks = list(range(100 * rank, 100 * rank + 5))
        allb = exchange_objects(my_dst_blocks)
        peer_blocks = allb[ri.send_to]
        mx = allreduce_max(1.5 + rank)
        q.put((rank, all(ok), peer_blocks == list(range(100 * ri.send_to, 100 * ri.send_to + 5)), mx))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, False, traceback.format_exc(), None))


def test_two_rank_control_plane_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=30)
    for rank, handles_ok, blocks_ok, mx in res:
        assert handles_ok is True, blocks_ok
        assert blocks_ok is True
        assert mx == 2.5  # max over ranks


def _ring_worker(rank, world, port, q):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2501_06709_b200.dist import RankInfo, collective_ring_exchange

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        ri = RankInfo(rank, world, rank)
        g = torch.Generator().manual_seed(rank)
        pool = torch.randint(-2 ** 15, 2 ** 15, (2, 2, 12, 16, 2, 8), generator=g, dtype=torch.int16)
        before = pool.clone()
        send = torch.tensor([1, 7, 3], dtype=torch.int64)
        recv = torch.tensor([10, 0, 5], dtype=torch.int64)
        collective_ring_exchange(pool, send, recv, ri)
        peer = torch.randint(-2 ** 15, 2 ** 15, (2, 2, 12, 16, 2, 8), generator=torch.Generator().manual_seed(
            ri.recv_from), dtype=torch.int16)
        ok = torch.equal(pool[:, :, recv], peer[:, :, send])
        untouched = [b for b in range(12) if b not in (10, 0, 5)]
        ok = ok and torch.equal(pool[:, :, untouched], before[:, :, untouched])
        q.put((rank, bool(ok), ""))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, False, traceback.format_exc()))


def test_collective_ring_baseline_gloo():
    """The NCCL-style comparison baseline (gather -> batch_isend_irecv ->
    scatter) moves each rank's request to its ring successor exactly."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    world = 3
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    for rank, ok, err in res:
        assert ok, err
