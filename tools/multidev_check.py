"""Cross-device correctness checks of the single-process multi-GPU path
(VERDICT r1 "next" #3), byte-exact where bytes are copied.  Used by
tests/test_gpu_multidev.py (>= 2 GPUs: devices 0 and 1) and by bench.py's
N > 1 run as its multi-device gate (rank 0, devices 0 and 1, reported as
`multi_device_checks`).  With dev_a == dev_b the same checks run on one
GPU (the harness itself is exercised on 1-GPU boxes).

Checks (insertion point of every executed move: sim.py:218-227):
  engine_push_over_peer        kvm_migrate on A storing into B's pool with each
                               copy engine (LDG/STG, TMA bulk), bytes + row +
                               flag, and each engine's push GB/s
  executor_cross_device        pools on two devices, one executor (kvm_init(1)
                               peer access), kv moves A -> B, bytes + table rows
  stream_ordered_cross_device  execute(stream_ordered=True) A -> B, then B -> A
                               writing into blocks A just freed, no host wait;
                               a consumer stream on B waits on report.done
  split_push_and_reprefill     split_transfer across devices: kvm_migrate on A
                               pushes the prefix while kvm_reprefill runs on B
  fused_split_pulls_over_peer  kvm_split_migrate on B pulling the prefix from
                               A's pool (A's pool registered on B via UVA)
  pipelined_decode_on_peer     layer-flag decode on B behind the A -> B copy,
                               equal to decoding the source on A

    python tools/multidev_check.py [--a 0 --b 1]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ATOL, RTOL = 1e-2, 1.6e-2


def _shape():
    from paper_2501_06709_b200.kvcache import ModelShape

    return ModelShape("md", layers=4, kv_heads=4, head_dim=128, q_heads=16, d_model=512)


def _fill(pool, seed):
    import torch

    g = torch.Generator(device=f"cuda:{pool.device}").manual_seed(seed)
    pool.tensor.view(torch.int16).copy_(torch.randint(-2 ** 15, 2 ** 15, pool.view_shape, generator=g,
                                                      device=f"cuda:{pool.device}", dtype=torch.int16))


def _gather(pool, blocks):
    import torch

    idx = torch.from_numpy(blocks.astype("int64")).to(f"cuda:{pool.device}")
    return pool.tensor.view(torch.int16)[:, :, idx].cpu()


def check_executor_cross_device(a, b):
    import numpy as np
    import torch

    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.kvcache import BlockTable, KVPool
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    sh = _shape()
    pools = {0: KVPool(sh, 128, device=a), 1: KVPool(sh, 128, device=b)}
    tables = {0: BlockTable(8, 32, device=a), 1: BlockTable(8, 32, device=b)}
    _fill(pools[0], 1)
    _fill(pools[1], 2)
    ex = MigrationExecutor(pools, tables)
    for rid, tok in ((1, 100), (2, 37), (3, 16 * 9)):
        ex.admit(rid, 0, tok)
    want = {r: _gather(pools[0], ex.where(r).blocks) for r in (1, 2, 3)}
    bpt = sh.kv_bytes_per_token
    rep = ex.execute([PlannedMove(PendingMove(r, 0, 1, t * bpt, t), KV_TRANSFER)
                      for r, t in ((1, 100), (2, 37), (3, 144))])
    torch.cuda.synchronize(a)
    torch.cuda.synchronize(b)
    for r in (1, 2, 3):
        res = ex.where(r)
        assert res.gpu == 1, f"request {r} not on GPU 1"
        assert torch.equal(_gather(pools[1], res.blocks), want[r]), f"request {r}: bytes differ"
        row = tables[1].rows[tables[1].slot(r), :len(res.blocks)].cpu().numpy()
        assert np.array_equal(row, res.blocks), f"request {r}: table row"
    assert pools[0].allocator.n_free == 128 and rep.launches == 1
    return {"moves": 3, "bytes": rep.bytes_moved}


def check_engine_push_over_peer(a, b):
    """kvm_migrate launched on A storing straight into B's pool (UVA peer
    mapping), once per copy engine: LDG/STG and the TMA bulk engine
    (cp.async.bulk smem -> peer global).  Bytes + table row bit-exact; each
    engine's push of 64 blocks of 7B KV (512 MiB) timed with CUDA events on
    A's stream (the single-process NVLink number beside the ring's IPC one)."""
    import ctypes

    import numpy as np
    import torch

    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.executor import ENGINES
    from paper_2501_06709_b200.kvcache import LLAMA2_7B, BlockTable, KVPool

    _native.check(_native.lib().kvm_init(1), "kvm_init")
    nb, n = 96, 64
    src, dst = KVPool(LLAMA2_7B, nb, device=a), KVPool(LLAMA2_7B, nb, device=b)
    _fill(src, 11)
    table = BlockTable(1, n, device=b)
    flag = torch.zeros(1, dtype=torch.int32, device=f"cuda:{b}")
    sb = np.random.default_rng(3).permutation(nb)[:n].astype(np.int32)
    db = np.random.default_rng(4).permutation(nb)[:n].astype(np.int32)
    want = _gather(src, sb)
    s = torch.cuda.Stream(device=a)
    out = {"bytes_per_push": n * LLAMA2_7B.block_tokens * LLAMA2_7B.kv_bytes_per_token}
    for name, eflag in ENGINES.items():
        _fill(dst, 12)
        torch.cuda.synchronize(b)    # the fill ran on b's current stream; the push runs on s (device a)
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, 1
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
        m.dst_table_row, m.done_flag = table.row_ptr(0), flag.data_ptr()

        def push():
            _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | eflag,
                                                    ctypes.c_void_p(s.cuda_stream)), f"kvm_migrate({name})")

        push()
        s.synchronize()
        assert torch.equal(_gather(dst, db), want), f"{name}: bytes differ on the peer"
        assert np.array_equal(table.rows[0].cpu().numpy(), db), f"{name}: table row"
        assert int(flag.item()) == 1, f"{name}: done flag"
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.device(a):
            for _ in range(3):
                push()
            ev[0].record(s)
            for _ in range(10):
                push()
            ev[1].record(s)
        s.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 10
        out[name] = {"ok": True, "ms": round(ms, 4), "GBps": round(out["bytes_per_push"] / ms / 1e6, 1)}
    return out


def check_stream_ordered_cross_device(a, b):
    import torch

    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.kvcache import BlockTable, KVPool
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    sh = _shape()
    pools = {0: KVPool(sh, 64, device=a), 1: KVPool(sh, 64, device=b)}
    tables = {0: BlockTable(8, 32, device=a), 1: BlockTable(8, 32, device=b)}
    _fill(pools[0], 3)
    _fill(pools[1], 4)
    ex = MigrationExecutor(pools, tables)
    ex.admit(1, 0, 300)
    ex.admit(2, 1, 200)
    w1, w2 = _gather(pools[0], ex.where(1).blocks), _gather(pools[1], ex.where(2).blocks)
    bpt = sh.kv_bytes_per_token
    r1 = ex.execute([PlannedMove(PendingMove(1, 0, 1, 300 * bpt, 300), KV_TRANSFER)], stream_ordered=True)
    # at once, no host wait: request 2 moves B -> A into the lowest free blocks of A, which are the
    # blocks request 1 was just read from (freed on the host at issue): the per-pool fence must order
    # this write behind the A -> B read
    r2 = ex.execute([PlannedMove(PendingMove(2, 1, 0, 200 * bpt, 200), KV_TRANSFER)], stream_ordered=True)
    consumer_b = torch.cuda.Stream(device=b)
    consumer_a = torch.cuda.Stream(device=a)
    consumer_b.wait_event(r1.done[b])
    consumer_a.wait_event(r2.done[a])
    consumer_b.synchronize()
    consumer_a.synchronize()
    torch.cuda.synchronize(a)
    torch.cuda.synchronize(b)
    assert torch.equal(_gather(pools[1], ex.where(1).blocks), w1), "request 1 bytes (A -> B)"
    assert torch.equal(_gather(pools[0], ex.where(2).blocks), w2), "request 2 bytes (B -> A)"
    return {"reused_freed_blocks": bool(set(ex.where(2).blocks.tolist()) & set(range(19)))}


def _engine(sh, devs):
    from paper_2501_06709_b200.reprefill import ReprefillEngine

    return ReprefillEngine(sh, sorted(set(devs)), with_q=False, seed=7)


def _check_suffix(ex, eng, rid, pre_blocks, sh):
    import torch

    r = ex.where(rid)
    n = r.tokens
    dev = ex.pool(r.gpu).device
    toks = torch.arange(pre_blocks * 16, n, device=f"cuda:{dev}")
    db = torch.from_numpy(r.blocks).long().to(f"cuda:{dev}")
    blk, slot = db[toks // 16], toks % 16
    x = eng.hidden(sh, rid, n, dev)[pre_blocks * 16:].float()
    w = eng.weights[(dev, sh.name)]
    pool = ex.pool(r.gpu)
    kvd = sh.kv_cols
    for l in range(sh.layers):
        ref = x @ w[l].float().t()
        torch.testing.assert_close(pool.tensor[l, 0, blk, slot].reshape(-1, kvd).float(), ref[:, :kvd],
                                   atol=ATOL, rtol=RTOL)
        torch.testing.assert_close(pool.tensor[l, 1, blk, slot].reshape(-1, kvd).float(), ref[:, kvd:],
                                   atol=ATOL, rtol=RTOL)


def check_split_push_and_reprefill(a, b, split_kernels="auto"):
    import numpy as np
    import torch

    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.kvcache import BlockTable, KVPool

    sh = _shape()
    pools = {0: KVPool(sh, 96, device=a, dtype=torch.bfloat16), 1: KVPool(sh, 96, device=b, dtype=torch.bfloat16)}
    tables = {0: BlockTable(4, 64, device=a), 1: BlockTable(4, 64, device=b)}
    _fill(pools[0], 5)
    eng = _engine(sh, [a, b])
    ex = MigrationExecutor(pools, tables, reprefill=eng, split_kernels=split_kernels)
    ex.admit(4, 0, 700)
    sb = ex.where(4).blocks.copy()
    want = _gather(pools[0], sb)
    rec = ex.split_move(4, 1, suffix=300)
    pre = rec.split_prefix_blocks[4]
    torch.cuda.synchronize(a)
    torch.cuda.synchronize(b)
    r = ex.where(4)
    assert r.gpu == 1 and pre == 25 and rec.tokens_recomputed == 300
    assert torch.equal(_gather(pools[1], r.blocks[:pre]), want[:, :, :pre]), "prefix bytes"
    _check_suffix(ex, eng, 4, pre, sh)
    row = tables[1].rows[tables[1].slot(4), :len(r.blocks)].cpu().numpy()
    assert np.array_equal(row, r.blocks), "table row"
    return {"prefix_blocks": pre, "suffix_tokens": rec.tokens_recomputed,
            "kernels": "kvm_migrate on A + kvm_reprefill on B" if (a != b or split_kernels == "two")
            else "fused (same device)"}


def check_fused_split_pulls_over_peer(a, b):
    import numpy as np
    import torch

    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.kvcache import BlockTable, KVPool
    from paper_2501_06709_b200.split import make_split, split_migrate_fused

    sh = _shape()
    src = KVPool(sh, 96, device=a, dtype=torch.bfloat16)
    dst = KVPool(sh, 96, device=b, dtype=torch.bfloat16)
    _fill(src, 6)
    _native.check(_native.lib().kvm_init(1), "kvm_init")
    # A's pool registered on B (UVA peer pointer): the kernel on B pulls the prefix over NVLink
    alias = KVPool(sh, 96, device=b, dtype=torch.bfloat16, allocator=False, _base_ptr=src.base_ptr)
    n, suffix = 640, 208
    plan = make_split(n, suffix)
    sb = np.random.default_rng(1).permutation(96)[:plan.total_blocks].astype(np.int32)
    db = dst.allocator.alloc(plan.total_blocks)
    eng = _engine(sh, [b])
    x = eng.hidden(sh, 9, n, b)[n - suffix:].contiguous()
    w = eng.weights[(b, sh.name)]
    table = BlockTable(1, plan.total_blocks, device=b)
    sbd, dbd = torch.from_numpy(sb).to(f"cuda:{b}"), torch.from_numpy(db).to(f"cuda:{b}")
    want = _gather(src, sb[:plan.prefix_blocks])
    split_migrate_fused(alias, dst, sbd, dbd, plan, x, w, table_row=table.row_ptr(0),
                        stream=torch.cuda.current_stream(b))
    torch.cuda.synchronize(b)
    assert torch.equal(_gather(dst, db[:plan.prefix_blocks]), want), "prefix pulled over the peer mapping"
    toks = torch.arange(plan.prefix_tokens, n, device=f"cuda:{b}")
    blk, slot = dbd.long()[toks // 16], toks % 16
    for l in range(sh.layers):
        ref = x.float() @ w[l].float().t()
        torch.testing.assert_close(dst.tensor[l, 0, blk, slot].reshape(suffix, sh.kv_cols).float(),
                                   ref[:, :sh.kv_cols], atol=ATOL, rtol=RTOL)
    assert np.array_equal(table.rows[0].cpu().numpy(), db), "table row"
    alias.close()
    return {"prefix_blocks": plan.prefix_blocks, "suffix_tokens": suffix}


def check_pipelined_decode_on_peer(a, b):
    import torch

    from paper_2501_06709_b200.attention import paged_decode
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.kvcache import KVPool, ModelShape
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    sh = ModelShape("mdd", layers=6, kv_heads=2, head_dim=128, q_heads=8, d_model=1024)
    pools = {0: KVPool(sh, 200, device=a, dtype=torch.bfloat16), 1: KVPool(sh, 200, device=b, dtype=torch.bfloat16)}
    g = torch.Generator(device=f"cuda:{a}").manual_seed(4)
    pools[0].tensor.copy_(torch.randn(pools[0].view_shape, generator=g, device=f"cuda:{a}").to(torch.bfloat16))
    ex = MigrationExecutor(pools)
    ex.admit(9, 0, 2500)
    q = torch.randn(sh.layers, 1, 8, 128, generator=g, device=f"cuda:{a}").to(torch.bfloat16)
    lens = torch.tensor([2500], dtype=torch.int32, device=f"cuda:{a}")
    with torch.cuda.device(a):
        ref = paged_decode(pools[0], q, torch.from_numpy(ex.where(9).blocks)[None].contiguous().to(f"cuda:{a}"),
                           lens)
    torch.cuda.synchronize(a)
    rep = ex.execute([PlannedMove(PendingMove(9, 0, 1, 2500 * sh.kv_bytes_per_token, 2500), KV_TRANSFER)],
                     stream_ordered=True, layer_flags=True)
    rec = rep.records[0]
    err = torch.zeros(1, dtype=torch.int32, device=f"cuda:{b}")
    dec = torch.cuda.Stream(device=b)
    qb, lb = q.to(f"cuda:{b}"), lens.to(f"cuda:{b}")
    torch.cuda.synchronize(b)
    with torch.cuda.device(b):
        out = paged_decode(pools[1], qb, torch.from_numpy(ex.where(9).blocks)[None].contiguous().to(f"cuda:{b}"),
                           lb, stream=dec, layer_flags=rec.layer_flags[9], timeout_ns=5_000_000_000, err_word=err)
    torch.cuda.synchronize(a)
    torch.cuda.synchronize(b)
    assert err.item() == 0, "layer wait timed out"
    assert rec.layer_flags[9].cpu().tolist() == [1] * sh.layers
    assert torch.equal(out.view(torch.int16).cpu(), ref.view(torch.int16).cpu()), "decode differs from the source"
    return {"layers": sh.layers}


CHECKS = {
    "engine_push_over_peer": check_engine_push_over_peer,
    "executor_cross_device": check_executor_cross_device,
    "stream_ordered_cross_device": check_stream_ordered_cross_device,
    "split_push_and_reprefill": check_split_push_and_reprefill,
    "split_two_kernels_forced": lambda a, b: check_split_push_and_reprefill(a, b, "two"),
    "fused_split_pulls_over_peer": check_fused_split_pulls_over_peer,
    "pipelined_decode_on_peer": check_pipelined_decode_on_peer,
}


def run_checks(a: int = 0, b: int = 1) -> dict:
    """{check: {"ok": bool, ...}} for devices a -> b."""
    import torch

    out = {"devices": [a, b], "cross_device": a != b}
    for name, fn in CHECKS.items():
        try:
            info = fn(a, b) or {}
            out[name] = {"ok": True, **info}
        except Exception as e:   # reported per check; the caller decides
            out[name] = {"ok": False, "error": f"{type(e).__name__}: {e}"[:400],
                         "where": traceback.format_exc().splitlines()[-3:]}
        torch.cuda.empty_cache()
    out["all_ok"] = all(v["ok"] for k, v in out.items() if isinstance(v, dict) and "ok" in v)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", type=int, default=0)
    ap.add_argument("--b", type=int, default=1)
    ap.add_argument("--out", default=None, help="also write the JSON result here (bench.py's subprocess probe)")
    args = ap.parse_args()
    import torch

    b = args.b if torch.cuda.device_count() > args.b else args.a
    res = run_checks(args.a, b)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
