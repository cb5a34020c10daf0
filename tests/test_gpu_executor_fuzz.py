"""Random operation sequences through the executor's public API on one B200:
admit / grow / release, planned kv moves (synchronous and stream-ordered),
compaction (synchronous and stream-ordered) and live migrations with decode
growth between pre-copy rounds, on three logical GPUs.  Every block a request
gains is fingerprinted (replay.Fingerprints); after every few operations all
resident requests must read back their own fingerprints wherever they now live,
their block-table rows must list exactly their blocks, and the allocators must
account for every block.  KVM_FUZZ_SEEDS sets the number of sequences."""
import os

import numpy as np
import pytest
import torch

from paper_2501_06709_b200.executor import MigrationExecutor
from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape
from paper_2501_06709_b200.live import LiveMigration
from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove
from paper_2501_06709_b200.replay import Fingerprints

pytestmark = pytest.mark.gpu
SHAPE = ModelShape("xf", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=128)
MAX_TOKENS = 640   # = the block tables' 40 blocks


def _check(ex, fp, pools, tables):
    torch.cuda.synchronize()
    fp.verify()
    for rid, r in ex.loc.items():
        t = tables[r.gpu]
        assert np.array_equal(t.rows[t.slot(rid), :len(r.blocks)].cpu().numpy(), r.blocks), rid
    for g, p in pools.items():
        used = sum(len(r.blocks) for r in ex.loc.values() if r.gpu == g)
        assert p.allocator.num_blocks - p.allocator.n_free == used, g


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVM_FUZZ_SEEDS", "30"))))
def test_executor_random_operations(seed):
    rng = np.random.default_rng(20000 + seed)
    pools = {g: KVPool(SHAPE, 1000) for g in range(3)}   # never full: every refusal would be a bug
    tables = {g: BlockTable(32, 40) for g in range(3)}
    ex = MigrationExecutor(pools, tables, engine="bulk" if rng.integers(2) else "ldg")
    fp = Fingerprints(ex)
    bpt = SHAPE.kv_bytes_per_token
    next_rid = 0
    for step in range(60):
        op = rng.choice(["admit", "admit", "grow", "release", "move", "move_async", "compact", "compact_async",
                         "live"])
        rids = sorted(ex.loc)
        if op == "admit" or not rids:
            g = int(rng.integers(3))
            ex.admit(next_rid, g, int(rng.integers(1, 200)))
            fp.stamp(next_rid)
            next_rid += 1
        elif op == "grow":
            rid = int(rng.choice(rids))
            ex.grow(rid, min(MAX_TOKENS, ex.where(rid).tokens + int(rng.integers(1, 40))))
            fp.stamp(rid)
        elif op == "release":
            rid = int(rng.choice(rids))
            ex.release(rid)
            fp.forget(rid)
        elif op in ("move", "move_async"):
            picked = [int(r) for r in rng.choice(rids, size=min(len(rids), int(rng.integers(1, 4))),
                                                replace=False)]
            plan = []
            for rid in picked:
                r = ex.where(rid)
                dst = int((r.gpu + rng.integers(1, 3)) % 3)
                plan.append(PlannedMove(PendingMove(rid, r.gpu, dst, r.tokens * bpt, r.tokens), KV_TRANSFER))
            ex.execute(plan, stream_ordered=(op == "move_async"))
        elif op in ("compact", "compact_async"):
            ex.compact(int(rng.choice(rids)), stream_ordered=(op == "compact_async"))
        else:  # live migration with decode growth between pre-copy rounds
            rid = int(rng.choice(rids))
            r = ex.where(rid)
            lm = LiveMigration(ex, rid, int((r.gpu + 1) % 3))
            for _ in range(int(rng.integers(1, 4))):
                lm.precopy()
                ex.grow(rid, min(MAX_TOKENS, ex.where(rid).tokens + int(rng.integers(1, 30))))
                fp.stamp(rid)
            lm.drain()
            lm.finish()
        if op in ("move_async", "compact_async"):
            # the stream-ordered contract: work that may reuse freed source blocks
            # (the next admit's fingerprint writes) queues behind the executor's stream
            torch.cuda.current_stream().wait_stream(ex.stream(0))
        if step % 5 == 4:
            _check(ex, fp, pools, tables)
    _check(ex, fp, pools, tables)
