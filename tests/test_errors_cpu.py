"""CPU-only error behaviour of the host objects (no GPU): the reference's
exception classes for the reference's kinds of misuse (errors.py:4-32)."""
import numpy as np
import pytest

from paper_2501_06709_b200 import ConfigError, KvPackError, NotPlaced, RequestTooLarge
from paper_2501_06709_b200.kvcache import BlockAllocator, ModelShape
from paper_2501_06709_b200.planner import KV_TRANSFER, TOKEN_TRANSFER, PendingMove, PlannedMove
from test_replay_cpu import MINI, HostExecutor, HostPool


def _ex():
    ex = HostExecutor({0: HostPool(MINI, 32, 0), 1: HostPool(MINI, 32, 1)})
    ex.reprefill = None
    return ex


def test_exception_hierarchy_matches_reference():
    for cls in (ConfigError, NotPlaced, RequestTooLarge):
        assert issubclass(cls, KvPackError)


def test_allocator_errors():
    a = BlockAllocator(4)
    with pytest.raises(ValueError):
        a.alloc(-1)
    with pytest.raises(RequestTooLarge):
        a.alloc(5)
    a.take([1])
    with pytest.raises(ValueError):
        a.take([1])
    with pytest.raises(ValueError):
        a.free([9])
    with pytest.raises(ConfigError):
        BlockAllocator(0)


def test_executor_misuse():
    ex = _ex()
    ex.admit(1, 0, 40)
    with pytest.raises(ValueError):
        ex.admit(1, 0, 40)
    with pytest.raises(NotPlaced):
        ex.where(2)
    with pytest.raises(NotPlaced):
        ex.admit(3, 7, 10)            # no pool on GPU 7
    with pytest.raises(RequestTooLarge):
        ex.admit(4, 1, 10 ** 6)       # pool too small
    ex.release(99)                     # releasing an unknown request is a no-op
    with pytest.raises(ConfigError):  # token_transfer needs a re-prefill engine
        ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 40), TOKEN_TRANSFER)])
    # a move whose item is not physically at src moves nothing (sim.py:209-213 semantics)
    rep = ex.execute([PlannedMove(PendingMove(1, 1, 0, 0, 40), KV_TRANSFER)])
    assert rep.records[0].requests == [] and ex.where(1).gpu == 0


def test_executor_bookkeeping_roundtrip():
    ex = _ex()
    ex.admit(5, 0, 33)                 # 3 blocks
    ex.grow(5, 48)                     # still 3
    assert len(ex.where(5).blocks) == 3
    ex.grow(5, 49)                     # 4th block
    assert len(ex.where(5).blocks) == 4
    rep = ex.execute([PlannedMove(PendingMove(5, 0, 1, 49 * MINI.kv_bytes_per_token, 49), KV_TRANSFER)])
    assert rep.records[0].requests == [5] and rep.tokens_moved == 49
    assert ex.where(5).gpu == 1 and ex.pool(0).allocator.n_free == 32
    assert ex.launched and ex.launched[-1][0][2] == 4   # one kvm_migrate, 4 blocks


def test_multi_model_executor_requires_model():
    other = ModelShape("other", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=128)
    ex = HostExecutor({0: {"mini": HostPool(MINI, 8, 0), "other": HostPool(other, 8, 1)}})
    with pytest.raises(ValueError):
        ex.admit(1, 0, 10)             # ambiguous: two models served
    ex.admit(1, 0, 10, model="other")
    assert ex.where(1).model == "other"
    with pytest.raises(ConfigError):
        HostExecutor({0: {"wrong-key": HostPool(MINI, 8, 0)}})


def test_residency_without_model_uses_the_single_model():
    """A Residency built by hand with the default model="" still resolves its
    pool and block table on a single-model executor (bench.py does this)."""
    from paper_2501_06709_b200.executor import Residency

    ex = _ex()
    ex.tables = {0: {"mini": "T0"}, 1: {"mini": "T1"}}
    ex.loc[7] = Residency(0, np.arange(2, dtype=np.int32), 20)
    assert ex.pool_of(7) is ex.pool(0)
    assert ex._table(0, ex.loc[7].model) == "T0"


def test_execute_is_all_or_nothing_when_a_pool_is_full():
    """A plan whose later move cannot get destination blocks raises before any
    launch and leaves every pool, residency and launch list untouched."""
    ex = _ex()
    ex.admit(1, 0, 100)                # 7 blocks on GPU 0
    ex.admit(2, 0, 60)                 # 4 blocks on GPU 0
    ex.admit(3, 1, 16 * 25)            # 25 of GPU 1's 32 blocks
    free0, free1 = ex.pools[0]["mini"].allocator.n_free, ex.pools[1]["mini"].allocator.n_free
    plan = [PlannedMove(PendingMove(2, 0, 1, 0, 60), KV_TRANSFER),     # fits (4 <= 7 free)
            PlannedMove(PendingMove(1, 0, 1, 0, 100), KV_TRANSFER)]    # does not (7 > 3 left)
    with pytest.raises(RequestTooLarge):
        ex.execute(plan)
    assert ex.pools[0]["mini"].allocator.n_free == free0 and ex.pools[1]["mini"].allocator.n_free == free1
    assert ex.where(1).gpu == 0 and ex.where(2).gpu == 0 and ex.launched == []


def test_deferred_commits_accumulate_and_guard():
    """Several wait=False executes before commit(): all are committed in order;
    a request with an uncommitted move cannot be moved again."""
    ex = _ex()
    ex.admit(1, 0, 40)
    ex.admit(2, 0, 40)
    ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER)], wait=False)
    ex.execute([PlannedMove(PendingMove(2, 0, 1, 0, 40), KV_TRANSFER)], wait=False)
    with pytest.raises(ValueError):
        ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER)], wait=False)
    ex.commit()
    assert ex.where(1).gpu == 1 and ex.where(2).gpu == 1
    assert ex.pools[0]["mini"].allocator.n_free == 32
