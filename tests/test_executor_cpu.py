"""CPU-only: the executor's placement invariant and its all-or-nothing issue
path, driven by the live slot loop (runtime.run_slots) with the native
scheduler on a B200-shaped trace; kernel launches are recorded, not run.

Invariant (the data plane follows the scheduler): after every slot, every
resident request whose item is not waiting in the backlog sits physically on
its item's logical GPU — including members whose member-level move never
reached the planner (sim.py:207-213 drops it; executor.reconcile moves the
bytes) and members that joined a group while its move was deferred."""
import pytest

from paper_2501_06709_b200 import ClusterState, ConfigError, MellScheduler, PriorityConfig, RequestTooLarge
from paper_2501_06709_b200.planner import KV_TRANSFER, TOKEN_TRANSFER, PendingMove, PlannedMove, Topology, \
    load_boundaries
from paper_2501_06709_b200.runtime import run_slots
from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson
from test_replay_cpu import MINI, HostExecutor, HostPool


def _run(seed, reconcile=True):
    trace = gen_poisson(0.5, 200, LengthDistribution(scale=10), seed).tuples()
    cl = ClusterState(48 << 30, gpus_per_machine=8)
    sch = MellScheduler(cl, priority_cfg=PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9, inter_bandwidth_bytes_per_s=50e9,
                    prefill_tokens_per_s=50_000.0)
    nb = int(1.5 * (48 << 30) / (16 * 524_288))
    ex = HostExecutor({g: HostPool(MINI, nb, g) for g in range(16)})
    bad = []

    def check(slot, rows):
        waiting = set()
        for r in rows:
            if r[6] == "deferred":
                item = r[1]
                waiting.update(cl.groups[item].members if item < 0 and item in cl.groups else (item,))
        for rid, res in ex.loc.items():
            item = cl.item_of_request(rid)
            if rid not in waiting and item is not None and cl.placement.get(item) != res.gpu:
                bad.append((slot, rid, res.gpu, cl.placement.get(item)))

    out = run_slots(trace, sch, cl, topo, load_boundaries(topo, 0.05, 0.2), bpt=524_288, tokens_per_slot=10,
                    duration_slots=200, executor=ex, on_slot=check, reconcile=reconcile)
    return out, bad, ex


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_physical_location_follows_the_scheduler(seed):
    out, bad, ex = _run(seed)
    assert bad == [], bad[:5]
    assert out.plan_rows, "trace must plan moves"
    # pools balance: every block is either free or owned by exactly one resident request
    for g, per in ex.pools.items():
        for pool in per.values():
            held = sum(len(r.blocks) for r in ex.loc.values() if r.gpu == g)
            assert pool.allocator.n_free + held == pool.num_blocks


def test_without_reconcile_member_moves_are_lost():
    """The reference's refresh drops member-level moves: without reconcile the
    bytes stay behind (this is what reconcile exists for)."""
    out, bad, _ = _run(0, reconcile=False)
    assert bad and out.reconciled_moves == 0
    out2, bad2, _ = _run(0)
    assert not bad2 and out2.reconciled_moves > 0
    assert out2.plan_rows == out.plan_rows          # decisions are untouched


def test_group_members_move_from_wherever_they_are():
    ex = HostExecutor({g: HostPool(MINI, 64, g) for g in range(3)})
    ex.admit(1, 0, 40)
    ex.admit(2, 1, 40)      # joined the group at an intermediate GPU while its move was pending
    ex.admit(3, 2, 40)      # already at the destination
    rep = ex.execute([PlannedMove(PendingMove(-7, 0, 2, 0, 120), KV_TRANSFER)], members_of=lambda g: [1, 2, 3])
    assert sorted(rep.records[0].requests) == [1, 2]
    assert {ex.where(r).gpu for r in (1, 2, 3)} == {2}
    # host pools all sit on device 0: one fused launch carrying both moves (src pools 0 and 1)
    assert [sorted(m[0] for m in l) for l in ex.launched] == [[0, 1]]


def test_issue_failure_rolls_back():
    class Failing(HostExecutor):
        def _launch_migrate(self, dev, moves, dst_pools=()):
            if dev == 0 and len(self.launched) >= 0 and self.fail:
                raise RuntimeError("launch failed")
            super()._launch_migrate(dev, moves, dst_pools)

    ex = Failing({g: HostPool(MINI, 32, g) for g in range(2)})
    ex.fail = True
    ex.admit(1, 0, 100)
    free = [ex.pool(g).allocator.n_free for g in range(2)]
    with pytest.raises(RuntimeError):
        ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 100), KV_TRANSFER)])
    assert [ex.pool(g).allocator.n_free for g in range(2)] == free and ex.where(1).gpu == 0
    ex.fail = False
    ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 100), KV_TRANSFER)])
    assert ex.where(1).gpu == 1


def test_validation_happens_before_any_reservation():
    class Engine:
        def validate(self, pool):
            raise ConfigError("re-prefill writes bf16 K/V: pool dtype must be bfloat16")

        def __call__(self, *a):
            raise AssertionError("must not be called")

    ex = HostExecutor({g: HostPool(MINI, 32, g) for g in range(2)})
    ex.reprefill = Engine()
    ex.admit(1, 0, 40)
    ex.admit(2, 0, 40)
    free = [ex.pool(g).allocator.n_free for g in range(2)]
    plan = [PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER),
            PlannedMove(PendingMove(2, 0, 1, 0, 40), TOKEN_TRANSFER)]
    with pytest.raises(ConfigError):
        ex.execute(plan)
    assert [ex.pool(g).allocator.n_free for g in range(2)] == free and ex.launched == []
    # mismatched KV geometry between the two pools of a move
    from paper_2501_06709_b200.kvcache import ModelShape

    other = ModelShape("mini", layers=16, kv_heads=2, head_dim=128, q_heads=2, d_model=512)
    ex2 = HostExecutor({0: HostPool(MINI, 32, 0), 1: HostPool(other, 32, 1)})
    ex2.admit(1, 0, 40)
    with pytest.raises(ConfigError):
        ex2.execute([PlannedMove(PendingMove(1, 0, 1, 0, 40), KV_TRANSFER)])


def test_table_width_checked_before_launch():
    class Table:
        max_blocks, free_slots = 2, 4

        def has(self, rid):
            return False

    ex = HostExecutor({g: HostPool(MINI, 32, g) for g in range(2)})
    ex.tables = {1: {"mini": Table()}}
    ex.admit(1, 0, 100)   # 7 blocks > table width 2
    with pytest.raises(RequestTooLarge):
        ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, 100), KV_TRANSFER)])
    assert ex.launched == [] and ex.pool(1).allocator.n_free == 32
