"""configs[4] end to end on one B200, nothing recorded: the trace generator ->
the NATIVE online scheduler (MellScheduler, csrc/scheduler.cpp) -> the
planner -> the GPU executor (kvm_migrate / kvm_reprefill) in the live slot
loop (runtime.run_slots).  The decisions must equal the reference simulator's
recorded run (plan rows, GPU-count series), and every resident request's KV
must read back its fingerprint after its migrations (checked every 100 slots).
8 logical GPUs = 8 pools on cuda:0 with a down-scaled KV shape (token counts,
hence every decision, unchanged)."""
import os
import sys

import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,seed", [("trace_7b_c48g_seed0.json", 0), ("trace_multillm_7b13b_seed0.json", 0)])
def test_online_loop_native_scheduler_on_gpu(name, seed):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from replay_trace import MINI, MINI_7B, build

    from paper_2501_06709_b200 import ClusterState, MellScheduler, PriorityConfig
    from paper_2501_06709_b200.planner import Topology, load_boundaries
    from paper_2501_06709_b200.replay import FingerprintedExecutor
    from paper_2501_06709_b200.runtime import run_slots
    from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson

    fx = load_golden(name)
    cfg = fx["config"]
    cl, wl = cfg["cluster"], cfg["workload"]
    trace = gen_poisson(wl["mean_interarrival_slots"], wl["duration_slots"], LengthDistribution(scale=wl["scale"]),
                        cfg["sim"]["seed"])
    assert [list(r) for r in trace.tuples()] == [list(r) for r in fx["trace"]]
    models = {int(k): v for k, v in fx.get("models", {}).items()}
    bpt = {rid: fx["model_bpt"][m] for rid, m in models.items()} if models else wl["kv_bytes_per_token"]
    inner, _ = build(fx, MINI_7B, "bulk", [0], MINI)
    ex = FingerprintedExecutor(inner)
    cluster = ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = MellScheduler(cluster, priority_cfg=PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, cfg["migration"]["epoch_seconds"], cfg["migration"]["budget_fraction"])
    checked = []
    misplaced = []

    def on_slot(slot, rows):
        if slot % 100 == 99:
            checked.append(ex.verify())
        # the bytes follow the scheduler: every request not waiting in the backlog sits on its
        # item's logical GPU (planned moves + executor.reconcile of member-level moves)
        waiting = set()
        for r in rows:
            if r[6] == "deferred":
                waiting.update(cluster.groups[r[1]].members if r[1] < 0 and r[1] in cluster.groups else (r[1],))
        for rid, res in ex.loc.items():
            item = cluster.item_of_request(rid)
            if rid not in waiting and item is not None and cluster.placement.get(item) != res.gpu:
                misplaced.append((slot, rid))

    out = run_slots(trace.tuples(), sched, cluster, topo, bounds, bpt=bpt,
                    tokens_per_slot=cfg["sim"]["tokens_per_slot"], max_defer=cfg["migration"]["max_defer"],
                    duration_slots=wl["duration_slots"], executor=ex,
                    models={rid: MINI[m].name for rid, m in models.items()}, on_slot=on_slot)
    assert out.plan_rows == [r[:7] for r in fx["plan_rows"]]
    assert out.active_gpus == fx["active_gpus"]
    assert out.bytes_moved > 0
    assert sum(checked) > 0
    assert misplaced == [] and out.reconciled_moves > 0
    assert sum(len(r.records) for r in ex.reports) > 0


def test_online_loop_split_mode_executes_splits():
    """Planner split mode on in the live loop: the B200
    figures for the cost terms (770 GB/s measured peer copy, the re-prefill
    kernel's ~400k tok/s for a 7B QKV projection) make the planner split moves
    that neither fit the link nor the compute budget whole; every split runs
    through the executor (fused kvm_split_migrate: both logical GPUs share this
    device).  Checked: the prefix blocks keep their fingerprints (bit-exact
    copy), the suffix K/V equals X.W^T within the bf16 tolerance, the block
    table lists every block, and with split off the plan rows are unchanged."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from replay_trace import MINI_7B

    from paper_2501_06709_b200 import ClusterState, MellScheduler, PriorityConfig
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.kvcache import BlockTable, KVPool
    from paper_2501_06709_b200.planner import SPLIT_TRANSFER, Topology, load_boundaries
    from paper_2501_06709_b200.replay import FingerprintedExecutor
    from paper_2501_06709_b200.reprefill import ReprefillEngine
    from paper_2501_06709_b200.runtime import run_slots
    from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson

    trace = gen_poisson(0.5, 200, LengthDistribution(scale=10), 0).tuples()
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=770e9, inter_bandwidth_bytes_per_s=50e9,
                    prefill_tokens_per_s=400_000.0)
    bounds = load_boundaries(topo, 0.05, 0.2)
    nb = int(1.5 * (48 << 30) / (16 * 524_288))
    pools = {g: KVPool(MINI_7B, nb, device=0, dtype=torch.bfloat16) for g in range(8)}
    tables = {g: BlockTable(512, 2048, device=0) for g in range(8)}
    eng = ReprefillEngine(MINI_7B, [0], with_q=False)
    inner = MigrationExecutor(pools, tables, reprefill=eng)
    ex = FingerprintedExecutor(inner)
    splits = []
    orig = ex.execute

    def execute(plan, members_of=None):
        rep = orig(plan, members_of=members_of)
        for rec in rep.records:
            if rec.mode != SPLIT_TRANSFER:
                continue
            torch.cuda.synchronize()
            for rid, pre in rec.split_prefix_blocks.items():
                r = inner.where(rid)
                n = r.tokens
                toks = torch.arange(pre * 16, n, device="cuda")
                db = torch.from_numpy(r.blocks).long().cuda()
                blk, slot = db[toks // 16], toks % 16
                x = eng.hidden(MINI_7B, rid, n, 0)[pre * 16:].float()
                w = eng.weights[(0, MINI_7B.name)]
                pool = inner.pool(r.gpu)
                kvd = MINI_7B.kv_cols
                for l in range(0, MINI_7B.layers, 7):
                    ref = x @ w[l].float().t()
                    torch.testing.assert_close(pool.tensor[l, 0, blk, slot].reshape(-1, kvd).float(), ref[:, :kvd],
                                               atol=1e-2, rtol=1.6e-2)
                    torch.testing.assert_close(pool.tensor[l, 1, blk, slot].reshape(-1, kvd).float(), ref[:, kvd:],
                                               atol=1e-2, rtol=1.6e-2)
                row = tables[r.gpu].rows[tables[r.gpu].slot(rid), :len(r.blocks)].cpu().numpy()
                assert (row == r.blocks).all()
                splits.append((rid, pre, n))
            assert ex.verify() >= 0      # prefix fingerprints of every resident request
        return rep

    ex.execute = execute
    cl = ClusterState(48 << 30, gpus_per_machine=8)
    out = run_slots(trace, MellScheduler(cl, priority_cfg=PriorityConfig(), batching=True), cl, topo, bounds,
                    bpt=524_288, tokens_per_slot=10, duration_slots=200, executor=ex, split=True)
    assert len(splits) >= 1 and all(0 < pre * 16 < n for _, pre, n in splits)
    assert sum(1 for r in out.plan_rows if r[6] == SPLIT_TRANSFER) == len(splits)
    cl2 = ClusterState(48 << 30, gpus_per_machine=8)
    ref = run_slots(trace, MellScheduler(cl2, priority_cfg=PriorityConfig(), batching=True), cl2, topo, bounds,
                    bpt=524_288, tokens_per_slot=10, duration_slots=200)
    assert not any(r[6] == SPLIT_TRANSFER for r in ref.plan_rows)


def test_online_loop_tool_dry_run_sizing():
    """tools/online_loop.run_online (the configs[4] driver bench.py runs at N=8
    with full shapes): pools sized from the host-only dry run hold the run
    (no RequestTooLarge), decisions over the slots run equal the reference's,
    fingerprints hold.  Mini shapes here (one GPU)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from online_loop import run_online

    res = run_online(os.path.join(ROOT, "tests", "golden", "trace_multillm_7b13b_seed0.json"), shape="mini",
                     verify_every=50, max_slots=700)
    assert res["decisions_match_reference"] is True and res["slots"] == 700
    assert res["fingerprint_checks"] > 0 and res["bytes_moved"] > 0
