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
