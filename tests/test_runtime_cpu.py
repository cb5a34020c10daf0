"""CPU-only: the live slot loop (runtime.run_slots) with the reference's own
MellScheduler plugged in through its step_epoch API reproduces the reference
simulator's plan rows and GPU-count series exactly (the recorded fixtures),
with this repo's planner and the executor's bookkeeping in the loop.

The reference scheduler is the *caller* of the hot path; it is imported from
/root/reference only when that tree is mounted (this container) — the test
skips elsewhere (the GPU box has no /root/reference).
"""
import os
import sys

import pytest

from conftest import load_golden
from paper_2501_06709_b200.planner import Topology, load_boundaries
from paper_2501_06709_b200.runtime import run_slots
from test_replay_cpu import MINI, HostExecutor, HostPool

REF = "/root/reference/pkg/src"


def _kvpack():
    if not os.path.isdir(REF):
        pytest.skip("reference tree not mounted (expected on the GPU box)")
    if REF not in sys.path:
        sys.path.append(REF)
    import kvpack  # noqa: F401
    return kvpack


@pytest.mark.parametrize("name", ["trace_7b_c48g_seed0.json", "trace_7b_mixed_seed0.json"])
def test_live_loop_with_reference_scheduler(name):
    kvpack = _kvpack()
    fx = load_golden(name)
    cfg = fx["config"]
    cl = cfg["cluster"]
    cluster = kvpack.ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = kvpack.MellScheduler(cluster, priority_cfg=kvpack.PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, cfg["migration"]["epoch_seconds"], cfg["migration"]["budget_fraction"])
    nb = 3 * (cl["capacity_bytes"] // cfg["workload"]["kv_bytes_per_token"]) // 16
    ex = HostExecutor({g: HostPool(MINI, nb, g) for g in range(16)})
    out = run_slots([tuple(r) for r in fx["trace"]], sched, cluster, topo, bounds,
                    bpt=cfg["workload"]["kv_bytes_per_token"], tokens_per_slot=cfg["sim"]["tokens_per_slot"],
                    max_defer=cfg["migration"]["max_defer"],
                    duration_slots=cfg["workload"]["duration_slots"], executor=ex)
    assert out.plan_rows == [r[:7] for r in fx["plan_rows"]]
    assert out.active_gpus == fx["active_gpus"]
    assert out.logical_moves == fx["migrations"]
    assert max(out.active_gpus) == fx["summary"]["peak_gpus"]
    assert out.completed == fx["summary"]["completed"]


def test_multi_llm_loop_matches_fixture():
    """configs[4] mixed 7B+13B: the reference scheduler with per-request byte
    sizes through the live loop reproduces the committed multi-LLM fixture."""
    kvpack = _kvpack()
    fx = load_golden("trace_multillm_7b13b_seed0.json")
    cfg = fx["config"]
    cl = cfg["cluster"]
    cluster = kvpack.ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = kvpack.MellScheduler(cluster, priority_cfg=kvpack.PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, cfg["migration"]["epoch_seconds"], cfg["migration"]["budget_fraction"])
    models = {int(k): v for k, v in fx["models"].items()}
    bpt = {rid: fx["model_bpt"][m] for rid, m in models.items()}
    out = run_slots([tuple(r) for r in fx["trace"]], sched, cluster, topo, bounds, bpt=bpt,
                    tokens_per_slot=cfg["sim"]["tokens_per_slot"], max_defer=cfg["migration"]["max_defer"],
                    duration_slots=cfg["workload"]["duration_slots"])
    assert out.plan_rows == [r[:7] for r in fx["plan_rows"]]
    assert out.active_gpus == fx["active_gpus"]
