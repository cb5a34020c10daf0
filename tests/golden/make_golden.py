"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (the container that has the read-only reference mounted):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (`kvpack`, pure Python) is imported only by this script; the
fixtures it writes are what the test-suite and the GPU box use, so nothing at
test time needs /root/reference.  Floats are stored with float.hex() so the
comparison is bit-exact.

Fixtures
  planner_cases.json   plan_hybrid / consensus_order / check_budgets on
                       seeded random move sets (migration.py:128-182),
                       including the verification.budget_safety generator
                       (verification.py:267-307) and forced/deferred cases.
  boundaries.json      load_boundaries (migration.py:77-91) incl. the
                       left-to-right float64 order.
  trace_7b_c48g_seed{0,2,3}.json
                       the slot loop's data-plane rows (sim.py:178-227) on the
                       B200-shaped run of SURVEY.md §8c: every plan row
                       (slot, item, src, dst, kv_bytes, tokens, mode), the
                       members of each group item at plan time, and the
                       per-slot active-GPU series.  Config 5's replay input
                       and the scheduler-parity target.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

import kvpack  # noqa: E402  (reference, via PYTHONPATH)
from kvpack import migration as refmig  # noqa: E402
from kvpack import sim as refsim  # noqa: E402
from kvpack.config import config_from_dict  # noqa: E402
from kvpack.workload import LengthDistribution, gen_poisson  # noqa: E402


def _hex(x: float) -> str:
    return float(x).hex()


def _plan_to_json(plan) -> dict:
    return {
        "assignments": [[p.move.item, p.mode, _hex(p.latency_s)] for p in plan.assignments],
        "link_bytes": [[list(k), _hex(v)] for k, v in plan.link_bytes.items()],
        "dest_tokens": [[k, _hex(v)] for k, v in plan.dest_tokens.items()],
        "forced": [m.item for m in plan.forced],
    }


def _topo_json(t) -> dict:
    return {"gpus_per_machine": t.gpus_per_machine,
            "intra_bandwidth_bytes_per_s": _hex(t.intra_bandwidth_bytes_per_s),
            "inter_bandwidth_bytes_per_s": _hex(t.inter_bandwidth_bytes_per_s),
            "prefill_tokens_per_s": _hex(t.prefill_tokens_per_s)}


def _bounds_json(b) -> dict:
    return {"comp_budget": _hex(b.comp_budget),
            "intra_comm_budget": _hex(b.intra_comm_budget),
            "inter_comm_budget": _hex(b.inter_comm_budget),
            "comm_budget": [[list(k), _hex(v)] for k, v in b.comm_budget.items()]}


def planner_cases() -> list:
    rng = random.Random(20250112)
    cases = []
    topologies = [
        refmig.Topology(),
        refmig.Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9,
                        inter_bandwidth_bytes_per_s=50e9, prefill_tokens_per_s=50_000.0),
        refmig.Topology(gpus_per_machine=2, intra_bandwidth_bytes_per_s=1e9,
                        inter_bandwidth_bytes_per_s=1e8, prefill_tokens_per_s=1000.0),
    ]
    # (1) the budget_safety generator, verbatim semantics, 200 sets
    for ci in range(200):
        topo = topologies[ci % len(topologies)]
        epoch_s = rng.choice([0.05, 0.25, 0.5, 1.0])
        fraction = rng.choice([0.05, 0.1, 0.2, 1.0])
        bounds = refmig.load_boundaries(topo, epoch_s, fraction)
        n = rng.randint(0, 30)
        moves, defer = [], {}
        for i in range(n):
            src, dst = rng.sample(range(16), 2)
            kv = rng.randint(1, int(bounds.inter_comm_budget * 2) + 1)
            moves.append(refmig.PendingMove(item=rng.choice([i, -i - 1]), src=src, dst=dst,
                                            kv_bytes=kv, tokens=kv // rng.choice([100, 524288]) + 1))
            if rng.random() < 0.3:
                defer[moves[-1].item] = rng.randint(0, 5)
        max_defer = rng.choice([0, 1, 3, 5])
        # dedupe items (PendingMove items are unique per backlog, sim.py:185-187)
        seen, uniq = set(), []
        for m in moves:
            if m.item not in seen:
                seen.add(m.item)
                uniq.append(m)
        moves = uniq
        rng.shuffle(moves)
        plan = refmig.plan_hybrid(moves, bounds, topo, defer_counts=defer, max_defer=max_defer)
        cases.append({
            "topology": _topo_json(topo),
            "epoch_seconds": _hex(epoch_s), "fraction": _hex(fraction),
            "boundaries": _bounds_json(bounds),
            "moves": [[m.item, m.src, m.dst, m.kv_bytes, m.tokens] for m in moves],
            "defer_counts": [[k, v] for k, v in defer.items()],
            "max_defer": max_defer,
            "consensus": [m.item for m in refmig.consensus_order(moves)],
            "plan": _plan_to_json(plan),
            "check_budgets": refmig.check_budgets(plan, bounds),
        })
    # (2) explicit per-link comm budgets (Boundaries.comm_budget override path)
    for ci in range(40):
        topo = topologies[ci % len(topologies)]
        comm = {("intra", 0): float(rng.randint(1, 10 ** 10)), ("inter",): float(rng.randint(1, 10 ** 9))}
        bounds = refmig.Boundaries(comm_budget=comm, comp_budget=float(rng.randint(0, 20_000)),
                                   intra_comm_budget=float(rng.randint(1, 10 ** 10)),
                                   inter_comm_budget=float(rng.randint(1, 10 ** 9)))
        moves = [refmig.PendingMove(item=i, src=rng.randrange(16), dst=rng.randrange(16),
                                    kv_bytes=rng.randint(0, 4 * 10 ** 9), tokens=rng.randint(0, 8000))
                 for i in range(rng.randint(1, 40))]
        plan = refmig.plan_hybrid(moves, bounds, topo)
        cases.append({
            "topology": _topo_json(topo),
            "boundaries": _bounds_json(bounds),
            "moves": [[m.item, m.src, m.dst, m.kv_bytes, m.tokens] for m in moves],
            "defer_counts": [], "max_defer": 3,
            "consensus": [m.item for m in refmig.consensus_order(moves)],
            "plan": _plan_to_json(plan),
            "check_budgets": refmig.check_budgets(plan, bounds),
        })
    return cases


def boundaries_cases() -> list:
    out = []
    for bw_intra, bw_inter, pf in [(50e9, 1.25e9, 10_000.0), (900e9, 50e9, 50_000.0),
                                   (10e9 / 8, 10e9 / 8, 1.0), (7.7e12, 3.3e10, 123_456.7)]:
        for epoch in [0.05, 0.1, 0.25, 1.0, 3.3]:
            for frac in [0.05, 0.1, 0.2, 0.5, 1.0]:
                t = refmig.Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=bw_intra,
                                    inter_bandwidth_bytes_per_s=bw_inter, prefill_tokens_per_s=pf)
                b = refmig.load_boundaries(t, epoch, frac)
                out.append({"topology": _topo_json(t), "epoch_seconds": _hex(epoch),
                            "fraction": _hex(frac), "boundaries": _bounds_json(b)})
    return out


# B200-shaped run: 7B KV (524 288 B/token), 48 GiB per GPU,
# 8 GPUs per machine, NVLink-class intra bandwidth.
B200_7B_DOC = {
    "cluster": {"capacity_bytes": 48 * 1024 ** 3, "gpus_per_machine": 8,
                "intra_bandwidth_bytes_per_s": 900e9, "inter_bandwidth_bytes_per_s": 50e9,
                "prefill_tokens_per_s": 50_000.0},
    "migration": {"epoch_seconds": 0.05, "budget_fraction": 0.2, "max_defer": 3},
    "workload": {"mean_interarrival_slots": 0.5, "duration_slots": 200, "scale": 10,
                 "kv_bytes_per_token": 524288},
    "sim": {"tokens_per_slot": 10},
}


# Same trace with tighter link budgets and a faster prefill so the planner
# also picks token_transfer (re-prefill) and defers more: exercises every mode.
MIXED_DOC = json.loads(json.dumps(B200_7B_DOC))
MIXED_DOC["cluster"]["intra_bandwidth_bytes_per_s"] = 200e9
MIXED_DOC["cluster"]["prefill_tokens_per_s"] = 500_000.0


def trace_fixture(seed: int, base: dict = B200_7B_DOC) -> dict:
    doc = json.loads(json.dumps(base))
    doc["sim"]["seed"] = seed
    cfg = config_from_dict(doc)
    w = cfg.workload
    dist = LengthDistribution(prompt_mean_log=w.prompt_mean_log, prompt_sigma_log=w.prompt_sigma_log,
                              response_mean_log=w.response_mean_log,
                              response_sigma_log=w.response_sigma_log, scale=w.scale)
    trace = gen_poisson(w.mean_interarrival_slots, w.duration_slots, dist, seed=seed)

    rows = []
    state = {"slot": -1, "cluster": None}
    orig_plan = refsim.plan_hybrid
    orig_cluster = refsim.ClusterState

    class SpyCluster(orig_cluster):  # capture the live ClusterState of the run
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            state["cluster"] = self

    def spy_plan(moves, boundaries, topology, defer_counts=None, max_defer=3):
        plan = orig_plan(moves, boundaries, topology, defer_counts=defer_counts, max_defer=max_defer)
        state["slot"] += 1
        cl = state["cluster"]
        for p in plan.assignments:
            m = p.move
            members = sorted(cl.groups[m.item].members) if m.item < 0 else [m.item]
            member_sizes = [cl.sizes[r] for r in members]
            rows.append([state["slot"], m.item, m.src, m.dst, m.kv_bytes, m.tokens, p.mode,
                         members, member_sizes])
        return plan

    slots = []
    orig_step = refsim.MellScheduler.step_epoch

    def spy_step(self, arrivals, completions, growths=None):
        res = orig_step(self, arrivals, completions, growths=growths)
        cl = state["cluster"]
        gone = [int(ev[1]) for ev in res.events if ev and ev[0] in ("rejected", "aborted")]
        arr = []
        for rid, size in arrivals:
            item = cl.item_of_request(rid)
            arr.append([rid, cl.placement.get(item, -1), size])
        slots.append({"arr": arr, "done": list(completions), "gone": gone})
        return res

    refsim.plan_hybrid = spy_plan
    refsim.ClusterState = SpyCluster
    refsim.MellScheduler.step_epoch = spy_step
    try:
        res = refsim.run(cfg, trace)
    finally:
        refsim.plan_hybrid = orig_plan
        refsim.ClusterState = orig_cluster
        refsim.MellScheduler.step_epoch = orig_step
    fp = hashlib.sha256(json.dumps([r[:7] for r in rows]).encode()).hexdigest()[:16]
    return {
        "config": doc,
        "trace": [[r.request_id, r.arrival_slot, r.prompt_tokens, r.response_tokens]
                  for r in trace.records],
        "plan_rows": rows,
        "slots": slots,
        "plan_rows_sha256_16": fp,
        "active_gpus": res.metrics.active_gpus,
        "migrations": res.metrics.migrations,
        "deferred": res.metrics.deferred,
        "forced": res.metrics.forced,
        "summary": {k: v for k, v in res.summary.items() if k != "config"},
    }


def multi_llm_fixture(seed: int = 0) -> dict:
    """configs[4]: multi-LLM Poisson trace (7B + 13B mix).  The reference sim
    has one kv_bytes_per_token (sim.py:105), so this run drives the REFERENCE
    MellScheduler through this repo's slot loop (runtime.run_slots, proven
    identical to sim.run on single-model traces by tests/test_runtime_cpu.py)
    with per-request byte sizes; model per request ~ seeded Bernoulli(0.5)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import numpy as np
    from paper_2501_06709_b200.planner import Topology, load_boundaries
    from paper_2501_06709_b200.runtime import run_slots

    doc = json.loads(json.dumps(B200_7B_DOC))
    doc["sim"]["seed"] = seed
    w = doc["workload"]
    dist = LengthDistribution(scale=w["scale"])
    trace = gen_poisson(w["mean_interarrival_slots"], w["duration_slots"], dist, seed=seed)
    rng = np.random.default_rng(1000 + seed)
    model_bpt = {"llama2-7b": 524288, "llama2-13b": 819200}
    models = {r.request_id: ("llama2-13b" if rng.random() < 0.5 else "llama2-7b") for r in trace.records}
    bpt = {rid: model_bpt[m] for rid, m in models.items()}
    cl = doc["cluster"]
    cluster = kvpack.ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = kvpack.MellScheduler(cluster, priority_cfg=kvpack.PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, doc["migration"]["epoch_seconds"], doc["migration"]["budget_fraction"])
    slots, rows = [], []
    orig_step = sched.step_epoch

    def spy_step(arrivals, completions, growths=None):
        res = orig_step(arrivals, completions, growths=growths)
        gone = [int(ev[1]) for ev in res.events if ev and ev[0] in ("rejected", "aborted")]
        arr = [[rid, cluster.placement.get(cluster.item_of_request(rid), -1), size] for rid, size in arrivals]
        slots.append({"arr": arr, "done": list(completions), "gone": gone})
        return res

    sched.step_epoch = spy_step

    def on_slot(slot, prow):
        for r in prow:
            item = r[1]
            members = sorted(cluster.groups[item].members) if item < 0 and item in cluster.groups else [item]
            rows.append(list(r) + [members, [cluster.sizes.get(m, 0) for m in members]])

    out = run_slots([(r.request_id, r.arrival_slot, r.prompt_tokens, r.response_tokens) for r in trace.records],
                    sched, cluster, topo, bounds, bpt=bpt, tokens_per_slot=doc["sim"]["tokens_per_slot"],
                    max_defer=doc["migration"]["max_defer"], duration_slots=w["duration_slots"],
                    on_slot=on_slot)
    doc["workload"]["kv_bytes_per_token"] = "per-request (models / model_bpt)"
    fp = hashlib.sha256(json.dumps([r[:7] for r in rows]).encode()).hexdigest()[:16]
    return {
        "config": doc, "models": {str(k): v for k, v in models.items()}, "model_bpt": model_bpt,
        "trace": [[r.request_id, r.arrival_slot, r.prompt_tokens, r.response_tokens] for r in trace.records],
        "plan_rows": rows, "slots": slots, "plan_rows_sha256_16": fp,
        "active_gpus": out.active_gpus, "migrations": out.logical_moves, "deferred": out.deferred,
        "forced": out.forced,
        "summary": {"peak_gpus": max(out.active_gpus), "completed": out.completed, "rejected": out.rejected,
                    "aborted": out.aborted, "total_migrations": sum(out.logical_moves)},
    }


def main() -> int:
    with open(os.path.join(HERE, "planner_cases.json"), "w") as fh:
        json.dump(planner_cases(), fh, separators=(",", ":"))
    with open(os.path.join(HERE, "boundaries.json"), "w") as fh:
        json.dump(boundaries_cases(), fh, separators=(",", ":"))
    for seed in (0, 2, 3):
        fx = trace_fixture(seed)
        with open(os.path.join(HERE, f"trace_7b_c48g_seed{seed}.json"), "w") as fh:
            json.dump(fx, fh, separators=(",", ":"))
        print(f"seed {seed}: {len(fx['trace'])} requests, {len(fx['plan_rows'])} plan rows, "
              f"peak {fx['summary']['peak_gpus']}, sha {fx['plan_rows_sha256_16']}")
    fx = trace_fixture(0, MIXED_DOC)
    with open(os.path.join(HERE, "trace_7b_mixed_seed0.json"), "w") as fh:
        json.dump(fx, fh, separators=(",", ":"))
    print(f"mixed seed 0: {len(fx['plan_rows'])} plan rows, modes "
          f"{sorted(set(r[6] for r in fx['plan_rows']))}, sha {fx['plan_rows_sha256_16']}")
    fx = multi_llm_fixture(0)
    with open(os.path.join(HERE, "trace_multillm_7b13b_seed0.json"), "w") as fh:
        json.dump(fx, fh, separators=(",", ":"))
    print(f"multi-LLM seed 0: {len(fx['trace'])} requests, {len(fx['plan_rows'])} plan rows, "
          f"peak {fx['summary']['peak_gpus']}, sha {fx['plan_rows_sha256_16']}")
    print("kvpack from", os.path.dirname(kvpack.__file__))
    return 0


if __name__ == "__main__":
    sys.exit(main())
