"""configs[4] live: Poisson trace -> native MellScheduler -> planner -> GPU executor.

    python tools/online_loop.py [--fixture tests/golden/trace_multillm_7b13b_seed0.json]
                                [--shape mini|full] [--engine bulk|ldg] [--verify-every 100]

Nothing recorded is replayed: the trace comes from the generator
(paper_2501_06709_b200.workload, seeded as the fixture's config), decisions
from the native scheduler, and the migrations run on the GPU through the
executor.  The fixture only supplies the config and the reference's recorded
decisions, which the run must reproduce (checked).  Logical GPU g maps to
device g % device_count.  Prints one JSON line: per-slot control-plane time
(scheduler, planner), executor time, bytes moved and fingerprint checks.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from paper_2501_06709_b200 import ClusterState, MellScheduler, PriorityConfig  # noqa: E402
from paper_2501_06709_b200 import runtime  # noqa: E402
from paper_2501_06709_b200.planner import Topology, load_boundaries, plan_hybrid  # noqa: E402
from paper_2501_06709_b200.replay import FingerprintedExecutor  # noqa: E402
from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson  # noqa: E402
from replay_trace import FULL, LLAMA2_7B, MINI, MINI_7B, build  # noqa: E402


class Clock:
    def __init__(self):
        self.t = {}

    def wrap(self, key, fn):
        def inner(*a, **k):
            t0 = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                self.t[key] = self.t.get(key, 0.0) + time.perf_counter() - t0
        return inner


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fixture", default=os.path.join(ROOT, "tests", "golden", "trace_multillm_7b13b_seed0.json"))
    ap.add_argument("--shape", choices=["mini", "full"], default="mini")
    ap.add_argument("--engine", choices=["bulk", "ldg"], default="bulk")
    ap.add_argument("--verify-every", type=int, default=100)
    ap.add_argument("--seed", type=int, default=None,
                    help="another trace seed (same config); decisions are then not checked against the fixture")
    a = ap.parse_args()
    with open(a.fixture) as fh:
        fx = json.load(fh)
    cfg = fx["config"]
    cl, wl = cfg["cluster"], cfg["workload"]
    seed = cfg["sim"]["seed"] if a.seed is None else a.seed
    same_seed = seed == cfg["sim"]["seed"]
    trace = gen_poisson(wl["mean_interarrival_slots"], wl["duration_slots"], LengthDistribution(scale=wl["scale"]),
                        seed)
    models = {int(k): v for k, v in fx.get("models", {}).items()}
    if models and not same_seed:   # the fixture generator's model draw (tests/golden/make_golden.py)
        import numpy as np

        rng = np.random.default_rng(1000 + seed)
        models = {r.request_id: ("llama2-13b" if rng.random() < 0.5 else "llama2-7b") for r in trace.records}
    bpt = {rid: fx["model_bpt"][m] for rid, m in models.items()} if models else wl["kv_bytes_per_token"]
    if not same_seed:   # size the logical GPUs from a dry run of the scheduler (no data plane)
        c0 = ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
        t0_ = Topology(gpus_per_machine=cl["gpus_per_machine"],
                       intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                       inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                       prefill_tokens_per_s=cl["prefill_tokens_per_s"])
        dry = runtime.run_slots(trace.tuples(), MellScheduler(c0, PriorityConfig(), batching=True), c0, t0_,
                                load_boundaries(t0_, cfg["migration"]["epoch_seconds"],
                                                cfg["migration"]["budget_fraction"]),
                                bpt=bpt, tokens_per_slot=cfg["sim"]["tokens_per_slot"],
                                max_defer=cfg["migration"]["max_defer"], duration_slots=wl["duration_slots"])
        fx = dict(fx, summary=dict(fx["summary"], peak_gpus=dry.peak_gpus))
    shapes = MINI if a.shape == "mini" else FULL
    devices = list(range(torch.cuda.device_count()))
    inner, nb = build(fx, MINI_7B if a.shape == "mini" else LLAMA2_7B, a.engine, devices, shapes)
    inner.timing = True          # per-call device time (CUDA events) in every ExecReport
    ex = FingerprintedExecutor(inner)
    clock = Clock()
    ex.execute = clock.wrap("executor", ex.execute)
    cluster = ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = MellScheduler(cluster, priority_cfg=PriorityConfig(), batching=True)
    sched.step_epoch = clock.wrap("scheduler", sched.step_epoch)
    runtime.plan_hybrid = clock.wrap("planner", plan_hybrid)
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, cfg["migration"]["epoch_seconds"], cfg["migration"]["budget_fraction"])
    checked = []

    def on_slot(slot, rows):
        if a.verify_every and slot % a.verify_every == a.verify_every - 1:
            checked.append(ex.verify())

    t0 = time.perf_counter()
    out = runtime.run_slots(trace.tuples(), sched, cluster, topo, bounds, bpt=bpt,
                            tokens_per_slot=cfg["sim"]["tokens_per_slot"], max_defer=cfg["migration"]["max_defer"],
                            duration_slots=wl["duration_slots"], executor=ex,
                            models={rid: shapes[m].name for rid, m in models.items()}, on_slot=on_slot)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    n = len(out.active_gpus)
    parity = (out.plan_rows == [r[:7] for r in fx["plan_rows"]] and out.active_gpus == fx["active_gpus"]
              if same_seed else None)
    print(json.dumps({
        "fixture": os.path.basename(a.fixture), "seed": seed, "shape": a.shape, "devices": len(devices),
        "logical_gpus": len(inner.pools), "slots": n, "requests": len(trace), "peak_gpus": max(out.active_gpus),
        "plan_rows": len(out.plan_rows), "executed_records": sum(len(r.records) for r in ex.reports),
        "bytes_moved": out.bytes_moved, "decisions_match_reference": parity,
        "fingerprint_checks": sum(checked),
        "ms_per_slot": {k: 1e3 * v / n for k, v in clock.t.items()} | {"loop": 1e3 * wall / n},
        "executor_GBps_while_moving": out.bytes_moved / clock.t.get("executor", 1e-9) / 1e9,
        "device_ms_total": round(sum(max(r.device_ms.values(), default=0.0) for r in ex.reports), 3),
        "device_copy_GBps": round(out.bytes_moved / max(1e-9, sum(max(r.device_ms.values(), default=0.0)
                                                                for r in ex.reports)) / 1e6, 1),
    }))
    if parity is False:
        raise SystemExit("decisions differ from the reference's recorded run")


if __name__ == "__main__":
    main()
