"""Control-plane timing: the native MellScheduler vs the reference's, per slot.

Runs the live slot loop (runtime.run_slots, planner included, no executor) on
(a) the reference's default run config (sim defaults: C = 120 000 B, 4 GPUs per
machine, 100 B/token, lambda = 0.5, 200 slots, batching on; SURVEY.md §6 quotes
1.62 ms/slot for the reference) and (b) the B200-shaped 7B config of SURVEY.md
§8c (C = 48 GiB, 8 GPUs per machine, scale 10), timing every step_epoch call.
The reference arm runs only where /root/reference is mounted.  Both arms must
produce the same plan rows (checked).

    python tools/bench_scheduler.py [--seeds 0 1 2]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2501_06709_b200 import cluster as ocl  # noqa: E402
from paper_2501_06709_b200 import scheduler as osch  # noqa: E402
from paper_2501_06709_b200.planner import Topology, load_boundaries  # noqa: E402
from paper_2501_06709_b200.runtime import run_slots  # noqa: E402
from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson  # noqa: E402

CONFIGS = {
    "reference-defaults": dict(capacity=120_000, gpm=4, bpt=100, scale=1, intra=50e9, inter=1.25e9,
                               prefill=10_000.0, epoch_s=1.0),
    "b200-7b-c48g": dict(capacity=48 << 30, gpm=8, bpt=524_288, scale=10, intra=900e9, inter=50e9,
                         prefill=50_000.0, epoch_s=0.05),
}


class Timed:
    """Wraps a scheduler; records wall time of every step_epoch."""

    def __init__(self, inner):
        self.inner, self.times = inner, []

    def step_epoch(self, *a, **k):
        t = time.perf_counter()
        r = self.inner.step_epoch(*a, **k)
        self.times.append(time.perf_counter() - t)
        return r


def run(kind: str, cfg: dict, seed: int, mod_cluster, mod_sched):
    trace = gen_poisson(0.5, 200, LengthDistribution(scale=cfg["scale"]), seed)
    cluster = mod_cluster.ClusterState(cfg["capacity"], gpus_per_machine=cfg["gpm"])
    sched = Timed(mod_sched.MellScheduler(cluster, priority_cfg=mod_sched.PriorityConfig(), batching=True))
    topo = Topology(gpus_per_machine=cfg["gpm"], intra_bandwidth_bytes_per_s=cfg["intra"],
                    inter_bandwidth_bytes_per_s=cfg["inter"], prefill_tokens_per_s=cfg["prefill"])
    bounds = load_boundaries(topo, cfg["epoch_s"], 0.2)
    t0 = time.perf_counter()
    out = run_slots(trace.tuples(), sched, cluster, topo, bounds, bpt=cfg["bpt"], tokens_per_slot=10,
                    duration_slots=200)
    wall = time.perf_counter() - t0
    st = sorted(sched.times)
    return {"impl": kind, "seed": seed, "requests": len(trace), "slots": len(st),
            "peak_gpus": max(out.active_gpus), "plan_rows": len(out.plan_rows),
            "step_epoch_ms_mean": 1e3 * statistics.fmean(st), "step_epoch_ms_p50": 1e3 * st[len(st) // 2],
            "step_epoch_ms_p99": 1e3 * st[min(len(st) - 1, int(0.99 * len(st)))],
            "loop_ms_per_slot": 1e3 * wall / len(st)}, out.plan_rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import sched_diff

    ref = sched_diff.kvpack()
    rows = []
    for name, cfg in CONFIGS.items():
        for seed in args.seeds:
            ours, rows_ours = run("native", cfg, seed, ocl, osch)
            ours["config"] = name
            rows.append(ours)
            print(json.dumps(ours))
            if ref is not None:
                theirs, rows_ref = run("reference", cfg, seed, ref, ref)
                theirs["config"] = name
                assert rows_ref == rows_ours, f"{name} seed {seed}: plan rows differ"
                theirs["speedup_step_epoch"] = theirs["step_epoch_ms_mean"] / ours["step_epoch_ms_mean"]
                rows.append(theirs)
                print(json.dumps(theirs))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
