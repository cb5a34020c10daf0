"""configs[4] live: Poisson trace -> native MellScheduler -> planner -> GPU executor.

    python tools/online_loop.py [--fixture tests/golden/trace_multillm_7b13b_seed0.json]
                                [--shape mini|full] [--engine bulk|ldg] [--verify-every 100]
                                [--max-slots N] [--split]

Nothing recorded is replayed: the trace comes from the generator
(paper_2501_06709_b200.workload, seeded as the fixture's config), decisions
from the native scheduler, and the migrations run on the GPU through the
executor.  The fixture only supplies the config and the reference's recorded
decisions, which the run must reproduce (checked, over the slots run).
Logical GPU g maps to device g % device_count: with 8 visible GPUs every
logical GPU of the trace is its own B200 and every kv move crosses NVLink.

--shape full uses the real Llama-2-7B / 13B KV geometry (512 / 800 KiB per
token).  Pools are sized from a dry run of the same loop on host-only pools
(the exact peak of blocks each logical GPU physically holds, which the
deferred-move skew puts above the logical capacity), plus a
small margin, instead of a blanket 1.5 x capacity.  Prints one JSON line:
per-slot control-plane time (scheduler, planner), executor time, bytes moved
and fingerprint checks.
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
from paper_2501_06709_b200.executor import MigrationExecutor  # noqa: E402
from paper_2501_06709_b200.kvcache import BlockAllocator, BlockTable, KVPool  # noqa: E402
from paper_2501_06709_b200.planner import Topology, load_boundaries, plan_hybrid  # noqa: E402
from paper_2501_06709_b200.replay import FingerprintedExecutor, pool_blocks_for  # noqa: E402
from paper_2501_06709_b200.reprefill import ReprefillEngine, sm_budget  # noqa: E402
from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson  # noqa: E402
from replay_trace import FULL, MINI  # noqa: E402


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


class _HostPool:
    """Block bookkeeping only (dry run): no device memory."""

    def __init__(self, shape, nb, pool_id):
        self.shape, self.num_blocks, self.device, self.pool_id = shape, nb, 0, pool_id
        self.allocator = BlockAllocator(nb)


class _NoStream:
    cuda_stream = 0

    def synchronize(self):
        pass

    def wait_stream(self, other):
        pass


class DryRunExecutor(MigrationExecutor):
    """The executor's bookkeeping with nothing launched: measures the peak
    number of blocks every logical GPU's pool physically holds."""

    def __init__(self, pools):
        super().__init__(pools, reprefill=lambda *a: None)
        self.peak = {(g, m): 0 for g, per in self.pools.items() for m in per}

    def _track(self):
        for g, per in self.pools.items():
            for m, p in per.items():
                used = p.num_blocks - p.allocator.n_free
                if used > self.peak[(g, m)]:
                    self.peak[(g, m)] = used

    def stream(self, device):
        return _NoStream()

    def ordered_stream(self, device):
        return _NoStream()

    def _launch_migrate(self, dev, moves, dst_pools=()):
        pass

    def _issue_split(self, pm, rec, rid, res, src_pool, dst_pool, dst_blocks, table_for):
        pass

    def admit(self, *a, **k):
        r = super().admit(*a, **k)
        self._track()
        return r

    def grow(self, *a, **k):
        r = super().grow(*a, **k)
        self._track()
        return r

    def _issue(self, *a, **k):
        self._track()            # destination blocks reserved, sources not yet freed: the true peak
        return super()._issue(*a, **k)

    def execute(self, *a, **k):
        r = super().execute(*a, **k)
        self._track()
        return r


def _setup(fx, seed):
    cfg = fx["config"]
    cl, wl = cfg["cluster"], cfg["workload"]
    trace = gen_poisson(wl["mean_interarrival_slots"], wl["duration_slots"], LengthDistribution(scale=wl["scale"]),
                        seed)
    models = {int(k): v for k, v in fx.get("models", {}).items()}
    if models and seed != cfg["sim"]["seed"]:   # the fixture generator's model draw (tests/golden/make_golden.py)
        import numpy as np

        rng = np.random.default_rng(1000 + seed)
        models = {r.request_id: ("llama2-13b" if rng.random() < 0.5 else "llama2-7b") for r in trace.records}
    bpt = {rid: fx["model_bpt"][m] for rid, m in models.items()} if models else wl["kv_bytes_per_token"]
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, cfg["migration"]["epoch_seconds"], cfg["migration"]["budget_fraction"])
    return trace, models, bpt, topo, bounds


def _loop(fx, trace, bpt, topo, bounds, executor, models, shapes, max_slots, split, on_slot=None, sched_wrap=None):
    cfg = fx["config"]
    cl, wl = cfg["cluster"], cfg["workload"]
    cluster = ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = MellScheduler(cluster, priority_cfg=PriorityConfig(), batching=True)
    if sched_wrap is not None:
        sched.step_epoch = sched_wrap(sched.step_epoch)
    return runtime.run_slots(trace.tuples(), sched, cluster, topo, bounds, bpt=bpt,
                             tokens_per_slot=cfg["sim"]["tokens_per_slot"], max_defer=cfg["migration"]["max_defer"],
                             duration_slots=wl["duration_slots"], executor=executor,
                             models={rid: shapes[m].name for rid, m in models.items()}, on_slot=on_slot,
                             split=split, max_slots=max_slots)


def dry_run_pool_blocks(fx, trace, models, bpt, topo, bounds, shapes, max_slots, split):
    """{(logical gpu, model name): peak blocks held} from a host-only run, and the peak GPU count."""
    mnames = sorted(set(models.values())) if models else [None]
    big = {m: pool_blocks_for(fx, 16, headroom=4.0, model=m) for m in mnames}
    n0 = max(fx["summary"]["peak_gpus"], 1) + 8
    pools = {}
    pid = 0
    for g in range(n0):
        per = {}
        for m in mnames:
            sh = shapes[m] if m else shapes["llama2-7b"]
            per[sh.name] = _HostPool(sh, big[m], pid)
            pid += 1
        pools[g] = per
    dry = DryRunExecutor(pools)
    out = _loop(fx, trace, bpt, topo, bounds, dry, models, shapes, max_slots, split)
    return dry.peak, out.peak_gpus


def run_online(fixture: str, shape: str = "mini", engine: str = "bulk", verify_every: int = 100,
               seed=None, max_slots=None, split: bool = False, devices=None, margin: float = 1.02,
               reprefill_sm_fraction: float = 1.0) -> dict:
    with open(fixture) as fh:
        fx = json.load(fh)
    cfg = fx["config"]
    seed = cfg["sim"]["seed"] if seed is None else seed
    same_seed = seed == cfg["sim"]["seed"]
    trace, models, bpt, topo, bounds = _setup(fx, seed)
    shapes = MINI if shape == "mini" else FULL
    devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    peak, peak_gpus = dry_run_pool_blocks(fx, trace, models, bpt, topo, bounds, shapes, max_slots, split)
    pools, tables = {}, {}
    per_dev_bytes = {}
    need = {}
    for (pg, name), blocks in peak.items():   # fail before allocating when the pools cannot fit
        sh = next(s for s in shapes.values() if s.name == name)
        d = devices[pg % len(devices)]
        need[d] = need.get(d, 0) + sh.pool_bytes(max(16, int(blocks * margin) + 64))
    for d, b in need.items():
        free = torch.cuda.mem_get_info(d)[0]
        if b > free - (2 << 30):
            raise SystemExit(f"online_loop: the pools of the logical GPUs on device {d} need {b / 2 ** 30:.1f} GiB, "
                             f"{free / 2 ** 30:.1f} GiB free: use more --devices or fewer --max-slots")
    for g in range(peak_gpus):
        dev = devices[g % len(devices)]
        pools[g], tables[g] = {}, {}
        for (pg, name), blocks in peak.items():
            if pg != g:
                continue
            sh = next(s for s in shapes.values() if s.name == name)
            nb = max(16, int(blocks * margin) + 64)
            per_dev_bytes[dev] = per_dev_bytes.get(dev, 0) + sh.pool_bytes(nb)
            pools[g][name] = KVPool(sh, nb, device=dev, dtype=torch.bfloat16)
            tables[g][name] = BlockTable(512, nb, device=dev)
    used = sorted({s.name for per in pools.values() for s in (p.shape for p in per.values())})
    # re-prefill on the budget fraction of the SMs (reprefill.sm_budget; 1.0 = every SM)
    max_sms = sm_budget(reprefill_sm_fraction, torch.cuda.get_device_properties(0).multi_processor_count)
    rp = ReprefillEngine([s for s in shapes.values() if s.name in used], sorted({p.device for per in pools.values()
                                                                               for p in per.values()}), with_q=False,
                         max_sms=max_sms)
    inner = MigrationExecutor(pools, tables, engine=engine, reprefill=rp, timing=True)
    ex = FingerprintedExecutor(inner)
    clock = Clock()
    inner.execute = clock.wrap("executor", inner.execute)   # the executor alone (not the stamps)
    runtime.plan_hybrid = clock.wrap("planner", plan_hybrid)
    # test harness, not the product: fingerprint stamps written into every block a request gains
    # (a stand-in for the prefill/decode that fills them in a server) and the periodic read-back checks
    ex.fp.flush = clock.wrap("fingerprint", ex.fp.flush)
    checked = []

    def timed_verify():
        f0, t0 = clock.t.get("fingerprint", 0.0), time.perf_counter()
        n_ok = ex.verify()                      # its own flush() is already counted by the wrapper
        dt = time.perf_counter() - t0 - (clock.t.get("fingerprint", 0.0) - f0)
        clock.t["fingerprint"] = clock.t.get("fingerprint", 0.0) + dt
        return n_ok

    def on_slot(slot, rows):
        if verify_every and slot % verify_every == verify_every - 1:
            checked.append(timed_verify())

    t0 = time.perf_counter()
    try:
        out = _loop(fx, trace, bpt, topo, bounds, ex, models, shapes, max_slots, split, on_slot=on_slot,
                    sched_wrap=lambda f: clock.wrap("scheduler", f))
    finally:
        runtime.plan_hybrid = plan_hybrid
    for d in sorted({p.device for per in pools.values() for p in per.values()}):
        torch.cuda.synchronize(d)
    wall = time.perf_counter() - t0
    checked.append(ex.verify())
    n = len(out.active_gpus)
    parity = None
    if same_seed and not split:
        ref_rows = [r[:7] for r in fx["plan_rows"] if r[0] < n]
        parity = out.plan_rows == ref_rows and out.active_gpus == fx["active_gpus"][:n]
    dev_ms = sum(max(r.device_ms.values(), default=0.0) for r in ex.reports)
    return {
        "fixture": os.path.basename(fixture), "seed": seed, "shape": shape, "devices": len(devices),
        "logical_gpus": len(inner.pools), "device_of_gpu": {g: devices[g % len(devices)] for g in pools},
        "pool_gib_per_device": {d: round(b / 2 ** 30, 2) for d, b in per_dev_bytes.items()},
        "slots": n, "requests": len(trace), "peak_gpus": max(out.active_gpus), "reprefill_max_sms": max_sms,
        "plan_rows": len(out.plan_rows), "executed_records": sum(len(r.records) for r in ex.reports),
        "bytes_moved": out.bytes_moved, "reconciled_moves": out.reconciled_moves,
        "splits": sum(1 for r in out.plan_rows if r[6] == "split_transfer"),
        "decisions_match_reference": parity, "fingerprint_checks": sum(checked),
        "ms_per_slot": {k: 1e3 * v / n for k, v in clock.t.items()} | {
            "loop": 1e3 * wall / n, "loop_minus_fingerprint": 1e3 * (wall - clock.t.get("fingerprint", 0.0)) / n},
        "executor_GBps_while_moving": out.bytes_moved / clock.t.get("executor", 1e-9) / 1e9,
        "device_ms_total": round(dev_ms, 3),
        "device_copy_GBps": round(out.bytes_moved / max(1e-9, dev_ms) / 1e6, 1),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fixture", default=os.path.join(ROOT, "tests", "golden", "trace_multillm_7b13b_seed0.json"))
    ap.add_argument("--shape", choices=["mini", "full"], default="mini")
    ap.add_argument("--engine", choices=["bulk", "ldg"], default="bulk")
    ap.add_argument("--verify-every", type=int, default=100)
    ap.add_argument("--max-slots", type=int, default=None)
    ap.add_argument("--split", action="store_true", help="planner split mode (extension)")
    ap.add_argument("--seed", type=int, default=None,
                    help="another trace seed (same config); decisions are then not checked against the fixture")
    ap.add_argument("--devices", type=int, default=None, help="spread logical GPUs over the first N devices")
    ap.add_argument("--out", default=None, help="also write the JSON result here (bench.py's subprocess run)")
    ap.add_argument("--reprefill-sm-fraction", type=float, default=1.0,
                    help="run token_transfer re-prefills on this fraction of the SMs (e.g. the run's budget_fraction)")
    a = ap.parse_args()
    res = run_online(a.fixture, a.shape, a.engine, a.verify_every, a.seed, a.max_slots, a.split,
                     devices=None if a.devices is None else list(range(a.devices)),
                     reprefill_sm_fraction=a.reprefill_sm_fraction)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh)
    print(json.dumps(res))
    if res["decisions_match_reference"] is False:
        raise SystemExit("decisions differ from the reference's recorded run")


if __name__ == "__main__":
    main()
