"""Live slot loop: any `step_epoch` scheduler -> planner -> GPU executor.

This is the reference's slot loop (sim.py:151-227) with the data plane filled
in.  The scheduler is the caller of the hot path and is used through the
reference's duck-typed plugin API:

    scheduler.step_epoch(arrivals: [(rid, size_bytes)], completions: [rid],
                         growths={rid: size_bytes}) -> EpochResult
                                                         (scheduler.py:979-981)
    result.logs[i].moves  -> Move(item, src|None, dst, reason)   (scheduler.py:24-45)
    result.logs[i].events -> ("rejected"|"aborted"|..., detail)

and the cluster object it mutates is read through `placement`, `item_size`,
`groups[gid].members` and `gpus[g].residents` (model.py:122-146).  So the
reference's own MellScheduler/ClusterState plug in unchanged; the physical
side (pools, blocks, bytes) is the executor's.

Reference line map for the loop body:
    growth / completions            sim.py:153-171
    step_epoch                      sim.py:177
    backlog + chain collapse        sim.py:179-187
    departures / arrivals           sim.py:196-205
    backlog refresh                 sim.py:207-217
    plan + execute + retire/defer   sim.py:218-227   (executor.execute is the new part)
"""
from __future__ import annotations

import os

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .planner import PendingMove, plan_hybrid


@dataclass
class LoopResult:
    """Per-slot series with the reference's MetricsSeries columns (sim.py:27-63):
    active_gpus, migrations (= logical_moves), deferred, forced, used_bytes,
    capacity_bytes; plus the executed plan rows and bytes physically moved."""
    plan_rows: List[list] = field(default_factory=list)   # (slot, item, src, dst, kv_bytes, tokens, mode)
    active_gpus: List[int] = field(default_factory=list)
    logical_moves: List[int] = field(default_factory=list)
    deferred: List[int] = field(default_factory=list)
    forced: List[int] = field(default_factory=list)
    used_bytes: List[int] = field(default_factory=list)      # sim.py:231-234 (KV bytes that exist)
    capacity_bytes: List[int] = field(default_factory=list)  # active GPUs x C
    bytes_moved: int = 0
    reconciled_moves: int = 0      # executor.reconcile moves (outside the plan)
    reconciled_bytes: int = 0
    completed: int = 0
    rejected: int = 0
    aborted: int = 0
    requests: int = 0
    config: Optional[Dict[str, dict]] = None   # the resolved run config (simulate)

    @property
    def peak_gpus(self) -> int:
        return max(self.active_gpus, default=0)

    # -- the reference's output files (sim.py:240-333) ------------------------------
    def metrics_csv(self) -> str:
        """metrics_to_csv: header + one row per slot (sim.py:312-321)."""
        import csv
        import io

        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["slot", "active_gpus", "migrations", "deferred", "forced", "used_bytes", "capacity_bytes"])
        w.writerows(zip(range(len(self.active_gpus)), self.active_gpus, self.logical_moves, self.deferred,
                        self.forced, self.used_bytes, self.capacity_bytes))
        return buf.getvalue()

    @property
    def summary(self) -> Dict[str, object]:
        """RunResult.summary (sim.py:240-257) for a Mell run."""
        cfg = self.config or resolve_config({})
        n = len(self.active_gpus)
        return {"schema_version": 1, "scheduler": cfg["scheduler"]["kind"],
                "batching": cfg["scheduler"]["batching"], "slots": n, "peak_gpus": self.peak_gpus,
                "total_migrations": sum(self.logical_moves), "total_deferred": sum(self.deferred),
                "total_forced": sum(self.forced), "mean_active_gpus": sum(self.active_gpus) / n if n else 0.0,
                "mean_utilization": self.mean_utilization, "requests": self.requests, "completed": self.completed,
                "rejected": self.rejected, "aborted": self.aborted,
                "config": {**{k: dict(v) for k, v in cfg.items()}, "schema_version": 1}}

    def write_metrics_csv(self, path: str) -> None:
        with open(path, "w", encoding="utf-8", newline="") as fh:
            fh.write(self.metrics_csv())

    def write_summary_json(self, path: str) -> None:
        """write_summary_json (sim.py:329-333): indent 2, sorted keys, newline."""
        import json

        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.summary, fh, indent=2, sort_keys=True)
            fh.write("\n")

    @property
    def mean_utilization(self) -> float:
        r = [u / c for u, c in zip(self.used_bytes, self.capacity_bytes) if c > 0]
        return sum(r) / len(r) if r else 0.0


def _completion_slot(arrival: int, response: int, tps: int) -> int:
    return arrival + math.ceil(response / tps)


def _size_at(rec, slot, tps, bpt) -> int:
    _, arrival, prompt, response = rec
    return (prompt + min(response, tps * (slot - arrival))) * bpt


def run_slots(records: Sequence[Tuple[int, int, int, int]], scheduler, cluster, topology, boundaries, *,
              bpt, tokens_per_slot: int = 10, epoch_slots: int = 1, max_defer: int = 3,
              duration_slots: int = 0, executor=None, reserve_final: bool = False,
              models: Optional[Dict[int, str]] = None,
              on_slot: Optional[Callable[[int, list], None]] = None, reconcile: bool = True,
              split: bool = False, max_slots: Optional[int] = None) -> LoopResult:
    """Run the slot loop; `records` are (request_id, arrival_slot, prompt, response).

    `bpt` is the reference's kv_bytes_per_token (config.py:92), or — multi-LLM
    extension — a dict request id -> bytes/token of that request's model
    (the reference Request already carries a per-request bpt, model.py:38;
    sim.run just sets them all equal).  `models` names each request's model
    for the executor's per-model pools.  With an executor, placements become
    executor.admit, growth executor.grow, departures executor.release and
    executed plan rows executor.execute.  reconcile: after the plan, requests
    whose physical GPU differs from their item's logical GPU and whose item
    is not in the backlog are moved there (executor.reconcile; member-level
    moves the reference's refresh drops, sim.py:207-213); counted in
    `reconciled_moves` / `reconciled_bytes`, not in the plan rows.  split:
    the planner's split mode (plan_hybrid(split=True), extension, off by
    default so the plan rows stay the reference's).  max_slots: stop after
    that many slots (a bounded prefix of the run; the rows so far are the
    reference's).
    """
    tps = tokens_per_slot
    recs = {r[0]: tuple(r) for r in records}
    per_req = isinstance(bpt, dict)
    bpt_of = (lambda rid: bpt[rid]) if per_req else (lambda rid: bpt)
    models = models or {}

    def item_tokens(item: int, size: int) -> int:
        """sim.py:217 (size // bpt); per member for a mixed-model group."""
        if not per_req:
            return size // bpt
        if item < 0:
            return sum(cluster.sizes[m] // bpt[m] for m in cluster.groups[item].members)
        return size // bpt[item]

    by_slot: Dict[int, List[int]] = {}
    for rid, (_, arrival, _p, _r) in recs.items():
        by_slot.setdefault(arrival, []).append(rid)
    last_arrival = max((r[1] for r in recs.values()), default=-1)
    horizon = max(duration_slots, last_arrival + 1)
    running: Dict[int, tuple] = {}
    buffered: List[Tuple[int, int]] = []
    pending: Dict[int, PendingMove] = {}
    defer_counts: Dict[int, int] = {}
    out = LoopResult()
    slot = 0
    while slot < horizon or running or buffered:
        growths, completions = {}, []
        size_now: Dict[int, int] = {}   # _size_at(request, this slot), computed once per request and slot

        def size_of(rid):
            v = size_now.get(rid)
            if v is None:
                v = size_now[rid] = _size_at(recs[rid], slot, tps, bpt_of(rid))
            return v

        for rid, rec in running.items():
            if _completion_slot(rec[1], rec[3], tps) <= slot:
                completions.append(rid)
            else:
                growths[rid] = size_of(rid)
        for rid in by_slot.get(slot, []):
            _, _a, prompt, response = recs[rid]
            size = (prompt + response) * bpt_of(rid) if reserve_final else prompt * bpt_of(rid)
            buffered.append((rid, size))
        if slot % epoch_slots == 0:
            arrivals, buffered = buffered, []
        else:
            arrivals = []
        result = scheduler.step_epoch(arrivals, completions, growths=growths)
        n_moves = 0
        gone = set(completions)
        for log in result.logs:
            for mv in log.moves:
                if mv.src is not None:
                    n_moves += 1
                    phys = pending[mv.item].src if mv.item in pending else mv.src
                    pending[mv.item] = PendingMove(mv.item, phys, mv.dst, 0, 0)
            for kind, *detail in log.events:
                if kind == "rejected":
                    out.rejected += 1
                    gone.add(int(detail[0]))
                elif kind == "aborted":
                    out.aborted += 1
                    gone.add(int(detail[0]))
        for rid in completions:
            running.pop(rid, None)
            out.completed += 1
        for rid in gone - set(completions):
            running.pop(rid, None)
        for rid, _size in arrivals:
            if rid not in gone:
                running[rid] = recs[rid]
        if executor is not None:
            for rid in gone:
                executor.release(rid)
            for rid in running:
                if rid in executor.loc:
                    tok = size_of(rid) // bpt_of(rid)
                    if tok > executor.loc[rid].tokens:
                        executor.grow(rid, tok)
            for rid, size in arrivals:
                if rid in running and rid not in executor.loc:
                    gpu = cluster.placement.get(cluster.item_of_request(rid))
                    if gpu is not None:
                        executor.admit(rid, gpu, size // bpt_of(rid), model=models.get(rid))
        # data plane: refresh backlog, plan, execute, retire
        for item in list(pending):
            loc = cluster.placement.get(item)
            if loc is None or loc == pending[item].src:
                del pending[item]
                defer_counts.pop(item, None)
                continue
            size = cluster.item_size(item)
            pending[item] = PendingMove(item, pending[item].src, loc, size, item_tokens(item, size))
        plan = plan_hybrid(list(pending.values()), boundaries, topology, defer_counts=defer_counts,
                           max_defer=max_defer, split=split)
        rows = [[slot, p.move.item, p.move.src, p.move.dst, p.move.kv_bytes, p.move.tokens, p.mode]
                for p in plan.assignments]
        out.plan_rows.extend(rows)
        if executor is not None and plan.executed:
            rep = executor.execute(plan, members_of=lambda gid: sorted(cluster.groups[gid].members)
                                   if gid in cluster.groups else [])
            out.bytes_moved += rep.bytes_moved
        for planned in plan.executed:
            del pending[planned.move.item]
            defer_counts.pop(planned.move.item, None)
        if executor is not None and reconcile:
            # bytes of requests whose logical move never reached the planner (member-level
            # moves, dropped at the refresh above) follow their item now; members of items
            # still pending travel with the item's planned move
            waiting = set()
            for item in pending:
                waiting.update(cluster.groups[item].members if item < 0 and item in cluster.groups else (item,))
            placement, rgroup = cluster.placement, cluster.request_group   # item_of_request, model.py:248-250
            rep = executor.reconcile(lambda rid: placement.get(rgroup.get(rid, rid)), skip=waiting)
            out.reconciled_moves += len(rep.records)
            out.reconciled_bytes += rep.bytes_moved
        for mv in plan.deferred:
            defer_counts[mv.item] = defer_counts.get(mv.item, 0) + 1
        active = sum(1 for g in cluster.gpus.values() if g.residents)
        out.active_gpus.append(active)
        sizes = cluster.sizes
        sizes = sizes.as_dict() if hasattr(sizes, "as_dict") else sizes
        out.used_bytes.append(sum(min(size_of(rid), cluster.capacity_bytes)
                                  for rid, rec in running.items() if rid in sizes))
        out.capacity_bytes.append(active * cluster.capacity_bytes)
        out.logical_moves.append(n_moves)
        out.deferred.append(len(plan.deferred))
        out.forced.append(len(plan.forced))
        if on_slot is not None:
            on_slot(slot, rows)
        slot += 1
        if max_slots is not None and slot >= max_slots:
            break
        if slot > horizon + 10 ** 6:
            raise RuntimeError("slot loop failed to drain")
    return out


# The reference's run-config schema (config.py:20-128): section -> {key: default}.
_CONFIG_DEFAULTS = {
    "cluster": {"capacity_bytes": 120_000, "gpus_per_machine": 4, "max_gpus": 1024,
                "intra_bandwidth_bytes_per_s": 50e9, "inter_bandwidth_bytes_per_s": 1.25e9,
                "prefill_tokens_per_s": 10_000.0},
    "scheduler": {"kind": "mell", "batching": True, "weight_free_mem": 1.0, "weight_request_count": 0.25,
                  "weight_same_machine": 0.5, "rebalance_period": 1, "imbalance_threshold": 0.25},
    "migration": {"epoch_seconds": 1.0, "budget_fraction": 0.2, "max_defer": 3},
    "workload": {"trace_path": None, "mean_interarrival_slots": 0.5, "duration_slots": 200,
                 "prompt_mean_log": 4.6, "prompt_sigma_log": 0.8, "response_mean_log": 5.3,
                 "response_sigma_log": 0.9, "scale": 1, "kv_bytes_per_token": 100},
    "sim": {"seed": 0, "tokens_per_slot": 10, "epoch_slots": 1},
}


# value checks of each section, in the reference's order (config.py:29-120)
_SCHEDULER_KINDS = ("mell", "bf", "wf", "lb")


def _check_section(name: str, c: dict) -> Optional[str]:
    if name == "cluster":
        if c["capacity_bytes"] <= 0:
            return "cluster.capacity_bytes must be > 0"
        if c["gpus_per_machine"] < 1:
            return "cluster.gpus_per_machine must be >= 1"
        if c["max_gpus"] < 1:
            return "cluster.max_gpus must be >= 1"
        for k in ("intra_bandwidth_bytes_per_s", "inter_bandwidth_bytes_per_s", "prefill_tokens_per_s"):
            if c[k] <= 0:
                return f"cluster.{k} must be > 0"
    elif name == "scheduler":
        if c["kind"] not in _SCHEDULER_KINDS:
            return f"scheduler.kind must be one of {_SCHEDULER_KINDS}"
        for k in ("weight_free_mem", "weight_request_count", "weight_same_machine"):
            if c[k] < 0:
                return f"scheduler.{k} must be >= 0"
        if c["rebalance_period"] < 1:
            return "scheduler.rebalance_period must be >= 1"
        if not 0.0 < c["imbalance_threshold"] < 1.0:
            return "scheduler.imbalance_threshold must be in (0, 1)"
    elif name == "migration":
        if c["epoch_seconds"] <= 0:
            return "migration.epoch_seconds must be > 0"
        if not 0.0 < c["budget_fraction"] <= 1.0:
            return "migration.budget_fraction must be in (0, 1]"
        if c["max_defer"] < 0:
            return "migration.max_defer must be >= 0"
    elif name == "workload":
        if c["mean_interarrival_slots"] <= 0:
            return "workload.mean_interarrival_slots must be > 0"
        if c["duration_slots"] < 0:
            return "workload.duration_slots must be >= 0"
        for k in ("prompt_sigma_log", "response_sigma_log"):
            if c[k] < 0:
                return f"workload.{k} must be >= 0"
        if c["scale"] < 1:
            return "workload.scale must be >= 1"
        if c["kv_bytes_per_token"] <= 0:
            return "workload.kv_bytes_per_token must be > 0"
    elif name == "sim":
        if c["tokens_per_slot"] < 1:
            return "sim.tokens_per_slot must be >= 1"
        if c["epoch_slots"] < 1:
            return "sim.epoch_slots must be >= 1"
    return None


def _type_error(name: str, key: str, default, value) -> Optional[str]:
    """The reference's per-key type rule (config.py:150-170), keyed on the
    declared type, which the defaults carry (trace_path: Optional, unchecked)."""
    if default is None:
        return None
    if isinstance(default, bool):
        return None if isinstance(value, bool) else f"{name}.{key} must be a boolean"
    if isinstance(default, int):
        return None if isinstance(value, int) and not isinstance(value, bool) else f"{name}.{key} must be an integer"
    if isinstance(default, float):
        ok = isinstance(value, (int, float)) and not isinstance(value, bool)
        return None if ok else f"{name}.{key} must be a number"
    if isinstance(default, str):
        return None if isinstance(value, str) else f"{name}.{key} must be a string"
    return None


def resolve_config(doc: Optional[dict] = None) -> Dict[str, dict]:
    """A reference run-config document (config.py's JSON schema, sections
    cluster / scheduler / migration / workload / sim) with the reference's
    defaults filled in and validated like config_from_dict (config.py:150-186,
    dataclass __post_init__ checks): unknown sections or keys, wrong types and
    out-of-range values raise ConfigError with the reference's messages.
    Idempotent (a resolved config resolves to itself)."""
    from .errors import ConfigError

    if doc is not None and not isinstance(doc, dict):
        raise ConfigError("config root must be a JSON object")
    doc = dict(doc or {})
    unknown = set(doc) - set(_CONFIG_DEFAULTS) - {"schema_version"}
    if unknown:
        raise ConfigError(f"unknown top-level keys: {sorted(unknown)}")
    version = doc.pop("schema_version", 1)
    if not isinstance(version, int) or isinstance(version, bool):
        raise ConfigError("schema_version must be an integer")
    out = {}
    for name, defaults in _CONFIG_DEFAULTS.items():
        sec = doc.get(name, {})
        if not isinstance(sec, dict):
            raise ConfigError(f"section {name!r} must be an object")
        bad = set(sec) - set(defaults)
        if bad:
            raise ConfigError(f"unknown keys in section {name!r}: {sorted(bad)}")
        for key, value in sec.items():
            err = _type_error(name, key, defaults[key], value)
            if err:
                raise ConfigError(err)
        out[name] = {**defaults, **sec}
        err = _check_section(name, out[name])
        if err:
            raise ConfigError(err)
    if version != 1:
        raise ConfigError(f"unsupported schema_version {version}, expected 1")
    return out


def load_config(path: str) -> Dict[str, dict]:
    """A run-config JSON file -> resolve_config (config.py:189-197); unreadable
    files and bad JSON raise ConfigError like the reference's loader."""
    import json

    from .errors import ConfigError

    try:
        with open(path, "r", encoding="utf-8") as fh:
            doc = json.load(fh)
    except OSError as exc:
        raise ConfigError(f"cannot read config {path!r}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigError(f"invalid JSON in {path!r}: {exc}") from exc
    return resolve_config(doc)


def simulate(doc: Optional[dict] = None, records=None, *,
             executor=None, bpt=None, models: Optional[Dict[int, str]] = None,
             on_slot: Optional[Callable[[int, list], None]] = None) -> LoopResult:
    """Drop-in for the Mell path of the reference's `sim.run(config, trace)`
    (sim.py:103-268): build ClusterState + the native MellScheduler, Topology
    and Boundaries from a reference config document, take the trace from
    `records` (a workload.Trace or (id, slot, prompt, response) rows), else from
    workload.trace_path (a trace CSV, workload.load_trace), else generate the
    Poisson trace from the workload section (cli.py:54-66), and run the live slot
    loop (optionally executing every plan on the GPUs through `executor`).
    `bpt` overrides workload.kv_bytes_per_token (an int, or a per-request dict
    for multi-LLM traces).  Returns the reference's metric series (LoopResult)."""
    from .cluster import ClusterState
    from .errors import ConfigError
    from .planner import Topology, load_boundaries
    from .scheduler import MellScheduler, PriorityConfig
    from .workload import LengthDistribution, Trace, gen_poisson, load_trace

    cfg = resolve_config(doc)   # idempotent: a load_config() result passes through
    cl, sc, mg, wl, sm = (cfg[k] for k in ("cluster", "scheduler", "migration", "workload", "sim"))
    if sc["kind"] != "mell":
        raise ConfigError(f"scheduler kind {sc['kind']!r}: only Mell's scheduler is provided "
                          "(the reference's bf/wf/lb baselines are out of scope)")
    if isinstance(records, Trace):
        records = records.tuples()
    if records is None and wl["trace_path"]:
        if not os.path.exists(wl["trace_path"]):
            raise ConfigError(f"trace file not found: {wl['trace_path']}")
        records = load_trace(wl["trace_path"]).tuples()
    if records is None:
        dist = LengthDistribution(prompt_mean_log=wl["prompt_mean_log"], prompt_sigma_log=wl["prompt_sigma_log"],
                                  response_mean_log=wl["response_mean_log"],
                                  response_sigma_log=wl["response_sigma_log"], scale=wl["scale"])
        records = gen_poisson(wl["mean_interarrival_slots"], wl["duration_slots"], dist, sm["seed"]).tuples()
    cluster = ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = MellScheduler(cluster, PriorityConfig(sc["weight_free_mem"], sc["weight_request_count"],
                                                  sc["weight_same_machine"]), batching=sc["batching"])
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, mg["epoch_seconds"], mg["budget_fraction"])
    records = list(records)
    res = run_slots(records, sched, cluster, topo, bounds, bpt=wl["kv_bytes_per_token"] if bpt is None else bpt,
                    tokens_per_slot=sm["tokens_per_slot"], epoch_slots=sm["epoch_slots"],
                    max_defer=mg["max_defer"], duration_slots=wl["duration_slots"], executor=executor,
                    models=models, on_slot=on_slot)
    res.requests, res.config = len(records), cfg
    return res
