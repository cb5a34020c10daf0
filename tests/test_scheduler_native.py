"""CPU-only: the native online scheduler (csrc/scheduler.cpp behind
paper_2501_06709_b200.scheduler / .cluster) makes the reference's decisions.

* Fixture replays (no reference needed, so they also run on the GPU box): the
  live slot loop with the NATIVE MellScheduler reproduces the reference
  simulator's recorded plan rows, GPU-count series and logical-move counts on
  every committed trace, including the multi-LLM (7B+13B) one.
* Lockstep differential runs against the reference MellScheduler (when
  /root/reference is mounted): identical EpochResults and identical cluster
  state after every epoch, over random traces that cover every size class,
  rejections, aborts, group churn, batching on/off, several epoch lengths and
  priority weights.
* Direct public operations (allocate / depart / update / handle_growth) on
  both, with identical results or identical exception classes.
"""
import json
import random

import pytest

import sched_diff as sd
from conftest import load_golden
from paper_2501_06709_b200 import cluster as ocl
from paper_2501_06709_b200 import scheduler as osch
from paper_2501_06709_b200.errors import NotPlaced, RequestTooLarge
from paper_2501_06709_b200.planner import Topology, load_boundaries
from paper_2501_06709_b200.runtime import run_slots


class _Ours:
    ClusterState = ocl.ClusterState
    MellScheduler = osch.MellScheduler
    PriorityConfig = osch.PriorityConfig


def _loop(fx, bpt):
    cfg = fx["config"]
    cl = cfg["cluster"]
    cluster = ocl.ClusterState(cl["capacity_bytes"], gpus_per_machine=cl["gpus_per_machine"])
    sched = osch.MellScheduler(cluster, priority_cfg=osch.PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=cl["gpus_per_machine"],
                    intra_bandwidth_bytes_per_s=cl["intra_bandwidth_bytes_per_s"],
                    inter_bandwidth_bytes_per_s=cl["inter_bandwidth_bytes_per_s"],
                    prefill_tokens_per_s=cl["prefill_tokens_per_s"])
    bounds = load_boundaries(topo, cfg["migration"]["epoch_seconds"], cfg["migration"]["budget_fraction"])
    return run_slots([tuple(r) for r in fx["trace"]], sched, cluster, topo, bounds, bpt=bpt,
                     tokens_per_slot=cfg["sim"]["tokens_per_slot"], max_defer=cfg["migration"]["max_defer"],
                     duration_slots=cfg["workload"]["duration_slots"])


@pytest.mark.parametrize("name", ["trace_7b_c48g_seed0.json", "trace_7b_c48g_seed2.json",
                                  "trace_7b_c48g_seed3.json", "trace_7b_mixed_seed0.json"])
def test_native_scheduler_reproduces_reference_run(name):
    fx = load_golden(name)
    out = _loop(fx, fx["config"]["workload"]["kv_bytes_per_token"])
    assert out.plan_rows == [r[:7] for r in fx["plan_rows"]]
    assert out.active_gpus == fx["active_gpus"]
    assert out.logical_moves == fx["migrations"]
    assert out.deferred == fx["deferred"] and out.forced == fx["forced"]
    assert max(out.active_gpus) == fx["summary"]["peak_gpus"]
    assert out.completed == fx["summary"]["completed"]


def test_native_scheduler_multi_llm_fixture():
    """configs[4]: mixed 7B+13B trace, per-request bytes/token."""
    fx = load_golden("trace_multillm_7b13b_seed0.json")
    models = {int(k): v for k, v in fx["models"].items()}
    out = _loop(fx, {rid: fx["model_bpt"][m] for rid, m in models.items()})
    assert out.plan_rows == [r[:7] for r in fx["plan_rows"]]
    assert out.active_gpus == fx["active_gpus"]


def _ref_or_skip():
    ref = sd.kvpack()
    if ref is None:
        pytest.skip("reference tree not mounted (expected on the GPU box)")
    return ref


@pytest.mark.parametrize("block", range(6))
def test_lockstep_random_traces(block):
    ref = _ref_or_skip()
    for seed in range(block * 25, block * 25 + 25):
        rng = random.Random(seed)
        recs = sd.random_trace(rng, rng.randint(5, 60), rng.randint(3, 40), rng.choice([50, 300, 700, 1300]),
                               rng.choice([20, 200, 900]))
        prio = rng.choice([(1.0, 0.25, 0.5), (0.0, 1.0, 0.0), (rng.random(), rng.random(), rng.random()),
                           (1.0, 0.0, 0.0)])
        sd.lockstep(ref, _Ours, recs, capacity=rng.choice([120000, 120001, 99991]), gpm=rng.choice([1, 2, 4, 8]),
                    prio=prio, batching=rng.random() < 0.5, bpt=100, tps=rng.choice([1, 10, 50]),
                    epoch_slots=rng.choice([1, 1, 3]))


def test_lockstep_b200_shaped_run():
    """The §8c B200-shaped config (7B bpt, C = 48 GiB, 8 GPUs/machine) on a
    synthetic trace long enough to reach several GPUs."""
    ref = _ref_or_skip()
    fx = load_golden("trace_7b_c48g_seed0.json")
    cfg = fx["config"]
    sd.lockstep(ref, _Ours, [tuple(r) for r in fx["trace"]], capacity=cfg["cluster"]["capacity_bytes"], gpm=8,
                prio=(1.0, 0.25, 0.5), batching=True, bpt=cfg["workload"]["kv_bytes_per_token"],
                tps=cfg["sim"]["tokens_per_slot"], check_state_every=5)


def _outcome(fn):
    try:
        return ("ok", fn())
    except Exception as e:  # the reference raises its own classes: compare names
        return ("err", type(e).__name__)


def test_direct_operations_match_reference():
    ref = _ref_or_skip()
    C = 120_000
    for seed in range(40):
        rng = random.Random(1000 + seed)
        rc, oc = ref.ClusterState(C), ocl.ClusterState(C)
        rs, os_ = ref.MellScheduler(rc), osch.MellScheduler(oc)
        live, next_id = [], 0
        for _ in range(60):
            op = rng.random()
            if op < 0.45 or not live:
                size = rng.choice([rng.randint(1, C // 8), rng.randint(C // 8, C // 2), rng.randint(C // 2, C),
                                   C + 1, 0])
                a = _outcome(lambda: sd.result_key(sd_wrap(rs.allocate(next_id, size))))
                b = _outcome(lambda: sd.result_key(sd_wrap(os_.allocate(next_id, size))))
                if a[0] == "ok":
                    live.append(next_id)
                next_id += 1
            elif op < 0.7:
                r = rng.choice(live + [10 ** 6])
                a = _outcome(lambda: sd.result_key(sd_wrap(rs.depart(r))))
                b = _outcome(lambda: sd.result_key(sd_wrap(os_.depart(r))))
                if r in live and a[0] == "ok":
                    live.remove(r)
            else:
                r = rng.choice(live)
                if r not in rc.sizes:
                    continue
                new = rc.sizes[r] + rng.randint(0, C // 3)
                rc.set_size(r, new)
                oc.set_size(r, new)
                a = _outcome(lambda: [sd.result_key(sd_wrap(x)) for x in rs.handle_growth([r])])
                b = _outcome(lambda: [sd.result_key(sd_wrap(x)) for x in os_.handle_growth([r])])
                live = [x for x in live if x in rc.sizes]
            assert a == b, (seed, a, b)
            assert sd.state_key(rc, rs, False) == sd.state_key(oc, os_, True)


class sd_wrap:
    """An OperationLog as a one-log EpochResult-like object for result_key."""

    def __init__(self, log):
        self.logs, self.terminated, self.batched = [log], [], False


def test_errors_and_views():
    c = ocl.ClusterState(120_000)
    s = osch.MellScheduler(c)
    with pytest.raises(RequestTooLarge):
        s.allocate(1, 120_001)
    with pytest.raises(ValueError):
        s.allocate(1, 0)
    with pytest.raises(NotPlaced):
        s.depart(7)
    with pytest.raises(ValueError):
        ocl.ClusterState(0)
    with pytest.raises(ValueError):
        osch.PriorityConfig(0.0, 0.0, 0.0)
    log = s.allocate(1, 72_000)
    assert log.moves == [osch.Move(1, None, 0, "allocate")]
    assert s.scheduled_class[1] is ocl.SizeClass.L and 2 not in s.scheduled_class
    c.sizes[5] = 10
    assert c.sizes[5] == 10 and 5 in c.sizes
    del c.sizes[5]
    assert 5 not in c.sizes
    g = c.gpus[0]
    g.activation_seq = 9
    assert c.gpus[0].activation_seq == 9
    assert osch.verify_properties(c) == []
    with pytest.raises(KeyError):
        c.place(3, 42)


def test_loop_metrics_match_reference_sim():
    """run_slots with the native scheduler reproduces kvpack.sim.run's whole
    MetricsSeries (active_gpus, migrations, deferred, forced, used_bytes,
    capacity_bytes) on the B200-shaped config, not only its plan rows."""
    ref = _ref_or_skip()
    from kvpack.config import config_from_dict
    from kvpack.sim import run as ref_run

    fx = load_golden("trace_7b_c48g_seed0.json")
    doc = {"schema_version": 1, **{k: v for k, v in fx["config"].items()}}
    cfg = config_from_dict(doc)
    trace = ref.Trace(records=[ref.ArrivalRecord(*r) for r in fx["trace"]])
    m = ref_run(cfg, trace).metrics
    out = _loop(fx, fx["config"]["workload"]["kv_bytes_per_token"])
    assert out.active_gpus == m.active_gpus and out.logical_moves == m.migrations
    assert out.deferred == m.deferred and out.forced == m.forced
    assert out.used_bytes == m.used_bytes and out.capacity_bytes == m.capacity_bytes
    assert out.peak_gpus == m.peak_gpus and out.mean_utilization == m.mean_utilization


def test_reference_default_run_fingerprint():
    """The reference's DEFAULT run (sim defaults: C = 120 000 B, 4 GPUs/machine,
    100 B/token, lambda 0.5, 200 slots, seed 0) from our generator + native
    scheduler + planner: the plan-row fingerprint recorded with the reference in
    SURVEY.md §8c (d0331a687103bf7e: 368 requests, peak 27 GPUs, 2 200 logical
    moves, 1 578 executed)."""
    import hashlib
    import json

    from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson

    tr = gen_poisson(0.5, 200, LengthDistribution(), 0)
    c = ocl.ClusterState(120_000, 4)
    s = osch.MellScheduler(c, osch.PriorityConfig(), batching=True)
    topo = Topology(gpus_per_machine=4)
    out = run_slots(tr.tuples(), s, c, topo, load_boundaries(topo, 1.0, 0.2), bpt=100, tokens_per_slot=10,
                    duration_slots=200)
    fp = hashlib.sha256(json.dumps([r[:7] for r in out.plan_rows]).encode()).hexdigest()[:16]
    assert (len(tr), out.peak_gpus, sum(out.logical_moves)) == (368, 27, 2200)
    assert sum(1 for r in out.plan_rows if r[6] != "deferred") == 1578
    assert fp == "d0331a687103bf7e"


@pytest.mark.parametrize("doc", [
    {},
    {"cluster": {"capacity_bytes": 200_000, "gpus_per_machine": 2}, "scheduler": {"batching": False},
     "sim": {"epoch_slots": 3, "seed": 4}},
    {"cluster": {"capacity_bytes": 48 << 30, "gpus_per_machine": 8, "intra_bandwidth_bytes_per_s": 900e9,
                 "inter_bandwidth_bytes_per_s": 50e9, "prefill_tokens_per_s": 50_000.0},
     "migration": {"epoch_seconds": 0.05}, "workload": {"scale": 10, "kv_bytes_per_token": 524288,
                                                        "duration_slots": 120},
     "scheduler": {"weight_request_count": 0.0}, "sim": {"seed": 2}},
])
def test_simulate_matches_reference_sim_run(doc):
    """runtime.simulate(config) == kvpack.sim.run(config, gen_poisson(...)) on the
    reference's own config schema: every metric column and the plan rows."""
    ref = _ref_or_skip()
    from kvpack.config import config_from_dict
    from kvpack.sim import run as ref_run

    from paper_2501_06709_b200.runtime import simulate

    cfg = config_from_dict(doc)
    w = cfg.workload
    trace = ref.gen_poisson(w.mean_interarrival_slots, w.duration_slots, ref.LengthDistribution(scale=w.scale),
                            cfg.sim.seed)
    rr = ref_run(cfg, trace)
    m = rr.metrics
    out = simulate(doc)
    assert out.active_gpus == m.active_gpus and out.logical_moves == m.migrations
    assert out.deferred == m.deferred and out.forced == m.forced
    assert out.used_bytes == m.used_bytes and out.capacity_bytes == m.capacity_bytes
    # the reference's output files, byte for byte
    from kvpack.sim import metrics_to_csv
    assert out.metrics_csv() == metrics_to_csv(m)
    assert json.dumps(out.summary, sort_keys=True, indent=2) == json.dumps(rr.summary, sort_keys=True, indent=2)


def test_simulate_rejects_unknown_config():
    from paper_2501_06709_b200.errors import ConfigError
    from paper_2501_06709_b200.runtime import simulate

    with pytest.raises(ConfigError):
        simulate({"cluster": {"bogus": 1}})
    with pytest.raises(ConfigError):
        simulate({"scheduler": {"kind": "lb"}})


_BAD_CONFIGS = [
    [], {"bogus": {}}, {"schema_version": 2}, {"schema_version": True}, {"cluster": []},
    {"cluster": {"capacity_bytes": 0}}, {"cluster": {"capacity_bytes": 1.5}}, {"cluster": {"gpus_per_machine": 0}},
    {"cluster": {"max_gpus": 0}}, {"cluster": {"intra_bandwidth_bytes_per_s": 0}},
    {"cluster": {"prefill_tokens_per_s": "fast"}}, {"cluster": {"capacity_bytes": True}},
    {"scheduler": {"kind": "rr"}}, {"scheduler": {"batching": 1}}, {"scheduler": {"weight_free_mem": -1}},
    {"scheduler": {"rebalance_period": 0}}, {"scheduler": {"imbalance_threshold": 1.0}}, {"scheduler": {"kind": 3}},
    {"migration": {"epoch_seconds": 0}}, {"migration": {"budget_fraction": 1.5}}, {"migration": {"max_defer": -1}},
    {"workload": {"mean_interarrival_slots": 0}}, {"workload": {"duration_slots": -1}},
    {"workload": {"prompt_sigma_log": -0.1}}, {"workload": {"scale": 0}}, {"workload": {"kv_bytes_per_token": 0}},
    {"workload": {"trace_path": 5, "scale": 0}}, {"sim": {"tokens_per_slot": 0}}, {"sim": {"epoch_slots": 0}},
    {"sim": {"seed": 1.0}}, {"cluster": {"capacity_bytes": 0}, "sim": {"epoch_slots": 0}},
]


@pytest.mark.parametrize("doc", _BAD_CONFIGS, ids=[str(i) for i in range(len(_BAD_CONFIGS))])
def test_config_validation_matches_reference(doc):
    """resolve_config rejects exactly what config_from_dict rejects, with the
    same ConfigError message."""
    from paper_2501_06709_b200.errors import ConfigError
    from paper_2501_06709_b200.runtime import resolve_config

    with pytest.raises(ConfigError) as ours:
        resolve_config(doc)
    ref = sd.kvpack()
    if ref is None:
        return
    from kvpack.config import config_from_dict
    from kvpack.errors import ConfigError as RefConfigError

    with pytest.raises(RefConfigError) as theirs:
        config_from_dict(doc)
    assert str(ours.value) == str(theirs.value)


def test_valid_configs_resolve_like_reference():
    ref = sd.kvpack()
    if ref is None:
        pytest.skip("reference tree not mounted")
    from kvpack.config import config_from_dict

    from paper_2501_06709_b200.runtime import resolve_config

    for doc in ({}, {"cluster": {"intra_bandwidth_bytes_per_s": 900_000_000_000}, "scheduler": {"kind": "bf"}},
                {"workload": {"trace_path": "x.csv", "scale": 3}, "sim": {"seed": 9}, "schema_version": 1}):
        r = config_from_dict(doc).to_dict()
        assert {**resolve_config(doc), "schema_version": 1} == r
        assert resolve_config(resolve_config(doc)) == resolve_config(doc)
