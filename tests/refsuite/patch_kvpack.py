"""pytest plugin: swap this repo's planner into the REFERENCE package before the
reference's own tests import it, so /root/reference/pkg/tests/test_migration.py
and test_sim.py exercise paper_2501_06709_b200.planner (and its ConfigError)
instead of kvpack.migration.  Loaded with `-p patch_kvpack` by
tests/test_reference_suite.py; never imported by the product."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import kvpack  # noqa: E402  (the reference, via PYTHONPATH)
import kvpack.migration as ref_migration  # noqa: E402
import kvpack.sim as ref_sim  # noqa: E402
import kvpack.verification as ref_verif  # noqa: E402

import paper_2501_06709_b200.errors as ours_errors  # noqa: E402
import paper_2501_06709_b200.planner as ours  # noqa: E402

NAMES = ["Topology", "Boundaries", "load_boundaries", "PendingMove", "PlannedMove", "MigrationPlan",
         "consensus_order", "plan_hybrid", "check_budgets", "KV_TRANSFER", "TOKEN_TRANSFER", "DEFERRED",
         "FORCED_KV_TRANSFER"]
for name in NAMES:
    setattr(ref_migration, name, getattr(ours, name))
    if hasattr(kvpack, name):
        setattr(kvpack, name, getattr(ours, name))
    for mod in (ref_sim, ref_verif):
        if hasattr(mod, name):
            setattr(mod, name, getattr(ours, name))
# the reference tests catch kvpack.ConfigError; ours must be that class for them
kvpack.ConfigError = ours_errors.ConfigError
ref_migration.ConfigError = ours_errors.ConfigError
os.environ["KVPACK_PLANNER_UNDER_TEST"] = ours.__file__

# With KVPACK_PATCH_SCHEDULER=1 the native scheduler and cluster model replace
# the reference's everywhere the reference modules bound them, so the
# reference's own scheduler/model/sim/acceptance tests drive csrc/scheduler.cpp.
if os.environ.get("KVPACK_PATCH_SCHEDULER") == "1":
    import importlib

    import paper_2501_06709_b200.cluster as ours_cluster  # noqa: E402
    import paper_2501_06709_b200.scheduler as ours_sched  # noqa: E402

    SCHED_NAMES = ["ClusterState", "GpuState", "MultiItemGroup", "SizeClass", "Request", "kv_size_at",
                   "classify_request", "classify_gpu", "request_weight", "total_weight", "active_gpu_count",
                   "WEIGHT_L_SINGLE", "WEIGHT_L_COMBINED", "WEIGHT_M", "WEIGHT_S",
                   "Move", "OperationLog", "EpochResult", "PriorityConfig", "DEFAULT_PRIORITY",
                   "allocation_priority", "migration_priority", "Violation", "verify_properties",
                   "MellScheduler", "batch_operations"]
    ERROR_NAMES = ["KvPackError", "RequestTooLarge", "NotPlaced", "NoCategory", "ConfigError", "ParseError"]
    ref_size_class = importlib.import_module("kvpack.model").SizeClass

    def _rekey(v):
        if isinstance(v, ref_size_class):
            return ours_cluster.SizeClass(v.value)
        if isinstance(v, tuple):
            return tuple(_rekey(x) for x in v)
        return v

    mods = [kvpack] + [importlib.import_module("kvpack." + m)
                       for m in ("sim", "verification", "baselines", "oracle", "cli", "config", "workload")]
    for mod in mods:
        for name in SCHED_NAMES:
            if hasattr(mod, name):
                setattr(mod, name, getattr(ours_cluster, name, None) or getattr(ours_sched, name))
        for name in ERROR_NAMES:
            if hasattr(mod, name):
                setattr(mod, name, getattr(ours_errors, name))
        # module-level tables keyed by the reference's SizeClass (e.g. MOVE_BOUNDS)
        for name, val in list(vars(mod).items()):
            if isinstance(val, dict) and any(_rekey(k) != k for k in val):
                setattr(mod, name, {_rekey(k): _rekey(v) for k, v in val.items()})
            elif isinstance(val, tuple) and val and any(isinstance(x, ref_size_class) for x in val):
                setattr(mod, name, _rekey(val))
    os.environ["KVPACK_SCHEDULER_UNDER_TEST"] = ours_sched.__file__
