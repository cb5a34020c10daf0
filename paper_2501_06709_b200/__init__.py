"""B200-native KV-cache migration for Mell (arXiv 2501.06709).

Drop-in for the reference's migration path (`kvpack.migration` +
the sim.py:207-227 data plane): the planner API keeps the reference's names;
the KV pools, block tables and executor carry out the plan on sm_100a kernels
in libkvmig.so (include/kvmig.h); the online scheduler that emits the moves
(`MellScheduler`, `ClusterState`) is the reference's, restated natively in
C++ in the same library.  See DESIGN.md.
"""
from .errors import (ConfigError, KvmCudaError, KvmUnsupported, KvPackError, NativeLibraryMissing,
                     NoCategory, NotPlaced, ParseError, RequestTooLarge)
from .planner import (DEFERRED, FORCED_KV_TRANSFER, KV_TRANSFER, TOKEN_TRANSFER, Boundaries,
                      MigrationPlan, PendingMove, PlannedMove, Topology, check_budgets,
                      consensus_order, load_boundaries, plan_hybrid)

__all__ = [
    "Boundaries", "ConfigError", "DEFERRED", "FORCED_KV_TRANSFER", "KV_TRANSFER", "KvPackError",
    "KvmCudaError", "KvmUnsupported", "MigrationPlan", "NativeLibraryMissing", "NoCategory",
    "NotPlaced", "ParseError", "PendingMove", "PlannedMove", "RequestTooLarge", "TOKEN_TRANSFER",
    "Topology", "check_budgets", "consensus_order", "load_boundaries", "plan_hybrid",
]


# the online scheduler and its cluster model (native, csrc/scheduler.cpp)
_CLUSTER_NAMES = ("ClusterState", "GpuState", "MultiItemGroup", "SizeClass", "Request", "kv_size_at",
                  "classify_request", "classify_gpu", "request_weight", "total_weight", "active_gpu_count")
_SCHED_NAMES = ("MellScheduler", "PriorityConfig", "DEFAULT_PRIORITY", "Move", "OperationLog", "EpochResult",
                "allocation_priority", "migration_priority", "Violation", "verify_properties",
                "batch_operations")


# the trace side (workload.py): generator and trace-file format
_WORKLOAD_NAMES = ("ArrivalRecord", "Trace", "LengthDistribution", "gen_poisson", "scale_trace", "load_trace",
                   "save_trace")


def __getattr__(name):  # data-path objects load the native library lazily
    if name in ("KVPool", "BlockTable", "BlockAllocator", "ModelShape", "LLAMA2_7B",
                "LLAMA2_13B", "LLAMA3_70B", "SHAPES"):
        from . import kvcache
        return getattr(kvcache, name)
    if name in _CLUSTER_NAMES:
        from . import cluster
        return getattr(cluster, name)
    if name in _SCHED_NAMES:
        from . import scheduler
        return getattr(scheduler, name)
    if name in ("MigrationExecutor", "ExecReport", "ExecRecord", "Residency"):
        from . import executor
        return getattr(executor, name)
    if name in _WORKLOAD_NAMES:
        from . import workload
        return getattr(workload, name)
    if name in ("simulate", "run_slots", "resolve_config", "load_config", "LoopResult"):
        from . import runtime
        return getattr(runtime, name)
    if name in ("StridedKVPool", "vllm_cache_shape"):
        from . import foreign
        return getattr(foreign, name)
    raise AttributeError(name)
