"""B200-native KV-cache migration for Mell (arXiv 2501.06709).

Drop-in for the reference's migration path (`kvpack.migration` +
the sim.py:207-227 data plane): the planner API keeps the reference's names;
the KV pools, block tables and executor carry out the plan on sm_100a kernels
in libkvmig.so (include/kvmig.h).  See DESIGN.md.
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


def __getattr__(name):  # data-path objects load the native library lazily
    if name in ("KVPool", "BlockTable", "BlockAllocator", "ModelShape", "LLAMA2_7B",
                "LLAMA2_13B", "LLAMA3_70B", "SHAPES"):
        from . import kvcache
        return getattr(kvcache, name)
    if name in ("MigrationExecutor", "ExecReport", "ExecRecord", "Residency"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
