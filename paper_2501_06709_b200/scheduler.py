"""Online multi-GPU scheduler that emits the migration decisions, native.

Drop-in for the reference's /root/reference/pkg/src/kvpack/scheduler.py:
`Move`, `OperationLog`, `EpochResult`, `PriorityConfig`, `DEFAULT_PRIORITY`,
`allocation_priority`, `migration_priority`, `Violation`,
`verify_properties`, `MellScheduler` (allocate / depart / update /
handle_growth / step_epoch, batching) and `batch_operations`, same names,
arguments, results and exceptions.  The decision logic runs in C++
(csrc/scheduler.cpp, `kvm_sched_*` in include/kvmig.h) on the native
`ClusterState`; one `step_epoch` is one ABI call.  This is the *caller* of
the migration data path: its cross-GPU moves become the planner's
PendingMoves (sim.py:177-187 -> runtime.run_slots).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Set, Tuple

from . import _native
from .cluster import (NONE, ClusterState, ItemId, SizeClass, class_of_code, classify_request,  # noqa: F401
                      code_of_class)

SM_CLASSES = (SizeClass.M, SizeClass.S)
T_CLASSES = (SizeClass.T, SizeClass.TINY)

_REASONS = ("allocate", "l-fill", "depart-refill", "update", "batch")
_LOG_KINDS = ("allocate", "depart", "update", "epoch")
_EVENTS = ("rejected", "aborted")
_REC_LOG, _REC_MOVE, _REC_EVENT, _REC_TERMINATED, _REC_BATCHED, _REC_EPOCH_COUNTS, _REC_CLASS = 1, 2, 3, 4, 5, 6, 7
_OP_ALLOCATE, _OP_DEPART, _OP_UPDATE, _OP_HANDLE_GROWTH, _OP_DUMP_CLASSES = 0, 1, 2, 3, 4
_VIOLATION_CODES = ("capacity", "P1", "P2", "P3", "P4", "P4", "P5")


@dataclass(frozen=True)
class Move:
    """One item relocation; src is None for a fresh placement (scheduler.py:24-31)."""

    item: ItemId
    src: Optional[int]
    dst: int
    reason: str


@dataclass
class OperationLog:
    """Moves and events of one scheduler invocation (scheduler.py:34-45)."""

    kind: str
    request_id: Optional[int]
    moves: List[Move] = field(default_factory=list)
    events: List[Tuple[str, ...]] = field(default_factory=list)

    @property
    def migration_count(self) -> int:
        return sum(1 for m in self.moves if m.src is not None)


@dataclass
class EpochResult:
    """scheduler.py:198-214."""

    logs: List[OperationLog]
    terminated: List[int]
    batched: bool = False

    @property
    def moves(self) -> List[Move]:
        return [m for log in self.logs for m in log.moves]

    @property
    def migration_count(self) -> int:
        return sum(log.migration_count for log in self.logs)

    @property
    def events(self) -> List[Tuple[str, ...]]:
        return [e for log in self.logs for e in log.events]


@dataclass(frozen=True)
class PriorityConfig:
    """Provider-tunable GPU priority weights (scheduler.py:48-62)."""

    weight_free_mem: float = 1.0
    weight_request_count: float = 0.25
    weight_same_machine: float = 0.5

    def __post_init__(self):
        if self.weight_free_mem < 0 or self.weight_request_count < 0 or self.weight_same_machine < 0:
            raise ValueError("priority weights must be non-negative")
        if not (self.weight_free_mem or self.weight_request_count or self.weight_same_machine):
            raise ValueError("at least one priority weight must be > 0")


DEFAULT_PRIORITY = PriorityConfig()


def _opt(v: int) -> Optional[int]:
    return None if v == NONE else v


def _parse_logs(words: list) -> Tuple[List[OperationLog], List[int], bool, Optional[Tuple[int, int]]]:
    logs: List[OperationLog] = []
    terminated: List[int] = []
    batched, counts = False, None
    for i in range(0, len(words), 5):
        tag, a, b, c, d = words[i:i + 5]
        if tag == _REC_MOVE:
            logs[-1].moves.append(Move(a, _opt(b), _opt(c), _REASONS[d]))
        elif tag == _REC_LOG:
            logs.append(OperationLog(_LOG_KINDS[a], _opt(b)))
        elif tag == _REC_EVENT:
            logs[-1].events.append((_EVENTS[a], str(b)))
        elif tag == _REC_TERMINATED:
            terminated.append(a)
        elif tag == _REC_BATCHED:
            batched = bool(a)
        elif tag == _REC_EPOCH_COUNTS:
            counts = (a, b)
    return logs, terminated, batched, counts


class _ScheduledClass:
    """`MellScheduler.scheduled_class` as a read-only mapping item -> SizeClass."""

    def __init__(self, sched: "MellScheduler"):
        self._s = sched

    def get(self, item, default=None):
        v = ctypes.c_int32()
        _native.check(self._s._lib.kvm_sched_class_of(self._s._h, int(item), ctypes.byref(v)))
        return default if v.value < 0 else class_of_code(v.value)

    def __getitem__(self, item):
        cls = self.get(item)
        if cls is None:
            raise KeyError(item)
        return cls

    def __contains__(self, item):
        return self.get(item) is not None

    def _dict(self) -> Dict[ItemId, SizeClass]:
        w = self._s._call(_native.lib().kvm_sched_op, _OP_DUMP_CLASSES, None, 0, 0)
        return {w[i + 1]: class_of_code(w[i + 2]) for i in range(0, len(w), 5)}

    def __iter__(self):
        return iter(self._dict())

    def __len__(self):
        return len(self._dict())

    def items(self):
        return self._dict().items()

    def __repr__(self):
        return repr(self._dict())


def _as_i64(values: Sequence[int]):
    arr = (ctypes.c_int64 * max(1, len(values)))(*values)
    return arr


class MellScheduler:
    """Category-aware online scheduler over one ClusterState (scheduler.py:217-1200)."""

    def __init__(self, cluster: ClusterState, priority_cfg: PriorityConfig = DEFAULT_PRIORITY,
                 batching: bool = False):
        if not isinstance(cluster, ClusterState):
            raise TypeError("MellScheduler needs this package's native ClusterState")
        self.cluster = cluster
        self.priority_cfg = priority_cfg
        self._batching = bool(batching)
        self._lib = _native.lib()
        p = _native.SchedParams(priority_cfg.weight_free_mem, priority_cfg.weight_request_count,
                                priority_cfg.weight_same_machine, int(self._batching), 0)
        h = ctypes.c_void_p()
        _native.check(self._lib.kvm_sched_create(cluster.handle, ctypes.byref(p), ctypes.byref(h)), "MellScheduler")
        self._h = h
        self.scheduled_class = _ScheduledClass(self)
        # (sequential, adopted) migration counts per batched epoch (scheduler.py:228-229)
        self.epoch_migration_counts: List[Tuple[int, int]] = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.kvm_sched_destroy(h)
            self._h = None

    @property
    def capacity(self) -> int:
        return self.cluster.capacity_bytes

    @property
    def batching(self) -> bool:
        return self._batching

    @batching.setter
    def batching(self, value: bool) -> None:
        self._batching = bool(value)
        _native.check(self._lib.kvm_sched_set_batching(self._h, int(self._batching)))

    def _call(self, fn, op, ids, n_ids, size) -> list:
        ptr, n = ctypes.c_void_p(), ctypes.c_int64()
        arr = _as_i64(ids or [])
        _native.check(fn(self._h, op, arr, n_ids, size, ctypes.byref(ptr), ctypes.byref(n)))
        return _native.records(ptr, n)

    def _op_logs(self, op: int, ids: Sequence[int], size: int = 0) -> List[OperationLog]:
        words = self._call(self._lib.kvm_sched_op, op, list(ids), len(ids), size)
        return _parse_logs(words)[0]

    # -- public operations (scheduler.py:641-876) ----------------------------------
    def allocate(self, request_id: int, size: int) -> OperationLog:
        return self._op_logs(_OP_ALLOCATE, [request_id], size)[0]

    def depart(self, request_id: int) -> OperationLog:
        return self._op_logs(_OP_DEPART, [request_id])[0]

    def update(self, request_id: int) -> OperationLog:
        return self._op_logs(_OP_UPDATE, [request_id])[0]

    def handle_growth(self, grown: Sequence[int]) -> List[OperationLog]:
        return self._op_logs(_OP_HANDLE_GROWTH, list(grown))

    def step_epoch(self, arrivals: Sequence[Tuple[int, int]], completions: Sequence[int],
                   growths: Optional[Dict[int, int]] = None) -> EpochResult:
        """One epoch of departs, updates and allocates (scheduler.py:979-1007):
        one native call; with batching, the batched outcome is adopted only if
        it needs no more migrations than the sequential one."""
        growths = growths or {}
        arr = [v for rid, size in arrivals for v in (int(rid), int(size))]
        grw = [v for rid, size in growths.items() for v in (int(rid), int(size))]
        comp = [int(r) for r in completions]
        ptr, n = ctypes.c_void_p(), ctypes.c_int64()
        _native.check(self._lib.kvm_sched_step_epoch(
            self._h, _as_i64(arr), len(arrivals), _as_i64(comp), len(comp), _as_i64(grw), len(growths),
            ctypes.byref(ptr), ctypes.byref(n)), "step_epoch")
        logs, terminated, batched, counts = _parse_logs(_native.records(ptr, n))
        if counts is not None:
            self.epoch_migration_counts.append(counts)
        return EpochResult(logs=logs, terminated=terminated, batched=batched)


def allocation_priority(cluster: ClusterState, gpu_id: int, cfg: PriorityConfig = DEFAULT_PRIORITY) -> float:
    """Workload-only score for a fresh allocation (scheduler.py:68-74), computed
    by the native scheduler's own arithmetic."""
    return _priority(cluster, NONE, gpu_id, cfg)


def migration_priority(cluster: ClusterState, src: int, dst: int, cfg: PriorityConfig = DEFAULT_PRIORITY) -> float:
    """Score of dst as a migration peer of src (scheduler.py:77-84)."""
    if src == dst:
        raise ValueError("src and dst must differ")
    return _priority(cluster, src, dst, cfg)


def _priority(cluster, src, dst, cfg) -> float:
    s = MellScheduler(cluster, cfg)
    out = ctypes.c_double()
    _native.check(s._lib.kvm_sched_priority(s._h, src, dst, ctypes.byref(out)))
    return out.value


@dataclass(frozen=True)
class Violation:
    """scheduler.py:91-95."""

    gpu_id: Optional[int]
    code: str
    detail: str


_DETAILS = {0: "residents exceed capacity", 3: "T-GPU below 75% utilization",
            4: "L-GPU lacks S/M though one fits", 5: "L-GPU holds multiple S/M",
            6: "L/M-GPU below 75% while T-GPUs exist"}


def verify_properties(cluster: ClusterState, exempt: Optional[Set[int]] = None) -> List[Violation]:
    """Canonical-shape check outside the exempt GPUs (scheduler.py:102-191)."""
    ex = sorted(exempt) if exempt is not None else []
    ptr, n = ctypes.c_void_p(), ctypes.c_int64()
    _native.check(cluster._lib.kvm_cluster_verify(cluster.handle, _as_i64(ex), len(ex) if exempt is not None else -1,
                                                   ctypes.byref(ptr), ctypes.byref(n)), "verify_properties")
    pairs = _native.records(ptr, n, width=2)
    out = []
    for i in range(0, len(pairs), 2):
        g, code = pairs[i], pairs[i + 1]
        if code in (1, 2):
            kinds = [cluster.item_class(it) for it in cluster.gpus[g].residents]
            detail = f"{'M' if code == 1 else 'S'}-GPU holds {kinds}"
        else:
            detail = _DETAILS[code]
        out.append(Violation(g, _VIOLATION_CODES[code], detail))
    return out


def batch_operations(scheduler: MellScheduler, departs: Sequence[int], updates: Dict[int, int],
                     allocates: Sequence[Tuple[int, int]]) -> EpochResult:
    """One epoch's depart/update/allocate sets as a batch (scheduler.py:1203-1213)."""
    was = scheduler.batching
    scheduler.batching = True
    try:
        return scheduler.step_epoch(allocates, departs, updates)
    finally:
        scheduler.batching = was
