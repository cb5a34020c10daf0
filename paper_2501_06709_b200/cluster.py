"""Cluster model of the online scheduler, backed by the native library.

Drop-in for the reference's domain model (/root/reference/pkg/src/kvpack/
model.py): `Request`, `kv_size_at`, `classify_request`, `SizeClass`,
`ClusterState`, `GpuState`, `MultiItemGroup`, `classify_gpu`,
`request_weight`, `total_weight`, `active_gpu_count` and the weights, with the
same names, argument meaning and exceptions.

`ClusterState` keeps its state in C++ (`kvm_cluster_*` in include/kvmig.h,
csrc/scheduler.cpp) so the native `MellScheduler` can mutate it without
crossing the ABI per decision.  Python reads it through views rebuilt from a
snapshot whenever the native mutation counter moves:

    gpus, placement, groups, request_group   read-only dict snapshots (the
                                             reference's insertion order)
    sizes                                    a write-through mapping, so
                                             `cluster.sizes[r] = n` works as
                                             in the reference (model.py:131)
    GpuState.activation_seq                  writable (write-through)

Mutating a snapshot container directly (e.g. `gpus[g].residents.add(x)`) does
not reach the native state; use the methods, as the reference's own code does.
"""
from __future__ import annotations

import ctypes
from collections.abc import MutableMapping
from dataclasses import dataclass
from enum import Enum
from fractions import Fraction
from typing import Dict, Iterator, List, Optional, Set

from . import _native
from .errors import NoCategory, NotPlaced, RequestTooLarge  # noqa: F401  (re-exported API)

ItemId = int
NONE = _native.KVM_NONE

_STATE_ORDER = {"pending": 0, "running": 1, "completed": 2}


class SizeClass(Enum):
    """model.py:23-28; `.code` is the native KVM_CLASS_* value."""

    L = "L"
    M = "M"
    S = "S"
    T = "T"
    TINY = "Tiny"


_CLASS_BY_CODE = (SizeClass.L, SizeClass.M, SizeClass.S, SizeClass.T, SizeClass.TINY)
_CODE_OF = {c: i for i, c in enumerate(_CLASS_BY_CODE)}


def class_of_code(code: int) -> SizeClass:
    return _CLASS_BY_CODE[code]


def code_of_class(cls: SizeClass) -> int:
    return _CODE_OF[cls]


@dataclass
class Request:
    """One LLM request (model.py:31-55)."""

    id: int
    arrival_slot: int
    prompt_tokens: int
    response_tokens: int
    kv_bytes_per_token: int
    state: str = "pending"

    def __post_init__(self):
        if self.prompt_tokens < 1:
            raise ValueError("prompt_tokens must be >= 1")
        if self.response_tokens < 1:
            raise ValueError("response_tokens must be >= 1")
        if self.kv_bytes_per_token <= 0:
            raise ValueError("kv_bytes_per_token must be > 0")
        if self.state not in _STATE_ORDER:
            raise ValueError(f"unknown state {self.state!r}")

    def advance_state(self, new_state: str) -> None:
        if _STATE_ORDER.get(new_state, -1) < _STATE_ORDER[self.state]:
            raise ValueError(f"illegal transition {self.state} -> {new_state}")
        self.state = new_state


def kv_size_at(request: Request, slot: int, tokens_per_slot: int) -> int:
    """KV bytes at a slot boundary (model.py:58-69): prompt plus the tokens
    generated so far, saturating at the response length."""
    if slot < request.arrival_slot:
        raise ValueError("slot precedes request arrival")
    done = min(request.response_tokens, tokens_per_slot * (slot - request.arrival_slot))
    return (request.prompt_tokens + done) * request.kv_bytes_per_token


def classify_request(size: int, capacity: int) -> SizeClass:
    """Size class with inclusive upper boundaries (model.py:72-86)."""
    if size <= 0:
        raise ValueError("size must be positive")
    if size > capacity:
        raise RequestTooLarge(f"size {size} exceeds capacity {capacity}")
    for k, cls in ((2, SizeClass.L), (3, SizeClass.M), (4, SizeClass.S), (8, SizeClass.T)):
        if k * size > capacity:
            return cls
    return SizeClass.TINY


class GpuState:
    """Snapshot of one active GPU (model.py:89-97); `activation_seq` writes
    through to the native cluster."""

    __slots__ = ("id", "capacity_bytes", "machine_id", "_seq", "residents", "_cluster")

    def __init__(self, cluster, gid, capacity, machine, seq, residents):
        self._cluster = cluster
        self.id, self.capacity_bytes, self.machine_id = gid, capacity, machine
        self._seq, self.residents = seq, residents

    @property
    def activation_seq(self) -> int:
        return self._seq

    @activation_seq.setter
    def activation_seq(self, value: int) -> None:
        self._cluster._op(_native_op("SET_ACTIVATION_SEQ"), self.id, int(value))
        self._seq = int(value)

    def __repr__(self):
        return (f"GpuState(id={self.id}, capacity_bytes={self.capacity_bytes}, machine_id={self.machine_id}, "
                f"activation_seq={self._seq}, residents={self.residents!r})")


@dataclass
class MultiItemGroup:
    """Snapshot of a group of sub-C/8 requests (model.py:100-106)."""

    group_id: ItemId
    members: Set[int]
    aggregate_bytes: int = 0


# KVM_CL_* op codes (include/kvmig.h)
_OPS = {name: i for i, name in enumerate((
    "ACTIVATE_GPU", "TERMINATE_GPU", "PLACE", "UNPLACE", "GPU_OF", "SET_SIZE", "PUT_SIZE", "DEL_SIZE",
    "NEW_GROUP", "GROUP_ADD", "GROUP_REMOVE", "DEL_GROUP", "ITEM_SIZE", "ITEM_CLASS", "USED_BYTES",
    "GPU_CLASS", "GPU_FAMILY", "LATEST_OF_FAMILY", "CHECK_CAPACITY", "ITEM_OF_REQUEST",
    "SET_ACTIVATION_SEQ", "SET_NEXT_ACTIVATION_SEQ", "VERSION", "CLASSIFY", "VERSION_ADDR"))}


def _native_op(name: str) -> int:
    return _OPS[name]


_SNAP_COUNTERS, _SNAP_GPU, _SNAP_RESIDENT, _SNAP_PLACEMENT, _SNAP_SIZE = 10, 11, 12, 13, 14
_SNAP_GROUP, _SNAP_MEMBER, _SNAP_REQUEST_GROUP, _SNAP_FREE_ID = 15, 16, 17, 18


class _Snapshot:
    __slots__ = ("version", "gpus", "placement", "sizes", "groups", "request_group", "free_ids",
                 "next_activation_seq", "next_group_id", "next_gpu_id")


class _Sizes(MutableMapping):
    """`cluster.sizes`: a dict-like write-through view (model.py:131)."""

    def __init__(self, cluster: "ClusterState"):
        self._c = cluster

    def __getitem__(self, rid):
        return self._c._snap().sizes[rid]

    def __setitem__(self, rid, value):
        self._c._op(_OPS["PUT_SIZE"], int(rid), int(value))

    def __delitem__(self, rid):
        self._c._op(_OPS["DEL_SIZE"], int(rid))

    def __iter__(self) -> Iterator[int]:
        return iter(list(self._c._snap().sizes))

    def __len__(self) -> int:
        return len(self._c._snap().sizes)

    def __contains__(self, rid) -> bool:
        return rid in self._c._snap().sizes

    def as_dict(self) -> Dict[int, int]:
        """The current sizes as a plain dict (read-only use; valid until the next mutation)."""
        return self._c._snap().sizes

    def __repr__(self):
        return repr(self._c._snap().sizes)


class ClusterState:
    """Placement of schedulable items on GPUs (model.py:116-305), native-backed.

    Single-writer, like the reference (model.py:119).
    """

    def __init__(self, capacity_bytes: int, gpus_per_machine: int = 4):
        if capacity_bytes <= 0:
            raise ValueError("capacity_bytes must be > 0")
        if gpus_per_machine < 1:
            raise ValueError("gpus_per_machine must be >= 1")
        self.capacity_bytes = int(capacity_bytes)
        self.gpus_per_machine = int(gpus_per_machine)
        self._lib = _native.lib()
        h = ctypes.c_void_p()
        _native.check(self._lib.kvm_cluster_create(self.capacity_bytes, self.gpus_per_machine, ctypes.byref(h)),
                      "ClusterState")
        self._h = h
        self._ret = ctypes.c_int64()
        self._cache: Optional[_Snapshot] = None
        self._sizes_view = _Sizes(self)
        # the native mutation counter, read in place (no call per view access)
        self._ver = ctypes.c_uint64.from_address(self._op(_OPS["VERSION_ADDR"]))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.kvm_cluster_destroy(h)
            self._h = None

    # -- native plumbing --------------------------------------------------------
    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def _op(self, op: int, a: int = 0, b: int = 0) -> int:
        rc = self._lib.kvm_cluster_op(self._h, op, a, b, ctypes.byref(self._ret))
        if rc < 0:
            _native.check(rc, "ClusterState")
        return self._ret.value

    def _version(self) -> int:
        return self._ver.value

    def _snap(self) -> _Snapshot:
        v = self._version()
        if self._cache is not None and self._cache.version == v:
            return self._cache
        ptr, n = ctypes.c_void_p(), ctypes.c_int64()
        _native.check(self._lib.kvm_cluster_snapshot(self._h, ctypes.byref(ptr), ctypes.byref(n)), "snapshot")
        w = _native.records(ptr, n)
        s = _Snapshot()
        s.version = v
        s.gpus, s.placement, s.sizes, s.groups, s.request_group, s.free_ids = {}, {}, {}, {}, {}, []
        cur = None
        for i in range(0, len(w), 5):
            tag, a, b, c, _d = w[i:i + 5]
            if tag == _SNAP_RESIDENT:
                cur.add(a)
            elif tag == _SNAP_MEMBER:
                cur.add(a)
            elif tag == _SNAP_PLACEMENT:
                s.placement[a] = b
            elif tag == _SNAP_SIZE:
                s.sizes[a] = b
            elif tag == _SNAP_GPU:
                cur = set()
                s.gpus[a] = GpuState(self, a, self.capacity_bytes, b, c, cur)
            elif tag == _SNAP_GROUP:
                cur = set()
                s.groups[a] = MultiItemGroup(a, cur, b)
            elif tag == _SNAP_REQUEST_GROUP:
                s.request_group[a] = b
            elif tag == _SNAP_FREE_ID:
                s.free_ids.append(a)
            elif tag == _SNAP_COUNTERS:
                s.next_activation_seq, s.next_group_id, s.next_gpu_id = a, b, c
        self._cache = s
        return s

    # -- state views (model.py:129-137) -------------------------------------------
    @property
    def gpus(self) -> Dict[int, GpuState]:
        return self._snap().gpus

    @property
    def placement(self) -> Dict[ItemId, int]:
        return self._snap().placement

    @property
    def sizes(self) -> _Sizes:
        return self._sizes_view

    @property
    def groups(self) -> Dict[ItemId, MultiItemGroup]:
        return self._snap().groups

    @property
    def request_group(self) -> Dict[int, ItemId]:
        return self._snap().request_group

    @property
    def next_activation_seq(self) -> int:
        return self._snap().next_activation_seq

    @next_activation_seq.setter
    def next_activation_seq(self, value: int) -> None:
        self._op(_OPS["SET_NEXT_ACTIVATION_SEQ"], int(value))

    # -- sizes and classes (model.py:143-187) ---------------------------------------
    def item_size(self, item: ItemId) -> int:
        return self._op(_OPS["ITEM_SIZE"], item)

    def set_size(self, request_id: int, size: int) -> None:
        self._op(_OPS["SET_SIZE"], request_id, size)

    def group_add(self, gid: ItemId, request_id: int) -> None:
        self._op(_OPS["GROUP_ADD"], gid, request_id)

    def group_remove(self, gid: ItemId, request_id: int) -> None:
        self._op(_OPS["GROUP_REMOVE"], gid, request_id)

    def item_class(self, item: ItemId) -> SizeClass:
        return _CLASS_BY_CODE[self._op(_OPS["ITEM_CLASS"], item)]

    def used_bytes(self, gpu_id: int) -> int:
        return self._op(_OPS["USED_BYTES"], gpu_id)

    def free_bytes(self, gpu_id: int) -> int:
        return self.capacity_bytes - self.used_bytes(gpu_id)

    # -- GPU lifecycle (model.py:191-219) --------------------------------------------
    def activate_gpu(self) -> GpuState:
        gid = self._op(_OPS["ACTIVATE_GPU"])
        return self.gpus[gid]

    def terminate_gpu(self, gpu_id: int) -> None:
        self._op(_OPS["TERMINATE_GPU"], gpu_id)

    def terminate_idle_gpus(self) -> List[int]:
        ptr, n = ctypes.c_void_p(), ctypes.c_int64()
        _native.check(self._lib.kvm_cluster_terminate_idle(self._h, ctypes.byref(ptr), ctypes.byref(n)),
                      "terminate_idle_gpus")
        return list(_native.records(ptr, n, width=1))

    # -- placement (model.py:223-250) -------------------------------------------------
    def place(self, item: ItemId, gpu_id: int) -> None:
        self._op(_OPS["PLACE"], item, gpu_id)

    def unplace(self, item: ItemId) -> int:
        return self._op(_OPS["UNPLACE"], item)

    def gpu_of(self, item: ItemId) -> Optional[int]:
        g = self._op(_OPS["GPU_OF"], item)
        return None if g == NONE else g

    def new_group(self) -> MultiItemGroup:
        gid = self._op(_OPS["NEW_GROUP"])
        return self.groups[gid]

    def item_of_request(self, request_id: int) -> ItemId:
        return self._op(_OPS["ITEM_OF_REQUEST"], request_id)

    # -- categories (model.py:254-289) -------------------------------------------------
    def gpu_class(self, gpu_id: int) -> SizeClass:
        return _CLASS_BY_CODE[self._op(_OPS["GPU_CLASS"], gpu_id)]

    def gpu_family(self, gpu_id: int) -> SizeClass:
        return _CLASS_BY_CODE[self._op(_OPS["GPU_FAMILY"], gpu_id)]

    def gpus_of_family(self, family: SizeClass) -> List[int]:
        return sorted(g for g, st in self.gpus.items() if st.residents and self.gpu_family(g) is family)

    def latest_gpu_of_family(self, family: SizeClass) -> Optional[int]:
        g = self._op(_OPS["LATEST_OF_FAMILY"], _CODE_OF[family])
        return None if g == NONE else g

    def exempt_gpus(self) -> Set[int]:
        out = set()
        for fam in (SizeClass.L, SizeClass.M, SizeClass.S, SizeClass.T):
            g = self.latest_gpu_of_family(fam)
            if g is not None:
                out.add(g)
        return out

    # -- invariants and aggregates (model.py:293-304) -----------------------------------
    def check_capacity(self) -> None:
        self._op(_OPS["CHECK_CAPACITY"])

    def running_requests(self) -> List[int]:
        placed = [r for r in self.placement if r >= 0]
        return sorted(set(placed) | set(self.request_group))


def classify_gpu(gpu: GpuState, cluster: ClusterState) -> SizeClass:
    """model.py:307-309."""
    return cluster.gpu_class(gpu.id)


WEIGHT_L_SINGLE = Fraction(1)
WEIGHT_L_COMBINED = Fraction(5, 6)
WEIGHT_M = Fraction(1, 2)
WEIGHT_S = Fraction(1, 3)


def request_weight(request_id: int, cluster: ClusterState) -> Fraction:
    """Analysis weight of a running request (model.py:312-332)."""
    if request_id in cluster.request_group:
        return Fraction(0)
    gpu_id = cluster.gpu_of(request_id)
    if gpu_id is None:
        raise NotPlaced(f"request {request_id} not placed")
    cls = cluster.item_class(request_id)
    if cls is SizeClass.M:
        return WEIGHT_M
    if cls is SizeClass.S:
        return WEIGHT_S
    if cls in (SizeClass.T, SizeClass.TINY):
        return Fraction(0)
    shares = any(other != request_id and cluster.item_class(other) in (SizeClass.M, SizeClass.S)
                 for other in cluster.gpus[gpu_id].residents)
    return WEIGHT_L_COMBINED if shares else WEIGHT_L_SINGLE


def total_weight(cluster: ClusterState) -> Fraction:
    return sum((request_weight(r, cluster) for r in cluster.placement if r >= 0), Fraction(0))


def active_gpu_count(cluster: ClusterState) -> int:
    return sum(1 for gpu in cluster.gpus.values() if gpu.residents)
