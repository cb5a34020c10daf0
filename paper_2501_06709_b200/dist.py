"""One process per GPU: peer-pool exchange over torch.distributed.

Each rank owns the KV pool in its own GPU's HBM.  To push a request to a
peer, the source rank maps the destination's pool into its address space
(CUDA IPC; the mapping routes stores over NVLink/NVSwitch) and launches the
migration kernel locally — no NCCL on the copy path.  torch.distributed is
plumbing only: it carries the 64-byte IPC handles and the destination block
ids (control plane), and the barriers of the benchmark.

Partitioning: every PendingMove is an independent src->dst
unit; the benchmark's concurrent pattern is the ring i -> (i+1) mod N, so
each GPU sends one request and receives one (weak scaling, no collective on
the data path).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import List, Optional, Tuple


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int

    @property
    def send_to(self) -> int:
        return (self.rank + 1) % self.world

    @property
    def recv_from(self) -> int:
        return (self.rank - 1) % self.world


def rank_info_from_env() -> RankInfo:
    return RankInfo(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                    int(os.environ.get("LOCAL_RANK", 0)))


def ring_pairs(world: int) -> List[Tuple[int, int]]:
    """(src, dst) for the i -> (i+1) mod N permutation; a 1-GPU world has no pairs."""
    return [(i, (i + 1) % world) for i in range(world)] if world > 1 else []


def exchange_handles(handle: bytes, offset: int, group=None) -> List[Tuple[bytes, int]]:
    """All-gather every rank's (ipc_handle, offset) for its pool."""
    import torch.distributed as dist

    out: List[Optional[Tuple[bytes, int]]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, (bytes(handle), int(offset)), group=group)
    return [(bytes(h), int(o)) for h, o in out]


def exchange_objects(obj, group=None) -> list:
    """All-gather small control-plane objects (e.g. destination block lists)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def allreduce_max(value: float, device=None) -> float:
    """Max over ranks (device-timed numbers are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def collective_ring_exchange(pool, send_blocks, recv_blocks, ri: RankInfo, group=None):
    """COMPARISON BASELINE ONLY, not the product path: the same
    ring exchange as bench.py's kvm_migrate push, done the library way —
    gather this rank's request into a contiguous buffer (`index_select` over the
    block axis of a native pool tensor [L][2][blocks][16][H][D]), one
    `batch_isend_irecv` (ncclSend / ncclRecv inside a group with the nccl
    backend) to ri.send_to / from ri.recv_from, then scatter the received
    request into `recv_blocks`.  send_blocks / recv_blocks: int64 tensors on
    the pool's device.  Returns the received buffer."""
    import torch
    import torch.distributed as dist

    out = pool.index_select(2, send_blocks)
    inc = torch.empty((pool.shape[0], pool.shape[1], recv_blocks.numel()) + tuple(pool.shape[3:]),
                      dtype=pool.dtype, device=pool.device)
    ops = [dist.P2POp(dist.isend, out, ri.send_to, group=group),
           dist.P2POp(dist.irecv, inc, ri.recv_from, group=group)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    pool.index_copy_(2, recv_blocks, inc)
    return inc
