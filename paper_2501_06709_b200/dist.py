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

import ctypes
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np


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


class PeerLink:
    """The one-process-per-GPU migration path (public API; bench.py's N > 1 e2e
    arm runs through it).  Insertion point: sim.py:221-223, where a planned
    kv_transfer between two GPUs would execute.

    Each rank publishes, once: its pool (CUDA-IPC handle), a control region
    [64 flag words | block-table row of the incoming request] and the pool
    blocks it will receive into (`recv_blocks`, ascending free-list order).
    `push(dst_rank, src_blocks, seq)` then launches kvm_migrate on this GPU:
    the kernel gathers the request's blocks from the local pool and stores
    them straight into the destination's mapped pool over NVLink/NVSwitch,
    rewrites the destination's block-table row and release-stores `seq` into
    its done flag (system scope).  `wait(seq)` makes the incoming move a
    stream dependency on this GPU (bounded device spin on the flag).  There
    is no NCCL on the copy path; torch.distributed only carries the handles.

    Construction is collective (all ranks of `group`); peer pools are mapped
    lazily on first push."""

    FLAG_WORDS = 64
    ERR_WORD = 63

    def __init__(self, pool, recv_blocks, ri: "RankInfo", group=None, max_row: Optional[int] = None):
        import torch

        from . import _native

        self._native = _native
        self.pool, self.ri, self.group = pool, ri, group
        self.recv_blocks = np.ascontiguousarray(recv_blocks, dtype=np.int32)
        width = max(int(max_row if max_row is not None else len(self.recv_blocks)), 1)
        dev = pool.device
        self.ctrl = torch.zeros(self.FLAG_WORDS + width, dtype=torch.int32, device=f"cuda:{dev}")
        self.mailbox, self.row = self.ctrl[:self.FLAG_WORDS], self.ctrl[self.FLAG_WORDS:]
        h_pool, o_pool = pool.ipc_handle()
        hb, ob = (ctypes.c_ubyte * 64)(), ctypes.c_int64()
        _native.check(_native.lib().kvm_ipc_export(ctypes.c_void_p(self.ctrl.data_ptr()), hb, ctypes.byref(ob)),
                      "kvm_ipc_export(ctrl)")
        self._info = exchange_objects((h_pool, o_pool, bytes(hb), ob.value, self.recv_blocks.tolist(),
                                       pool.num_blocks), group=group)
        self._peers: Dict[int, tuple] = {}

    def peer(self, rank: int) -> tuple:
        """(mapped pool, flag address, table-row address, host blocks, device blocks) of `rank`."""
        p = self._peers.get(rank)
        if p is None:
            import torch

            from .kvcache import KVPool

            h_pool, o_pool, h_ctrl, o_ctrl, blocks, nb = self._info[rank]
            dev = self.pool.device
            mapped = KVPool.from_ipc(self.pool.shape, nb, dev, h_pool, o_pool, dtype=self.pool.dtype)
            ptr = ctypes.c_void_p()
            self._native.check(self._native.lib().kvm_ipc_import(
                dev, (ctypes.c_ubyte * 64).from_buffer_copy(h_ctrl), o_ctrl, ctypes.byref(ptr)),
                "kvm_ipc_import(ctrl)")
            hb = np.asarray(blocks, dtype=np.int32)
            p = (mapped, ptr.value, ptr.value + 4 * self.FLAG_WORDS, hb,
                 torch.from_numpy(hb).to(f"cuda:{dev}"), (ptr.value, o_ctrl))
            self._peers[rank] = p
        return p

    def push(self, dst_rank: int, src_blocks, seq: int, engine: str = "bulk", stream=None,
             layer_flags: int = 0, max_sms: int = 0) -> None:
        """Migrate the request held in `src_blocks` (host int32 array -> host
        block lists, or an int32 CUDA tensor) into `dst_rank`'s advertised
        receive blocks; asynchronous on `stream`.  max_sms > 0: the push runs
        on at most that many SMs (KVM_F_MAX_SMS; the link, not the SMs, bounds it)."""
        import torch

        from .executor import ENGINES

        if engine not in ENGINES:
            raise ValueError(f"engine must be one of {sorted(ENGINES)}")
        mapped, flag, row, hb, db, _ = self.peer(dst_rank)
        n = len(hb)
        m = self._native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = self.pool.pool_id, mapped.pool_id, n, int(seq)
        flags = ENGINES[engine] | self._native.KVM_F_MAX_SMS(max_sms)
        if isinstance(src_blocks, np.ndarray):
            sb = np.ascontiguousarray(src_blocks, dtype=np.int32)
            if len(sb) != n:
                raise ValueError(f"request has {len(sb)} blocks, rank {dst_rank} receives {n}")
            m.src_blocks, m.dst_blocks = sb.ctypes.data, hb.ctypes.data
            flags |= self._native.KVM_F_BLOCKS_ON_HOST
        else:
            if src_blocks.numel() != n or src_blocks.dtype != torch.int32:
                raise ValueError("device block list must be int32 with one entry per received block")
            m.src_blocks, m.dst_blocks = src_blocks.data_ptr(), db.data_ptr()
        m.dst_table_row, m.done_flag, m.layer_flags = row, flag, layer_flags or None
        s = stream if stream is not None else torch.cuda.current_stream(self.pool.device)
        self._native.check(self._native.lib().kvm_migrate(ctypes.byref(m), 1, flags,
                                                          ctypes.c_void_p(s.cuda_stream)), "kvm_migrate(peer)")

    def wait(self, seq: int, stream=None, timeout_ns: int = 30_000_000_000) -> None:
        """Queue on `stream` a bounded wait until the incoming move's done flag
        reaches `seq` (ld.acquire.sys); a lost peer sets the error word
        instead of hanging the GPU (see check())."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.pool.device)
        base = self.mailbox.data_ptr()
        self._native.check(self._native.lib().kvm_wait_flag_timeout(
            ctypes.c_void_p(base), int(seq), int(timeout_ns), ctypes.c_void_p(base + 4 * self.ERR_WORD),
            ctypes.c_void_p(s.cuda_stream)), "kvm_wait_flag_timeout")

    def check(self) -> None:
        """Raise if a wait() timed out (synchronises on the error word)."""
        if int(self.mailbox[self.ERR_WORD].item()) != 0:
            raise TimeoutError(f"rank {self.ri.rank}: incoming migration from rank {self.ri.recv_from} "
                               "did not land before the timeout")

    def reset(self) -> None:
        """Zero the flags (sequence numbers restart at 1); callers barrier after."""
        self.mailbox.zero_()

    def close(self) -> None:
        for mapped, *_rest, ctrl in self._peers.values():
            mapped.close()
            self._native.lib().kvm_ipc_close(ctypes.c_void_p(ctrl[0]), ctrl[1])
        self._peers = {}


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
