"""Live migration: pre-copy while decode keeps appending,
then a short stop-and-copy of the tail.

The paper builds on Llumnix-style live migration of a running request's KV
cache: since decode only ever *appends* K/V, every
block that is full is immutable, so full blocks can be copied while the
request keeps decoding on the source; only the partially filled last block
(and blocks completed since the last round) must be copied with decode paused.
The downtime is therefore one short copy, independent of the request's size.

Protocol (driven by the serving loop, single scheduler thread):

    lm = LiveMigration(executor, rid, dst_gpu)
    while lm.remaining_blocks() > threshold:     # decode continues meanwhile
        lm.precopy()                             # async copy of newly-full blocks
        ... decode steps on the source (executor.grow(rid, tokens)) ...
    lm.finish()                                  # pause: copy the tail, rewrite the
                                                 # dst block table, switch residency

Every copy is one kvm_migrate launch (bulk engine) on the source device's
migration stream; `precopy` does not wait, so decode and copy overlap.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native
from .errors import ConfigError
from .executor import Residency


@dataclass
class LiveStats:
    rounds: int = 0
    blocks_precopied: int = 0
    blocks_stopcopied: int = 0
    downtime_s: float = 0.0      # host wall time of finish(): pause -> switched (-> issued, stream-ordered)
    done: Optional[object] = None  # stream-ordered finish: CUDA event after the tail copy + table rewrite
    total_s: float = 0.0
    round_blocks: List[int] = field(default_factory=list)


class LiveMigration:
    def __init__(self, executor, rid: int, dst_gpu: int, engine_flags: int = _native.KVM_F_ENGINE_BULK):
        self.ex = executor
        self.rid = rid
        res = executor.where(rid)
        if res.gpu == dst_gpu:
            raise ConfigError("live migration needs a different destination GPU")
        self.src_gpu, self.dst_gpu = res.gpu, dst_gpu
        self.model = res.model
        self.src_pool = executor.pool(res.gpu, res.model)
        self.dst_pool = executor.pool(dst_gpu, res.model)
        self.bt = self.src_pool.shape.block_tokens
        self.dst_blocks = np.zeros(0, dtype=np.int32)   # dst block for logical block i (i < copied)
        self.copied = 0                                 # logical blocks already copied (all full)
        self.flags = engine_flags
        self.stats = LiveStats()
        self._t0 = time.perf_counter()
        self._keep = []
        self._last = None   # event after the latest launched copy
        self._table = executor._table(dst_gpu, res.model)

    def _res(self) -> Residency:
        return self.ex.where(self.rid)

    def full_blocks(self) -> int:
        return self._res().tokens // self.bt

    def remaining_blocks(self) -> int:
        """Blocks a stop-and-copy would still have to move right now."""
        return len(self._res().blocks) - self.copied

    def _copy(self, lo: int, hi: int) -> None:
        if hi <= lo:
            return
        res = self._res()
        new = self.dst_pool.allocator.alloc(hi - lo)
        self.dst_blocks = np.concatenate([self.dst_blocks, new])
        sb = np.ascontiguousarray(res.blocks[lo:hi], dtype=np.int32)
        db = np.ascontiguousarray(new, dtype=np.int32)
        self._keep += [sb, db]
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = self.src_pool.pool_id, self.dst_pool.pool_id, hi - lo, 1
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
        if self._table is not None:  # fused: this launch fills entries [lo, hi) of the dst row
            self._table.set_host(self.rid, self.dst_blocks)
            m.dst_table_row = self._table.row_ptr(self.rid) + 4 * lo
        s = self.ex.ordered_stream(self.src_pool.device)
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | self.flags,
                                                ctypes.c_void_p(s.cuda_stream)), "kvm_migrate (live)")
        import torch

        self._last = torch.cuda.Event()
        self._last.record(s)

    def precopy_done(self) -> bool:
        """Have all pre-copy rounds launched so far landed?  (Non-blocking: the
        serving loop keeps decoding until this is true, then pauses.)"""
        return self._last is None or self._last.query()

    def drain(self) -> None:
        """Wait (decode still running) until the launched pre-copy rounds landed."""
        if self._last is not None:
            self._last.synchronize()

    def precopy(self, after=None) -> int:
        """Asynchronously copy every block that became full since the last
        round.  Decode on the source may continue; returns blocks launched.
        `after`: a CUDA event recorded after the decode writes that filled
        those blocks (the copy stream waits on it; no host sync)."""
        if after is not None:
            self.ex.stream(self.src_pool.device).wait_event(after)
        full = self.full_blocks()
        n = full - self.copied
        self._copy(self.copied, full)
        self.copied = max(self.copied, full)
        if n > 0:
            self.stats.rounds += 1
            self.stats.blocks_precopied += n
            self.stats.round_blocks.append(n)
        return n

    def finish(self, after=None, stream_ordered: bool = False) -> LiveStats:
        """Pause point (decode stopped): copy the tail incl. the partial last
        block, switch residency, free the source blocks.  The destination
        block-table row was filled piecewise by the copy kernels themselves.

        stream_ordered: do not wait on the host; `stats.done` is an event the
        destination's decode stream waits on (`wait_event`), so the GPU goes from
        the last source decode step to the tail copy to the first destination
        decode step without a host round trip."""
        import torch

        t0 = time.perf_counter()
        if after is not None:
            self.ex.stream(self.src_pool.device).wait_event(after)
        res = self._res()
        n_all = len(res.blocks)
        tail = n_all - self.copied
        self._copy(self.copied, n_all)
        self.copied = n_all
        if stream_ordered:
            self.stats.done = torch.cuda.Event(enable_timing=True)
            self.stats.done.record(self.ex.stream(self.src_pool.device))
        else:
            self.ex.stream(self.src_pool.device).synchronize()
        self.ex._commit([(self.rid, self.dst_gpu, res.tokens, self.dst_blocks)])
        t1 = time.perf_counter()
        self.stats.blocks_stopcopied = tail
        self.stats.downtime_s = t1 - t0
        self.stats.total_s = t1 - self._t0
        self._keep.clear()
        return self.stats
