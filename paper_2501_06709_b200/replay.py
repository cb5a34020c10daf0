"""Trace-replay executor: the reference's slot loop with the bytes moved.

Input is a recorded run of the reference simulator (tests/golden/trace_*.json,
written by tests/golden/make_golden.py from `kvpack.sim.run`): per slot, the
arrivals and the GPU the scheduler placed each on, completions / rejections /
aborts, and every plan row (item, src, dst, kv_bytes, tokens, mode) with the
group members at plan time.  The replay reproduces sim.py:151-227 physically:

  1. completions / rejected / aborted requests release their blocks;
  2. decode growth: every resident request's KV grows to
     prompt + min(response, tokens_per_slot * (slot - arrival)) tokens
     (model.py:58-69), allocating blocks on the GPU that *physically* holds it;
  3. arrivals are admitted on the GPU the scheduler placed them on;
  4. the slot's executed plan rows (plan.executed, migration.py:119-121) run on
     the GPUs: kv_transfer / forced_kv_transfer -> kvm_migrate,
     token_transfer -> kvm_reprefill.  Group items move the members that are
     physically on the row's src (SURVEY.md §7 hard part 5).

Each logical GPU of the trace gets its own KV pool; several logical GPUs may
share one physical device (the whole 8-GPU trace replays on one B200 with a
down-scaled KV shape; token counts and therefore every decision are unchanged,
bytes scale by shape.kv_bytes_per_token / reference bpt).

Correctness: every block a request owns carries a fingerprint that depends on
(request, logical block, layer, K|V); `verify()` checks every resident request
still reads back its own fingerprint wherever it now lives.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from .planner import DEFERRED, TOKEN_TRANSFER, PendingMove, PlannedMove


@dataclass
class SlotStats:
    slot: int
    rows: int
    executed: int
    kv_moves: int
    token_moves: int
    bytes_moved: int          # bytes physically copied by kvm_migrate (whole blocks)
    tokens_moved: int         # tokens of the requests copied (algorithmic bytes = x bpt)
    ref_kv_bytes: int         # sum of the reference's kv_bytes over executed kv rows (at its bpt)
    seconds: float


@dataclass
class ReplayReport:
    slots: List[SlotStats] = field(default_factory=list)
    verified_requests: int = 0     # request fingerprints checked (summed over checks)
    recomputed_requests: int = 0

    @property
    def bytes_moved(self) -> int:
        return sum(s.bytes_moved for s in self.slots)

    @property
    def executed(self) -> int:
        return sum(s.executed for s in self.slots)

    @property
    def tokens_moved(self) -> int:
        return sum(s.tokens_moved for s in self.slots)

    @property
    def migrate_seconds(self) -> float:
        return sum(s.seconds for s in self.slots)


def tokens_at(rec, slot: int, tokens_per_slot: int) -> int:
    """model.py:58-69 in tokens."""
    _, arrival, prompt, response = rec
    return prompt + min(response, tokens_per_slot * max(0, slot - arrival))


def _sync_devices(executor) -> None:
    """Wait for every device the executor's pools live on (torch.cuda.synchronize()
    alone waits for the current device only)."""
    import torch

    for dev in sorted({p.device for per in executor.pools.values() for p in per.values()}):
        torch.cuda.synchronize(dev)


class Fingerprints:
    """Per-request KV fingerprints on an executor's pools: every block a
    request owns holds a value that depends on (request, logical block, layer,
    K|V), written when the block is gained; `verify()` checks every resident
    request still reads back its own values wherever it now lives (requests
    whose KV was re-prefilled are skipped: their bytes are recomputed, not
    copied)."""

    def __init__(self, executor):
        self.ex = executor
        self.recomputed: set = set()
        self.prefix_only: Dict[int, int] = {}  # split_transfer: rid -> leading blocks still carrying copies
        self._stamped: Dict[int, int] = {}   # rid -> number of blocks stamped
        self._marked: set = set()            # stamps awaiting flush()

    def stamp(self, rid: int) -> None:
        """Write the fingerprint into blocks the request gained since last time (now)."""
        self.mark(rid)
        self.flush()

    def mark(self, rid: int) -> None:
        """Like stamp(), but batched: written at the next flush() (one write per
        pool for every marked request).  Call flush() before anything copies or
        reads the request's blocks."""
        if rid not in self.recomputed:
            self._marked.add(rid)

    def flush(self) -> None:
        import torch

        marked, self._marked = self._marked, set()
        by_pool: Dict[int, list] = {}
        for rid in marked:
            r = self.ex.loc.get(rid)
            if r is None or rid in self.recomputed:
                continue
            start = self._stamped.get(rid, 0)
            if start >= len(r.blocks):
                continue
            pool = self.ex.pool(r.gpu, r.model)
            by_pool.setdefault(id(pool), [pool, [], [], []])
            e = by_pool[id(pool)]
            e[1].append(np.full(len(r.blocks) - start, rid, dtype=np.int64))
            e[2].append(np.arange(start, len(r.blocks), dtype=np.int64))
            e[3].append(r.blocks[start:].astype(np.int64))
            self._stamped[rid] = len(r.blocks)
        for pool, rids, idx, blocks in by_pool.values():
            dev = pool.tensor.device
            rids_t = torch.from_numpy(np.concatenate(rids)).to(dev)
            idx_t = torch.from_numpy(np.concatenate(idx)).to(dev)
            blk_t = torch.from_numpy(np.concatenate(blocks)).to(dev)
            v = self._values(rids_t, idx_t, pool)                  # [L][2][n]
            pool.tensor.view(torch.int16)[:, :, blk_t] = v[..., None, None, None].expand(
                *v.shape, *pool.view_shape[3:])

    def forget(self, rid: int) -> None:
        self._stamped.pop(rid, None)
        self.recomputed.discard(rid)
        self.prefix_only.pop(rid, None)
        self._marked.discard(rid)

    @staticmethod
    def _values(rids, idx, pool):
        """Fingerprint of (request, logical block, layer, K|V): int16 [L][2][n]."""
        import torch

        L = pool.shape.layers
        dev = rids.device
        base = (rids * 7919 + idx * 104729) % 16381
        lay = torch.arange(L, device=dev, dtype=torch.int64)[:, None, None] * 2
        kv = torch.arange(2, device=dev, dtype=torch.int64)[None, :, None]
        return ((base[None, None, :] * 2 + lay * 3 + kv) % 32749 - 16374).to(torch.int16)

    @staticmethod
    def values(rid, lo, hi, pool):
        import torch

        dev = pool.tensor.device
        i = torch.arange(lo, hi, device=dev, dtype=torch.int64)
        v = Fingerprints._values(torch.full_like(i, rid), i, pool)
        return v[..., None, None, None].expand(*v.shape, *pool.view_shape[3:])

    def verify(self) -> int:
        """Number of resident requests checked; raises on the first mismatch."""
        import torch

        self.flush()
        n = 0
        for rid, r in self.ex.loc.items():
            if rid in self.recomputed:
                continue
            pool = self.ex.pool(r.gpu, r.model)
            k = min(len(r.blocks), self.prefix_only.get(rid, len(r.blocks)))   # split: the copied prefix only
            got = pool.tensor.view(torch.int16)[:, :, torch.from_numpy(r.blocks[:k].astype(np.int64)).to(
                pool.tensor.device)]
            if not torch.equal(got, self.values(rid, 0, k, pool)):
                raise AssertionError(f"request {rid} on GPU {r.gpu}: KV bytes differ from its fingerprint")
            n += 1
        return n


class FingerprintedExecutor:
    """Executor proxy for the live loop (runtime.run_slots): the same
    admit / grow / release / execute calls, with every block a request gains
    fingerprinted so `verify()` can prove the migrated bytes are intact."""

    def __init__(self, executor):
        self.ex = executor
        self.fp = Fingerprints(executor)
        self.reports: list = []

    @property
    def loc(self):
        return self.ex.loc

    def admit(self, rid, gpu, tokens, model=None):
        r = self.ex.admit(rid, gpu, tokens, model=model)
        self.fp.mark(rid)
        return r

    def grow(self, rid, tokens):
        r = self.ex.grow(rid, tokens)
        self.fp.mark(rid)
        return r

    def release(self, rid):
        self.ex.release(rid)
        self.fp.forget(rid)

    def execute(self, plan, members_of=None):
        self.fp.flush()              # the stamps must be in the blocks before they are copied
        report = self.ex.execute(plan, members_of=members_of)
        for rec in report.records:
            if rec.mode == TOKEN_TRANSFER:
                self.fp.recomputed.update(rec.requests)
            for rid, k in rec.split_prefix_blocks.items():
                self.fp.prefix_only[rid] = min(self.fp.prefix_only.get(rid, k), k)
        self.reports.append(report)
        return report

    def reconcile(self, target_of, skip=()):
        self.fp.flush()
        report = self.ex.reconcile(target_of, skip=skip)
        self.reports.append(report)
        return report

    def verify(self) -> int:
        _sync_devices(self.ex)
        return self.fp.verify()


class TraceReplay:
    """Drive a MigrationExecutor with a recorded reference run."""

    def __init__(self, fixture: dict, executor, ref_bpt: Optional[int] = None, fingerprint: bool = True,
                 model_map: Optional[Dict[str, str]] = None):
        self.fx = fixture
        self.ex = executor
        wl_bpt = fixture["config"]["workload"]["kv_bytes_per_token"]
        self.ref_bpt = ref_bpt or (wl_bpt if isinstance(wl_bpt, int) else None)
        self.tps = fixture["config"]["sim"].get("tokens_per_slot", 10)
        self.trace = {r[0]: tuple(r) for r in fixture["trace"]}
        self.rows_by_slot: Dict[int, list] = {}
        for row in fixture["plan_rows"]:
            self.rows_by_slot.setdefault(row[0], []).append(row)
        self.fingerprint = fingerprint
        # multi-LLM fixtures carry the model of every request and its bytes/token
        self.models: Dict[int, str] = {int(k): v for k, v in fixture.get("models", {}).items()}
        self.model_bpt: Dict[str, int] = dict(fixture.get("model_bpt", {}))
        # fixture model name -> executor pool key (e.g. a down-scaled shape's name)
        self.model_map: Dict[str, str] = dict(model_map or {})
        self.fp = Fingerprints(executor)
        self.recomputed = self.fp.recomputed
        self.reports: list = []              # per-slot ExecReport (None if nothing executed)

    def bpt_of(self, rid: int) -> int:
        m = self.models.get(rid)
        return self.model_bpt[m] if m is not None else self.ref_bpt

    # -- fingerprints ------------------------------------------------------------
    def _stamp(self, rid: int) -> None:
        if self.fingerprint:
            self.fp.mark(rid)

    def verify(self) -> int:
        return self.fp.verify() if self.fingerprint else 0

    # -- the slot loop -------------------------------------------------------------
    def run(self, max_slots: Optional[int] = None, verify_every: int = 0) -> ReplayReport:
        if self.fingerprint:
            import torch

        rep = ReplayReport()
        ex = self.ex
        slots = self.fx["slots"]
        n_slots = len(slots) if max_slots is None else min(max_slots, len(slots))
        for s in range(n_slots):
            ev = slots[s]
            # 1. departures (completed, rejected, aborted)
            for rid in list(ev["done"]) + list(ev["gone"]):
                if rid in ex.loc:
                    ex.release(rid)
                    self.fp.forget(rid)
            # 2. decode growth of resident requests on their physical GPU
            for rid in list(ex.loc):
                if rid in self.trace:
                    tok = tokens_at(self.trace[rid], s, self.tps)
                    if tok > ex.loc[rid].tokens:
                        ex.grow(rid, tok)
                        self._stamp(rid)
            # 3. arrivals at the scheduler's placement
            for rid, gpu, size in ev["arr"]:
                if gpu < 0 or rid in ex.loc:
                    continue
                model = self.models.get(rid)
                ex.admit(rid, gpu, size // self.bpt_of(rid),
                         model=self.model_map.get(model, model) if model else None)
                self._stamp(rid)
            # 4. the slot's executed plan rows
            rows = self.rows_by_slot.get(s, [])
            planned, members = [], {}
            ref_bytes = 0
            for (_slot, item, src, dst, kvb, tok, mode, mem, _sizes) in rows:
                if mode == DEFERRED:
                    continue
                planned.append(PlannedMove(PendingMove(item, src, dst, kvb, tok), mode))
                members[item] = mem
                if mode != TOKEN_TRANSFER:
                    ref_bytes += kvb
            if self.fingerprint and planned:
                self.fp.flush()
            t0 = time.perf_counter()
            report = ex.execute(planned, members_of=lambda it: members.get(it, [it])) if planned else None
            dt = time.perf_counter() - t0
            if report is not None:
                for rec in report.records:
                    if rec.mode == TOKEN_TRANSFER:
                        self.recomputed.update(rec.requests)
            rep.slots.append(SlotStats(
                s, len(rows), len(planned),
                sum(1 for p in planned if p.mode != TOKEN_TRANSFER),
                sum(1 for p in planned if p.mode == TOKEN_TRANSFER),
                report.bytes_moved if report else 0, report.tokens_moved if report else 0,
                ref_bytes, dt))
            self.reports.append(report)
            if self.fingerprint and verify_every and (s + 1) % verify_every == 0:
                _sync_devices(self.ex)
                rep.verified_requests += self.verify()
        if self.fingerprint:
            _sync_devices(self.ex)
            rep.verified_requests += self.verify()
        rep.recomputed_requests = len(self.recomputed)
        return rep


def pool_blocks_for(fixture: dict, shape_block_tokens: int = 16, headroom: float = 1.5,
                    model: Optional[str] = None) -> int:
    """Blocks per logical GPU (per model): capacity in tokens
    (capacity_bytes / bpt) with headroom for the physical-vs-logical skew of
    deferred moves (the physical source can hold ~1.2 C)."""
    bpt = fixture["model_bpt"][model] if model else fixture["config"]["workload"]["kv_bytes_per_token"]
    cap_tokens = fixture["config"]["cluster"]["capacity_bytes"] // bpt
    return int(math.ceil(headroom * cap_tokens / shape_block_tokens))
