"""The data plane the reference leaves out: execute a MigrationPlan on GPUs.

Insertion point: /root/reference/pkg/src/kvpack/sim.py:218-227, where the
reference takes `plan.executed` (migration.py:119-121) and simply deletes the
records.  `MigrationExecutor.execute(plan)` is called at exactly that spot,
once per slot, from the single scheduler thread (model.py:119);
it is asynchronous on per-device CUDA streams and, by default, awaited before
returning so the slot's metrics row (sim.py:229-238) stays truthful.

Physical vs logical placement.  The scheduler moves items logically at once,
but a deferred move's bytes stay where they were for epochs (sim.py:207-227),
and a group item's members drift while its move is pending.  The executor
therefore keeps its own physical location map per *request* and, for a move
of item I from GPU s to GPU d, migrates exactly the members of I that are
physically on s (SURVEY.md §7 hard part 5).  Source blocks are released only
after the copy has completed.

Modes (migration.py:19-22):
  kv_transfer, forced_kv_transfer -> kvm_migrate (gather -> push -> table rewrite)
  token_transfer                  -> kvm_reprefill on the destination
  split_transfer (extension, plan_hybrid(split=True)) -> the prefix's blocks by
      KV copy and the suffix's tokens by re-prefill: one fused
      kvm_split_migrate launch on the destination when both pools share a
      device, else kvm_migrate on the source in parallel with kvm_reprefill
      on the destination
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .errors import ConfigError, NotPlaced, RequestTooLarge
from .kvcache import BlockTable, KVPool
from .planner import (FORCED_KV_TRANSFER, KV_TRANSFER, SPLIT_TRANSFER, TOKEN_TRANSFER, MigrationPlan, PendingMove,
                      PlannedMove)

ENGINES = {"ldg": 0, "bulk": _native.KVM_F_ENGINE_BULK}


@dataclass
class Residency:
    """Where a request's KV physically lives right now."""

    gpu: int
    blocks: np.ndarray  # int32, logical block i -> pool block id
    tokens: int
    model: str = ""     # ModelShape.name of the pool it lives in (multi-LLM)


@dataclass
class ExecRecord:
    item: int
    src: int
    dst: int
    mode: str
    requests: List[int]
    blocks: int
    bytes_moved: int      # KV bytes physically copied (members found at src), whole blocks
    tokens_recomputed: int
    tokens_moved: int = 0  # tokens of the members copied: algorithmic bytes = tokens_moved * bpt
    request_tokens: Dict[int, int] = field(default_factory=dict)  # per moved request: its tokens
    done: Optional[object] = None  # stream-ordered calls: CUDA event recorded after the move (and read-back)
    # execute(layer_flags=True): per moved request, an int32 device tensor [layers] on the destination
    # GPU; entry l reaches 1 once layer l landed (paged_decode(..., layer_flags=...) pipelines on it)
    layer_flags: Dict[int, object] = field(default_factory=dict)
    # split_transfer: per moved request, how many of its blocks (from the front) were copied
    split_prefix_blocks: Dict[int, int] = field(default_factory=dict)


@dataclass
class ExecReport:
    records: List[ExecRecord] = field(default_factory=list)
    launches: int = 0
    # with MigrationExecutor(timing=True) and wait=True: device time per GPU from
    # the first launch of this call to the last (CUDA events on the executor's
    # stream), in ms
    device_ms: Dict[int, float] = field(default_factory=dict)
    # stream_ordered execute(): destination device -> event after its incoming
    # moves landed; source device -> event after its launches
    done: Dict[int, object] = field(default_factory=dict)
    src_done: Dict[int, object] = field(default_factory=dict)

    @property
    def copy_GBps(self) -> Optional[float]:
        """Payload bytes copied / the slowest GPU's device time (None without timing)."""
        if not self.device_ms:
            return None
        ms = max(self.device_ms.values())
        return self.bytes_moved / ms / 1e6 if ms > 0 else None

    @property
    def bytes_moved(self) -> int:
        return sum(r.bytes_moved for r in self.records)

    @property
    def tokens_moved(self) -> int:
        return sum(r.tokens_moved for r in self.records)


class MigrationExecutor:
    """Executes planned moves over registered per-GPU pools.

    pools:  logical GPU id -> KVPool, or -> {model name: KVPool} when the GPU
            serves several LLMs (multi-LLM: a request lives in the pool of its
            model's shape).  Several logical GPUs may share one physical
            device (e.g. replaying an 8-GPU trace on one B200).
    tables: same keys -> BlockTable (optional; when present the kernel
            rewrites the destination row in place).
    reprefill: callable(executor, request_id, dst_gpu, dst_blocks, tokens,
            stream) that recomputes KV on the destination (token_transfer);
            see reprefill.ReprefillEngine.  Without it, token_transfer raises.
    """

    def __init__(self, pools: Dict[int, KVPool], tables: Optional[Dict[int, BlockTable]] = None,
                 engine: str = "bulk", reprefill: Optional[Callable] = None, timing: bool = False,
                 split_kernels: str = "auto", copy_sms: int = 0):
        import torch

        if split_kernels not in ("auto", "fused", "two"):
            raise ConfigError("split_kernels must be 'auto', 'fused' or 'two'")
        # split_transfer: "auto" = one fused kvm_split_migrate when source and destination pools share a
        # device, else kvm_migrate (source) + kvm_reprefill (destination); "two" forces the latter
        self.split_kernels = split_kernels

        self.timing = timing
        self._events: Dict[int, list] = {}
        self._pending: List[Tuple[list, bool]] = []   # wait=False calls awaiting commit()
        if engine not in ENGINES:
            raise ConfigError(f"engine must be one of {sorted(ENGINES)}")
        if not pools:
            raise ConfigError("executor needs at least one pool")
        self.pools: Dict[int, Dict[str, KVPool]] = {g: _by_model(p) for g, p in pools.items()}
        self.tables: Dict[int, Dict[str, BlockTable]] = {}
        for g, t in (tables or {}).items():
            if isinstance(t, dict):
                self.tables[g] = dict(t)
            else:  # one table per GPU: shared by the GPU's (single) model
                self.tables[g] = {m: t for m in self.pools[g]}
        models = {m for per in self.pools.values() for m in per}
        self.default_model = next(iter(models)) if len(models) == 1 else None
        if not 0 <= copy_sms <= 255:
            raise ConfigError("copy_sms must be in [0, 255] (0 = the whole GPU)")
        # copy_sms > 0: every kvm_migrate / kvm_compact of this executor runs on at most that many SMs
        # (KVM_F_MAX_SMS): a push bound by a link needs far fewer SMs than the HBM-bound compaction
        self.engine_flag = ENGINES[engine] | _native.KVM_F_MAX_SMS(copy_sms)
        self.reprefill = reprefill
        self.loc: Dict[int, Residency] = {}
        self._streams: Dict[int, "torch.cuda.Stream"] = {}
        self._fences: Dict[int, Dict[int, object]] = {}   # pool id -> {device: event of a pending read}
        _native.lib()  # fail loudly now if the native library is missing
        devices = {p.device for per in self.pools.values() for p in per.values()}
        if len(devices) > 1:
            # single process, several GPUs: kernels on the source device store straight
            # into the destination device's pool and block table (UVA peer access)
            _native.check(_native.lib().kvm_init(1), "kvm_init(enable_peer_access)")
        for d in sorted(devices):   # created now: the first torch stream of a process costs ~0.5 s
            self.stream(d)

    # -- streams ---------------------------------------------------------------
    def stream(self, device: int):
        import torch

        s = self._streams.get(device)
        if s is None:
            s = torch.cuda.Stream(device=device)
            self._streams[device] = s
        return s

    def ordered_stream(self, device: int):
        """The executor's stream for `device`, made to wait for everything the
        caller has queued on its current stream (pool fills, hidden states,
        weights...): the usual side-stream contract, so a migration or
        re-prefill never reads data that is still being produced."""
        import torch

        s = self.stream(device)
        s.wait_stream(torch.cuda.current_stream(device))
        if self.timing and device not in self._events:   # first launch on this GPU in this call
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            self._events[device] = [e0, None]
        return s

    def _close_timing(self, report: "ExecReport") -> None:
        import torch

        for dev, ev in self._events.items():
            ev[1] = torch.cuda.Event(enable_timing=True)
            ev[1].record(self.stream(dev))
        self.synchronize()
        for dev, (e0, e1) in self._events.items():
            report.device_ms[dev] = e0.elapsed_time(e1)
        self._events = {}

    def synchronize(self) -> None:
        for s in self._streams.values():
            s.synchronize()

    # -- residency ---------------------------------------------------------------
    def pool(self, gpu: int, model: Optional[str] = None) -> KVPool:
        """The pool of `model` on logical GPU `gpu` (model may be omitted when
        the executor serves a single model)."""
        per = self.pools.get(gpu)
        if per is None:
            raise NotPlaced(f"no KV pool registered for GPU {gpu}")
        key = model or self.default_model
        if key is None:
            raise ValueError("several models are served: pass model=")
        try:
            return per[key]
        except KeyError:
            raise NotPlaced(f"GPU {gpu} has no pool for model {key!r}") from None

    def pool_of(self, rid: int) -> KVPool:
        r = self._res(rid)
        return self.pool(r.gpu, r.model)

    def admit(self, rid: int, gpu: int, tokens: int, model: Optional[str] = None) -> np.ndarray:
        """Allocate blocks for a new request on `gpu` (prefill happens elsewhere)."""
        if rid in self.loc:
            raise ValueError(f"request {rid} already resident")
        pool = self.pool(gpu, model)
        blocks = pool.allocator.alloc(pool.shape.blocks_for(tokens))
        self.loc[rid] = Residency(gpu, blocks, tokens, pool.shape.name)
        self._table_set(gpu, pool.shape.name, rid, blocks)
        return blocks

    def grow(self, rid: int, tokens: int) -> None:
        """Decode appended tokens: extend the block table when a block fills."""
        r = self._res(rid)
        pool = self.pool(r.gpu, r.model)
        need = pool.shape.blocks_for(tokens) - len(r.blocks)
        if need > 0:
            old = len(r.blocks)
            r.blocks = np.concatenate([r.blocks, pool.allocator.alloc(need)])
            self._table_set(r.gpu, r.model, rid, r.blocks, start=old)
        r.tokens = tokens

    def release(self, rid: int) -> None:
        r = self.loc.pop(rid, None)
        if r is None:
            return
        self.pool(r.gpu, r.model).allocator.free(r.blocks)
        t = self._table(r.gpu, r.model)
        if t is not None:
            t.drop(rid)

    def where(self, rid: int) -> Residency:
        return self._res(rid)

    # -- execution ---------------------------------------------------------------
    def execute(self, plan, members_of: Optional[Callable[[int], Sequence[int]]] = None,
                wait: bool = True, stream_ordered: bool = False, layer_flags: bool = False) -> ExecReport:
        """Carry out `plan.executed` (or a list of PlannedMove) in plan order.

        members_of(item) -> request ids of a group item (negative id); the
        default treats every item as a single request.  Every member that is
        not physically on the move's dst moves there, from whichever GPU holds
        it now: a group's members drift while its move is pending (a member
        that joined at an intermediate GPU, sim.py:207-217), and the item's
        logical GPU is where its bytes must end up.

        All-or-nothing: every move is validated and every destination block
        reserved before anything launches (unknown mode, missing or mismatched
        pools, a re-prefill engine that cannot write the pool, a full pool or
        block table all raise with nothing changed); a failure while issuing
        rolls the reservations and new table rows back before re-raising.

        layer_flags: kv moves publish per-layer completion into `rec.layer_flags[rid]`
        (value 1), so a destination decode can start layer by layer
        (attention.paged_decode(..., layer_flags=...)) while the copy runs.

        stream_ordered: return right after issuing, with residencies already
        switched on the host.  Each destination GPU's executor stream waits
        (cudaStreamWaitEvent, no host round trip) on the copy launched on every
        source GPU that feeds it, and `report.done[dst_device]` / `rec.done`
        is an event after which the destination's blocks and table row are
        final: a decode stream `wait_event`s on it.  Freed source blocks may
        be reallocated by the host at once: every later executor launch that
        writes into that pool, from any device, first waits on the source's
        copy (per-pool fences); a caller's own stream that writes into the
        pool waits on `report.src_done[src_device]`.
        """
        executed: List[PlannedMove] = plan.executed if isinstance(plan, MigrationPlan) else [
            p for p in plan if p.mode != "deferred"]
        report = ExecReport()
        self._events = {}
        # phase 1: validate every move and reserve all destination blocks; nothing is
        # launched yet, so a failure leaves the pools and tables exactly as they were
        work = []  # (pm, rec, [(rid, res, src_pool, dst_pool, dst_blocks)])
        taken = []  # (pool, blocks) reserved in this call, for rollback
        new_rows: Dict[int, int] = {}   # id(table) -> slots this call will newly take
        try:
            for pm in executed:
                mv = pm.move
                if pm.mode not in (KV_TRANSFER, FORCED_KV_TRANSFER, TOKEN_TRANSFER, SPLIT_TRANSFER):
                    raise ValueError(f"cannot execute mode {pm.mode!r}")
                if pm.mode == SPLIT_TRANSFER and mv.item < 0:
                    raise ValueError("split_transfer applies to single requests, not groups")
                rids = list(members_of(mv.item)) if (members_of and mv.item < 0) else [mv.item]
                if self._pending:
                    self._check_not_pending(rids)
                movers = [r for r in rids if r in self.loc and self.loc[r].gpu != mv.dst]
                if pm.mode in (TOKEN_TRANSFER, SPLIT_TRANSFER) and self.reprefill is None and movers:
                    raise ConfigError(f"{pm.mode} planned but executor has no re-prefill engine")
                rec = ExecRecord(mv.item, mv.src, mv.dst, pm.mode, movers, 0, 0, 0)
                items = []
                for rid in movers:
                    res = self.loc[rid]
                    src_pool, dst_pool = self.pool(res.gpu, res.model), self.pool(mv.dst, res.model)
                    if _geometry(src_pool) != _geometry(dst_pool):
                        raise ConfigError(f"request {rid}: pools of GPU {res.gpu} and GPU {mv.dst} have different "
                                          f"KV geometry {_geometry(src_pool)} vs {_geometry(dst_pool)}")
                    if pm.mode in (TOKEN_TRANSFER, SPLIT_TRANSFER):
                        check = getattr(self.reprefill, "validate", None)
                        if check is not None:
                            check(dst_pool)
                    table = self._table(mv.dst, res.model)
                    if table is not None:
                        if len(res.blocks) > table.max_blocks:
                            raise RequestTooLarge(f"request {rid}: {len(res.blocks)} blocks > block-table width "
                                                  f"{table.max_blocks} on GPU {mv.dst}")
                        if not table.has(rid):
                            new_rows[id(table)] = new_rows.get(id(table), 0) + 1
                            if new_rows[id(table)] > table.free_slots:
                                raise ConfigError(f"block table of GPU {mv.dst} is full")
                    dst_blocks = dst_pool.allocator.alloc(len(res.blocks))
                    taken.append((dst_pool, dst_blocks))
                    items.append((rid, res, src_pool, dst_pool, dst_blocks))
                work.append((pm, rec, items))
        except Exception:
            for pool, blocks in taken:
                pool.allocator.free(blocks)
            raise
        # phase 2: issue; on failure undo the reservations and the rows this call created
        created: List[Tuple[BlockTable, int]] = []
        try:
            self._issue(work, report, created, layer_flags)
        except BaseException:
            try:
                self.synchronize()      # nothing issued may still be writing the blocks we release
            finally:
                for pool, blocks in taken:
                    pool.allocator.free(blocks)
                for table, rid in created:
                    table.drop(rid)
            raise
        post = [(rid, pm.move.dst, res.tokens, dst_blocks)
                for pm, rec, items in work for rid, res, src_pool, dst_pool, dst_blocks in items]
        if stream_ordered:
            self._order_across_devices(report, work)
            self._commit(post)
        elif wait:
            if self.timing:
                self._close_timing(report)
            self.synchronize()
            self._commit(post)
        else:
            self._pending.append((post, False))
        return report

    def _issue(self, work, report: "ExecReport", created: list, layer_flags: bool) -> None:
        """Phase 2 of execute(): re-prefills on their destination streams, then
        one fused kvm_migrate launch per source device."""
        by_dev: Dict[int, List[_native.Move]] = {}
        writes: Dict[int, Dict[int, object]] = {}   # src device -> {dst pool id: dst pool}
        keep = []  # host arrays must outlive the kvm_migrate call

        def table_for(gpu, model, rid):
            table = self._table(gpu, model)
            if table is not None and not table.has(rid):
                table.slot(rid)
                created.append((table, rid))
            return table

        for pm, rec, items in work:
            mv = pm.move
            for rid, res, src_pool, dst_pool, dst_blocks in items:
                nb = len(res.blocks)
                if pm.mode in (KV_TRANSFER, FORCED_KV_TRANSFER):
                    m = _native.Move()
                    m.src_pool, m.dst_pool, m.n_blocks = src_pool.pool_id, dst_pool.pool_id, nb
                    m.done_value = 1
                    sb = np.ascontiguousarray(res.blocks, dtype=np.int32)
                    db = np.ascontiguousarray(dst_blocks, dtype=np.int32)
                    keep += [sb, db]
                    m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
                    table = table_for(mv.dst, res.model, rid)
                    if table is not None:
                        table.set_host(rid, db)
                        m.dst_table_row = table.row_ptr(rid)
                    if layer_flags:
                        import torch

                        fl = torch.zeros(src_pool.shape.layers, dtype=torch.int32, device=f"cuda:{dst_pool.device}")
                        rec.layer_flags[rid] = fl
                        m.layer_flags = fl.data_ptr()
                    by_dev.setdefault(src_pool.device, []).append(m)
                    writes.setdefault(src_pool.device, {})[dst_pool.pool_id] = dst_pool
                    rec.bytes_moved += nb * src_pool.shape.piece_bytes * 2 * src_pool.shape.layers
                    rec.tokens_moved += res.tokens
                elif pm.mode == SPLIT_TRANSFER:
                    self._issue_split(pm, rec, rid, res, src_pool, dst_pool, dst_blocks, table_for)
                    report.launches += 1 if (src_pool.device == dst_pool.device and self.split_kernels != "two") else 2
                else:  # TOKEN_TRANSFER
                    s = self.ordered_stream(dst_pool.device)
                    self._wait_fences(s, dst_pool.device, [dst_pool])
                    self.reprefill(self, rid, mv.dst, dst_blocks, res.tokens, s)
                    table = table_for(mv.dst, res.model, rid)
                    if table is not None:
                        table.set_host(rid, dst_blocks)
                        table.rows[table.slot(rid), :len(dst_blocks)].copy_(
                            _as_i32_tensor(dst_blocks, dst_pool.device), non_blocking=False)
                    rec.tokens_recomputed += res.tokens
                    report.launches += 1
                rec.blocks += nb
                rec.request_tokens[rid] = res.tokens
            report.records.append(rec)
        for dev, moves in by_dev.items():
            self._launch_migrate(dev, moves, list(writes[dev].values()))
            report.launches += 1

    def reconcile(self, target_of: Callable[[int], Optional[int]], skip=(), **kw) -> ExecReport:
        """Move every resident request whose physical GPU differs from
        `target_of(rid)` (its item's logical GPU) there, as kv_transfer —
        except requests in `skip` (members of items still in the backlog,
        which travel with their item's planned move).

        Why: the reference's planner never sees member-level moves (a member
        shed from its group and re-placed, scheduler.py:944-975, or a request
        absorbed into another GPU's group): at the backlog refresh the moved
        id is no longer an item, so its PendingMove is dropped
        (sim.py:207-213) and its bytes would stay on the old GPU for good.
        These moves are outside the plan (no budget, no plan row); the
        decisions stay the reference's."""
        moves = []
        for rid in sorted(self.loc):
            if rid in skip:
                continue
            res = self.loc[rid]
            g = target_of(rid)
            if g is None or g == res.gpu:
                continue
            moves.append(PlannedMove(PendingMove(rid, res.gpu, g, 0, res.tokens), KV_TRANSFER))
        if not moves:
            return ExecReport()
        return self.execute(moves, **kw)

    def _order_across_devices(self, report: "ExecReport", work) -> None:
        """Stream-ordered completion: one event per source device after its
        launches; each destination device's stream waits on the events of the
        sources that feed it, then records its own done event."""
        import torch

        feeds: Dict[int, set] = {}
        for pm, rec, items in work:
            for rid, res, src_pool, dst_pool, dst_blocks in items:
                feeds.setdefault(dst_pool.device, set()).add(src_pool.device)
        for dev in sorted({d for srcs in feeds.values() for d in srcs}):
            ev = torch.cuda.Event()
            ev.record(self.stream(dev))
            report.src_done[dev] = ev
        for pm, rec, items in work:   # the source blocks are freed now; writers elsewhere wait on the read
            for rid, res, src_pool, dst_pool, dst_blocks in items:
                self._fence(src_pool, src_pool.device, report.src_done[src_pool.device])
        for dst, srcs in sorted(feeds.items()):
            s = self.stream(dst)
            for src in sorted(srcs):
                if src != dst:
                    s.wait_event(report.src_done[src])
            ev = torch.cuda.Event(enable_timing=self.timing)
            ev.record(s)
            report.done[dst] = ev
        for pm, rec, items in work:
            if items:
                rec.done = report.done[items[0][3].device]

    def compact(self, rid: int, wait: bool = True, row_out=None, stream_ordered: bool = False) -> ExecRecord:
        """1-GPU case: move a request into the lowest free blocks of its own
        pool (defragmentation; kvm_compact = migrate with src pool == dst pool).

        row_out: optional pinned host int32 tensor; the rewritten block-table
        row is copied into it on the same stream right after the kernel, so one
        synchronize covers the move and the read-back.

        stream_ordered: return right after issuing, with the residency already
        updated on the host and `rec.done` an event that completes after the
        move (and read-back).  Safe because every later launch touching this
        pool is queued behind it on the executor's ordered stream; it lets the
        host prepare the next call while the GPU copies."""
        if self._pending:
            self._check_not_pending([rid])
        res = self._res(rid)
        pool = self.pool(res.gpu, res.model)
        nb = len(res.blocks)
        dst = pool.allocator.alloc(nb)
        sb = np.ascontiguousarray(res.blocks, dtype=np.int32)
        table = self._table(res.gpu, res.model)
        row = 0
        if table is not None:
            table.set_host(rid, dst)
            row = table.row_ptr(rid)
        if row_out is not None and table is None:
            raise ConfigError("row_out needs a block table on this GPU")
        s = self.ordered_stream(pool.device)
        self._wait_fences(s, pool.device, [pool])
        lib = _native.lib()
        sp = ctypes.c_void_p(s.cuda_stream)
        _native.check(lib.kvm_compact(pool.pool_id, sb.ctypes.data, dst.ctypes.data, nb, ctypes.c_void_p(row),
                                      _native.KVM_F_BLOCKS_ON_HOST | self.engine_flag, sp), "kvm_compact")
        if row_out is not None:   # D2H of the rewritten row, ordered after the kernel on the same stream
            if row_out.numel() < nb or row_out.element_size() != 4 or not row_out.is_pinned():
                raise ValueError("row_out must be a pinned host int32 tensor with >= n_blocks entries")
            _native.check(lib.kvm_read_back(ctypes.c_void_p(row_out.data_ptr()), ctypes.c_void_p(row), 4 * nb, sp),
                          "kvm_read_back")
        rec = ExecRecord(rid, res.gpu, res.gpu, "compact", [rid], nb,
                         nb * pool.shape.piece_bytes * 2 * pool.shape.layers, 0)
        post = [(rid, res.gpu, res.tokens, dst)]
        if stream_ordered:
            import torch

            rec.done = torch.cuda.Event()
            rec.done.record(s)
            self._fence(pool, pool.device, rec.done)
            self._commit(post, keep_table=True)
        elif wait:
            s.synchronize()
            self._commit(post, keep_table=True)
        else:
            self._pending.append((post, True))
        return rec

    def split_move(self, rid: int, dst_gpu: int, suffix: Optional[int] = None, *, topology=None,
                   **execute_kw) -> ExecRecord:
        """One split_transfer through execute() (the planner's split mode does
        this for every split it plans): copy the first n - s tokens' blocks,
        re-prefill the last s tokens on `dst_gpu`.  s is `suffix`, or — with a
        `topology` — the planner's balanced point from the topology's own link
        bandwidth and prefill rate (planner.split_suffix, the reference's cost
        terms migration.py:158-163), without budget limits."""
        from .planner import split_suffix

        res = self._res(rid)
        sh = self.pool(res.gpu, res.model).shape
        n = res.tokens
        kv = n * sh.kv_bytes_per_token
        if suffix is None:
            if topology is None:
                raise ConfigError("split_move needs suffix= or topology= (the split point comes from its link "
                                  "bandwidth and prefill rate)")
            link = topology.link_of(res.gpu, dst_gpu)
            suffix = split_suffix(n, kv, topology.bandwidth_of(link), topology.prefill_tokens_per_s,
                                  float("inf"), float("inf"), sh.block_tokens)
            if suffix is None:
                suffix = n
        if not 0 <= suffix <= n:
            raise ValueError("suffix must be in [0, tokens]")
        pm = PlannedMove(PendingMove(rid, res.gpu, dst_gpu, kv, n), SPLIT_TRANSFER, 0.0, suffix)
        return self.execute([pm], **execute_kw).records[0]

    def commit(self) -> None:
        """Finish every wait=False execute()/compact(): await streams, then free
        the sources and switch residencies (in call order)."""
        self.synchronize()
        pending, self._pending = self._pending, []
        for post, keep_table in pending:
            self._commit(post, keep_table=keep_table)

    def _check_not_pending(self, rids) -> None:
        busy = {rid for post, _ in self._pending for rid, *_ in post}
        hit = busy.intersection(rids)
        if hit:
            raise ValueError(f"requests {sorted(hit)} have an uncommitted move: call commit() first")

    # -- internals ---------------------------------------------------------------
    def _issue_split(self, pm, rec, rid, res, src_pool, dst_pool, dst_blocks, table_for) -> None:
        """One split_transfer: the first n - s tokens' blocks are copied, the
        last s tokens re-prefilled on the destination (s = pm.suffix_tokens,
        re-based on the request's current length; the prefix stays whole
        blocks).  Same device: ONE fused kvm_split_migrate launch (idle GEMM
        warps stream the prefix while the tensor cores recompute the suffix).
        Across devices: kvm_migrate on the source pushes the prefix over
        NVLink while kvm_reprefill runs on the destination, whose stream then
        waits for the prefix's done flag (device side) and gets the full
        block-table row."""
        import torch

        from .reprefill import reprefill
        from .split import make_split, split_migrate_fused

        sh = dst_pool.shape
        n = res.tokens
        prefix = max(0, min(n, pm.move.tokens - pm.suffix_tokens))
        prefix -= prefix % sh.block_tokens
        plan = make_split(n, n - prefix, sh.block_tokens)
        eng = self.reprefill
        dev = dst_pool.device
        cross = src_pool.device != dev or self.split_kernels == "two"
        if self.split_kernels == "fused" and src_pool.device != dev:
            raise ConfigError("split_kernels='fused' needs the source pool on the destination's device")
        flags = torch.zeros(2, dtype=torch.int32, device=f"cuda:{dev}") if cross else None
        s = self.ordered_stream(dev)
        self._wait_fences(s, dev, [dst_pool])
        w = eng.weights[(dev, sh.name)]
        table = table_for(pm.move.dst, res.model, rid)
        row = 0
        if table is not None:
            table.set_host(rid, dst_blocks)
            row = table.row_ptr(rid)
        rope = float(getattr(eng, "rope_theta", None) or 0.0)
        db_np = np.ascontiguousarray(dst_blocks, dtype=np.int32)
        with torch.cuda.stream(s):
            x = eng.hidden(sh, rid, n, dev)[prefix:].contiguous() if plan.suffix else None
            dbd = torch.from_numpy(db_np).to(f"cuda:{dev}")
        keep = [t for t in (x, dbd, flags) if t is not None]
        if not cross:
            with torch.cuda.stream(s):
                sbd = torch.from_numpy(np.ascontiguousarray(res.blocks, dtype=np.int32)).to(f"cuda:{dev}")
            keep.append(sbd)
            split_migrate_fused(src_pool, dst_pool, sbd, dbd, plan, x, w, stream=s, table_row=row, rope_theta=rope)
        else:
            if plan.prefix_blocks:
                xs = self.ordered_stream(src_pool.device)
                xs.wait_stream(torch.cuda.current_stream(dev))   # the flag words / table row reset live there
                self._wait_fences(xs, src_pool.device, [dst_pool])
                m = _native.Move()
                m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src_pool.pool_id, dst_pool.pool_id, \
                    plan.prefix_blocks, 1
                sb = np.ascontiguousarray(res.blocks[:plan.prefix_blocks], dtype=np.int32)
                m.src_blocks, m.dst_blocks, m.done_flag = sb.ctypes.data, db_np.ctypes.data, flags.data_ptr()
                _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1,
                                                        _native.KVM_F_BLOCKS_ON_HOST | self.engine_flag,
                                                        ctypes.c_void_p(xs.cuda_stream)), "kvm_migrate(split prefix)")
            if plan.suffix:
                reprefill(dst_pool, x, w, dbd, tok0=prefix, stream=s, rope_theta=rope or None)
            if plan.prefix_blocks:
                _native.check(_native.lib().kvm_wait_flag(ctypes.c_void_p(flags.data_ptr()), 1,
                                                          ctypes.c_void_p(s.cuda_stream)), "kvm_wait_flag")
            if table is not None:
                with torch.cuda.stream(s):
                    table.rows[table.slot(rid), :len(db_np)].copy_(dbd)
        for t in keep:
            t.record_stream(s)
        rec.bytes_moved += plan.prefix_blocks * src_pool.shape.piece_bytes * 2 * src_pool.shape.layers
        rec.tokens_moved += plan.prefix_tokens
        rec.tokens_recomputed += plan.suffix
        rec.split_prefix_blocks[rid] = plan.prefix_blocks

    def _launch_migrate(self, dev: int, moves: List[_native.Move], dst_pools=()) -> None:
        """One fused kvm_migrate launch for every move leaving `dev` this slot.

        The kernel (on `dev`) also writes the destination devices' memory: the
        pools, the block-table rows (reset to -1 on slot reuse) and the layer
        flags (zeroed) — the latter two queued by this call on the destination
        devices' current streams.  So the launch stream waits on those streams
        and on the fences of every destination pool first."""
        import torch

        arr = (_native.Move * len(moves))(*moves)
        s = self.ordered_stream(dev)
        for d in sorted({p.device for p in dst_pools} - {dev}):
            s.wait_stream(torch.cuda.current_stream(d))
        self._wait_fences(s, dev, dst_pools)
        _native.check(_native.lib().kvm_migrate(arr, len(moves),
                                                _native.KVM_F_BLOCKS_ON_HOST | self.engine_flag,
                                                ctypes.c_void_p(s.cuda_stream)), "kvm_migrate")

    def _wait_fences(self, s, dev: int, pools) -> None:
        """Make stream `s` (on `dev`) wait for outstanding stream-ordered moves
        that READ blocks of `pools` and were issued on another device: their
        source blocks are already free on the host and may be handed out
        again to the write `s` is about to issue."""
        for p in pools:
            fences = self._fences.get(p.pool_id)
            if not fences:
                continue
            for d, ev in list(fences.items()):
                if ev.query():
                    del fences[d]
                elif d != dev:
                    s.wait_event(ev)

    def _fence(self, pool, dev: int, ev) -> None:
        self._fences.setdefault(pool.pool_id, {})[dev] = ev

    def _commit(self, post, keep_table: bool = False) -> None:
        for rid, dst, tokens, dst_blocks in post:
            old = self.loc[rid]
            self.pool(old.gpu, old.model).allocator.free(old.blocks)
            t = self._table(old.gpu, old.model)
            if t is not None and not keep_table:
                t.drop(rid)
            self.loc[rid] = Residency(dst, np.asarray(dst_blocks, dtype=np.int32), tokens, old.model)

    def _table(self, gpu: int, model: str) -> Optional[BlockTable]:
        return self.tables.get(gpu, {}).get(model or self.default_model)

    def _res(self, rid: int) -> Residency:
        try:
            return self.loc[rid]
        except KeyError:
            raise NotPlaced(f"request {rid} is not resident") from None

    def _table_set(self, gpu: int, model: str, rid: int, blocks: np.ndarray, start: int = 0) -> None:
        """Host mirror now; the device row entries [start, len) are batched with
        every other admission / growth and written at the table's next flush
        (before any kernel or reader uses the rows)."""
        t = self._table(gpu, model)
        if t is None:
            return
        t.stage(rid, blocks, start)


def _geometry(pool) -> tuple:
    sh = pool.shape
    return (sh.layers, sh.kv_heads, sh.head_dim, sh.block_tokens, sh.elem_bytes)


def _by_model(p) -> Dict[str, KVPool]:
    if isinstance(p, dict):
        for name, pool in p.items():
            if pool.shape.name != name:
                raise ConfigError(f"pool keyed {name!r} has shape {pool.shape.name!r}")
        return dict(p)
    return {p.shape.name: p}


def _as_i32_tensor(a: np.ndarray, device: int):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(f"cuda:{device}")
