#!/usr/bin/env python
"""KV-migration benchmark (BASELINE.json metric: KV migration GB/s & p50
latency vs NVLink/HBM roofline; bit-exact).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 7b-4k|13b-8k|70b-16k] [--engine ldg|bulk]

A step = one migration of one request's full paged KV cache (every layer, K
and V) on every rank.
  N = 1 : intra-GPU migration (compaction) of the request into fresh blocks of
          the same pool: HBM -> HBM, bound = HBM copy bandwidth.
  N > 1 : one process per GPU (torchrun), ring i -> (i+1) mod N; each rank
          pushes its request into the next rank's pool over NVLink (CUDA-IPC
          mapped peer memory, stores issued by the kernel), weak scaling.
`value` is payload GB/s (kv_bytes, sim.py:214 definition) over all ranks,
device-timed with CUDA events, max over ranks; the roofline object counts the
kernel's algorithmic traffic (read + write for HBM; bytes crossing the link
for NVLink).  `e2e` is the same metric through the public API with host block
lists (pinned staging + H2D inside the call) and a D2H read of the rewritten
destination block-table row every step.

--impl reference: the reference has no data path (it deletes executed moves,
sim.py:221-223), so its CPU implementation of the path is the oracle port
(oracle/kvmig_oracle.c, the C restatement) timed on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (shape name, tokens, BASELINE.json config it is quoted on)
    "7b-4k": ("llama2-7b", 4096, "configs[1]: Llama-2-7B KV, 4k-token request"),
    "13b-8k": ("llama2-13b", 8192, "configs[2] shape: Llama-2-13B KV, 8k tokens (full transfer)"),
    "70b-16k": ("llama3-70b-gqa", 16384, "configs[3]: Llama-3-70B GQA KV, 16k tokens"),
    "7b-512": ("llama2-7b", 512, "test size (contract tests only; not a BASELINE config)"),
}
NVLINK_PEAK_GBS = 900.0        # nominal per direction per GPU
NVLINK_MEASURED_GBS = 770.0    # B200_PROFILING.md: measured peer copy per direction


def _kernel_extras(device: int) -> dict:
    """Fresh measurements of the path's other kernels on the same box, reported
    beside the headline (not part of the timed region): K3 re-prefill on the
    CTA-pair tcgen05 kernel (configs[2]'s 13B suffix of 1 360 tokens, QKV, 40
    layers) and K5 paged decode over a 7B 4k-token cache (32 layers), each with
    its roofline fraction against MEASURED_PEAKS.json."""
    import torch

    from paper_2501_06709_b200.attention import paged_decode
    from paper_2501_06709_b200.kvcache import SHAPES, KVPool
    from paper_2501_06709_b200.reprefill import reprefill, reprefill_flops, synthetic_hidden, synthetic_weights

    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        tflops_peak, tsrc = float(pk["bf16_tflops_sustained"]), "measured (MEASURED_PEAKS.json bf16 sustained)"
        hbm_peak = float(pk["hbm_gbs"])
    except Exception:
        tflops_peak, tsrc, hbm_peak = 2250.0, "fallback (nominal dense bf16)", 6650.0
    st = torch.cuda.Stream(device=device)

    def timed(fn, reps=5, iters=3):
        st.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(st):
            for _ in range(2):
                fn()
            ms = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(iters):
                    fn()
                e1.record(st)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1) / iters)
        return statistics.median(ms)

    out = {}
    try:
        sh, rows = SHAPES["llama2-13b"], 1360
        nblk = (rows + 15) // 16
        pool = KVPool(sh, nblk + 4, device=device, dtype=torch.bfloat16)
        blocks = torch.arange(nblk, dtype=torch.int32, device=f"cuda:{device}")
        x, w = synthetic_hidden(sh, rows, device), synthetic_weights(sh, device, with_q=True)
        ms = timed(lambda: reprefill(pool, x, w, blocks, stream=st))
        tf = reprefill_flops(sh, rows, with_q=True) / ms / 1e9
        out["reprefill_13b_s1360"] = {"kernel": "reprefill_pair_kernel (tcgen05 cta_group::2)", "ms": round(ms, 4),
                                      "achieved": round(tf, 1), "peak": tflops_peak, "unit": "TFLOP/s",
                                      "frac": round(tf / tflops_peak, 4), "peak_source": tsrc}
        del pool, x, w
    except Exception as e:  # reported, never fatal for the headline
        out["reprefill_13b_s1360"] = {"error": str(e)[:300]}
    try:
        sh, seq = SHAPES["llama2-7b"], 4096
        nblk = seq // 16
        pool = KVPool(sh, nblk + 8, device=device)
        pool.tensor.normal_()
        g = torch.Generator().manual_seed(0)
        table = torch.randperm(nblk + 8, generator=g)[:nblk].to(torch.int32).view(1, nblk).to(f"cuda:{device}")
        lens = torch.full((1,), seq, dtype=torch.int32, device=f"cuda:{device}")
        q = torch.randn(sh.layers, 1, sh.q_heads, 128, device=f"cuda:{device}").half()
        o = torch.empty_like(q)
        ms = timed(lambda: paged_decode(pool, q, table, lens, o, max_seq_len=seq, stream=st), iters=10)
        gbs = 2 * seq * sh.kv_heads * 128 * 2 * sh.layers / ms / 1e6
        out["decode_7b_4k_32l"] = {"kernel": "decode_gqa_kernel (mma.sync)", "ms": round(ms, 4),
                                   "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                                   "frac": round(gbs / hbm_peak, 4),
                                   "note": "read-only stream vs the read+write copy peak"}
        del pool, q, o
    except Exception as e:
        out["decode_7b_4k_32l"] = {"error": str(e)[:300]}
    try:   # live-migration tail: one 7B block (8 MiB) with host block lists, table row + done flag
        import ctypes

        import numpy as np

        from paper_2501_06709_b200 import _native
        from paper_2501_06709_b200.kvcache import BlockTable

        sh = SHAPES["llama2-7b"]
        src, dst = KVPool(sh, 4, device=device), KVPool(sh, 4, device=device)
        table = BlockTable(1, 4, device=device)
        flag = torch.zeros(1, dtype=torch.int32, device=f"cuda:{device}")
        sb, db = np.array([1], dtype=np.int32), np.array([2], dtype=np.int32)
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, 1, 1
        m.src_blocks, m.dst_blocks, m.dst_table_row, m.done_flag = sb.ctypes.data, db.ctypes.data, \
            table.row_ptr(0), flag.data_ptr()
        sp = ctypes.c_void_p(st.cuda_stream)
        lib = _native.lib()
        fl = _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK
        lat = []
        for r in range(60):
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _native.check(lib.kvm_migrate(ctypes.byref(m), 1, fl, sp))
            e1.record(st)
            e1.synchronize()
            if r >= 10:
                lat.append(e0.elapsed_time(e1) * 1e3)
        out["small_move_7b_1block"] = {"kernel": "migrate_bulk_kernel (one-move, 2-stage)",
                                       "issue_to_landed_us_p50": round(statistics.median(lat), 2),
                                       "bytes": sh.kv_bytes_per_token * 16,
                                       "definition": "event before the kvm_migrate call -> event after it, stream "
                                                     "idle: host issue (host block lists, table row, done flag) "
                                                     "+ kernel"}
        del src, dst
    except Exception as e:
        out["small_move_7b_1block"] = {"error": str(e)[:300]}
    torch.cuda.empty_cache()
    return out


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.BITS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _traffic_for(kernel: str, workload: str, engine: str):
    """dram read+write bytes per launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d[f"{workload}/{engine}"]["dram_bytes_per_launch"]
    except Exception:
        return None


# ----------------------------------------------------------------------------------
# CPU baseline (oracle port) — only here and in --impl reference
# ----------------------------------------------------------------------------------
def _cpu_setup(shape, tokens, seed=0):
    import numpy as np

    from oracle import kvmig_oracle as orc

    orc.lib()
    n = tokens // shape.block_tokens
    nb = 3 * n
    rng = np.random.default_rng(seed)
    # content is irrelevant to a byte copy's speed: a memset touches every page (no first-touch
    # faults inside the timed copies) far faster than generating random bits
    pool = np.full((shape.layers, 2, nb, shape.block_tokens, shape.kv_heads, shape.head_dim), 0x3C01,
                   dtype=np.int16)
    src = rng.permutation(nb)[:n].astype(np.int32)
    free = np.ones(nb, dtype=np.uint8)
    free[src] = 0
    rest = np.flatnonzero(free)
    free[rng.permutation(rest)[: len(rest) // 2]] = 0
    dst = orc.alloc_ascending(free, n)
    d = orc.desc(shape.layers, shape.kv_heads, shape.head_dim, shape.block_tokens, nb)
    return pool, d, src, dst


def cpu_migrate_rate(shape, tokens, threads, budget_s=6.0, min_reps=2, max_reps=None):
    """Time the oracle port migrating the request inside a host pool."""
    from oracle import kvmig_oracle as orc

    pool, d, src, dst = _cpu_setup(shape, tokens)
    kv_bytes = tokens * shape.kv_bytes_per_token
    orc.migrate(pool, d, pool, d, src, dst, threads=threads)  # warm (page-in)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < min_reps or (time.perf_counter() < t_end and (max_reps is None or len(times) < max_reps)):
        t0 = time.perf_counter()
        orc.migrate(pool, d, pool, d, src, dst, threads=threads)
        times.append(time.perf_counter() - t0)
        src, dst = dst, src
    return kv_bytes, times


def run_reference(args) -> int:
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    from paper_2501_06709_b200.kvcache import SHAPES

    shape_name, tokens, cfg_desc = WORKLOADS[args.workload]
    shape = SHAPES[shape_name]
    threads = os.cpu_count() or 1
    kv_bytes, _ = cpu_migrate_rate(shape, tokens, threads, budget_s=0.0, min_reps=max(args.warmup, 1),
                                   max_reps=max(args.warmup, 1))
    kv_bytes, times = cpu_migrate_rate(shape, tokens, threads, budget_s=0.0, min_reps=args.steps,
                                       max_reps=args.steps)
    total = sum(times)
    value = kv_bytes * len(times) / total / 1e9
    sample = (f"{len(times)} full {args.workload} migrations ({kv_bytes} B each) inside one host pool, "
              f"oracle C port, {threads} pthreads")
    line = {
        "impl": "reference", "metric": "kv_migration_GBps", "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp16 bytes", "data": "synthetic",
        "config": {"workload": f"{args.workload} CPU reference path (oracle port)", "baseline_config": cfg_desc,
                   "kv_bytes_per_step": kv_bytes},
        "latency_ms": {"p50": round(1e3 * statistics.median(times), 3),
                       "p99": round(1e3 * sorted(times)[max(0, int(0.99 * len(times)) - 1)], 3)},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference kvpack moves no bytes (sim.py:221-223); its CPU path is the oracle port",
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------
def _fill_random(t, seed):
    import torch

    g = torch.Generator(device=t.device).manual_seed(seed)
    v = t.view(torch.int16).view(-1)
    step = 1 << 28
    for i in range(0, v.numel(), step):
        n = min(step, v.numel() - i)
        v[i:i + n] = torch.randint(-2 ** 15, 2 ** 15, (n,), generator=g, device=t.device, dtype=torch.int16)


def _layout(shape, tokens, seed):
    """Recipe of SURVEY.md §8d: src table = first n of randperm(NB) (seed), dst
    pre-occupied at 50% so the free blocks it receives are scattered."""
    import numpy as np
    import torch

    n = tokens // shape.block_tokens
    nb = 4 * n
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(seed))[:n].to(torch.int32).numpy()
    rng = np.random.default_rng(seed + 100)
    used = np.zeros(nb, dtype=bool)
    used[sb] = True
    rest = np.flatnonzero(~used)
    used[rng.permutation(rest)[: len(rest) // 2]] = True
    return n, nb, sb, used


def run_ours(args) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.dist import allreduce_max, exchange_objects, rank_info_from_env
    from paper_2501_06709_b200.executor import ENGINES, MigrationExecutor, Residency
    from paper_2501_06709_b200.kvcache import SHAPES, BlockTable, KVPool

    ri = rank_info_from_env()
    world = ri.world
    ndev = torch.cuda.device_count()
    shared_gpu = world > 1 and ndev < world
    device = ri.local_rank % max(ndev, 1)
    torch.cuda.set_device(device)
    if world > 1:
        backend = "nccl" if ndev >= world else "gloo"   # gloo: N ranks sharing one GPU (test mode)
        dist.init_process_group(backend=backend, device_id=torch.device(f"cuda:{device}")
                                if backend == "nccl" else None)
    shape_name, tokens, cfg_desc = WORKLOADS[args.workload]
    shape = SHAPES[shape_name]
    kv_bytes = tokens * shape.kv_bytes_per_token
    n, nb, sb_np, used = _layout(shape, tokens, seed=1 + ri.rank)
    eng = ENGINES[args.engine] | (_native.KVM_F_L2_EVICT_FIRST if args.l2_evict_first else 0)
    lib = _native.lib()

    pool = KVPool(shape, nb, device=device)
    _fill_random(pool.tensor, 1234 + ri.rank)
    pool.allocator.take(np.flatnonzero(used))
    db_np = pool.allocator.alloc(n)          # blocks this rank RECEIVES into
    table = BlockTable(4, n, device=device)
    # one control allocation per rank, exported once: [0, 64) done flags, [64, 64 + n) the block-table
    # row the incoming transfer rewrites (N > 1)
    ctrl = torch.zeros(64 + n, dtype=torch.int32, device=f"cuda:{device}")
    mailbox, rowbuf = ctrl[:64], ctrl[64:]
    stream = torch.cuda.Stream(device=device)
    sptr = ctypes.c_void_p(stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- peers ----------------
    if world > 1:
        h_pool, o_pool = pool.ipc_handle()
        from paper_2501_06709_b200 import kvcache as kvc
        hb = (ctypes.c_ubyte * 64)()
        ob = ctypes.c_int64()
        _native.check(lib.kvm_ipc_export(ctypes.c_void_p(ctrl.data_ptr()), hb, ctypes.byref(ob)))
        info = exchange_objects((h_pool, o_pool, bytes(hb), ob.value, db_np.tolist()))
        peer = info[ri.send_to]
        dst_pool = kvc.KVPool.from_ipc(shape, nb, device, peer[0], peer[1])
        mb = ctypes.c_void_p()
        _native.check(lib.kvm_ipc_import(device, (ctypes.c_ubyte * 64).from_buffer_copy(peer[2]), peer[3],
                                         ctypes.byref(mb)))
        peer_flag, peer_row = mb.value, mb.value + 64 * 4
        peer_db = np.asarray(peer[4], dtype=np.int32)
    else:
        dst_pool, peer_flag, peer_row, peer_db = pool, mailbox.data_ptr(), table.row_ptr(0), db_np

    sb_dev = torch.from_numpy(sb_np).to(f"cuda:{device}")
    db_dev = torch.from_numpy(peer_db).to(f"cuda:{device}")
    seq = [0]

    def make_move(host: bool, fwd: bool):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks = pool.pool_id, dst_pool.pool_id, n
        if world == 1 and not fwd:       # compaction ping-pong: back into the original blocks
            m.src_blocks = (db_np.ctypes.data if host else db_dev.data_ptr())
            m.dst_blocks = (sb_np.ctypes.data if host else sb_dev.data_ptr())
        else:
            m.src_blocks = (sb_np.ctypes.data if host else sb_dev.data_ptr())
            m.dst_blocks = (peer_db.ctypes.data if host else db_dev.data_ptr())
        m.dst_table_row = peer_row
        m.done_flag = peer_flag
        seq[0] += 1
        m.done_value = seq[0]
        return m

    def step(i, host: bool):
        m = make_move(host, fwd=(i % 2 == 0))
        _native.check(lib.kvm_migrate(ctypes.byref(m), 1, eng | (_native.KVM_F_BLOCKS_ON_HOST if host else 0),
                                      sptr))
        if world > 1 and shared_gpu:
            # test mode, several ranks on ONE GPU: a device-side spin on the incoming flag can starve
            # the peer process's context (no time-slicing of a running kernel was observed), so the
            # receive completes on the host: own push done, then every rank has pushed.
            stream.synchronize()
            barrier()
        elif world > 1:   # wait for the incoming transfer from recv_from (dst-visible completion);
            # bounded (30 s) so a lost peer write fails the run instead of wedging the GPU
            _native.check(lib.kvm_wait_flag_timeout(ctypes.c_void_p(mailbox.data_ptr()), seq[0],
                                                    30_000_000_000, ctypes.c_void_p(mailbox.data_ptr() + 4 * 63),
                                                    sptr))

    # ---------------- correctness gate (bit-exact) before timing ----------------
    def gathered_checksum(blocks_np):
        idx = torch.from_numpy(blocks_np).long().to(pool.tensor.device)
        w = torch.arange(1, shape.piece_bytes // 2 + 1, device=idx.device, dtype=torch.int64)
        acc = torch.zeros((), dtype=torch.int64, device=idx.device)
        for l in range(shape.layers):
            g = pool.tensor[l][:, idx].reshape(2, n, -1).view(torch.int16).to(torch.int64)
            acc += (g * w).sum() + (g.sum(-1) * torch.arange(1, n + 1, device=idx.device)).sum()
        return int(acc.item())

    sent = gathered_checksum(sb_np)
    # every rank's pool (and the blocks it receives into) is initialised before any peer pushes into it
    torch.cuda.synchronize()
    barrier()
    with torch.cuda.stream(stream):
        step(0, host=False)
    stream.synchronize()
    barrier()
    got = gathered_checksum(db_np)
    if world == 1:
        ok = got == sent
    else:   # what this rank received must equal what recv_from sent
        sums = exchange_objects(sent)
        ok = got == sums[ri.recv_from] and bool(torch.equal(rowbuf.cpu(), torch.from_numpy(db_np)))
    if world > 1 and int(mailbox[63].item()) != 0:
        raise RuntimeError(f"rank {ri.rank}: incoming transfer from rank {ri.recv_from} timed out")
    if not ok:
        print(f"rank {ri.rank}: parity gate failed: received checksum {got}, sent "
              f"{sums[ri.recv_from] if world > 1 else sent}, table row ok "
              f"{bool(torch.equal(rowbuf.cpu(), torch.from_numpy(db_np))) if world > 1 else None}",
              file=sys.stderr)
    bit_exact = allreduce_max(0.0 if ok else 1.0, device) == 0.0
    seq[0] = 0
    mailbox.zero_()
    torch.cuda.synchronize()
    barrier()

    # ---------------- warmup ----------------
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i, host=False)
    stream.synchronize()
    barrier()

    # ---------------- timed: device-resident ----------------
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(device) as clk:
        with torch.cuda.stream(stream):
            t_start.record(stream)
            for i in range(K):
                ev[i][0].record(stream)
                step(args.warmup + i, host=False)
                ev[i][1].record(stream)
            t_end.record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
    barrier()
    launches = _native.launch_count() - launches0
    elapsed_ms = allreduce_max(t_start.elapsed_time(t_end), device)
    per = sorted(a.elapsed_time(b) for a, b in ev)
    avg_launch_ms = sum(per) / len(per)
    p50 = statistics.median(per)
    p99 = per[max(0, int(round(0.99 * len(per))) - 1)]
    p50 = allreduce_max(p50, device)
    p99 = allreduce_max(p99, device)
    avg_launch_ms = allreduce_max(avg_launch_ms, device)
    value = world * kv_bytes * K / (elapsed_ms / 1e3) / 1e9

    # ---------------- timed: e2e through the public API ----------------
    h2d = d2h = 0
    if world == 1:
        ex = MigrationExecutor({0: pool}, {0: table}, engine=args.engine)
        pool.allocator.free(db_np)   # the request is resident in sb; db is free again
        ex.loc[0] = Residency(0, sb_np.copy(), tokens, pool.shape.name)
        table.set_host(0, sb_np)
        # make device bytes consistent with the residency (content is irrelevant to timing)
        rows = [torch.empty(n, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        for i in range(args.warmup):
            ex.compact(0, row_out=rows[0])
        torch.cuda.synchronize()
        e2e_lat = []
        # every step: host block lists -> H2D -> kernel -> D2H of the rewritten block-table row,
        # and the host waits for that row; the call is stream-ordered, so the host prepares step
        # i+1 while the GPU still copies step i (double-buffered pinned rows)
        t0 = time.perf_counter()
        prev = None
        e2e_ok = True
        for i in range(K):
            ts = time.perf_counter()
            rec = ex.compact(0, row_out=rows[i & 1], stream_ordered=True)
            if prev is not None:
                prev[0].done.synchronize()
                e2e_lat.append(time.perf_counter() - prev[1])
                e2e_ok &= bool(np.array_equal(rows[(i - 1) & 1].numpy(), prev[2]))
            prev = (rec, ts, ex.where(0).blocks.copy())
        prev[0].done.synchronize()
        e2e_lat.append(time.perf_counter() - prev[1])
        e2e_s = time.perf_counter() - t0
        torch.cuda.synchronize()
        h2d, d2h = 2 * n * 4, n * 4
        assert e2e_ok and np.array_equal(rows[(K - 1) & 1].numpy(), ex.where(0).blocks)
        # per-call latency of one synchronous call (issue -> row on the host), not pipelined
        e2e_lat = []
        for i in range(min(K, 30)):
            ts = time.perf_counter()
            ex.compact(0, row_out=rows[0])
            e2e_lat.append(time.perf_counter() - ts)
    else:
        row = torch.empty(n, dtype=torch.int32, pin_memory=True)
        torch.cuda.synchronize()
        barrier()
        e2e_lat = []
        t0 = time.perf_counter()
        for i in range(K):
            ts = time.perf_counter()
            with torch.cuda.stream(stream):
                step(i, host=True)
                # D2H of the block-table row the incoming kernel rewrote, ordered after the wait
                row.copy_(rowbuf[:n], non_blocking=True)
            stream.synchronize()
            e2e_lat.append(time.perf_counter() - ts)
        torch.cuda.synchronize()
        e2e_s = allreduce_max(time.perf_counter() - t0, device)
        barrier()
        h2d, d2h = 2 * n * 4, n * 4
    e2e = world * kv_bytes * K / e2e_s / 1e9

    # ---------------- roofline ----------------
    hbm_peak, hbm_src = _peaks()
    if world == 1:
        alg_bytes = 2 * kv_bytes  # read + write, same HBM
        roof = {"bound": "hbm", "achieved": round(alg_bytes / (avg_launch_ms / 1e3) / 1e9, 1),
                "peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src,
                "kernel": "migrate_ldg_kernel" if args.engine == "ldg" else "migrate_bulk_kernel",
                "algorithmic_bytes_per_launch": alg_bytes,
                "traffic": _traffic_for("migrate", args.workload, args.engine)}
    elif ndev < world:
        # test mode: ranks share one GPU, so the "peer" stores stay in local HBM
        alg_bytes = 2 * kv_bytes
        roof = {"bound": "hbm", "achieved": round(alg_bytes / (avg_launch_ms / 1e3) / 1e9, 1),
                "peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src,
                "kernel": "migrate_ldg_kernel" if args.engine == "ldg" else "migrate_bulk_kernel",
                "algorithmic_bytes_per_launch": alg_bytes, "traffic": None,
                "note": f"{world} ranks share {ndev} GPU(s): IPC path exercised without NVLink"}
    else:
        alg_bytes = kv_bytes  # bytes crossing this GPU's NVLink egress per launch
        roof = {"bound": "nvlink", "achieved": round(alg_bytes / (avg_launch_ms / 1e3) / 1e9, 1),
                "peak": NVLINK_MEASURED_GBS, "unit": "GB/s",
                "peak_source": "B200_PROFILING.md measured peer copy per direction (nominal 900)",
                "kernel": "migrate_ldg_kernel" if args.engine == "ldg" else "migrate_bulk_kernel",
                "algorithmic_bytes_per_launch": alg_bytes, "traffic": None}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)

    line = None
    if ri.rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            cb, times = cpu_migrate_rate(shape, tokens, threads, budget_s=args.cpu_budget_s)
            cpu = {"value": round(cb * len(times) / sum(times) / 1e9, 3), "unit": "GB/s", "cores": threads,
                   "kind": "port",
                   "sample": f"{len(times)} x {args.workload} migrations ({cb} B each, same workload) inside "
                             f"one host pool, oracle C port (oracle/kvmig_oracle.c), {threads} pthreads, "
                             f"~{args.cpu_budget_s:.0f} s budget"}
        line = {
            "metric": "kv_migration_GBps", "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(elapsed_ms / K, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16 bytes (u16 copy)",
            "data": "synthetic (seeded random KV bits, NaN payloads included)",
            "config": {"workload": (f"{args.workload} intra-GPU migration (compaction into fresh blocks of the "
                                    f"same pool)" if world == 1 else
                                    (f"{args.workload} ring push i->(i+1) mod {world} over NVLink (CUDA IPC)"
                                     if ndev >= world else
                                     f"{args.workload} ring push i->(i+1) mod {world}, ranks sharing "
                                     f"{ndev} GPU (CUDA IPC test mode, no NVLink hop)")),
                       "baseline_config": cfg_desc, "kv_bytes_per_rank_per_step": kv_bytes, "blocks": n,
                       "pool_blocks": nb, "engine": args.engine, "l2_evict_first": bool(args.l2_evict_first),
                       "l2": "inputs larger than L2 (%.1f GiB per step per rank)" % (kv_bytes / 2 ** 30),
                       "parallelism": f"{world} ranks, one process per GPU" if world > 1 else "1 GPU"},
            "latency_ms": {"p50": round(p50, 4), "p99": round(p99, 4),
                           "definition": "kernel launch -> done flag on dst stream (CUDA events)"},
            "bit_exact": bool(bit_exact),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "latency_ms_p50": round(1e3 * statistics.median(e2e_lat), 4),
                    "latency_definition": "one synchronous call through the API: issue -> result row on the host",
                    "path": "MigrationExecutor.compact(stream_ordered) -> kvm_compact(host block lists) -> "
                            "table row D2H -> host waits for the row (next step issued meanwhile)"
                    if world == 1 else "kvm_migrate(host block lists) -> kvm_wait_flag -> table row D2H"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_extras:
            line["kernels"] = _kernel_extras(device)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="7b-4k")
    ap.add_argument("--engine", choices=["ldg", "bulk"], default=None,
                    help="copy engine; default bulk (TMA) for local HBM at N=1, ldg (128-bit peer "
                         "stores, the proven NVLink pattern) for N>1")
    ap.add_argument("--l2-evict-first", type=int, choices=[0, 1], default=0,
                    help="stream KV through L2 with an evict-first policy (KVM_F_L2_EVICT_FIRST)")
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the re-prefill / decode measurements reported beside the headline")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    if args.engine is None:
        args.engine = "bulk" if int(os.environ.get("WORLD_SIZE", args.gpus)) == 1 else "ldg"
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
