#!/usr/bin/env python
"""KV-migration benchmark (BASELINE.json metric: KV migration GB/s & p50
latency vs NVLink/HBM roofline; bit-exact).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 7b-4k|13b-8k|70b-16k] [--engine ldg|bulk]

A step = one migration of one request's full paged KV cache (every layer, K
and V) on every rank.
  N = 1 : intra-GPU migration (compaction) of the request into fresh blocks of
          the same pool: HBM -> HBM, bound = HBM copy bandwidth.
  N > 1 : one process per GPU, ring i -> (i+1) mod N; each rank pushes its
          request into the next rank's pool over NVLink (CUDA-IPC mapped peer
          memory, stores issued by the kernel; dist.PeerLink), weak scaling.
          Launched by torchrun, or — when WORLD_SIZE is unset — bench.py
          re-launches itself under torch.distributed.run with N ranks, so a
          plain `python bench.py --gpus N` measures N GPUs.  N larger than
          the visible GPU count is an error unless --shared-gpu (test mode:
          ranks share one GPU, no NVLink hop, labelled as such).
`value` is payload GB/s (kv_bytes, sim.py:214 definition) over all ranks,
device-timed with CUDA events, max over ranks; the roofline object counts the
kernel's algorithmic traffic (read + write for HBM; bytes leaving the GPU for
NVLink) and, at N > 1, the NVLink bytes NVML saw cross the ports.  `e2e` is
the same metric through the public API with host block lists (pinned staging
+ H2D inside the call) and a D2H read of the rewritten destination block-table
row every step.  At N > 1 the same ring done the library way (NCCL
batch_isend_irecv of the gathered request) is timed in the same run
(`library`), and the 70B-GQA 16k-token ring (configs[3]) is measured beside
the headline (`extra_workloads`), with the push on 32 / 64 SMs
(`config.push_sm_budget_ab`) and, on rank 0, GPU 0 -> 1 split and
time-to-first-decode extras.  At N = 1 the line's `kernels` object adds the
re-prefill (vs cuBLAS, with energy per launch), decode, the configs[2] split,
the one-block move latency, the push over PCIe to pinned host memory, decode
beside a migration / re-prefill, and the copy SM-budget sweep.

--impl reference: the reference has no data path (it deletes executed moves,
sim.py:221-223), so its CPU implementation of the path is the oracle port
(oracle/kvmig_oracle.c, the C restatement) timed on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import datetime
import json
import os
import platform
import random
import socket
import statistics
import subprocess
import sys
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
WAIT_NS = 5_000_000_000        # bound on one receive wait in the ring (a 5 GB push takes ~7 ms over NVLink)
NVLINK_MEASURED_GBS = 770.0    # B200_PROFILING.md: measured peer copy per direction


def _peaks():
    """(hbm GB/s, bf16 burst TF/s, bf16 sustained TF/s, source)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return (float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d["bf16_tflops_sustained"]),
                "measured (MEASURED_PEAKS.json)")
    except Exception:
        return 6650.0, 2250.0, 2250.0, "fallback (B200_PROFILING.md / nominal dense bf16)"


def _kernel_extras(device: int) -> dict:
    """Fresh measurements of the path's other kernels on the same box, reported
    beside the headline (not part of the timed region): K3 re-prefill on the
    CTA-pair tcgen05 kernel (configs[2]'s 13B suffix of 1 360 tokens, QKV, 40
    layers) against the burst bf16 peak (a ~6 ms launch timed alone) with
    cuBLAS on the same shape in the same session; K5 paged decode over a 7B
    4k-token cache (32 layers); and the one-block move latency."""
    import torch

    from paper_2501_06709_b200.attention import paged_decode
    from paper_2501_06709_b200.kvcache import SHAPES, KVPool
    from paper_2501_06709_b200.reprefill import reprefill, reprefill_flops, synthetic_hidden, synthetic_weights

    hbm_peak, burst, sustained, psrc = _peaks()
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
    # the latency-bound small move first, before the ms-long power-capped GEMMs below lower the clocks
    try:   # live-migration tail: one 7B block (8 MiB) with host block lists, table row + done flag
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
                                       "definition": "the one small-move latency this repo quotes: CUDA event "
                                                     "recorded on the idle stream right before the kvm_migrate "
                                                     "call -> event right after it; covers host issue (host "
                                                     "block lists, table row, done flag) + kernel"}
        del src, dst
    except Exception as e:
        out["small_move_7b_1block"] = {"error": str(e)[:300]}
    try:
        sh, rows = SHAPES["llama2-13b"], 1360
        nblk = (rows + 15) // 16
        pool = KVPool(sh, nblk + 4, device=device, dtype=torch.bfloat16)
        blocks = torch.arange(nblk, dtype=torch.int32, device=f"cuda:{device}")
        x, w = synthetic_hidden(sh, rows, device), synthetic_weights(sh, device, with_q=True)
        flops = reprefill_flops(sh, rows, with_q=True)
        outs = torch.empty(rows, w.shape[1], dtype=torch.bfloat16, device=f"cuda:{device}")

        def cublas():
            for l in range(sh.layers):
                torch.matmul(x, w[l].t(), out=outs)

        # interleaved rounds: both arms see the same power / thermal state
        ours_ms, lib_ms = [], []
        for _ in range(3):
            ours_ms.append(timed(lambda: reprefill(pool, x, w, blocks, stream=st), reps=3))
            lib_ms.append(timed(cublas, reps=3))
        ms, lms = statistics.median(ours_ms), statistics.median(lib_ms)
        tf, ltf = flops / ms / 1e9, flops / lms / 1e9
        # power roofline: board energy per launch (NVML counter) over ~1 s of back-to-back launches of
        # each arm; at the board limit, time = energy per launch / limit (tools/power_roofline.py)
        power = None
        try:
            from paper_2501_06709_b200.telemetry import ClockSampler, EnergyMeter

            em = EnergyMeter(device)
            if em.error is None:
                power = {"limit_w": em.limit_w}
                for name, fn, t in (("ours", lambda: reprefill(pool, x, w, blocks, stream=st), ms),
                                    ("cublas", cublas, lms)):
                    with torch.cuda.stream(st), ClockSampler(device) as clk:
                        r = em.measure(fn, max(5, int(1000 / t)), st.synchronize)
                    if "joules_per_call" in r:
                        r["tflop_per_joule"] = round(flops / 1e12 / r["joules_per_call"], 3)
                        r["cap_bound_ms"] = round(r["joules_per_call"] / em.limit_w * 1e3, 4)
                    r["sm_mhz"] = clk.summary()["sm_mhz"]
                    power[name] = r
                if "tflop_per_joule" in power["ours"] and "tflop_per_joule" in power["cublas"]:
                    power["ours_over_cublas_energy_eff"] = round(power["ours"]["tflop_per_joule"] /
                                                                 power["cublas"]["tflop_per_joule"], 4)
                power["definition"] = ("NVML board energy per launch over ~1 s of back-to-back launches; "
                                       "cap_bound_ms = joules per launch / enforced power limit: the "
                                       "shortest time at that energy per launch")
            else:
                power = {"error": em.error}
        except Exception as e:
            power = {"error": repr(e)[:200]}
        out["reprefill_13b_s1360"] = {
            "kernel": "reprefill_pair_kernel (tcgen05 cta_group::2)", "ms": round(ms, 4),
            "achieved": round(tf, 1), "peak": burst, "unit": "TFLOP/s", "frac": round(tf / burst, 4),
            "peak_source": psrc + " bf16 burst (kernel timed alone)",
            "frac_vs_sustained": round(tf / sustained, 4),
            "cublas_same_shape": {"impl": "torch.matmul per layer (cuBLAS), GEMM only, no K/V scatter",
                                  "ms": round(lms, 4), "achieved": round(ltf, 1),
                                  "frac": round(ltf / burst, 4), "ours_over_cublas": round(lms / ms, 4)},
            "power": power}
        del pool, x, w, outs
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
                                   "frac_of_nominal_7700": round(gbs / 7700.0, 4),
                                   "note": "read-only stream vs the read+write copy peak; torch's own read-only "
                                           "reductions reach 5.9-6.8 TB/s on this GPU, so the nominal 7.7 TB/s "
                                           "(B200_PROFILING.md) is the read ceiling quoted beside it"}
        del pool, q, o
    except Exception as e:
        out["decode_7b_4k_32l"] = {"error": str(e)[:300]}
    try:   # configs[2]: 13B 8k adaptive split on this GPU (fused kernel, two kernels, full transfer)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from bench_split import run_split_bench

        out["split_13b_8k"] = run_split_bench(iters=5, warmup=3, src_dev=device, dst_dev=device)
        out["split_13b_8k"]["kernel"] = "kvm_split_migrate (reprefill_pair_kernel<kCopy>) / kvm_migrate + kvm_reprefill"
        torch.cuda.empty_cache()
    except Exception as e:
        out["split_13b_8k"] = {"error": repr(e)[:300]}
    torch.cuda.empty_cache()
    # the push over a remote link this box has: PCIe to / from pinned host memory (system-scope completion,
    # as for a peer pool) vs the link's contiguous-copy roofline and vLLM swap_blocks (child process)
    if device == 0:
        out["remote_link_pcie"] = _tool_json("bench_host_link.py", ["--iters", "5"], timeout_s=300)
        # decode of resident requests beside an incoming migration / a re-prefill on every SM / on an SM budget
        out["decode_interference"] = _tool_json("bench_interference.py", ["--steps", "30"], timeout_s=300)
        # copy throughput against the SM budget (KVM_F_MAX_SMS): per-SM rate, SMs to saturate HBM / PCIe
        out["copy_sm_budget"] = _tool_json("bench_copy_sms.py", [], timeout_s=300)
    return out


def _traffic_for(workload: str, engine: str):
    """dram read+write bytes per launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d[f"{workload}/{engine}"]["dram_bytes_per_launch"]
    except Exception:
        return None


# ----------------------------------------------------------------------------------
# CPU baselines — only here and in --impl reference (the checker and the
# reference itself are never on the measured GPU path)
# ----------------------------------------------------------------------------------
def _cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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


def _reference_kvpack():
    """The reference package for the control-plane baseline: baseline/_ref
    (pip-installed from /root/reference, travels to the GPU box), else the
    read-only source tree when mounted; None when neither exists."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "kvpack")):
            if p not in sys.path:
                sys.path.append(p)
            try:
                import kvpack

                return kvpack, p
            except Exception:
                return None, None
    return None, None


def control_plane_baseline(budget_s: float = 8.0) -> dict:
    """BASELINE.md CPU baseline 1: the reference's control plane (kvpack
    plan_hybrid, migration.py:137-170, and MellScheduler.step_epoch,
    scheduler.py:979-1007) timed on ONE core beside this repo's native
    planner / scheduler on the same inputs; decisions checked identical."""
    kp, where = _reference_kvpack()
    out = {"cores": 1}
    if kp is None:
        out["reference"] = "unavailable (baseline/_ref not installed and /root/reference not mounted)"
    else:
        out["reference"] = f"kvpack from {os.path.relpath(where, ROOT) if where.startswith(ROOT) else where}"
    from paper_2501_06709_b200 import cluster as ocl
    from paper_2501_06709_b200 import scheduler as osch
    from paper_2501_06709_b200.planner import PendingMove, Topology, load_boundaries, plan_hybrid, plan_hybrid_native
    from paper_2501_06709_b200.runtime import run_slots
    from paper_2501_06709_b200.workload import LengthDistribution, gen_poisson

    old_aff = None
    try:
        old_aff = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {sorted(old_aff)[0]})   # this thread only: one core
    except Exception:
        pass
    t_stop = time.perf_counter() + budget_s
    try:
        rng = random.Random(0)
        topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9)
        bounds = load_boundaries(topo, 0.05, 0.2)
        plans = {}
        for n in (8, 64, 1024):
            moves = [PendingMove(i, rng.randrange(16), rng.randrange(16), rng.randint(1, 4 * 10 ** 9),
                                 rng.randint(1, 8000)) for i in range(n)]
            defer = {i: rng.randint(0, 4) for i in range(0, n, 3)}
            reps = max(3, 400 // n)
            from paper_2501_06709_b200 import planner as _pl

            plan_hybrid_native(moves, bounds, topo, defer)   # warm (buffers sized)
            sc = _pl._scratch
            arms = {"ours_us": lambda: plan_hybrid(moves, bounds, topo, defer),           # the drop-in API
                    "ours_native_us": lambda: plan_hybrid_native(moves, bounds, topo, defer),
                    # the C ABI call alone on the marshalled buffers (what a C/C++ host pays)
                    "ours_c_abi_call_us": lambda: sc.fn(sc.a_arr, n, sc.pp_addr, sc.a_out, sc.led_addr)}
            if kp is not None:
                rtopo = kp.Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9)
                rb = kp.load_boundaries(rtopo, 0.05, 0.2)
                rmoves = [kp.PendingMove(m.item, m.src, m.dst, m.kv_bytes, m.tokens) for m in moves]
                arms["reference_us"] = lambda: kp.plan_hybrid(rmoves, rb, rtopo, defer)
            # interleaved trials, best of 9 per arm: host timing noise hits every arm alike
            best = {k: float("inf") for k in arms}
            for _ in range(9):
                for k, fn in arms.items():
                    t0 = time.perf_counter()
                    for _ in range(reps):
                        fn()
                    best[k] = min(best[k], (time.perf_counter() - t0) / reps * 1e6)
            row = {k: round(v, 2) for k, v in best.items()}
            row["timing"] = f"best of 9 interleaved trials of {reps} calls"
            if kp is not None:
                ours, ref = plan_hybrid(moves, bounds, topo, defer), kp.plan_hybrid(rmoves, rb, rtopo, defer)
                row["identical"] = [(a.move.item, a.mode, a.latency_s) for a in ours.assignments] == \
                    [(a.move.item, a.mode, a.latency_s) for a in ref.assignments]
            plans[n] = row
        out["plan_hybrid"] = plans

        class Timed:
            def __init__(self, inner):
                self.inner, self.times = inner, []

            def step_epoch(self, *a, **k):
                t = time.perf_counter()
                r = self.inner.step_epoch(*a, **k)
                self.times.append(time.perf_counter() - t)
                return r

        # SURVEY.md §8c B200-shaped 7B run: C = 48 GiB, 8 GPUs/machine, 900e9 B/s, lambda 0.5, scale 10
        trace = gen_poisson(0.5, 200, LengthDistribution(scale=10), 0).tuples()
        stopo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9,
                         inter_bandwidth_bytes_per_s=50e9, prefill_tokens_per_s=50_000.0)
        sb = load_boundaries(stopo, 0.05, 0.2)
        arms = [("ours_native", ocl, osch)] + ([("reference", kp, kp)] if kp is not None else [])
        sched = {}
        rows = {}
        for name, mc, ms in arms:
            if time.perf_counter() > t_stop and name == "reference":
                sched["reference"] = "skipped (budget)"
                continue
            cl = mc.ClusterState(48 << 30, gpus_per_machine=8)
            s = Timed(ms.MellScheduler(cl, priority_cfg=ms.PriorityConfig(), batching=True))
            res = run_slots(trace, s, cl, stopo, sb, bpt=524_288, tokens_per_slot=10, duration_slots=200)
            t = sorted(s.times)
            rows[name] = res.plan_rows
            sched[name] = {"step_epoch_ms_mean": round(1e3 * statistics.fmean(t), 4),
                           "step_epoch_ms_p50": round(1e3 * t[len(t) // 2], 4), "epochs": len(t),
                           "peak_gpus": max(res.active_gpus)}
        if "reference" in rows:
            sched["identical_plan_rows"] = rows["reference"] == rows["ours_native"]
        sched["workload"] = "gen_poisson(0.5, 200 slots, scale 10, seed 0), C 48 GiB, 7B bpt, 8 GPUs/machine"
        out["step_epoch"] = sched
    finally:
        if old_aff is not None:
            try:
                os.sched_setaffinity(0, old_aff)
            except Exception:
                pass
    return out


def cpu_baseline(args, shape, tokens) -> dict:
    threads = os.cpu_count() or 1
    cb, times = cpu_migrate_rate(shape, tokens, threads, budget_s=args.cpu_budget_s)
    # 1 thread on a bounded 2k-token sample of the same shape (BASELINE.md CPU baseline 2)
    t1_tokens = min(tokens, 2048)
    cb1, times1 = cpu_migrate_rate(shape, t1_tokens, 1, budget_s=min(4.0, args.cpu_budget_s / 2), min_reps=2)
    out = {"value": round(cb * len(times) / sum(times) / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
           "sample": f"{len(times)} x {args.workload} migrations ({cb} B each, same workload) inside one host "
                     f"pool, oracle C port (oracle/kvmig_oracle.c), {threads} pthreads, "
                     f"~{args.cpu_budget_s:.0f} s budget",
           "cpu_model": _cpu_model(), "os_cpu_count": os.cpu_count(),
           "one_thread": {"value": round(cb1 * len(times1) / sum(times1) / 1e9, 3), "unit": "GB/s", "cores": 1,
                          "sample": f"{len(times1)} x {t1_tokens}-token migrations of the same shape "
                                    f"({cb1} B each), oracle C port, 1 thread"}}
    try:
        out["control_plane"] = control_plane_baseline()
    except Exception as e:
        out["control_plane"] = {"error": repr(e)[:300]}
    return out


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
                         "sample": sample, "cpu_model": _cpu_model()},
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


def _checksum(pool, blocks_np, n):
    """Order-sensitive int64 checksum of the request's pieces (every layer, K
    and V) gathered by `blocks_np`: equal sums <=> equal bytes in practice."""
    import torch

    shape = pool.shape
    idx = torch.from_numpy(blocks_np).long().to(pool.tensor.device)
    w = torch.arange(1, shape.piece_bytes // 2 + 1, device=idx.device, dtype=torch.int64)
    acc = torch.zeros((), dtype=torch.int64, device=idx.device)
    for l in range(shape.layers):
        g = pool.tensor[l][:, idx].reshape(2, n, -1).view(torch.int16).to(torch.int64)
        acc += (g * w).sum() + (g.sum(-1) * torch.arange(1, n + 1, device=idx.device)).sum()
    return int(acc.item())


def _pcts(xs):
    s = sorted(xs)
    return statistics.median(s), s[max(0, int(round(0.99 * len(s))) - 1)]


class Ring:
    """One workload on the ring i -> (i+1) mod N (N > 1): this rank's pool,
    its request, the PeerLink to its neighbours, and the measurements."""

    def __init__(self, ctx, workload: str):
        import numpy as np
        import torch

        from paper_2501_06709_b200.dist import PeerLink
        from paper_2501_06709_b200.kvcache import SHAPES, KVPool

        self.ctx, self.workload = ctx, workload
        ri, dev = ctx["ri"], ctx["device"]
        shape_name, self.tokens, self.cfg_desc = WORKLOADS[workload]
        self.shape = shape = SHAPES[shape_name]
        self.kv_bytes = self.tokens * shape.kv_bytes_per_token
        self.n, self.nb, self.sb_np, used = _layout(shape, self.tokens, seed=1 + ri.rank)
        self.pool = KVPool(shape, self.nb, device=dev)
        _fill_random(self.pool.tensor, 1234 + ri.rank)
        self.pool.allocator.take(np.flatnonzero(used))
        self.db_np = self.pool.allocator.alloc(self.n)          # blocks this rank RECEIVES into
        self.link = PeerLink(self.pool, self.db_np, ri)
        self.sb_dev = torch.from_numpy(self.sb_np).to(f"cuda:{dev}")
        self.stream = torch.cuda.Stream(device=dev)
        self.seq = 0
        self.link.peer(ri.send_to)      # map the neighbour's pool now, not inside a timed region

    def reset(self):
        import torch

        torch.cuda.synchronize()
        self.ctx["barrier"]()
        self.seq = 0
        self.link.reset()
        torch.cuda.synchronize()
        self.ctx["barrier"]()

    def step(self, engine: str, host: bool, ev=None, max_sms: int = 0):
        """Push this rank's request to send_to, then make the incoming one (from
        recv_from) a dependency of this rank's stream."""
        ri, shared = self.ctx["ri"], self.ctx["shared"]
        self.seq += 1
        if ev is not None:
            ev[0].record(self.stream)
        self.link.push(ri.send_to, self.sb_np if host else self.sb_dev, self.seq, engine=engine,
                       stream=self.stream, max_sms=max_sms)
        if ev is not None:
            ev[1].record(self.stream)
        if shared:
            # test mode, several ranks on ONE GPU: a device-side spin on the incoming flag can starve
            # the peer process's context, so the receive completes on the host: own push done, then
            # every rank has pushed
            self.stream.synchronize()
            self.ctx["barrier"]()
        else:
            self.link.wait(self.seq, self.stream, timeout_ns=WAIT_NS)
        if ev is not None:
            ev[2].record(self.stream)

    def landed(self) -> bool:
        """False if a receive wait timed out (the peer's move never became
        visible); never raises, so every rank reaches the next collective."""
        try:
            self.link.check()
            return True
        except TimeoutError as e:
            print(f"bench.py: {e}", file=sys.stderr)
            return False

    def gate(self, engine: str) -> bool:
        """One migration, then bit-exact check: what this rank received equals
        what recv_from sent, and the table row lists the receive blocks."""
        import numpy as np
        import torch

        from paper_2501_06709_b200.dist import exchange_objects

        ri = self.ctx["ri"]
        sent = _checksum(self.pool, self.sb_np, self.n)
        self.reset()
        with torch.cuda.stream(self.stream):
            self.step(engine, host=False)
        self.stream.synchronize()
        self.ctx["barrier"]()
        arrived = self.landed()
        got = _checksum(self.pool, self.db_np, self.n)
        sums = exchange_objects(sent)
        row_ok = bool(np.array_equal(self.link.row[:self.n].cpu().numpy(), self.db_np))
        ok = arrived and got == sums[ri.recv_from] and row_ok
        if not ok:
            print(f"rank {ri.rank}: parity gate failed ({engine}): received checksum {got}, sent "
                  f"{sums[ri.recv_from]}, table row ok {row_ok}", file=sys.stderr)
        return self.ctx["all_ok"](ok)

    def timed(self, engine: str, K: int, W: int, meter=None, clocks=None, max_sms: int = 0) -> dict:
        import torch

        from paper_2501_06709_b200 import _native
        from paper_2501_06709_b200.dist import allreduce_max

        dev = self.ctx["device"]
        self.reset()
        with torch.cuda.stream(self.stream):
            for _ in range(W):
                self.step(engine, host=False, max_sms=max_sms)
        self.stream.synchronize()
        self.ctx["barrier"]()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = _native.launch_count()
        torch.cuda.synchronize()
        self.ctx["barrier"]()
        if meter is not None:
            meter.start()
        if clocks is not None:
            clocks.__enter__()
        # throughput: K steps back to back (no per-launch events in the region, as at N = 1)
        with torch.cuda.stream(self.stream):
            t0.record(self.stream)
            for i in range(K):
                self.step(engine, host=False, max_sms=max_sms)
            t1.record(self.stream)
        self.stream.synchronize()
        torch.cuda.synchronize()
        if clocks is not None:
            clocks.__exit__()
        if meter is not None:
            meter.stop()
        launches = _native.launch_count() - launches0
        self.ctx["barrier"]()
        # latency: the same step with an event pair around the push and one after the wait, after the region
        KL = min(K, 30)
        ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(KL)]
        with torch.cuda.stream(self.stream):
            for i in range(KL):
                self.step(engine, host=False, ev=ev[i], max_sms=max_sms)
        self.stream.synchronize()
        torch.cuda.synchronize()
        self.ctx["barrier"]()
        arrived = self.ctx["all_ok"](self.landed())
        elapsed = allreduce_max(t0.elapsed_time(t1), dev)
        push = [a.elapsed_time(b) for a, b, _ in ev]
        stepms = [a.elapsed_time(c) for a, _, c in ev]
        p50, p99 = _pcts(push)
        s50, s99 = _pcts(stepms)
        return {"elapsed_ms": elapsed, "push_ms_mean": allreduce_max(statistics.fmean(push), dev),
                "push_p50": allreduce_max(p50, dev), "push_p99": allreduce_max(p99, dev),
                "step_p50": allreduce_max(s50, dev), "step_p99": allreduce_max(s99, dev),
                "launches": launches, "K": K, "all_landed": arrived,
                "value": self.ctx["world"] * self.kv_bytes * K / (elapsed / 1e3) / 1e9}

    def e2e(self, engine: str, K: int) -> dict:
        """The same ring through the public API (dist.PeerLink) with host block
        lists every step and a D2H of the rewritten block-table row."""
        import torch

        from paper_2501_06709_b200.dist import allreduce_max

        dev = self.ctx["device"]
        self.reset()
        row = torch.empty(self.n, dtype=torch.int32, pin_memory=True)
        torch.cuda.synchronize()
        self.ctx["barrier"]()
        lat = []
        t0 = time.perf_counter()
        for i in range(K):
            ts = time.perf_counter()
            with torch.cuda.stream(self.stream):
                self.step(engine, host=True)
                # D2H of the block-table row the incoming kernel rewrote, ordered after the wait
                row.copy_(self.link.row[:self.n], non_blocking=True)
            self.stream.synchronize()
            lat.append(time.perf_counter() - ts)
        torch.cuda.synchronize()
        e2e_s = allreduce_max(time.perf_counter() - t0, dev)
        self.ctx["barrier"]()
        ok = self.landed() and bool((row.numpy() == self.db_np).all())
        return {"value": self.ctx["world"] * self.kv_bytes * K / e2e_s / 1e9, "h2d_bytes_per_step": 2 * self.n * 4,
                "d2h_bytes_per_step": self.n * 4, "latency_ms_p50": 1e3 * allreduce_max(statistics.median(lat), dev),
                "row_ok": self.ctx["all_ok"](ok)}

    def library(self, K: int) -> dict:
        """COMPARISON ONLY: the same ring exchange done the library way —
        index_select gather, NCCL batch_isend_irecv (ncclSend/ncclRecv in one
        group), index_copy_ scatter (dist.collective_ring_exchange)."""
        import torch

        from paper_2501_06709_b200.dist import allreduce_max, collective_ring_exchange, exchange_objects

        ri, dev = self.ctx["ri"], self.ctx["device"]
        t = self.pool.tensor
        sbl = self.sb_dev.long()
        dbl = torch.from_numpy(self.db_np).long().to(f"cuda:{dev}")
        sent = _checksum(self.pool, self.sb_np, self.n)
        self.reset()
        collective_ring_exchange(t, sbl, dbl, ri)
        torch.cuda.synchronize()
        self.ctx["barrier"]()
        got = _checksum(self.pool, self.db_np, self.n)
        sums = exchange_objects(sent)
        ok = self.ctx["all_ok"](got == sums[ri.recv_from])
        collective_ring_exchange(t, sbl, dbl, ri)
        torch.cuda.synchronize()
        self.ctx["barrier"]()
        cs = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for _ in range(K):
            collective_ring_exchange(t, sbl, dbl, ri)
        e1.record(cs)
        torch.cuda.synchronize()
        ms = allreduce_max(e0.elapsed_time(e1), dev)
        self.ctx["barrier"]()
        return {"impl": "NCCL batch_isend_irecv ring (torch.distributed nccl) with index_select gather + "
                        "index_copy_ scatter (dist.collective_ring_exchange)",
                "value": round(self.ctx["world"] * self.kv_bytes * K / (ms / 1e3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(ms / K, 4), "steps": K, "bit_exact": ok}

    def library_gloo(self, K: int, group) -> dict:
        """COMPARISON ONLY: the paper prototype's transport (Gloo P2P for KV,
        PAPER.md:672): gather on the GPU, D2H into pinned memory, Gloo
        isend/irecv between the processes, H2D, scatter."""
        import torch
        import torch.distributed as dist

        from paper_2501_06709_b200.dist import allreduce_max, exchange_objects

        ri, dev = self.ctx["ri"], self.ctx["device"]
        t = self.pool.tensor
        sbl = self.sb_dev.long()
        dbl = torch.from_numpy(self.db_np).long().to(f"cuda:{dev}")
        out_h = torch.empty((t.shape[0], t.shape[1], self.n) + tuple(t.shape[3:]), dtype=t.dtype, pin_memory=True)
        in_h = torch.empty_like(out_h, pin_memory=True)

        def step():
            out_h.copy_(t.index_select(2, sbl))
            ops = [dist.P2POp(dist.isend, out_h, ri.send_to, group=group),
                   dist.P2POp(dist.irecv, in_h, ri.recv_from, group=group)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            t.index_copy_(2, dbl, in_h.to(t.device))
            torch.cuda.synchronize()

        sent = _checksum(self.pool, self.sb_np, self.n)
        self.reset()
        step()
        got = _checksum(self.pool, self.db_np, self.n)
        ok = self.ctx["all_ok"](got == exchange_objects(sent)[ri.recv_from])
        self.ctx["barrier"]()
        t0 = time.perf_counter()
        for _ in range(K):
            step()
        s = allreduce_max(time.perf_counter() - t0, dev)
        self.ctx["barrier"]()
        return {"impl": "Gloo P2P with host staging (gather -> D2H pinned -> gloo isend/irecv -> H2D -> scatter), "
                        "the paper prototype's transport (PAPER.md:672)",
                "value": round(self.ctx["world"] * self.kv_bytes * K / s / 1e9, 3), "unit": "GB/s",
                "ms_per_step": round(1e3 * s / K, 2), "steps": K, "bit_exact": ok, "timing": "host wall clock"}

    def close(self):
        import torch

        torch.cuda.synchronize()
        self.ctx["barrier"]()
        self.link.close()
        self.ctx["barrier"]()     # no peer maps this pool any more
        self.pool.close()
        del self.pool
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


def _roofline_nvlink(kv_bytes: int, push_ms: float, engine: str, traffic) -> dict:
    ach = kv_bytes / (push_ms / 1e3) / 1e9
    return {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_MEASURED_GBS, "unit": "GB/s",
            "frac": round(ach / NVLINK_MEASURED_GBS, 4),
            "peak_source": "B200_PROFILING.md measured peer copy per direction per GPU",
            "peak_nominal": NVLINK_PEAK_GBS, "frac_nominal": round(ach / NVLINK_PEAK_GBS, 4),
            "kernel": "migrate_ldg_kernel" if engine == "ldg" else "migrate_bulk_kernel",
            "algorithmic_bytes_per_launch": kv_bytes,
            "definition": "kv_bytes leaving this GPU per launch / mean launch time (launch -> done flag "
                          "release-stored to the peer after a system-scope fence), max over ranks",
            "traffic": traffic}


def _tool_json(script: str, argv: list, timeout_s: float) -> dict:
    """Run tools/<script> in a child process (its own CUDA contexts) and return
    the JSON it writes to --out.  A fault there (illegal address, hang until
    the timeout) is reported in the line instead of killing this rank."""
    import tempfile

    fd, out = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    t0 = time.perf_counter()
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", script), *argv, "--out", out],
                           capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
        try:
            with open(out) as f:
                res = json.load(f)
        except (OSError, ValueError):
            res = {"all_ok": False, "error": f"rc={r.returncode}: " + (r.stderr or r.stdout)[-400:]}
    except subprocess.TimeoutExpired:
        res = {"all_ok": False, "error": f"timed out after {timeout_s:.0f} s"}
    finally:
        try:
            os.unlink(out)
        except OSError:
            pass
    res["subprocess_s"] = round(time.perf_counter() - t0, 1)
    return res


def _peer_probe(args, ctx) -> dict:
    """Rank 0, before any timing, in a child process: the single-process
    cross-device checks on GPUs 0 and 1 (tools/multidev_check.py), including a
    push with each copy engine into the peer's pool.  Every rank then waits on
    a CPU (gloo) barrier and receives the result, so the engine A/B only
    offers the TMA bulk engine if its peer stores were bit-exact here."""
    import torch.distributed as dist

    md = None
    if ctx["ri"].rank == 0 and not args.no_multidev_checks:
        # ranks sharing one GPU (test mode): the same checks with both 'devices' = cuda:0
        b = "1" if ctx["ndev"] >= 2 else "0"
        md = _tool_json("multidev_check.py", ["--a", "0", "--b", b], timeout_s=600)
    box = [md]
    dist.broadcast_object_list(box, src=0, group=ctx["cpu_group"])
    return box[0]


def ring_engines(requested, md) -> list:
    """Copy engines the ring's start-up A/B may try: the one requested, else
    both, except that the TMA bulk engine is only offered when the cross-device
    probe pushed into a peer pool with it bit-exact (or no probe ran)."""
    if requested:
        return [requested]
    if md is None:
        return ["bulk", "ldg"]
    bulk_ok = bool(((md.get("engine_push_over_peer") or {}).get("bulk") or {}).get("ok", False))
    return ["bulk", "ldg"] if bulk_ok else ["ldg"]


def run_ring(args, ctx) -> int:
    """N > 1: the ring measurement, its evidence and extras."""
    import torch

    from paper_2501_06709_b200.dist import exchange_objects
    from paper_2501_06709_b200.telemetry import ClockSampler, NvlinkMeter, merge_clocks

    ri, world, dev, shared = ctx["ri"], ctx["world"], ctx["device"], ctx["shared"]
    md = _peer_probe(args, ctx)
    ring = Ring(ctx, args.workload)
    engines = ring_engines(args.engine, md)
    gates = {e: ring.gate(e) for e in engines}
    ab = {}
    if len(engines) > 1:   # start-up A/B to the peer, behind the bit-exact gate: keep the faster engine
        for e in engines:
            if gates[e]:
                r = ring.timed(e, K=5, W=3)
                ab[e] = {"push_ms_mean": round(r["push_ms_mean"], 4), "bit_exact": True}
            else:
                ab[e] = {"bit_exact": False}
        ok_eng = [e for e in engines if gates[e]]
        engine = min(ok_eng, key=lambda e: ab[e]["push_ms_mean"]) if ok_eng else engines[0]
    else:
        engine = engines[0]
    if not any(gates.values()):
        # nothing landed bit-exact on the peer: no throughput is reported for a path that is wrong
        if ri.rank == 0:
            print(json.dumps({"metric": "kv_migration_GBps", "value": 0.0, "unit": "GB/s", "n_gpus": world,
                              "steps": 0, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                              "scaling": "weak", "vs_baseline": None, "dtype": "fp16 bytes (u16 copy)",
                              "data": "synthetic", "bit_exact": False, "engines_tried": engines,
                              "multi_device_checks": md,
                              "error": "no copy engine passed the bit-exact gate to the peer pool"}), flush=True)
        ring.close()
        return 1
    bit_exact = gates[engine]
    # how many SMs the link-bound push needs: the chosen engine on 32 and 64 SMs (KVM_F_MAX_SMS) beside
    # the whole GPU (the timed run below uses the whole GPU); one SM's bulk pipeline moves ~37 GB/s
    # (tools/bench_copy_sms.py), so ~21 SMs' worth saturates 0.77 TB/s
    sm_ab = {}
    for cap in (32, 64, 0):
        r = ring.timed(engine, K=5, W=2, max_sms=cap)
        sm_ab[str(cap or "all")] = {"push_ms_mean": round(r["push_ms_mean"], 4),
                                    "GBps_per_gpu": round(ring.kv_bytes / (r["push_ms_mean"] / 1e3) / 1e9, 1),
                                    "all_landed": r["all_landed"]}
    meter = NvlinkMeter(dev)
    clocks = ClockSampler(dev)
    main = ring.timed(engine, args.steps, args.warmup, meter=meter, clocks=clocks)
    nv = exchange_objects(meter.result())
    clk = merge_clocks(exchange_objects(clocks.summary()))
    e2e = ring.e2e(engine, args.steps)
    lib = None
    if not shared and not args.no_library:
        try:
            lib = ring.library(min(args.steps, 20))
            lib["ours_over_library"] = round(main["value"] / lib["value"], 3)
        except Exception as e:
            lib = {"error": repr(e)[:300]}
        try:
            import torch.distributed as dist

            gl = ring.library_gloo(2 if world <= 2 else 1, dist.new_group(backend="gloo"))
            gl["ours_over_library"] = round(main["value"] / gl["value"], 1)
            lib = dict(lib or {}, paper_transport=gl)
        except Exception as e:
            lib = dict(lib or {}, paper_transport={"error": repr(e)[:300]})
    elif shared:
        lib = {"skipped": "ranks share one GPU (gloo control plane; NCCL needs one GPU per rank)"}
        if not args.no_library:
            try:
                import torch.distributed as dist

                lib["paper_transport"] = ring.library_gloo(2, dist.new_group(backend="gloo"))
            except Exception as e:
                lib["paper_transport"] = {"error": repr(e)[:300]}
    kv_bytes = ring.kv_bytes
    n, nb = ring.n, ring.nb
    cfg_desc = ring.cfg_desc
    ring.close()
    extras = {}
    extra_list = [w for w in (args.extra_workloads or "").split(",") if w and w != args.workload]
    for w in extra_list:
        try:
            r2 = Ring(ctx, w)
            ok2 = r2.gate(engine)
            m2 = r2.timed(engine, min(args.steps, 20), args.warmup)
            extras[w] = {"config": WORKLOADS[w][2], "kv_bytes_per_rank_per_step": r2.kv_bytes,
                         "value": round(m2["value"], 2), "unit": "GB/s", "ms_per_step": round(m2["elapsed_ms"] / m2["K"], 4),
                         "steps": m2["K"], "bit_exact": ok2, "engine": engine,
                         "latency_ms": {"p50": round(m2["push_p50"], 4), "p99": round(m2["push_p99"], 4)},
                         "roofline": _roofline_nvlink(r2.kv_bytes, m2["push_ms_mean"], engine, None)
                         if not shared else None}
            r2.close()
        except Exception as e:
            extras[w] = {"error": repr(e)[:300]}
    # NVLink bytes NVML saw (per rank), as roofline.traffic per launch
    tx = [r.get("tx_bytes") for r in nv]
    traffic = None
    if all(t is not None for t in tx):
        traffic = round(statistics.fmean(tx) / main["K"])
    if shared:
        hbm_peak, _, _, psrc = _peaks()
        ach = 2 * kv_bytes / (main["push_ms_mean"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "peak_source": psrc + " hbm_gbs",
                "kernel": "migrate_ldg_kernel" if engine == "ldg" else "migrate_bulk_kernel",
                "algorithmic_bytes_per_launch": 2 * kv_bytes, "traffic": None,
                "note": f"{world} ranks share {ctx['ndev']} GPU(s): IPC path exercised without NVLink"}
    else:
        roof = _roofline_nvlink(kv_bytes, main["push_ms_mean"], engine, traffic)
    roof["nvlink_counters"] = {"per_rank": nv,
                               "definition": "NVML NVLink TX/RX bytes over the timed region per rank; traffic = "
                                             "mean TX bytes per launch (null when the box does not expose them)"}
    line = None
    if ri.rank == 0:
        if not shared and ctx["ndev"] >= 2 and not args.no_extras:
            # configs[2] across two GPUs: the prefix pushed 0 -> 1 over NVLink while GPU 1 re-prefills
            # the suffix (and the fused kernel pulling the prefix), child process, others wait on the CPU
            extras["split_13b_8k_2gpu"] = _tool_json("bench_split.py", ["--src-dev", "0", "--dst-dev", "1",
                                                                        "--iters", "5"], timeout_s=600)
            # time to the first decode step after a 7B-4k migration GPU 0 -> GPU 1: sequential vs the decode
            # of layer l starting when the copy released layer l's flag on GPU 1
            extras["pipelined_decode_7b_4k_2gpu"] = _tool_json(
                "bench_pipelined_decode.py", ["--src-dev", "0", "--dst-dev", "1", "--reps", "10"], timeout_s=300)
        if not shared and ctx["ndev"] >= 8 and world >= 8 and args.config5_slots > 0:
            # configs[4] at real shapes: the live loop (native scheduler -> planner -> executor) with one
            # logical GPU per B200, full Llama-2-7B KV, slot-limited; bytes fingerprint-checked.  A child
            # process (the other ranks wait on a CPU barrier, their GPUs idle)
            torch.cuda.empty_cache()
            extras["config5_online_full_7b"] = _tool_json(
                "online_loop.py", ["--fixture", os.path.join(ROOT, "tests", "golden", "trace_7b_c48g_seed0.json"),
                                   "--shape", "full", "--engine", engine, "--verify-every", "100",
                                   "--max-slots", str(args.config5_slots), "--devices", "8"], timeout_s=900)
        cpu = None if args.no_cpu_baseline else cpu_baseline(args, ring.shape, ring.tokens)
        line = {
            "metric": "kv_migration_GBps", "value": round(main["value"], 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(main["elapsed_ms"] / main["K"], 4),
            "higher_is_better": True, "scaling": "weak", "scaling_note": "N=1 is intra-GPU compaction bound by HBM (configs[1] needs two GPUs); N>1 is the ring push bound by NVLink (one link crossing per byte): compare roofline.frac per N, not value(N)/(N*value(1))", "vs_baseline": None, "dtype": "fp16 bytes (u16 copy)",
            "data": "synthetic (seeded random KV bits, NaN payloads included)",
            "config": {"workload": (f"{args.workload} ring push i->(i+1) mod {world} over NVLink (CUDA IPC)"
                                    if not shared else
                                    f"{args.workload} ring push i->(i+1) mod {world}, ranks sharing "
                                    f"{ctx['ndev']} GPU (CUDA IPC test mode, no NVLink hop)"),
                       "baseline_config": cfg_desc, "kv_bytes_per_rank_per_step": kv_bytes, "blocks": n,
                       "pool_blocks": nb, "engine": engine, "engine_ab": ab or None,
                       "push_sm_budget_ab": sm_ab or None,
                       "l2": "inputs larger than L2 (%.1f GiB per step per rank)" % (kv_bytes / 2 ** 30),
                       "parallelism": f"{world} ranks, one process per GPU" +
                                      (f" ({ctx['ndev']} physical GPU, shared)" if shared else ""),
                       "launcher": ctx["launcher"]},
            "latency_ms": {"p50": round(main["push_p50"], 4), "p99": round(main["push_p99"], 4),
                           "definition": "per step on each rank: event before the push launch -> event after the "
                                         "push kernel, whose last CTA release-stores the done flag into the "
                                         "destination (system scope) after the block-table row; max over ranks; "
                                         "up to 30 steps timed one by one after the throughput region",
                           "step_p50": round(main["step_p50"], 4), "step_p99": round(main["step_p99"], 4),
                           "step_definition": "push + wait until the incoming move's done flag is visible here "
                                              "(ld.acquire.sys)"},
            "bit_exact": bool(bit_exact and main["all_landed"] and e2e["row_ok"]
                              and (md is None or md.get("all_ok", False))),
            "multi_device_checks": md,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e["value"], 2), "unit": "GB/s", "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                    "latency_ms_p50": round(e2e["latency_ms_p50"], 4), "row_ok": e2e["row_ok"],
                    "path": "dist.PeerLink.push(host block lists) -> PeerLink.wait(done flag) -> "
                            "block-table row D2H -> host waits"},
            "library": lib,
            "extra_workloads": extras or None,
            "gpu_launches": int(main["launches"]),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    return 0


def run_compact(args, ctx) -> int:
    """N = 1: intra-GPU migration (compaction) of the request, HBM -> HBM."""
    import numpy as np
    import torch

    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.executor import ENGINES, MigrationExecutor, Residency
    from paper_2501_06709_b200.kvcache import SHAPES, BlockTable, KVPool
    from paper_2501_06709_b200.telemetry import ClockSampler

    device = ctx["device"]
    engine = args.engine or "bulk"
    shape_name, tokens, cfg_desc = WORKLOADS[args.workload]
    shape = SHAPES[shape_name]
    kv_bytes = tokens * shape.kv_bytes_per_token
    n, nb, sb_np, used = _layout(shape, tokens, seed=1)
    eng = ENGINES[engine] | (_native.KVM_F_L2_EVICT_FIRST if args.l2_evict_first else 0)
    lib = _native.lib()
    pool = KVPool(shape, nb, device=device)
    _fill_random(pool.tensor, 1234)
    pool.allocator.take(np.flatnonzero(used))
    db_np = pool.allocator.alloc(n)
    table = BlockTable(4, n, device=device)
    mailbox = torch.zeros(64, dtype=torch.int32, device=f"cuda:{device}")
    stream = torch.cuda.Stream(device=device)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    sb_dev = torch.from_numpy(sb_np).to(f"cuda:{device}")
    db_dev = torch.from_numpy(db_np).to(f"cuda:{device}")
    seq = [0]

    def step(i):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks = pool.pool_id, pool.pool_id, n
        fwd = i % 2 == 0         # compaction ping-pong: forward into db, then back into the original blocks
        m.src_blocks = sb_dev.data_ptr() if fwd else db_dev.data_ptr()
        m.dst_blocks = db_dev.data_ptr() if fwd else sb_dev.data_ptr()
        m.dst_table_row = table.row_ptr(0)
        m.done_flag = mailbox.data_ptr()
        seq[0] += 1
        m.done_value = seq[0]
        _native.check(lib.kvm_migrate(ctypes.byref(m), 1, eng, sptr))

    sent = _checksum(pool, sb_np, n)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        step(0)
    stream.synchronize()
    bit_exact = _checksum(pool, db_np, n) == sent and \
        bool(np.array_equal(table.rows[0, :n].cpu().numpy(), db_np)) and int(mailbox[0].item()) == 1
    seq[0] = 0
    with torch.cuda.stream(stream):   # sb and db now hold the same bytes: the ping-pong keeps them equal
        for i in range(args.warmup):
            step(i)
    stream.synchronize()
    K = args.steps
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    torch.cuda.synchronize()
    with ClockSampler(device) as clk:
        with torch.cuda.stream(stream):
            t_start.record(stream)
            for i in range(K):
                step(args.warmup + i)
            t_end.record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    elapsed_ms = t_start.elapsed_time(t_end)
    avg_launch_ms = elapsed_ms / K    # the launches run back to back: mean launch time over the timed region
    value = kv_bytes * K / (elapsed_ms / 1e3) / 1e9
    # latency: the same step timed one launch at a time, after the throughput region (an event pair around
    # each launch keeps the next launch from starting under this one's tail, ~5 us per launch, so per-launch
    # events stay out of the throughput loop)
    KL = min(K, 50)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(KL)]
    with torch.cuda.stream(stream):
        for i in range(KL):
            ev[i][0].record(stream)
            step(args.warmup + K + i)
            ev[i][1].record(stream)
    stream.synchronize()
    per = [a.elapsed_time(b) for a, b in ev]
    p50, p99 = _pcts(per)

    # ---------------- e2e through the public API ----------------
    ex = MigrationExecutor({0: pool}, {0: table}, engine=engine)
    pool.allocator.free(db_np)   # the request is resident in sb; db is free again
    ex.loc[0] = Residency(0, sb_np.copy(), tokens, pool.shape.name)
    table.set_host(0, sb_np)
    rows = [torch.empty(n, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    for i in range(args.warmup):
        ex.compact(0, row_out=rows[0])
    torch.cuda.synchronize()
    # every step: host block lists -> H2D -> kernel -> D2H of the rewritten block-table row, and the
    # host waits for that row; the call is stream-ordered, so the host prepares step i+1 while the
    # GPU still copies step i (double-buffered pinned rows)
    t0 = time.perf_counter()
    prev = None
    e2e_ok = True
    for i in range(K):
        ts = time.perf_counter()
        rec = ex.compact(0, row_out=rows[i & 1], stream_ordered=True)
        if prev is not None:
            prev[0].done.synchronize()
            e2e_ok &= bool(np.array_equal(rows[(i - 1) & 1].numpy(), prev[2]))
        prev = (rec, ts, ex.where(0).blocks.copy())
    prev[0].done.synchronize()
    e2e_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    e2e_ok &= bool(np.array_equal(rows[(K - 1) & 1].numpy(), ex.where(0).blocks))
    # content check after the e2e loop: the request's bytes are still the ones it started with
    e2e_ok &= _checksum(pool, ex.where(0).blocks, n) == sent
    e2e_lat = []
    for i in range(min(K, 30)):   # per-call latency of one synchronous call (issue -> row on the host)
        ts = time.perf_counter()
        ex.compact(0, row_out=rows[0])
        e2e_lat.append(time.perf_counter() - ts)
    e2e = kv_bytes * K / e2e_s / 1e9

    # ---------------- the library path on the same workload ----------------
    lib_line = None
    if not args.no_library:
        try:
            v = pool.tensor.view(2 * shape.layers, nb, -1)
            planes = [v[i] for i in range(2 * shape.layers)]
            tmp = torch.empty(n, v.shape[2], dtype=v.dtype, device=v.device)
            sl, dl = sb_dev.long(), db_dev.long()

            def view_arm(a, b):      # one gather + one scatter over the [layers*2, blocks, piece] view
                v.index_copy_(1, b, v.index_select(1, a))

            def plane_arm(a, b):     # per (layer, K|V) plane: dim-0 index ops (torch's contiguous-row path)
                for pv in planes:
                    torch.index_select(pv, 0, a, out=tmp)
                    pv.index_copy_(0, b, tmp)

            arms = {}
            for name, fn in (("index_select+index_copy_ on the [layers*2, blocks, piece] view", view_arm),
                             ("index_select+index_copy_ per [blocks, piece] plane", plane_arm)):
                torch.cuda.synchronize()
                sent_now = _checksum(pool, sb_np, n)
                with torch.cuda.stream(stream):
                    fn(sl, dl)
                stream.synchronize()
                ok = _checksum(pool, db_np, n) == sent_now
                KL = min(K, 20)
                with torch.cuda.stream(stream):
                    for _ in range(2):
                        fn(sl, dl)
                    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    l0.record(stream)
                    for i in range(KL):
                        fn(*((sl, dl) if i % 2 == 0 else (dl, sl)))
                    l1.record(stream)
                stream.synchronize()
                lms = l0.elapsed_time(l1) / KL
                arms[name] = {"value": round(kv_bytes / lms / 1e6, 2), "ms_per_step": round(lms, 4), "steps": KL,
                              "bit_exact": bool(ok)}
            best = max(arms, key=lambda k: arms[k]["value"])
            lib_line = {"impl": f"torch {best} (the faster torch arm; both below)", "unit": "GB/s",
                        **arms[best], "arms": arms,
                        "ours_over_library": round((kv_bytes / (elapsed_ms / K) / 1e6) / arms[best]["value"], 3)}
            del tmp
        except Exception as e:
            lib_line = {"error": repr(e)[:300]}

    hbm_peak, _, _, psrc = _peaks()
    alg_bytes = 2 * kv_bytes  # read + write, same HBM
    ach = alg_bytes / (avg_launch_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(ach / hbm_peak, 4), "peak_source": psrc + " hbm_gbs",
            "kernel": "migrate_ldg_kernel" if engine == "ldg" else "migrate_bulk_kernel",
            "algorithmic_bytes_per_launch": alg_bytes, "traffic": _traffic_for(args.workload, engine)}
    cpu = None if args.no_cpu_baseline else cpu_baseline(args, shape, tokens)
    line = {
        "metric": "kv_migration_GBps", "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(elapsed_ms / K, 4),
        "higher_is_better": True, "scaling": "weak", "scaling_note": "N=1 is intra-GPU compaction bound by HBM (configs[1] needs two GPUs); N>1 is the ring push bound by NVLink (one link crossing per byte): compare roofline.frac per N, not value(N)/(N*value(1))", "vs_baseline": None, "dtype": "fp16 bytes (u16 copy)",
        "data": "synthetic (seeded random KV bits, NaN payloads included)",
        "config": {"workload": f"{args.workload} intra-GPU migration (compaction into fresh blocks of the same pool)",
                   "baseline_config": cfg_desc, "kv_bytes_per_rank_per_step": kv_bytes, "blocks": n,
                   "pool_blocks": nb, "engine": engine, "l2_evict_first": bool(args.l2_evict_first),
                   "l2": "inputs larger than L2 (%.1f GiB per step)" % (kv_bytes / 2 ** 30),
                   "parallelism": "1 GPU", "launcher": ctx["launcher"]},
        "latency_ms": {"p50": round(p50, 4), "p99": round(p99, 4), "launches": KL,
                       "definition": "kernel launch -> done flag on dst stream (CUDA events around each "
                                     "launch, one launch at a time after the timed region)"},
        "bit_exact": bool(bit_exact and e2e_ok),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": 2 * n * 4, "d2h_bytes_per_step": n * 4,
                "latency_ms_p50": round(1e3 * statistics.median(e2e_lat), 4),
                "latency_definition": "one synchronous call through the API: issue -> result row on the host",
                "path": "MigrationExecutor.compact(stream_ordered) -> kvm_compact(host block lists: <= 256 blocks "
                        "travel H2D inside the kernel's parameter block, more are staged by a pinned copy) -> "
                        "table row D2H -> host waits for the row (next step issued meanwhile)"},
        "library": lib_line,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if not args.no_extras:
        line["kernels"] = _kernel_extras(device)
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args) -> int:
    import torch
    import torch.distributed as dist

    from paper_2501_06709_b200.dist import allreduce_max, rank_info_from_env

    ri = rank_info_from_env()
    world = ri.world
    ndev = torch.cuda.device_count()
    if ndev == 0:
        print("bench.py: no CUDA device visible (the GPU arm has no CPU fallback)", file=sys.stderr)
        return 3
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    shared = world > 1 and ndev < world
    if shared and not args.shared_gpu:
        print(f"bench.py: --gpus {world} needs {world} visible GPUs, found {ndev} (pass --shared-gpu to run the "
              f"ranks on shared GPUs as a functional test; no NVLink is measured then)", file=sys.stderr)
        return 2
    device = ri.local_rank % ndev
    torch.cuda.set_device(device)
    ctx = {"ri": ri, "world": world, "device": device, "ndev": ndev, "shared": shared,
           "launcher": os.environ.get("KVM_BENCH_LAUNCHER", "torchrun" if world > 1 else "python")}
    if world > 1:
        backend = "gloo" if shared else "nccl"   # gloo: N ranks sharing one GPU (test mode)
        dist.init_process_group(backend=backend, device_id=torch.device(f"cuda:{device}")
                                if backend == "nccl" else None)
        ctx["barrier"] = dist.barrier
        ctx["all_ok"] = lambda ok: allreduce_max(0.0 if ok else 1.0, device) == 0.0
        # control-plane group on the host: ranks that wait while rank 0 runs its child-process checks
        # and CPU baselines block here on the CPU, not in a spinning NCCL kernel on their GPU, and no
        # NCCL watchdog fires during rank 0's minutes of extras
        ctx["cpu_group"] = dist.new_group(backend="gloo", timeout=datetime.timedelta(minutes=60))
        try:
            rc = run_ring(args, ctx)
        finally:
            dist.barrier(group=ctx["cpu_group"])
            dist.destroy_process_group()
        return rc
    ctx["barrier"] = lambda: None
    ctx["all_ok"] = bool
    return run_compact(args, ctx)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv) -> int:
    """`python bench.py --gpus N` without torchrun: re-launch this script under
    torch.distributed.run with N ranks (one process per GPU) on 127.0.0.1;
    rank 0's JSON line is the output."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *argv]
    env = dict(os.environ, KVM_BENCH_LAUNCHER="self-launched torch.distributed.run")
    return subprocess.call(cmd, env=env)


def launch_check(args) -> int:
    """--launch-check: the launcher path without a GPU (CPU tests): every rank
    joins a gloo group, checks WORLD_SIZE == --gpus, reduces a max over ranks
    and rank 0 prints one line."""
    import torch.distributed as dist

    from paper_2501_06709_b200.dist import allreduce_max, exchange_objects, rank_info_from_env

    ri = rank_info_from_env()
    if ri.world != args.gpus:
        print(f"bench.py: WORLD_SIZE={ri.world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if ri.world > 1:
        dist.init_process_group("gloo")
    ranks = exchange_objects(ri.rank) if ri.world > 1 else [0]
    mx = allreduce_max(float(ri.rank))
    if ri.rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": ri.world, "ranks": ranks, "max_rank": mx,
                          "launcher": os.environ.get("KVM_BENCH_LAUNCHER", "torchrun" if ri.world > 1 else "python")}),
              flush=True)
    if ri.world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="7b-4k")
    ap.add_argument("--engine", choices=["ldg", "bulk"], default=None,
                    help="copy engine; default bulk (TMA) at N=1; at N>1 a start-up A/B of both engines to the "
                         "peer, behind the bit-exact gate, keeps the faster")
    ap.add_argument("--l2-evict-first", type=int, choices=[0, 1], default=0,
                    help="stream KV through L2 with an evict-first policy (KVM_F_L2_EVICT_FIRST), N=1")
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the re-prefill / decode measurements reported beside the headline (N=1)")
    ap.add_argument("--no-library", action="store_true",
                    help="skip the library-path comparison (torch index_select/index_copy_ at N=1, NCCL ring at N>1)")
    ap.add_argument("--extra-workloads", default=None,
                    help="comma list of workloads measured beside the headline at N>1 (default 70b-16k)")
    ap.add_argument("--no-multidev-checks", action="store_true",
                    help="skip rank 0's single-process cross-device checks (tools/multidev_check.py) at N>1")
    ap.add_argument("--config5-slots", type=int, default=400,
                    help="at N>=8: slots of the configs[4] live loop at full 7B shapes run by rank 0 (0: skip)")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="allow N ranks on fewer GPUs (functional test of the IPC path; no NVLink)")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.extra_workloads is None:
        args.extra_workloads = "70b-16k" if args.workload != "7b-512" else ""
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return self_launch(args, argv)
    if args.launch_check:
        return launch_check(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
