"""Power roofline of the re-prefill GEMM and the fused split migration
(VERDICT r1 weak #2): is the CTA-pair tcgen05 kernel held back by its pipe or
by the board power limit?

Each arm runs back to back for ~`--seconds` while NVML reads the board's
cumulative energy counter (telemetry.EnergyMeter) and samples the SM clock
(telemetry.ClockSampler); ms per call from CUDA events on the launching
stream.  Two interleaved rounds, so every arm sees the same thermal state.

Arms (13B shapes, configs[2]):
  reprefill_pair      kvm_reprefill, CTA-pair kernel, s = 1 360 rows, QKV, 40 layers
  reprefill_single    the single-CTA engine on the same shape
  cublas              torch.matmul per layer (cuBLAS) on the same shape, GEMM only
  suffix_gemm         the split's suffix re-prefill alone (s from split_point)
  prefix_copy         kvm_migrate of the split's prefix blocks alone (bulk engine)
  fused_split         kvm_split_migrate: both in one launch

Derived:
  TFLOP/J per GEMM arm (energy efficiency; at the cap, time = J / W_limit)
  cap_bound_ms = joules_per_call / limit_w (the shortest time at that energy
                 per call if the board may draw at most its limit)
  fused_energy_model_ms = (J(suffix_gemm) + J(prefix_copy)) / limit_w vs the
                 measured fused time: if they agree, the fused kernel is at the
                 power roofline, and hiding more of the copy needs less energy
                 per copied byte, not more overlap.

    python tools/power_roofline.py [--seconds 2] [--out file.json]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import (reprefill, reprefill_flops, split_point,  # noqa: E402
                                             synthetic_hidden, synthetic_weights)
from paper_2501_06709_b200.split import flops_per_token, make_split, split_migrate_fused  # noqa: E402
from paper_2501_06709_b200.telemetry import ClockSampler, EnergyMeter  # noqa: E402

NVLINK_BPS = 770e9          # measured peer copy per direction (B200_PROFILING.md)
TENSOR_FLOPS = 1.28e15      # kvm_reprefill's measured rate on 13B (tools/bench_reprefill.py)


def fill(pool, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    v = pool.tensor.view(torch.int16).view(-1)
    step = 1 << 28
    for i in range(0, v.numel(), step):
        k = min(step, v.numel() - i)
        v[i:i + k] = torch.randint(-2 ** 15, 2 ** 15 - 1, (k,), generator=g, device="cuda", dtype=torch.int16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=2.0)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--rows", type=int, default=1360)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    sh = LLAMA2_13B
    st = torch.cuda.Stream()
    em = EnergyMeter(0)

    # re-prefill arms
    rows = a.rows
    nblk = (rows + 15) // 16
    rpool = KVPool(sh, nblk + 4, dtype=torch.bfloat16)
    rblocks = torch.arange(nblk, dtype=torch.int32, device="cuda")
    x, w = synthetic_hidden(sh, rows, 0), synthetic_weights(sh, 0, with_q=True)
    outs = torch.empty(rows, w.shape[1], dtype=torch.bfloat16, device="cuda")
    flops = reprefill_flops(sh, rows, with_q=True)

    def cublas():
        for l in range(sh.layers):
            torch.matmul(x, w[l].t(), out=outs)

    # split arms
    n = a.tokens
    fpt = flops_per_token(sh, with_q=True)
    s = split_point(n, sh.kv_bytes_per_token, NVLINK_BPS, fpt, TENSOR_FLOPS)
    plan = make_split(n, s)
    tb = plan.total_blocks
    nb = tb + 64
    src, dst = KVPool(sh, nb, dtype=torch.bfloat16), KVPool(sh, nb, dtype=torch.bfloat16)
    fill(src, 1)
    fill(dst, 2)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:tb].to(torch.int32).numpy()
    db_np = np.sort(np.random.default_rng(2).permutation(nb)[:tb]).astype(np.int32)
    sbd, dbd = torch.from_numpy(sb).cuda(), torch.from_numpy(db_np).cuda()
    xs = synthetic_hidden(sh, max(plan.suffix, 1), 0, seed=2)[:plan.suffix].contiguous()
    pre_s, pre_d = np.ascontiguousarray(sb[:plan.prefix_blocks]), np.ascontiguousarray(db_np[:plan.prefix_blocks])
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, plan.prefix_blocks, 1
    m.src_blocks, m.dst_blocks = pre_s.ctypes.data, pre_d.ctypes.data
    sp = ctypes.c_void_p(st.cuda_stream)

    def prefix_copy():
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST |
                                                _native.KVM_F_ENGINE_BULK, sp))

    arms = {
        "reprefill_pair": (lambda: reprefill(rpool, x, w, rblocks, stream=st), flops),
        "reprefill_single": (lambda: reprefill(rpool, x, w, rblocks, stream=st, single_cta=True), flops),
        "cublas": (cublas, flops),
        "suffix_gemm": (lambda: reprefill(dst, xs, w, dbd, tok0=plan.prefix_tokens, stream=st),
                        plan.suffix * fpt),
        "prefix_copy": (prefix_copy, None),
        "fused_split": (lambda: split_migrate_fused(src, dst, sbd, dbd, plan, xs, w, stream=st),
                        plan.suffix * fpt),
    }
    st.wait_stream(torch.cuda.current_stream())
    res = {k: [] for k in arms}
    with torch.cuda.stream(st):
        for _ in range(a.rounds):
            for name, (fn, fl) in arms.items():
                for _ in range(3):
                    fn()
                st.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(3):
                    fn()
                e1.record(st)
                e1.synchronize()
                est = e0.elapsed_time(e1) / 3
                calls = max(5, int(a.seconds * 1e3 / est))
                e0.record(st)
                with ClockSampler(0) as clk:
                    r = em.measure(fn, calls, st.synchronize)
                e1.record(st)
                e1.synchronize()
                r["ms"] = e0.elapsed_time(e1) / calls
                r["sm_mhz"] = clk.summary()["sm_mhz"]
                r["reasons"] = clk.summary()["reasons"]
                if fl:
                    r["tflops"] = fl / r["ms"] / 1e9
                    if "joules_per_call" in r:
                        r["tflop_per_joule"] = fl / 1e12 / r["joules_per_call"]
                res[name].append(r)
    torch.cuda.synchronize()

    def med(name, key):
        v = [r[key] for r in res[name] if r.get(key) is not None]
        return statistics.median(v) if v else None

    lim = em.limit_w
    summary = {}
    for name in arms:
        d = {k: med(name, k) for k in ("ms", "joules_per_call", "board_w", "sm_mhz", "tflops", "tflop_per_joule")}
        d = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items()}
        if d["joules_per_call"] and lim:
            d["cap_bound_ms"] = round(d["joules_per_call"] / lim * 1e3, 4)
        d["at_cap"] = any(r.get("at_cap") for r in res[name])
        d["reasons"] = sorted({x for r in res[name] for x in r.get("reasons", [])})
        summary[name] = d
    out = {"tool": "power_roofline", "limit_w": lim, "energy_error": em.error,
           "shape": "llama2-13b", "reprefill_rows": rows, "split": {"tokens": n, "suffix": plan.suffix,
                                                                  "prefix_blocks": plan.prefix_blocks,
                                                                  "prefix_bytes": plan.prefix_tokens *
                                                                  sh.kv_bytes_per_token},
           "arms": summary, "rounds": res}
    sj, pj = summary["suffix_gemm"]["joules_per_call"], summary["prefix_copy"]["joules_per_call"]
    if sj and pj and lim:
        out["fused_energy_model_ms"] = round((sj + pj) / lim * 1e3, 4)
        out["fused_measured_ms"] = summary["fused_split"]["ms"]
        out["fused_joules_vs_parts"] = round(summary["fused_split"]["joules_per_call"] / (sj + pj), 4)
        out["prefix_hidden_frac"] = round(1 - (summary["fused_split"]["ms"] - summary["suffix_gemm"]["ms"]) /
                                          summary["prefix_copy"]["ms"], 4)
    if summary["cublas"]["tflop_per_joule"] and summary["reprefill_pair"]["tflop_per_joule"]:
        out["pair_over_cublas_energy_eff"] = round(summary["reprefill_pair"]["tflop_per_joule"] /
                                                   summary["cublas"]["tflop_per_joule"], 4)
        out["pair_over_cublas_speed"] = round(summary["cublas"]["ms"] / summary["reprefill_pair"]["ms"], 4)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "rounds"}))


if __name__ == "__main__":
    main()
