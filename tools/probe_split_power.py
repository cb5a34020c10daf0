"""Is the fused split migration's overhead over the bare suffix GEMM a power /
clock effect?  Runs each arm back to back for ~3 s while nvidia-smi samples SM
clock and board power, and reports ms per call with the median clock/power.

    python tools/probe_split_power.py [--seconds 3]

Arms (13B, 8k tokens, s = 1 456): suffix re-prefill alone (CTA-pair GEMM);
fused split (same GEMM + 5.5 GB prefix copy in the same kernel); prefix copy
alone (kvm_migrate of the prefix blocks, bulk engine).
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights  # noqa: E402
from paper_2501_06709_b200.split import make_split, split_migrate_fused  # noqa: E402


def sampled(fn, seconds):
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                             "-lms", "100"], stdout=subprocess.PIPE, text=True)
    torch.cuda.synchronize()
    t0, n = time.perf_counter(), 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    proc.terminate()
    out = proc.communicate()[0]
    rows = [tuple(float(x) for x in line.split(",")) for line in out.strip().splitlines() if "," in line]
    rows = rows[2:] if len(rows) > 4 else rows   # drop the ramp
    return {"ms_per_call": round(e0.elapsed_time(e1) / n, 4),
            "sm_mhz_median": statistics.median(r[0] for r in rows) if rows else None,
            "power_w_median": statistics.median(r[1] for r in rows) if rows else None, "samples": len(rows)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    sh = LLAMA2_13B
    n_tok, s = 8192, 1456
    plan = make_split(n_tok, s)
    nb = plan.total_blocks + 16
    src, dst = KVPool(sh, nb, dtype=torch.bfloat16), KVPool(sh, nb, dtype=torch.bfloat16)
    src.tensor.view(torch.int16).view(-1)[: 1 << 28].random_()
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:plan.total_blocks].to(torch.int32).cuda()
    db = torch.arange(plan.total_blocks, dtype=torch.int32, device="cuda")
    x = synthetic_hidden(sh, s, 0)
    w = synthetic_weights(sh, 0, with_q=True)
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, plan.prefix_blocks, 1
    m.src_blocks, m.dst_blocks = sb.data_ptr(), db.data_ptr()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    arms = {
        "suffix_gemm": lambda: reprefill(dst, x, w, db, tok0=plan.prefix_tokens),
        "fused_split": lambda: split_migrate_fused(src, dst, sb, db, plan, x, w),
        "prefix_copy": lambda: _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1,
                                                                      _native.KVM_F_ENGINE_BULK, st)),
    }
    out = {}
    for rnd in range(2):
        for name, fn in arms.items():
            out.setdefault(name, []).append(sampled(fn, a.seconds))
    print(json.dumps({"workload": "13B 8k tokens, suffix 1456", "arms": out}))


if __name__ == "__main__":
    main()
