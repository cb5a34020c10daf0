"""Time kvm_reprefill (tcgen05) against cuBLAS (torch.matmul) on the same
projection, 13B shape by default.  Prints one JSON line.

    python tools/bench_reprefill.py [--rows 1360] [--shape llama2-13b] [--kv-only] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import (reprefill, reprefill_flops, synthetic_hidden,  # noqa: E402
                                             synthetic_weights)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1360)
    ap.add_argument("--shape", default="llama2-13b")
    ap.add_argument("--kv-only", action="store_true")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cublas", action="store_true")
    a = ap.parse_args()
    shape = SHAPES[a.shape]
    rows = a.rows
    nblk = (rows + 15) // 16
    pool = KVPool(shape, nblk + 4, dtype=torch.bfloat16)
    blocks = torch.arange(nblk, dtype=torch.int32, device="cuda")
    x = synthetic_hidden(shape, rows, 0)
    w = synthetic_weights(shape, 0, with_q=not a.kv_only)
    flops = reprefill_flops(shape, rows, with_q=not a.kv_only)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # x, w, pool were produced on the default stream

    def timeit(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(s)
        for _ in range(a.iters):
            fn()
        ev[1].record(s)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / a.iters

    y = torch.empty(rows, w.shape[1], dtype=torch.bfloat16, device="cuda")

    def cublas():
        for l in range(shape.layers):
            torch.matmul(x, w[l].t(), out=y)

    arms = {"pair": lambda: reprefill(pool, x, w, blocks, stream=s),
            "single": lambda: reprefill(pool, x, w, blocks, stream=s, single_cta=True)}
    if not a.no_cublas:
        arms["cublas"] = cublas
    # interleaved rounds (pair, single, cuBLAS, pair, ...) so every arm sees the same
    # thermal / power state; the median round per arm is reported
    samples = {k: [] for k in arms}
    with torch.cuda.stream(s):
        for _ in range(a.rounds):
            for k, fn in arms.items():
                samples[k].append(timeit(fn))
    med = {k: sorted(v)[len(v) // 2] for k, v in samples.items()}
    ms, ms1 = med["pair"], med["single"]
    out = {"kernel": "reprefill_pair_kernel (tcgen05 cta_group::2)", "shape": a.shape, "rows": rows,
           "kv_only": a.kv_only, "flops": flops, "ms": round(ms, 4),
           "tflops": round(flops / ms / 1e9, 1),
           "single_cta_ms": round(ms1, 4), "single_cta_tflops": round(flops / ms1 / 1e9, 1),
           "rounds": a.rounds, "iters_per_round": a.iters}
    if "cublas" in med:
        out["cublas_ms"] = round(med["cublas"], 4)
        out["cublas_tflops"] = round(flops / med["cublas"] / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
