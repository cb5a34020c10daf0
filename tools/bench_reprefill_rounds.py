"""Re-prefill (13B, 1 360-token suffix, QKV, 40 layers) vs cuBLAS on the same shape, in rounds from a
cool start: how the comparison moves as the board settles at its power limit.

    python tools/bench_reprefill_rounds.py

Three interleaved rounds of (ours, cuBLAS) on a side stream and on the default stream; per arm the
median ms of 3 reps x 3 back-to-back launches.  One JSON line of per-round ms.
"""
import sys, os, time, json, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool
from paper_2501_06709_b200.reprefill import reprefill, reprefill_flops, synthetic_hidden, synthetic_weights
sh, rows = LLAMA2_13B, 1360
nblk = (rows + 15) // 16
pool = KVPool(sh, nblk + 4, dtype=torch.bfloat16)
blocks = torch.arange(nblk, dtype=torch.int32, device="cuda")
x, w = synthetic_hidden(sh, rows, 0), synthetic_weights(sh, 0, with_q=True)
flops = reprefill_flops(sh, rows, with_q=True)
outs = torch.empty(rows, w.shape[1], dtype=torch.bfloat16, device="cuda")
st = torch.cuda.Stream()
def timed(fn, reps=5, iters=3, stream=None):
    s = stream or torch.cuda.current_stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2): fn()
        ms = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(iters): fn()
            e1.record(s); e1.synchronize()
            ms.append(e0.elapsed_time(e1) / iters)
    return statistics.median(ms)
def ours(): reprefill(pool, x, w, blocks, stream=torch.cuda.current_stream())
def cublas():
    for l in range(sh.layers): torch.matmul(x, w[l].t(), out=outs)
def cublas_T():
    wt = w  # [L][n_out][d] -> x @ w^T via mm with transposed view
    for l in range(sh.layers): torch.mm(x, w[l].t(), out=outs)
res = {}
for rnd in range(3):
    for name, fn, strm in (("ours_side", ours, st), ("cublas_side", cublas, st), ("ours_default", ours, None), ("cublas_default", cublas, None)):
        ms = timed(fn, reps=3, stream=strm)
        res.setdefault(name, []).append(round(ms, 3))
print(json.dumps(res))
