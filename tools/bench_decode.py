"""Paged-attention decode bandwidth (kvm_paged_decode) on the frozen pool layout.

    python tools/bench_decode.py [--shape llama2-7b] [--batch 1] [--seq 4096] [--layers all]

One launch covers n_layers x batch; algorithmic bytes = K+V of every token
read once = 2 * seq * kv_heads * 128 * 2 * layers * batch.  Reports GB/s and
the fraction of the measured HBM copy bandwidth (MEASURED_PEAKS.json).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200.attention import paged_decode  # noqa: E402
from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama2-7b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    sh = SHAPES[a.shape]
    L = a.layers or sh.layers
    nblk = (a.seq + 15) // 16
    nb = nblk * a.batch + 8
    pool = KVPool(sh, nb)
    pool.tensor.normal_()
    perm = torch.randperm(nb)[: nblk * a.batch].to(torch.int32).view(a.batch, nblk).cuda()
    lens = torch.full((a.batch,), a.seq, dtype=torch.int32, device="cuda")
    q = torch.randn(L, a.batch, sh.q_heads, 128, device="cuda").half()
    out = torch.empty_like(q)
    for _ in range(3):
        paged_decode(pool, q, perm, lens, out, max_seq_len=a.seq)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        paged_decode(pool, q, perm, lens, out, max_seq_len=a.seq)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    byts = 2 * a.seq * sh.kv_heads * 128 * 2 * L * a.batch
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(json.dumps({"kernel": "decode_split_kernel", "shape": a.shape, "batch": a.batch, "seq": a.seq,
                      "layers": L, "bytes": byts, "ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1),
                      "frac_of_hbm_copy_peak": round(byts / ms / 1e6 / peak, 3)}))


if __name__ == "__main__":
    main()
