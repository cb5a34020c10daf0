"""Paged decode on the migrated cache: kvm_paged_decode vs flashinfer's paged
decode (the library path; vLLM-style PagedAttention) on the SAME pool memory.

The pool's per-layer K and V planes are [blocks][16][kv_heads][128], which is
flashinfer's NHD paged layout, so flashinfer reads our blocks in place through
the same block table (CSR page indices).  flashinfer runs one layer per call;
ours covers every layer in one launch.  Outputs are compared (fp32 reference
tolerance of an fp16 softmax-attention) and both are timed with CUDA events.

    python tools/bench_decode_vs_flashinfer.py [--shape llama2-7b] [--batch 1] [--seq 4096]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2501_06709_b200.attention import paged_decode  # noqa: E402
from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama2-7b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    sh = SHAPES[a.shape]
    L = sh.layers
    nblk = (a.seq + 15) // 16
    nb = nblk * a.batch + 8
    pool = KVPool(sh, nb)
    pool.tensor.normal_()
    g = torch.Generator().manual_seed(0)
    table = torch.randperm(nb, generator=g)[: nblk * a.batch].to(torch.int32).view(a.batch, nblk).cuda()
    lens = torch.full((a.batch,), a.seq, dtype=torch.int32, device="cuda")
    q = torch.randn(L, a.batch, sh.q_heads, 128, device="cuda").half()
    out = torch.empty_like(q)
    byts = 2 * a.seq * sh.kv_heads * 128 * 2 * L * a.batch

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters

    res = {"shape": a.shape, "batch": a.batch, "seq": a.seq, "layers": L, "bytes": byts}
    ms = timeit(lambda: paged_decode(pool, q, table, lens, out, max_seq_len=a.seq))
    res["ours"] = {"ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1), "launches": 1}
    try:
        import flashinfer
    except Exception as e:  # library absent: report, do not fail
        res["flashinfer"] = {"unavailable": str(e)[:200]}
        print(json.dumps(res))
        return
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dec = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    indptr = torch.arange(0, (a.batch + 1) * nblk, nblk, dtype=torch.int32, device="cuda")
    last = torch.full((a.batch,), a.seq - (nblk - 1) * 16, dtype=torch.int32, device="cuda")
    dec.plan(indptr, table.reshape(-1).contiguous(), last, sh.q_heads, sh.kv_heads, 128, 16,
             pos_encoding_mode="NONE", q_data_type=torch.float16, kv_data_type=torch.float16)
    fi_out = torch.empty_like(q)

    def fi():
        for l in range(L):
            fi_out[l] = dec.run(q[l], (pool.tensor[l, 0], pool.tensor[l, 1]))

    ms_fi = timeit(fi)
    res["flashinfer"] = {"version": flashinfer.__version__, "ms": round(ms_fi, 4),
                         "GBps": round(byts / ms_fi / 1e6, 1), "launches": L}
    paged_decode(pool, q, table, lens, out, max_seq_len=a.seq)
    fi()
    torch.cuda.synchronize()
    diff = (out.float() - fi_out.float()).abs().max().item()
    res["max_abs_diff_vs_flashinfer"] = diff
    res["agree"] = bool(torch.allclose(out.float(), fi_out.float(), atol=2e-3, rtol=2e-2))
    res["speedup_vs_flashinfer"] = round(ms_fi / ms, 3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
