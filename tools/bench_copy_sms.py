"""How many SMs the push needs: copy throughput against the SM budget
(KVM_F_MAX_SMS), for the HBM-bound compaction and for a link-bound push.

    python tools/bench_copy_sms.py [--out f.json]

Arms, bulk engine (or --engine ldg: n x 4 CTAs of 256 threads), 7B KV: a 7B-4k compaction inside one pool (HBM: 2 bytes
of traffic per payload byte) and a 1 024-token push into pinned host memory
(PCIe: the only link a one-GPU box has), each with the copy capped at
1 .. 148 SMs.  The per-SM rate of the HBM arm at small budgets is what one
SM's bulk-copy pipeline sustains; the link arm shows how few SMs saturate a
link (NVLink's ~0.77 TB/s per direction then needs ~770 / per-SM rate).
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B, KVPool  # noqa: E402

SMS = (1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--engine", choices=["bulk", "ldg"], default="bulk")
    a = ap.parse_args()
    eng = _native.KVM_F_ENGINE_BULK if a.engine == "bulk" else 0
    lib = _native.lib()
    st = torch.cuda.Stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    sh = LLAMA2_7B

    def timed(fn, iters=5):
        fn()
        st.synchronize()
        out = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return statistics.median(out)

    def mover(src, dst, sb, db, cap):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks = src.pool_id, dst.pool_id, len(sb)
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
        flags = _native.KVM_F_BLOCKS_ON_HOST | eng | _native.KVM_F_MAX_SMS(cap)
        return lambda: _native.check(lib.kvm_migrate(ctypes.byref(m), 1, flags, sp))

    res = {"engine": a.engine, "hbm_compaction_7b_4k": {}, "pcie_push_7b_1k": {}}
    n = 256
    pool = KVPool(sh, 2 * n + 8)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    sb = np.arange(n, dtype=np.int32)
    db = np.arange(n + 8, 2 * n + 8, dtype=np.int32)
    kv = n * 16 * sh.kv_bytes_per_token
    for cap in SMS:
        ms = timed(mover(pool, pool, sb, db, cap), iters=3 if cap and cap < 8 else 5)
        res["hbm_compaction_7b_4k"][str(cap or "all")] = {"ms": round(ms, 4), "GBps_payload": round(kv / ms / 1e6, 1)}
    del pool
    n = 64
    gpu = KVPool(sh, n + 8)
    gpu.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    host_t = torch.empty((sh.layers, 2, n + 8) + gpu.view_shape[3:], dtype=torch.float16).pin_memory()
    host = KVPool(sh, n + 8, device=0, tensor=host_t)
    sb = np.arange(n, dtype=np.int32)
    kv = n * 16 * sh.kv_bytes_per_token
    dbuf = torch.empty(kv // 2, dtype=torch.float16, device="cuda")
    hbuf = torch.empty(kv // 2, dtype=torch.float16).pin_memory()
    with torch.cuda.stream(st):
        roof = timed(lambda: hbuf.copy_(dbuf, non_blocking=True))
    res["pcie_contiguous_d2h_GBps"] = round(kv / roof / 1e6, 2)
    for cap in SMS:
        ms = timed(mover(gpu, host, sb, sb, cap), iters=3)
        res["pcie_push_7b_1k"][str(cap or "all")] = {"ms": round(ms, 4), "GBps_payload": round(kv / ms / 1e6, 2)}
    ok = torch.equal(host.tensor[:, :, :n].view(torch.int16), gpu.tensor[:, :, :n].cpu().view(torch.int16))
    res["pcie_bit_exact"] = bool(ok)
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
