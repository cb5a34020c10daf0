"""configs[3] analogue on one GPU: K concurrent moves (default 8 x 70B-GQA
16k-token requests, 5 GiB each) in ONE fused kvm_migrate launch, versus K
separate launches.  Each move has its own src and dst pool.

    python tools/bench_concurrent.py [--moves 8] [--workload 70b-16k] [--iters 5]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402

WL = {"70b-16k": ("llama3-70b-gqa", 16384), "7b-4k": ("llama2-7b", 4096), "13b-8k": ("llama2-13b", 8192)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--moves", type=int, default=8)
    ap.add_argument("--workload", default="70b-16k", choices=sorted(WL))
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per request")
    a = ap.parse_args()
    shape, tokens = SHAPES[WL[a.workload][0]], a.tokens or WL[a.workload][1]
    n = tokens // 16
    pools = [(KVPool(shape, n), KVPool(shape, n)) for _ in range(a.moves)]
    sb = np.arange(n, dtype=np.int32)[::-1].copy()
    db = np.arange(n, dtype=np.int32)
    sbd, dbd = torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()
    moves = []
    for s, d in pools:
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = s.pool_id, d.pool_id, n, 1
        m.src_blocks, m.dst_blocks = sbd.data_ptr(), dbd.data_ptr()
        moves.append(m)
    arr = (_native.Move * len(moves))(*moves)
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    L = _native.lib()

    def fused():
        _native.check(L.kvm_migrate(arr, len(moves), _native.KVM_F_ENGINE_BULK, sp))

    def separate():
        for i in range(len(moves)):
            _native.check(L.kvm_migrate(ctypes.byref(arr[i]), 1, _native.KVM_F_ENGINE_BULK, sp))

    def t(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters

    kv = tokens * shape.kv_bytes_per_token * a.moves
    tf, ts = t(fused), t(separate)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(json.dumps({"workload": f"{a.moves} x {shape.name} {tokens}-token moves, one GPU", "kv_bytes": kv,
                      "fused_ms": round(tf, 3), "separate_ms": round(ts, 3),
                      "fused_payload_GBps": round(kv / tf / 1e6, 1),
                      "fused_hbm_frac": round(2 * kv / tf / 1e6 / peak, 3)}))


if __name__ == "__main__":
    main()
