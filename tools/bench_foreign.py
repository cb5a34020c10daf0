"""7B-4k migration between vLLM-layout caches vs native pools (one B200).

    python tools/bench_foreign.py [--reps 30]

Same move (256 scattered blocks, 2 GiB of KV) for: native -> native,
vLLM FlashAttention layout -> same, FlashInfer -> same, FlashAttention ->
native.  Device time per move with CUDA events (block lists on the device,
bulk engine), median over reps; inputs (2 GiB per move) exceed L2.
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
from paper_2501_06709_b200.foreign import StridedKVPool, vllm_cache_shape  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B, KVPool  # noqa: E402


def pool(kind, nb):
    s = LLAMA2_7B
    if kind == "native":
        p = KVPool(s, nb)
        p.tensor.view(torch.int16).random_()
        return p
    caches = [torch.empty(vllm_cache_shape(kind, nb, 16, s.kv_heads, s.head_dim), dtype=torch.float16,
                          device="cuda") for _ in range(s.layers)]
    for c in caches:
        c.view(torch.int16).random_()
    return StridedKVPool.from_vllm(caches, kind)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    nb, n = 640, 256
    rng = np.random.default_rng(0)
    sb = torch.from_numpy(rng.permutation(nb)[:n].astype(np.int32)).cuda()
    db = torch.from_numpy(rng.permutation(nb)[:n].astype(np.int32)).cuda()
    kv_bytes = n * 16 * LLAMA2_7B.kv_bytes_per_token
    out = []
    for src_kind, dst_kind in (("native", "native"), ("flash_attn", "flash_attn"), ("flashinfer", "flashinfer"),
                               ("flash_attn", "native")):
        src, dst = pool(src_kind, nb), pool(dst_kind, nb)
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, 1
        m.src_blocks, m.dst_blocks = sb.data_ptr(), db.data_ptr()
        st = torch.cuda.current_stream()
        times = []
        for r in range(a.reps + 5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_ENGINE_BULK,
                                                    ctypes.c_void_p(st.cuda_stream)))
            e1.record(st)
            e1.synchronize()
            if r >= 5:
                times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        row = {"src": src_kind, "dst": dst_kind, "kv_bytes": kv_bytes, "ms": round(ms, 4),
               "GBps_payload": round(kv_bytes / ms / 1e6, 1), "GBps_rw": round(2 * kv_bytes / ms / 1e6, 1)}
        print(json.dumps(row), flush=True)
        out.append(row)
        del src, dst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
