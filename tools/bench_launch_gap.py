"""Back-to-back kvm_migrate launches with and without a CUDA event pair around each launch
(and with / without completion tracking): what per-launch timing events cost a throughput loop.

    python tools/bench_launch_gap.py

7B compaction ping-pong, 32 and 256 blocks, 200 launches; prints one JSON object of us/step and GB/s.
"""
import ctypes, sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2501_06709_b200 import _native
from paper_2501_06709_b200.kvcache import LLAMA2_7B, KVPool, BlockTable
lib = _native.lib(); st = torch.cuda.Stream(); sp = ctypes.c_void_p(st.cuda_stream)
out = {}
for n in (32, 256):
    pool = KVPool(LLAMA2_7B, 4 * n + 8); pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    sb = torch.arange(n, dtype=torch.int32, device="cuda"); db = torch.arange(2 * n, 3 * n, dtype=torch.int32, device="cuda")
    table = BlockTable(2, n); flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    kv = n * 16 * LLAMA2_7B.kv_bytes_per_token
    for tracked in (False, True):
        seq = [0]
        def step(i):
            m = _native.Move(); m.src_pool = m.dst_pool = pool.pool_id; m.n_blocks = n
            a, b = (sb, db) if i % 2 == 0 else (db, sb)
            m.src_blocks, m.dst_blocks = a.data_ptr(), b.data_ptr()
            if tracked:
                seq[0] += 1; m.dst_table_row, m.done_flag, m.done_value = table.row_ptr(0), flag.data_ptr(), seq[0]
            _native.check(lib.kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_ENGINE_BULK, sp))
        for ev_between in (False, True):
            for i in range(10): step(i)
            st.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(400)]
            t0.record(st)
            for i in range(200):
                if ev_between: evs[2 * i].record(st)
                step(i)
                if ev_between: evs[2 * i + 1].record(st)
            t1.record(st); t1.synchronize()
            ms = t0.elapsed_time(t1) / 200
            out[f"{n}blk tracked={tracked} events={ev_between}"] = {"us_per_step": round(ms * 1e3, 2), "GBps": round(kv / ms / 1e6, 1)}
    del pool
print(json.dumps(out))
