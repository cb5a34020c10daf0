"""Break down the e2e step of bench.py (MigrationExecutor.compact with host block
lists + D2H of the table row) into host phases, to see what the ~50 us above the
kernel time is.  Diagnostic only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200.executor import MigrationExecutor, Residency  # noqa: E402
from paper_2501_06709_b200.kvcache import SHAPES, BlockTable, KVPool  # noqa: E402

shape = SHAPES["llama2-7b"]
n, nb = 256, 1024
pool = KVPool(shape, nb)
table = BlockTable(4, n)
ex = MigrationExecutor({0: pool}, {0: table})
sb = np.arange(0, 2 * n, 2, dtype=np.int32)
pool.allocator.take(sb)
ex.loc[0] = Residency(0, sb.copy(), n * 16, shape.name)
table.set_host(0, sb)
row = torch.empty(n, dtype=torch.int32, pin_memory=True)
for _ in range(5):
    ex.compact(0, row_out=row)
torch.cuda.synchronize()
K = 50
t_total = 0.0
t_launch = 0.0
for i in range(K):
    t0 = time.perf_counter()
    rec = ex.compact(0, wait=False, row_out=row)
    t1 = time.perf_counter()
    ex.stream(0).synchronize()
    ex.commit()
    t2 = time.perf_counter()
    t_launch += t1 - t0
    t_total += t2 - t0
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = ex.stream(0)
ev0.record(s)
for i in range(K):
    ex.compact(0, wait=False)
    ex.commit()
ev1.record(s)
torch.cuda.synchronize()
print({"host_issue_us": 1e6 * t_launch / K, "step_us": 1e6 * t_total / K,
       "device_back_to_back_us": 1e3 * ev0.elapsed_time(ev1) / K})


def timed(fn, k=200):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    dt = (time.perf_counter() - t) / k
    torch.cuda.synchronize()
    return round(1e6 * dt, 2)


import ctypes  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402

a = pool.allocator
blocks = ex.where(0).blocks


def alloc_free():
    x = a.alloc(n)
    a.free(x)


db = np.arange(1, 2 * n, 2, dtype=np.int32)
lib = _native.lib()
sp = ctypes.c_void_p(s.cuda_stream)


def raw_compact_tiny():   # 1 block: launch + staging cost without the copy itself
    lib.kvm_compact(pool.pool_id, sb.ctypes.data, db.ctypes.data, 1, None,
                    _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK, sp)


def row_copy():
    with torch.cuda.stream(s):
        row[:n].copy_(table.rows[table.slot(0), :n], non_blocking=True)


print({"alloc_free_us": timed(alloc_free), "ordered_stream_us": timed(lambda: ex.ordered_stream(0)),
       "kvm_compact_1block_us": timed(raw_compact_tiny), "row_copy_us": timed(row_copy),
       "set_host_us": timed(lambda: table.set_host(0, blocks))})
