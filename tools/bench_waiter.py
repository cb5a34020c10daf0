"""A flag waiter beside the copy kernel: kvm_migrate of a 13B 8k prefix / 7B-4k
request with and without a done flag / table row, with and without a
kvm_wait_flag kernel spinning on that flag on a second stream of the same GPU.
ms per move (10 back-to-back after 3 warm-ups).  profiles/r2_reentry/waiter_interference.md

    python tools/bench_waiter.py
"""
import ctypes, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2501_06709_b200 import _native
from paper_2501_06709_b200.kvcache import LLAMA2_13B, LLAMA2_7B, KVPool, BlockTable
res = {}
for shape, nblk in ((LLAMA2_13B, 421), (LLAMA2_7B, 256)):
    nb = nblk + 64
    src, dst = KVPool(shape, nb), KVPool(shape, nb)
    sb = np.random.default_rng(1).permutation(nb)[:nblk].astype(np.int32)
    db = np.sort(np.random.default_rng(2).permutation(nb)[:nblk]).astype(np.int32)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    table = BlockTable(1, nblk)
    s = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    def run(flag, row, eng, wait, seq=[0]):
        seq[0] += 1
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, nblk, seq[0]
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
        m.done_flag = flags.data_ptr() if flag else None
        m.dst_table_row = table.row_ptr(0) if row else None
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | eng, ctypes.c_void_p(s.cuda_stream)))
        if wait:
            _native.check(_native.lib().kvm_wait_flag(ctypes.c_void_p(flags.data_ptr()), seq[0], ctypes.c_void_p(s2.cuda_stream)))
    for name, args in (("untracked", (0,0)), ("flag", (1,0)), ("row", (0,1)), ("flag+row", (1,1))):
        for eng_name, eng in (("bulk", _native.KVM_F_ENGINE_BULK), ("ldg", 0)):
            for wait in ((False, True) if args[0] else (False,)):
                for _ in range(3): run(*args, eng, wait)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(10): run(*args, eng, wait)
                e1.record(s); torch.cuda.synchronize()
                res[f"{shape.name}/{name}/{eng_name}/wait={wait}"] = round(e0.elapsed_time(e1)/10, 4)
    del src, dst
    torch.cuda.empty_cache()
print(json.dumps(res, indent=0))
