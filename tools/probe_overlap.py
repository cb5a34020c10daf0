"""Probe: does the capped LDG copy co-run with the persistent re-prefill GEMM?"""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2501_06709_b200 import _native
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights

shape = LLAMA2_13B
nblk = 421
src = KVPool(shape, 512, dtype=torch.bfloat16); dst = KVPool(shape, 1100, dtype=torch.bfloat16)
sb = np.arange(0, 421, dtype=np.int32); db = np.arange(600, 1021, dtype=np.int32)
rows = 1456
dbt = torch.arange(0, 600, dtype=torch.int32, device="cuda")
x = synthetic_hidden(shape, rows, 0); w = synthetic_weights(shape, 0)
sa, sbs = torch.cuda.Stream(), torch.cuda.Stream()
def copy(stream, flags):
    m = _native.Move(); m.src_pool, m.dst_pool, m.n_blocks = src.pool_id, dst.pool_id, nblk
    m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
    _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | flags, ctypes.c_void_p(stream.cuda_stream)))
def gemm(stream):
    reprefill(dst, x, w, dbt, tok0=8192 - rows, stream=stream)
def t(fn, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sbs)
    for _ in range(it): fn()
    e1.record(sbs); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / it, 3)
def both(cap, first, eng):
    def f():
        ev = torch.cuda.Event(); ev.record(sbs); sa.wait_event(ev)
        if first == "gemm": gemm(sbs); copy(sa, _native.KVM_F_CTAS_PER_SM(cap) | eng)
        else: copy(sa, _native.KVM_F_CTAS_PER_SM(cap) | eng); gemm(sbs)
        ev2 = torch.cuda.Event(); ev2.record(sa); sbs.wait_event(ev2)
    return f
out = {"gemm": t(lambda: gemm(sbs)), "copy_bulk": t(lambda: copy(sbs, _native.KVM_F_ENGINE_BULK))}
EF = _native.KVM_F_L2_EVICT_FIRST
out["copy_bulk_ef"] = t(lambda: copy(sbs, _native.KVM_F_ENGINE_BULK | EF))
for cap in (2, 3):
    out[f"copy_ldg_ef_cap{cap}"] = t(lambda: copy(sbs, _native.KVM_F_CTAS_PER_SM(cap) | EF))
    out[f"both_ef_cap{cap}_gemmfirst"] = t(both(cap, "gemm", EF))
for cap in (1, 2, 3):
    out[f"copy_ldg_cap{cap}"] = t(lambda: copy(sbs, _native.KVM_F_CTAS_PER_SM(cap)))
    for first in ("gemm", "copy"):
        out[f"both_cap{cap}_{first}first"] = t(both(cap, first, 0))
print(json.dumps(out))
