"""Small-move issue cost of kvm_migrate (DESIGN.md §11 item 3).

    python tools/bench_issue.py [--calls 2000] [--json out.json]

One move of n blocks of a 7B pool (512 KiB per block) between two pools on
cuda:0, block lists on the host (KVM_F_BLOCKS_ON_HOST, the live-migration
path) or on the device.  Reports per call:
  host_us   host time of one ctypes kvm_migrate call in a back-to-back loop
            (the GPU keeps up for small n, so this is the issue cost);
  lat_us    device time from an event recorded just before the call to one
            recorded just after it, one call at a time with the stream idle
            (what a paused request waits for, minus host issue);
  ctypes_us an empty ctypes call (kvm_version) for scale.
"""
import argparse
import ctypes
import itertools
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B, KVPool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    lib = _native.lib()
    nb = 600
    src, dst = KVPool(LLAMA2_7B, nb), KVPool(LLAMA2_7B, nb)
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    t0 = time.perf_counter()
    for _ in range(a.calls):
        lib.kvm_version()
    ctypes_us = (time.perf_counter() - t0) / a.calls * 1e6
    rows = []
    engines = {"bulk": _native.KVM_F_ENGINE_BULK, "ldg": 0}
    for n, (eng, eflag), on_host in itertools.product((1, 4, 16, 64, 256), engines.items(), (True, False)):
        sb = np.arange(n, dtype=np.int32)
        db = np.arange(nb - n, nb, dtype=np.int32)
        if on_host:
            ps, pd = sb.ctypes.data, db.ctypes.data
            flags = _native.KVM_F_BLOCKS_ON_HOST | eflag
        else:
            tsb, tdb = torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()
            ps, pd = tsb.data_ptr(), tdb.data_ptr()
            flags = eflag
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, n, 1
        m.src_blocks, m.dst_blocks = ps, pd
        mp = ctypes.byref(m)
        calls = a.calls if n <= 16 else max(50, a.calls // (n // 8))
        for _ in range(20):
            lib.kvm_migrate(mp, 1, flags, sp)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(calls):
            lib.kvm_migrate(mp, 1, flags, sp)
        host_us = (time.perf_counter() - t0) / calls * 1e6
        torch.cuda.synchronize()
        gpu_us = (time.perf_counter() - t0) / calls * 1e6
        lats = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(50):
            torch.cuda.synchronize()
            e0.record(s)
            lib.kvm_migrate(mp, 1, flags, sp)
            e1.record(s)
            e1.synchronize()
            lats.append(e0.elapsed_time(e1) * 1e3)
        row = {"n_blocks": n, "engine": eng, "blocks_on_host": on_host, "host_us": round(host_us, 2),
               "throughput_us": round(gpu_us, 2), "lat_us": round(statistics.median(lats), 2),
               "MiB": n * LLAMA2_7B.kv_bytes_per_token * 16 / 2 ** 20}
        rows.append(row)
        print(json.dumps(row), flush=True)
    # one block, host lists, with completion consumers (table row + done flag):
    # .gpu scope derived per call (pointer checks) vs forced .sys (no checks)
    from paper_2501_06709_b200.kvcache import BlockTable

    table = BlockTable(1, 4)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    sb, db = np.array([1], dtype=np.int32), np.array([nb - 1], dtype=np.int32)
    for label, extra in (("tracked_gpu_scope", 0), ("tracked_sys_scope", _native.KVM_F_SYS_SCOPE)):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, 1, 1
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
        m.dst_table_row, m.done_flag = table.row_ptr(0), flag.data_ptr()
        mp = ctypes.byref(m)
        flags = _native.KVM_F_BLOCKS_ON_HOST | _native.KVM_F_ENGINE_BULK | extra
        for _ in range(20):
            lib.kvm_migrate(mp, 1, flags, sp)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.calls):
            lib.kvm_migrate(mp, 1, flags, sp)
        host_us = (time.perf_counter() - t0) / a.calls * 1e6
        torch.cuda.synchronize()
        lats = []
        for _ in range(50):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            lib.kvm_migrate(mp, 1, flags, sp)
            e1.record(s)
            e1.synchronize()
            lats.append(e0.elapsed_time(e1) * 1e3)
        row = {"n_blocks": 1, "variant": label, "host_us": round(host_us, 2),
               "lat_us": round(statistics.median(lats), 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    out = {"ctypes_us": round(ctypes_us, 3), "rows": rows, "device": torch.cuda.get_device_name(0)}
    print(json.dumps({"ctypes_us": out["ctypes_us"]}))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
