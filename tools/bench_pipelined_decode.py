"""Migration -> first decode step, sequential vs layer-pipelined.

    python tools/bench_pipelined_decode.py [--shape llama2-7b] [--seq 4096] [--reps 20]
                                           [--src-dev 0 --dst-dev 1] [--out f.json]

sequential: kvm_migrate of the request, then kvm_paged_decode over the
destination, on one stream.  pipelined: the copy on one stream publishing
per-layer flags, the decode on another with KVM_DECODE_WAIT_LAYERS (layer l
decoded as soon as its KV landed).  Time = event before the copy -> event
after the decode (both streams joined), median over reps.  On one GPU both
kernels are HBM-bound, so the overlap has little to hide; across GPUs
(--src-dev != --dst-dev: one process, peer access, the copy kernel on the
source GPU storing into the destination's pool over NVLink and releasing the
layer flags there) the copy is link-bound and the decode of layer l runs on
the destination under the copy of later layers.  Every event of a timed
interval is recorded on the destination GPU (the copy stream waits on the
start event), so time-to-first-token is measured on one device clock.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.attention import paged_decode  # noqa: E402
from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama2-7b")
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    sh = SHAPES[a.shape]
    k = (a.seq + 15) // 16
    nb = k + 8
    lib = _native.lib()
    if a.src_dev != a.dst_dev:
        _native.check(lib.kvm_init(1), "kvm_init(enable_peer_access)")
    S, Dd = f"cuda:{a.src_dev}", f"cuda:{a.dst_dev}"
    src, dst = KVPool(sh, nb, device=a.src_dev), KVPool(sh, nb, device=a.dst_dev)
    src.tensor.normal_()
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:k].to(torch.int32).to(S)
    db = torch.randperm(nb, generator=torch.Generator().manual_seed(2))[:k].to(torch.int32).to(Dd)
    q = torch.randn(sh.layers, 1, sh.q_heads, 128, device=Dd).half()
    lens = torch.tensor([a.seq], dtype=torch.int32, device=Dd)
    table = db[None].contiguous()
    flags = torch.zeros(sh.layers, dtype=torch.int32, device=Dd)
    err = torch.zeros(1, dtype=torch.int32, device=Dd)
    out = torch.empty_like(q)
    cs, ds = torch.cuda.Stream(device=a.src_dev), torch.cuda.Stream(device=a.dst_dev)
    # the copy reads the destination's block list from the source GPU (peer read of 4 KiB)

    def sync():
        torch.cuda.synchronize(a.src_dev)
        torch.cuda.synchronize(a.dst_dev)

    def migrate(stream, value):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, k, value
        m.src_blocks, m.dst_blocks, m.layer_flags = sb.data_ptr(), db.data_ptr(), flags.data_ptr()
        _native.check(lib.kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_ENGINE_BULK, ctypes.c_void_p(stream.cuda_stream)))

    seq_ms, pipe_ms, copy_ms, dec_ms = [], [], [], []
    value = 0
    for r in range(a.reps + 3):
        # sequential: the copy (source GPU), then the decode (destination GPU) after it
        value += 1
        sync()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(ds)
        cs.wait_event(e0)
        migrate(cs, value)
        c1 = torch.cuda.Event()
        c1.record(cs)
        ds.wait_event(c1)
        e1.record(ds)
        paged_decode(dst, q, table, lens, out, max_seq_len=a.seq, stream=ds)
        e2.record(ds)
        e2.synchronize()
        # pipelined: the decode of layer l starts when the copy released layer l's flag
        value += 1
        sync()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(ds)
        cs.wait_event(p0)
        migrate(cs, value)
        paged_decode(dst, q, table, lens, out, max_seq_len=a.seq, stream=ds, layer_flags=flags, layer_value=value,
                     timeout_ns=5_000_000_000, err_word=err)
        c2 = torch.cuda.Event()
        c2.record(cs)
        ds.wait_event(c2)
        p1.record(ds)
        p1.synchronize()
        if r >= 3:
            seq_ms.append(e0.elapsed_time(e2))
            copy_ms.append(e0.elapsed_time(e1))
            dec_ms.append(e1.elapsed_time(e2))
            pipe_ms.append(p0.elapsed_time(p1))
    assert err.item() == 0, "layer wait timed out"
    med = statistics.median
    line = json.dumps({"shape": a.shape, "seq": a.seq, "layers": sh.layers, "src_dev": a.src_dev,
                       "dst_dev": a.dst_dev, "kv_bytes": a.seq * sh.kv_bytes_per_token,
                       "copy_ms": round(med(copy_ms), 4), "decode_ms": round(med(dec_ms), 4),
                       "sequential_ms": round(med(seq_ms), 4), "pipelined_ms": round(med(pipe_ms), 4),
                       "saved_ms": round(med(seq_ms) - med(pipe_ms), 4),
                       "copy_GBps": round(a.seq * sh.kv_bytes_per_token / med(copy_ms) / 1e6, 1),
                       "definition": "event on the destination GPU before the copy -> event there after the decode "
                                     "of every layer (time to the first decode step after the migration)"})
    print(line)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
