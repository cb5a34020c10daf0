"""The push kernel against a REMOTE link it can measure on a one-GPU box: PCIe
to pinned host memory (KV swap-out / swap-in).

Every gpurun box has one B200, so the NVLink hop of the N > 1 push has no
measurement here.  This tool runs the same kvm_migrate kernels with the
destination (or source) pool in pinned host memory: the stores (loads) then
leave the GPU over a link, system-scope completion included, exactly the
code path of a peer pool except for the link.  Question answered: does the
SM-driven push saturate a link that is ~100x slower than HBM, against the
link's own roofline (one contiguous cudaMemcpyAsync of the same byte count,
copy engine) and the library way vLLM swaps KV blocks (swap_blocks per
(layer, K|V) plane, one cudaMemcpyAsync per block)?

    python tools/bench_host_link.py [--tokens 1024] [--iters 5] [--out f.json]

One JSON line: GB/s of payload per arm and direction, the contiguous-copy
roofline, each arm's fraction of it, and bit-exactness of every arm.
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
from paper_2501_06709_b200.kvcache import LLAMA2_7B, BlockTable, KVPool  # noqa: E402


def timed(fn, iters, warmup=2, stream=None):
    s = stream or torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    s.synchronize()
    out = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    shape = LLAMA2_7B
    n = a.tokens // shape.block_tokens
    kv_bytes = n * shape.block_tokens * shape.kv_bytes_per_token
    lib = _native.lib()
    st = torch.cuda.Stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    g = torch.Generator().manual_seed(0)
    gpu_nb, host_nb = 3 * n, n + 8
    gpu = KVPool(shape, gpu_nb, device=0)
    gpu.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    host_t = torch.empty((shape.layers, 2, host_nb) + gpu.view_shape[3:], dtype=torch.float16).pin_memory()
    host_t.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    host = KVPool(shape, host_nb, device=0, tensor=host_t)
    gb = torch.randperm(gpu_nb, generator=g)[:n].numpy().astype(np.int32)     # scattered GPU blocks
    hb = torch.randperm(host_nb, generator=g)[:n].numpy().astype(np.int32)    # scattered host blocks
    table = BlockTable(2, n)
    flag = torch.zeros(4, dtype=torch.int32).pin_memory()                     # host-visible done flag
    seq = [0]

    def ours(engine, out_dir):
        def run():
            m = _native.Move()
            src, dst, sb, db = (gpu, host, gb, hb) if out_dir else (host, gpu, hb, gb)
            m.src_pool, m.dst_pool, m.n_blocks = src.pool_id, dst.pool_id, n
            m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
            seq[0] += 1
            m.dst_table_row, m.done_flag, m.done_value = table.row_ptr(0), flag.data_ptr(), seq[0]
            _native.check(lib.kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST | engine, sp))
        return run

    def scramble(out_dir):
        # the destination blocks get fresh bits first, so an arm that moved nothing cannot pass
        if out_dir:
            host.tensor[:, :, torch.from_numpy(hb).long()] = torch.randn(
                shape.layers, 2, n, *gpu.view_shape[3:], generator=g).half()
        else:
            gpu.tensor[:, :, torch.from_numpy(gb).long().cuda()] = torch.randn(
                shape.layers, 2, n, *gpu.view_shape[3:], device="cuda").half()
        torch.cuda.synchronize()

    def expect_out():
        return torch.equal(host.tensor[:, :, torch.from_numpy(hb).long()].view(torch.int16),
                           gpu.tensor[:, :, torch.from_numpy(gb).long().cuda()].cpu().view(torch.int16))

    res = {"workload": f"7B KV, {a.tokens} tokens ({n} blocks, {kv_bytes} B) between a B200 pool and a "
                       f"pinned-host pool, scattered blocks both sides", "kv_bytes": kv_bytes, "ms": {},
           "GBps": {}, "bit_exact": {}}
    # link roofline: one contiguous copy of kv_bytes each way (copy engine)
    dbuf = torch.empty(kv_bytes // 2, dtype=torch.float16, device="cuda")
    hbuf = torch.empty(kv_bytes // 2, dtype=torch.float16).pin_memory()
    with torch.cuda.stream(st):
        res["ms"]["contiguous_d2h"] = timed(lambda: hbuf.copy_(dbuf, non_blocking=True), a.iters, stream=st)
        res["ms"]["contiguous_h2d"] = timed(lambda: dbuf.copy_(hbuf, non_blocking=True), a.iters, stream=st)
    arms = [("ours_bulk_d2h", ours(_native.KVM_F_ENGINE_BULK, True), True),
            ("ours_ldg_d2h", ours(0, True), True),
            ("ours_bulk_h2d", ours(_native.KVM_F_ENGINE_BULK, False), False),
            ("ours_ldg_h2d", ours(0, False), False)]
    for name, fn, out_dir in arms:
        try:
            scramble(out_dir)
            res["ms"][name] = timed(fn, a.iters, stream=st)
            st.synchronize()
            if out_dir:
                res["bit_exact"][name] = expect_out() and int(flag[0]) == seq[0] and \
                    np.array_equal(table.rows[0, :n].cpu().numpy(), hb)
            else:
                res["bit_exact"][name] = expect_out() and int(flag[0]) == seq[0] and \
                    np.array_equal(table.rows[0, :n].cpu().numpy(), gb)
        except Exception as e:   # an engine the link refuses is reported, not fatal
            res.setdefault("errors", {})[name] = repr(e)[:300]
    try:
        import vllm._custom_ops as vops
        piece = shape.piece_bytes
        m_out = torch.from_numpy(np.stack([gb, hb], 1).astype(np.int64))
        m_in = torch.from_numpy(np.stack([hb, gb], 1).astype(np.int64))
        gplanes = [gpu.tensor[l, kv] for l in range(shape.layers) for kv in range(2)]
        hplanes = [host.tensor[l, kv] for l in range(shape.layers) for kv in range(2)]

        def vllm_out():
            for gpl, hpl in zip(gplanes, hplanes):
                vops.swap_blocks(gpl, hpl, piece, m_out)

        def vllm_in():
            for gpl, hpl in zip(gplanes, hplanes):
                vops.swap_blocks(hpl, gpl, piece, m_in)
        with torch.cuda.stream(st):
            scramble(True)
            res["ms"]["vllm_swap_blocks_d2h"] = timed(vllm_out, a.iters, stream=st)
            st.synchronize()
            res["bit_exact"]["vllm_swap_blocks_d2h"] = expect_out()
            scramble(False)
            res["ms"]["vllm_swap_blocks_h2d"] = timed(vllm_in, a.iters, stream=st)
            st.synchronize()
            res["bit_exact"]["vllm_swap_blocks_h2d"] = expect_out()
    except Exception as e:
        res.setdefault("errors", {})["vllm"] = repr(e)[:300]
    for k, ms in res["ms"].items():
        res["ms"][k] = round(ms, 4)
        res["GBps"][k] = round(kv_bytes / ms / 1e6, 2)
    roof = {"d2h": res["GBps"]["contiguous_d2h"], "h2d": res["GBps"]["contiguous_h2d"]}
    res["link_roofline_GBps"] = roof
    res["frac_of_link"] = {k: round(v / roof["d2h" if "d2h" in k else "h2d"], 3)
                           for k, v in res["GBps"].items() if not k.startswith("contiguous")}
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
