"""BASELINE configs[2]: Llama-2-13B KV, 8k tokens, adaptive split (partial KV
transfer + tcgen05 re-prefill, overlapped).  One JSON line.

    python tools/bench_split.py [--tokens 8192] [--suffix S] [--iters 10]

On one B200 both halves share the GPU: the persistent re-prefill GEMM is
launched first (1 CTA/SM, tensor-bound) and the prefix copy (LDG engine, capped
CTAs/SM, HBM-bound) fills the remaining SM slots.  On two GPUs the halves run
on different devices (K1 on the source, K3 on the destination).  The split
point comes from reprefill.split_point with the NVLink link rate (so the
suffix is what a 2-GPU deployment would re-prefill) unless --suffix is given.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import reprefill, split_point, synthetic_hidden, synthetic_weights  # noqa: E402
from paper_2501_06709_b200.split import (flops_per_token, make_split, split_migrate,  # noqa: E402
                                         split_migrate_fused, wait_split)

NVLINK_GBS = 770e9
TENSOR_FLOPS = 1.28e15  # measured kvm_reprefill rate on 13B (tools/bench_reprefill.py)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--suffix", type=int, default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ctas-per-sm", type=int, default=3)
    a = ap.parse_args()
    shape = LLAMA2_13B
    n = a.tokens
    fpt = flops_per_token(shape, with_q=True)
    s = a.suffix if a.suffix is not None else split_point(n, shape.kv_bytes_per_token, NVLINK_GBS, fpt,
                                                          TENSOR_FLOPS)
    plan = make_split(n, s)
    nblk = plan.total_blocks
    nb = nblk + 64
    src = KVPool(shape, nb, dtype=torch.bfloat16)
    dst = KVPool(shape, nb, dtype=torch.bfloat16)
    for p, seed in ((src, 1), (dst, 2)):
        g = torch.Generator(device="cuda").manual_seed(seed)
        v = p.tensor.view(torch.int16).view(-1)
        step = 1 << 28
        for i in range(0, v.numel(), step):
            k = min(step, v.numel() - i)
            v[i:i + k] = torch.randint(-2 ** 15, 2 ** 15 - 1, (k,), generator=g, device="cuda", dtype=torch.int16)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:nblk].to(torch.int32).numpy()
    dst.allocator.take(np.random.default_rng(2).permutation(nb)[: 32])
    db = torch.from_numpy(dst.allocator.alloc(nblk)).cuda()
    x = synthetic_hidden(shape, max(plan.suffix, 1), 0, seed=2)[:plan.suffix].contiguous()
    w = synthetic_weights(shape, 0, with_q=True, seed=3)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    sa, sbs = torch.cuda.Stream(), torch.cuda.Stream()
    kv_bytes = n * shape.kv_bytes_per_token
    cap = _native.KVM_F_CTAS_PER_SM(a.ctas_per_sm)
    seq = [0]

    def run_split(overlap=True):
        seq[0] += 1
        start = torch.cuda.Event()
        start.record(sbs)
        sa.wait_event(start)
        split_migrate(src, dst, sb, db, plan, x, w, xfer_stream=sa if overlap else sbs, rp_stream=sbs,
                      flags_dev=flags, seq=seq[0], engine_flags=cap)
        wait_split(flags, plan, seq[0], sbs)

    def run_full():
        sbh = np.ascontiguousarray(sb)
        dbh = db.cpu().numpy()
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, nblk, 1
        m.src_blocks, m.dst_blocks = sbh.ctypes.data, dbh.ctypes.data
        _native.check(_native.lib().kvm_migrate(ctypes_byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST |
                                                _native.KVM_F_ENGINE_BULK, ctypes_stream(sbs)))

    def run_prefix_only():
        sbh = np.ascontiguousarray(sb[:plan.prefix_blocks])
        dbh = db[:plan.prefix_blocks].cpu().numpy()
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, plan.prefix_blocks, 1
        m.src_blocks, m.dst_blocks = sbh.ctypes.data, dbh.ctypes.data
        _native.check(_native.lib().kvm_migrate(ctypes_byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST |
                                                _native.KVM_F_ENGINE_BULK, ctypes_stream(sbs)))

    sbd = torch.from_numpy(sb).cuda()

    def run_fused():
        split_migrate_fused(src, dst, sbd, db, plan, x, w, stream=sbs)

    def run_suffix_only():
        reprefill(dst, x, w, db, tok0=plan.prefix_tokens, stream=sbs)

    def timeit(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sbs)
        for _ in range(a.iters):
            fn()
        e1.record(sbs)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters

    sbs.wait_stream(torch.cuda.current_stream())   # pools, x and w were produced on the default stream
    sa.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(sbs):
        # parity first: prefix bit-exact, suffix within bf16 tolerance
        run_split(True)
        torch.cuda.synchronize()
        pi = torch.from_numpy(sb[:plan.prefix_blocks]).long().cuda()
        exact = bool(torch.equal(dst.tensor[:, :, db[:plan.prefix_blocks].long()].view(torch.int16),
                                 src.tensor[:, :, pi].view(torch.int16)))
        worst = 0.0
        if plan.suffix:
            kvd, qc = shape.kv_cols, shape.q_cols
            toks = torch.arange(plan.prefix_tokens, n, device="cuda")
            blk, slot = db.long()[toks // 16], toks % 16
            for l in (0, shape.layers // 2, shape.layers - 1):
                ref = x.float() @ w[l].float().t()
                for kv, lo in ((0, qc), (1, qc + kvd)):
                    got = dst.tensor[l, kv, blk, slot].reshape(plan.suffix, kvd).float()
                    r = ref[:, lo:lo + kvd]
                    worst = max(worst, float(((got - r).abs() - 1.6e-2 * r.abs()).max()))
        # fused one-launch variant: parity again, then timing
        dst.tensor.view(torch.int16).zero_()
        run_fused()
        torch.cuda.synchronize()
        exact_fused = bool(torch.equal(dst.tensor[:, :, db[:plan.prefix_blocks].long()].view(torch.int16),
                                       src.tensor[:, :, pi].view(torch.int16)))
        t_fused = timeit(run_fused)
        t_fused_single = timeit(lambda: split_migrate_fused(src, dst, sbd, db, plan, x, w, stream=sbs,
                                                            single_cta=True))
        t_split = timeit(lambda: run_split(True))
        t_serial = timeit(lambda: run_split(False))
        t_full = timeit(run_full)
        t_prefix = timeit(run_prefix_only)
        t_suffix = timeit(run_suffix_only) if plan.suffix else 0.0
    out = {
        "config": "configs[2]: Llama-2-13B KV, 8k tokens, adaptive split", "tokens": n,
        "suffix_reprefilled": plan.suffix, "prefix_blocks": plan.prefix_blocks,
        "kv_bytes": kv_bytes, "prefix_bytes": plan.prefix_tokens * shape.kv_bytes_per_token,
        "suffix_flops": plan.suffix * fpt,
        "ms": {"split_fused_one_kernel": round(t_fused, 4),
               "split_fused_one_kernel_single_cta_gemm": round(t_fused_single, 4),
               "split_overlapped_1gpu": round(t_split, 4), "split_serialized_1gpu": round(t_serial, 4),
               "full_transfer_1gpu": round(t_full, 4), "prefix_transfer_only": round(t_prefix, 4),
               "suffix_reprefill_only": round(t_suffix, 4)},
        "overlap_efficiency_two_streams": round((t_prefix + t_suffix) / t_split, 3) if t_split else None,
        "overlap_efficiency_fused": round((t_prefix + t_suffix) / t_fused, 3) if t_fused else None,
        "fused_prefix_bit_exact": exact_fused,
        "suffix_tflops": round(plan.suffix * fpt / t_suffix / 1e9, 1) if t_suffix else None,
        "model_2gpu_ms": {"full_transfer_nvlink": round(kv_bytes / NVLINK_GBS * 1e3, 3),
                          "split": round(max(plan.prefix_tokens * shape.kv_bytes_per_token / NVLINK_GBS,
                                             plan.suffix * fpt / TENSOR_FLOPS) * 1e3, 3)},
        "prefix_bit_exact": exact, "suffix_within_tolerance": worst <= 1e-2, "suffix_worst_excess": worst,
    }
    print(json.dumps(out))


def ctypes_byref(m):
    import ctypes
    return ctypes.byref(m)


def ctypes_stream(s):
    import ctypes
    return ctypes.c_void_p(s.cuda_stream)


if __name__ == "__main__":
    main()
