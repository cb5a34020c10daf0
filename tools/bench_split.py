"""BASELINE configs[2]: Llama-2-13B KV, 8k tokens, adaptive split (partial KV
transfer + tcgen05 re-prefill, overlapped).  One JSON line.

    python tools/bench_split.py [--tokens 8192] [--suffix S] [--iters 10]
                                [--src-dev 0 --dst-dev 1] [--out file.json]

Source pool on --src-dev, destination pool, hidden states and weights on
--dst-dev.  Arms (CUDA events; on two devices the timed region starts with an
event on the destination stream that the source stream waits on, and ends on
the destination stream after it has waited for both halves' done flags):

  split_fused_one_kernel   kvm_split_migrate on the destination: its idle warp
                           copies (same device) or PULLS (peer device, the
                           source pool registered on the destination through
                           UVA peer access) the prefix while the tensor cores
                           recompute the suffix
  split_two_kernels        kvm_migrate pushing the prefix from the source (its
                           stream) + kvm_reprefill on the destination (its
                           stream), overlapped; serialized variant beside it
  full_transfer            kvm_migrate of every block (the reference's kv_transfer)
  prefix_transfer_only / suffix_reprefill_only

The split point comes from reprefill.split_point with the measured NVLink
peer-copy rate (so the suffix is what a 2-GPU deployment re-prefills) unless
--suffix is given.  Parity first: prefix bit-exact, suffix within the bf16
tolerance of an fp32 torch reference (three layers).
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
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import reprefill, split_point, synthetic_hidden, synthetic_weights  # noqa: E402
from paper_2501_06709_b200.split import (flops_per_token, make_split, split_migrate,  # noqa: E402
                                         split_migrate_fused, wait_split)

NVLINK_BPS = 770e9       # measured peer copy per direction (B200_PROFILING.md)
TENSOR_FLOPS = 1.28e15   # measured kvm_reprefill rate on 13B (tools/bench_reprefill.py)


def _fill(pool, seed):
    dev = pool.device
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(seed)
    v = pool.tensor.view(torch.int16).view(-1)
    step = 1 << 28
    for i in range(0, v.numel(), step):
        k = min(step, v.numel() - i)
        v[i:i + k] = torch.randint(-2 ** 15, 2 ** 15 - 1, (k,), generator=g, device=f"cuda:{dev}",
                                   dtype=torch.int16)


def run_split_bench(tokens: int = 8192, suffix=None, iters: int = 10, warmup: int = 3, src_dev: int = 0,
                    dst_dev: int = 0, force_two: bool = False) -> dict:
    """force_two: run the two-device code path (peer alias of the source pool,
    done-flag waits, two-kernel overlap) even when src_dev == dst_dev, so a
    1-GPU box exercises it."""
    shape = LLAMA2_13B
    n = tokens
    two = src_dev != dst_dev or force_two
    if two:
        _native.check(_native.lib().kvm_init(1), "kvm_init(enable_peer_access)")
    fpt = flops_per_token(shape, with_q=True)
    s = suffix if suffix is not None else split_point(n, shape.kv_bytes_per_token, NVLINK_BPS, fpt, TENSOR_FLOPS)
    plan = make_split(n, s)
    nblk = plan.total_blocks
    nb = nblk + 64
    D = f"cuda:{dst_dev}"
    src = KVPool(shape, nb, device=src_dev, dtype=torch.bfloat16)
    dst = KVPool(shape, nb, device=dst_dev, dtype=torch.bfloat16)
    _fill(src, 1)
    _fill(dst, 2)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:nblk].to(torch.int32).numpy()
    dst.allocator.take(np.random.default_rng(2).permutation(nb)[:32])
    db_np = dst.allocator.alloc(nblk)
    db = torch.from_numpy(db_np).to(D)
    x = synthetic_hidden(shape, max(plan.suffix, 1), dst_dev, seed=2)[:plan.suffix].contiguous()
    w = synthetic_weights(shape, dst_dev, with_q=True, seed=3)
    flags = torch.zeros(4, dtype=torch.int32, device=D)
    s_src = torch.cuda.Stream(device=src_dev)     # the prefix push (source GPU)
    s_dst = torch.cuda.Stream(device=dst_dev)     # re-prefill, waits, timing (destination GPU)
    kv_bytes = n * shape.kv_bytes_per_token
    seq = [0]
    # the fused kernel reads the source pool through a mapping registered on the destination device
    alias = (KVPool(shape, nb, device=dst_dev, dtype=torch.bfloat16, allocator=False, _base_ptr=src.base_ptr)
             if two else src)
    sbd = torch.from_numpy(sb).to(D)

    def push(blocks_s, blocks_d, value):
        m = _native.Move()
        m.src_pool, m.dst_pool, m.n_blocks, m.done_value = src.pool_id, dst.pool_id, len(blocks_s), value
        m.src_blocks, m.dst_blocks = blocks_s.ctypes.data, blocks_d.ctypes.data
        m.done_flag = flags.data_ptr() if two else None
        _native.check(_native.lib().kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_BLOCKS_ON_HOST |
                                                _native.KVM_F_ENGINE_BULK, ctypes.c_void_p(s_src.cuda_stream)))

    # two GPUs: the bulk (TMA) engine on the source; one GPU: the LDG engine capped at 3 CTAs/SM so the
    # copy fits beside the persistent GEMM's CTAs (the bulk engine's 128 KiB ring does not)
    xfer_flags = _native.KVM_F_ENGINE_BULK if two else _native.KVM_F_CTAS_PER_SM(3)
    pre_s = np.ascontiguousarray(sb[:plan.prefix_blocks])
    pre_d = np.ascontiguousarray(db_np[:plan.prefix_blocks])
    all_s, all_d = np.ascontiguousarray(sb), np.ascontiguousarray(db_np)

    def begin():
        """The source stream starts when the destination's stream reaches this
        point (one split at a time: iteration i+1's push cannot run ahead)."""
        e = torch.cuda.Event()
        e.record(s_dst)
        s_src.wait_event(e)

    def end_copy(value):
        """The destination stream waits for a push's done flag (two devices) or
        the source stream (one device)."""
        if two:
            _native.check(_native.lib().kvm_wait_flag(ctypes.c_void_p(flags.data_ptr()), value,
                                                      ctypes.c_void_p(s_dst.cuda_stream)))
        else:
            s_dst.wait_stream(s_src)

    def run_split(overlap=True):
        seq[0] += 1
        begin()
        split_migrate(src, dst, sb, db, plan, x, w, xfer_stream=s_src if overlap else s_dst, rp_stream=s_dst,
                      flags_dev=flags, seq=seq[0], engine_flags=xfer_flags)
        wait_split(flags, plan, seq[0], s_dst)

    def run_full():
        seq[0] += 1
        begin()
        push(all_s, all_d, seq[0])
        end_copy(seq[0])

    def run_prefix_only():
        seq[0] += 1
        begin()
        push(pre_s, pre_d, seq[0])
        end_copy(seq[0])

    def run_fused():
        split_migrate_fused(alias, dst, sbd, db, plan, x, w, stream=s_dst)

    def run_suffix_only():
        reprefill(dst, x, w, db, tok0=plan.prefix_tokens, stream=s_dst)

    def timeit(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(src_dev)
        torch.cuda.synchronize(dst_dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_dst)
        for _ in range(iters):
            fn()
        e1.record(s_dst)
        torch.cuda.synchronize(src_dev)
        torch.cuda.synchronize(dst_dev)
        return e0.elapsed_time(e1) / iters

    def prefix_exact():
        pi = torch.from_numpy(sb[:plan.prefix_blocks].astype(np.int64)).to(f"cuda:{src_dev}")
        want = src.tensor[:, :, pi].view(torch.int16).to(D)      # compared on the destination device
        got = dst.tensor[:, :, db[:plan.prefix_blocks].long()].view(torch.int16)
        ok = bool(torch.equal(got, want))
        del want, got
        return ok

    def suffix_worst():
        if not plan.suffix:
            return 0.0
        kvd, qc = shape.kv_cols, shape.q_cols
        toks = torch.arange(plan.prefix_tokens, n, device=D)
        blk, slot = db.long()[toks // 16], toks % 16
        worst = 0.0
        for l in (0, shape.layers // 2, shape.layers - 1):
            ref = x.float() @ w[l].float().t()
            for kv, lo in ((0, qc), (1, qc + kvd)):
                got = dst.tensor[l, kv, blk, slot].reshape(plan.suffix, kvd).float()
                r = ref[:, lo:lo + kvd]
                worst = max(worst, float(((got - r).abs() - 1.6e-2 * r.abs()).max()))
        return worst

    for st in (s_src, s_dst):   # pools, x and w were produced on the default streams
        st.wait_stream(torch.cuda.current_stream(st.device))
    torch.cuda.synchronize(src_dev)
    torch.cuda.synchronize(dst_dev)
    # parity first: two-kernel split, then the fused one-launch split (destination zeroed between)
    run_split(True)
    torch.cuda.synchronize(src_dev)
    torch.cuda.synchronize(dst_dev)
    exact, worst = prefix_exact(), suffix_worst()
    dst.tensor.view(torch.int16).zero_()
    torch.cuda.synchronize(dst_dev)
    run_fused()
    torch.cuda.synchronize(dst_dev)
    exact_fused, worst_fused = prefix_exact(), suffix_worst()
    t_fused = timeit(run_fused)
    # two kernels only overlap across GPUs: on one GPU the persistent GEMM holds every SM (223 KB smem,
    # 57 K registers per CTA) so a copy kernel cannot co-reside, and the fused kernel is the split
    t_split = timeit(lambda: run_split(True)) if two else None
    t_serial = timeit(lambda: run_split(False))
    t_full = timeit(run_full)
    t_prefix = timeit(run_prefix_only)
    t_suffix = timeit(run_suffix_only) if plan.suffix else 0.0
    if two:
        alias.close()
    where = f"src cuda:{src_dev} -> dst cuda:{dst_dev}" + (" (NVLink)" if src_dev != dst_dev else
                                                           " (same GPU, two-device code path)" if two else " (same GPU)")
    return {
        "config": "configs[2]: Llama-2-13B KV, 8k tokens, adaptive split", "devices": where, "tokens": n,
        "suffix_reprefilled": plan.suffix, "prefix_blocks": plan.prefix_blocks,
        "kv_bytes": kv_bytes, "prefix_bytes": plan.prefix_tokens * shape.kv_bytes_per_token,
        "suffix_flops": plan.suffix * fpt,
        "ms": {"split_fused_one_kernel": round(t_fused, 4),
               "split_two_kernels": round(t_split, 4) if t_split is not None else None,
               "split_two_kernels_serialized": round(t_serial, 4), "full_transfer": round(t_full, 4),
               "prefix_transfer_only": round(t_prefix, 4), "suffix_reprefill_only": round(t_suffix, 4)},
        "split_over_full_transfer": round(t_full / min(t_fused, t_split or t_fused), 3),   # > 1 only across GPUs
        "note": None if two else ("one GPU: the full transfer is an HBM copy (no link), so only the fused "
                                  "kernel's overlap is meaningful here; split vs full transfer needs two GPUs"),
        "prefix_GBps": round(plan.prefix_tokens * shape.kv_bytes_per_token / t_prefix / 1e6, 1) if t_prefix else None,
        "full_transfer_GBps": round(kv_bytes / t_full / 1e6, 1),
        "suffix_tflops": round(plan.suffix * fpt / t_suffix / 1e9, 1) if t_suffix else None,
        "model_ms": {"full_transfer_at_770GBps": round(kv_bytes / NVLINK_BPS * 1e3, 3),
                     "split_balanced": round(max(plan.prefix_tokens * shape.kv_bytes_per_token / NVLINK_BPS,
                                                 plan.suffix * fpt / TENSOR_FLOPS) * 1e3, 3)},
        "prefix_bit_exact": exact and exact_fused,
        "suffix_within_tolerance": max(worst, worst_fused) <= 1e-2,
        "suffix_worst_excess": max(worst, worst_fused),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--suffix", type=int, default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--force-two", action="store_true", help="two-device code path on one device (test)")
    a = ap.parse_args()
    res = run_split_bench(a.tokens, a.suffix, a.iters, a.warmup, a.src_dev, a.dst_dev, a.force_two)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
