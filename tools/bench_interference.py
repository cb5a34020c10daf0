"""What an incoming migration costs the requests already decoding on the
destination GPU, and what the re-prefill SM budget buys back.

The paper's case for choosing KV transfer over re-prefill includes the
slowdown a co-running prefill inflicts on decode (up to 2.5x);
the reference's planner bounds re-prefill per epoch with a compute budget
(Boundaries.comp_budget, migration.py:77-91).  On a B200 the re-prefill GEMM
is a persistent kernel that fills every SM it is given for milliseconds, so a
decode step launched beside it waits for it -- unless the re-prefill runs on
an SM budget (KVM_REPREFILL_MAX_SMS), which leaves the other SMs to decode.

    python tools/bench_interference.py [--steps 40] [--out f.json]

Foreground: decode steps of 8 resident 7B requests x 2 048 tokens (32 layers,
one kvm_paged_decode launch per step) on a high-priority stream, timed one by
one with CUDA events.  Background (another stream, launched back to back for
the whole window): nothing; an incoming 7B-4k kvm_migrate into this GPU's
pool; the 13B 1 360-token re-prefill (QKV, 40 layers) on every SM, then on
an SM budget of 112 / 96 / 64 SMs.  Reported per arm: decode step p50 / p90
(and slowdown vs alone) with the background running for the whole window,
and each background launch's time alone.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.attention import paged_decode  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B, LLAMA2_13B, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lib = _native.lib()
    fg = torch.cuda.Stream(priority=-1)
    bg = torch.cuda.Stream()

    # foreground: 8 resident requests decoding
    sh, B, seq = LLAMA2_7B, 8, 2048
    nblk = seq // 16
    dec_pool = KVPool(sh, B * nblk + 8)
    dec_pool.tensor.normal_()
    table = torch.randperm(B * nblk, generator=torch.Generator().manual_seed(0)).to(torch.int32).view(B, nblk).cuda()
    lens = torch.full((B,), seq, dtype=torch.int32, device="cuda")
    q = torch.randn(sh.layers, B, sh.q_heads, 128, device="cuda").half()
    out = torch.empty_like(q)

    def decode_step():
        paged_decode(dec_pool, q, table, lens, out, max_seq_len=seq, stream=fg)

    # background 1: an incoming 7B-4k migration (into this GPU's pool)
    mig_n = 256
    src, dst = KVPool(sh, mig_n + 8), KVPool(sh, mig_n + 8)
    src.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    sb = torch.arange(mig_n, dtype=torch.int32, device="cuda")
    db = torch.arange(8, mig_n + 8, dtype=torch.int32, device="cuda")

    def migrate_on(max_sms):
        def migrate():
            m = _native.Move()
            m.src_pool, m.dst_pool, m.n_blocks = src.pool_id, dst.pool_id, mig_n
            m.src_blocks, m.dst_blocks = sb.data_ptr(), db.data_ptr()
            _native.check(lib.kvm_migrate(ctypes.byref(m), 1, _native.KVM_F_ENGINE_BULK | _native.KVM_F_MAX_SMS(max_sms),
                                          ctypes.c_void_p(bg.cuda_stream)))
        return migrate
    migrate = migrate_on(0)

    # background 2: the 13B re-prefill of a 1 360-token suffix
    rows = 1360
    rblk = (rows + 15) // 16
    rp_pool = KVPool(LLAMA2_13B, rblk + 4, dtype=torch.bfloat16)
    x = synthetic_hidden(LLAMA2_13B, rows, 0)
    w = synthetic_weights(LLAMA2_13B, 0, with_q=True)
    rp_blocks = torch.arange(rblk, dtype=torch.int32, device="cuda")

    def rp(max_sms):
        return lambda: reprefill(rp_pool, x, w, rp_blocks, stream=bg, max_sms=max_sms)

    torch.cuda.synchronize()

    def bg_time(fn, n=5):
        fn()
        bg.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(bg)
        for _ in range(n):
            fn()
        e1.record(bg)
        e1.synchronize()
        return e0.elapsed_time(e1) / n

    def decode_alone_ms():
        for _ in range(3):
            decode_step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(fg)
        for _ in range(5):
            decode_step()
        e1.record(fg)
        e1.synchronize()
        return e0.elapsed_time(e1) / 5

    def run_arm(fn, bg_one=None):
        """Background launched back to back on `bg` for the whole window; decode steps timed on `fg`."""
        for _ in range(3):
            decode_step()
        fg.synchronize()
        per, bg_ms = [], None
        if fn is not None:
            # enough background to outlast the decode window: each decode step at worst 4x slower than alone
            # plus one whole background launch
            n_bg = int(a.steps * (4 * dec_alone + bg_one) / bg_one) + 3
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(bg)
            for _ in range(n_bg):
                fn()
            b1.record(bg)
        evs = []
        for _ in range(a.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(fg)
            decode_step()
            e1.record(fg)
            evs.append((e0, e1))
        fg.synchronize()
        bg.synchronize()
        per = [e0.elapsed_time(e1) for e0, e1 in evs]
        window = evs[0][0].elapsed_time(evs[-1][1])
        if fn is not None:
            bg_ms = b0.elapsed_time(b1) / n_bg
            assert bg_ms * n_bg >= window, "background ended before the decode window"
        s = sorted(per)
        return {"decode_ms_p50": round(statistics.median(s), 4), "decode_ms_p90": round(s[int(0.9 * (len(s) - 1))], 4),
                "decode_ms_max": round(s[-1], 4), "background_launches": n_bg if fn is not None else 0}

    res = {"decode": f"8 x 7B requests x {seq} tokens, 32 layers, one paged-decode launch per step, high-priority "
                     f"stream", "steps": a.steps, "arms": {}}
    dec_alone = decode_alone_ms()
    alone_bg = {"incoming_migrate_7b_4k": bg_time(migrate), "incoming_migrate_7b_4k_32_sms": bg_time(migrate_on(32)),
                "reprefill_all_sms": bg_time(rp(0))}
    for cap in (112, 96, 64):
        alone_bg[f"reprefill_{cap}_sms"] = bg_time(rp(cap))
    arms = [("alone", None), ("incoming_migrate_7b_4k", migrate), ("incoming_migrate_7b_4k_32_sms", migrate_on(32)),
            ("reprefill_all_sms", rp(0)),
            ("reprefill_112_sms", rp(112)), ("reprefill_96_sms", rp(96)), ("reprefill_64_sms", rp(64))]
    for name, fn in arms:
        res["arms"][name] = run_arm(fn, alone_bg.get(name))
    base = res["arms"]["alone"]["decode_ms_p50"]
    for name, r in res["arms"].items():
        r["decode_slowdown_p50"] = round(r["decode_ms_p50"] / base, 2)
    res["background_alone_ms_per_launch"] = {k: round(v, 4) for k, v in alone_bg.items()}
    res["decode_alone_ms"] = round(dec_alone, 4)
    res["reading"] = ("the re-prefill GEMM is persistent: on every SM it holds them for its whole launch and a "
                      "decode step waits for it; on an SM budget (KVM_REPREFILL_MAX_SMS) decode keeps the rest. "
                      "An incoming migration shares HBM bandwidth only.")
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
