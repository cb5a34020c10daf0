"""Live migration downtime vs stop-and-copy, 7B request.

    python tools/bench_live.py [--tokens 4096] [--decode-steps 64] [--reps 5]

Both on one B200 (two pools).  Stop-and-copy: the request is paused for one
full kvm_migrate of all its blocks.  Live: full blocks are pre-copied while
(mock) decode keeps appending; once the launched rounds have landed
(`LiveMigration.drain`, decode still running) the request pauses and only the
tail is copied.  Times
are host wall clock around the paused section (what a serving loop sees),
median over reps.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200.executor import MigrationExecutor  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B, BlockTable, KVPool  # noqa: E402
from paper_2501_06709_b200.live import LiveMigration  # noqa: E402
from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--decode-steps", type=int, default=70)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    shape = LLAMA2_7B
    nb = 2 * (a.tokens + a.decode_steps) // 16 + 8
    pools = {0: KVPool(shape, nb), 1: KVPool(shape, nb)}
    tables = {0: BlockTable(4, nb), 1: BlockTable(4, nb)}
    ex = MigrationExecutor(pools, tables)
    dec = torch.cuda.Stream()
    stop, live, rounds, gpu_pause, issue_pause = [], [], [], [], []
    rid = 1
    for rep in range(a.reps + 1):
        ex.admit(rid, 0, a.tokens)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ex.execute([PlannedMove(PendingMove(rid, 0, 1, a.tokens * shape.kv_bytes_per_token, a.tokens),
                                KV_TRANSFER)])
        t1 = time.perf_counter()
        ex.release(rid)
        ex.admit(rid, 0, a.tokens)
        lm = LiveMigration(ex, rid, 1)
        ev = torch.cuda.Event()
        tokens = a.tokens
        lm.precopy()
        for step in range(a.decode_steps):
            tokens += 1
            ex.grow(rid, tokens)
            r = ex.where(rid)
            with torch.cuda.stream(dec):  # mock decode write of the new token
                pools[0].tensor[:, :, int(r.blocks[(tokens - 1) // 16]), (tokens - 1) % 16].fill_(step)
            if (tokens % 16) == 0:
                ev.record(dec)
                lm.precopy(after=ev)
        ev.record(dec)
        dec.synchronize()
        lm.drain()                    # decode keeps running until the pre-copy rounds landed ...
        st = lm.finish(after=ev)      # ... then pause: only the tail is copied
        ex.release(rid)
        # stream-ordered variant: no host round trip; GPU-side pause = last source decode
        # write -> tail copy + table rewrite landed (CUDA events)
        ex.admit(rid, 0, a.tokens)
        lm2 = LiveMigration(ex, rid, 1)
        lm2.precopy()
        lm2.drain()
        stop_ev = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(dec):
            r = ex.where(rid)
            pools[0].tensor[:, :, int(r.blocks[-1]), (a.tokens - 1) % 16].fill_(1)   # last source decode write
            stop_ev.record(dec)
        st2 = lm2.finish(after=stop_ev, stream_ordered=True)
        st2.done.synchronize()
        ex.release(rid)
        if rep:
            gpu_pause.append(stop_ev.elapsed_time(st2.done) / 1e3)
            issue_pause.append(st2.downtime_s)
        if rep:  # first rep warms up
            stop.append(t1 - t0)
            live.append(st.downtime_s)
            rounds.append((st.rounds, st.blocks_precopied, st.blocks_stopcopied))
    out = {"workload": f"7b request, {a.tokens} tokens + {a.decode_steps} decode steps during pre-copy",
           "kv_bytes": a.tokens * shape.kv_bytes_per_token,
           "stop_and_copy_pause_ms": round(1e3 * statistics.median(stop), 4),
           "live_pause_ms": round(1e3 * statistics.median(live), 4),
           "pause_reduction_x": round(statistics.median(stop) / statistics.median(live), 1),
           "stream_ordered": {"gpu_pause_ms": round(1e3 * statistics.median(gpu_pause), 4),
                              "host_issue_ms": round(1e3 * statistics.median(issue_pause), 4),
                              "definition": "last source decode write -> tail copy + table rewrite landed "
                                            "(CUDA events); the host never waits"},
           "rounds_precopied_stopcopied_blocks": rounds[-1]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
