"""Replay a recorded reference run (tests/golden/trace_*.json) on GPU pools.

    python tools/replay_trace.py [--fixture tests/golden/trace_7b_c48g_seed0.json]
                                 [--shape mini|full] [--max-slots N] [--engine bulk|ldg]

Logical GPU g of the trace maps to physical device g % device_count.  With
--shape mini (default) the KV shape is Llama-2-7B's layer count with 2 KV
heads (32 KiB/token, 1/16 of 7B) so all 8 logical pools fit one B200; token
counts, and therefore every scheduler/planner decision, are the reference's.
Prints one JSON line with the totals.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200.executor import MigrationExecutor  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B, LLAMA2_13B, BlockTable, KVPool, ModelShape  # noqa: E402
from paper_2501_06709_b200.replay import TraceReplay, pool_blocks_for  # noqa: E402
from paper_2501_06709_b200.reprefill import ReprefillEngine  # noqa: E402

MINI_7B = ModelShape("llama2-7b-mini", layers=32, kv_heads=2, head_dim=128, q_heads=2, d_model=512)
MINI_13B = ModelShape("llama2-13b-mini", layers=40, kv_heads=2, head_dim=128, q_heads=2, d_model=512)
MINI = {"llama2-7b": MINI_7B, "llama2-13b": MINI_13B}
FULL = {"llama2-7b": LLAMA2_7B, "llama2-13b": LLAMA2_13B}


def build(fx, shape, engine, devices, shapes=None):
    """One pool (per model, for multi-LLM fixtures) per logical GPU of the trace."""
    n_gpus = fx["summary"]["peak_gpus"]
    models = sorted(set(fx.get("models", {}).values()))
    pools, tables = {}, {}
    nb = 0
    for g in range(n_gpus):
        dev = devices[g % len(devices)]
        if models:
            pools[g], tables[g] = {}, {}
            for m in models:
                sh = shapes[m]
                nbm = pool_blocks_for(fx, sh.block_tokens, model=m)
                nb = max(nb, nbm)
                pools[g][sh.name] = KVPool(sh, nbm, device=dev, dtype=torch.bfloat16)
                tables[g][sh.name] = BlockTable(512, nbm, device=dev)
        else:
            nb = pool_blocks_for(fx, shape.block_tokens)
            pools[g] = KVPool(shape, nb, device=dev, dtype=torch.bfloat16)
            tables[g] = BlockTable(512, nb, device=dev)
    used = [shapes[m] for m in models] if models else [shape]
    rp = ReprefillEngine(used, sorted(set(devices[g % len(devices)] for g in range(n_gpus))), with_q=False)
    return MigrationExecutor(pools, tables, engine=engine, reprefill=rp), nb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fixture", default=os.path.join("tests", "golden", "trace_7b_c48g_seed0.json"))
    ap.add_argument("--shape", choices=["mini", "full"], default="mini")
    ap.add_argument("--max-slots", type=int, default=None)
    ap.add_argument("--engine", choices=["bulk", "ldg"], default="bulk")
    ap.add_argument("--verify-every", type=int, default=50)
    a = ap.parse_args()
    with open(a.fixture) as fh:
        fx = json.load(fh)
    shape = MINI_7B if a.shape == "mini" else LLAMA2_7B
    shapes = MINI if a.shape == "mini" else FULL
    devices = list(range(torch.cuda.device_count()))
    ex, nb = build(fx, shape, a.engine, devices, shapes)
    rp = TraceReplay(fx, ex, model_map={m: s.name for m, s in shapes.items()})
    rep = rp.run(max_slots=a.max_slots, verify_every=a.verify_every)
    wl = fx["config"]["workload"]["kv_bytes_per_token"]
    scale = shape.kv_bytes_per_token / wl if isinstance(wl, int) else None
    ref_bytes = sum(s.ref_kv_bytes for s in rep.slots)
    out = {
        "fixture": os.path.basename(a.fixture), "shape": shape.name, "devices": len(devices),
        "logical_gpus": len(ex.pools), "models": sorted({m for per in ex.pools.values() for m in per}),
        "pool_blocks": nb, "slots": len(rep.slots),
        "executed_rows": rep.executed,
        "kv_moves": sum(s.kv_moves for s in rep.slots), "token_moves": sum(s.token_moves for s in rep.slots),
        "bytes_moved": rep.bytes_moved, "tokens_moved": rep.tokens_moved,
        "ref_kv_bytes": ref_bytes, "ref_kv_bytes_scaled": int(ref_bytes * scale) if scale else None,
        "execute_seconds": round(rep.migrate_seconds, 4),
        "verified_requests": rep.verified_requests, "recomputed_requests": rep.recomputed_requests,
        "fixture_sha": fx["plan_rows_sha256_16"],
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
