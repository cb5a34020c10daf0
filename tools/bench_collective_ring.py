"""NCCL comparison baseline for the ring push: the same
per-rank request (7B-4k: 256 scattered blocks, 2 GiB) moved to the ring
successor with index_select -> ncclSend/ncclRecv (batch_isend_irecv) ->
index_copy_, instead of bench.py's one kvm_migrate kernel storing over NVLink.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_collective_ring.py [--steps 20]

Device time per step with CUDA events, max over ranks; one JSON line on rank
0.  Needs N >= 2 GPUs (NCCL does not run two ranks on one device).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2501_06709_b200.dist import allreduce_max, collective_ring_exchange, rank_info_from_env  # noqa: E402
from paper_2501_06709_b200.kvcache import LLAMA2_7B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--blocks", type=int, default=256)
    a = ap.parse_args()
    ri = rank_info_from_env()
    if ri.world < 2:
        print(json.dumps({"impl": "nccl_ring_baseline", "unavailable": "needs >= 2 GPUs (one rank per GPU)"}))
        return
    torch.cuda.set_device(ri.local_rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{ri.local_rank}"))
    s = LLAMA2_7B
    nb = 4 * a.blocks
    pool = torch.empty((s.layers, 2, nb, 16, s.kv_heads, s.head_dim), dtype=torch.float16, device="cuda")
    pool.view(torch.int16).random_(generator=torch.Generator(device="cuda").manual_seed(ri.rank))
    g = torch.Generator().manual_seed(100 + ri.rank)
    perm = torch.randperm(nb, generator=g)
    send, recv = perm[:a.blocks].cuda(), perm[a.blocks:2 * a.blocks].cuda()
    for _ in range(a.warmup):
        collective_ring_exchange(pool, send, recv, ri)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        collective_ring_exchange(pool, send, recv, ri)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = allreduce_max(e0.elapsed_time(e1) / a.steps, device=f"cuda:{ri.local_rank}")
    kv_bytes = a.blocks * 16 * s.kv_bytes_per_token
    if ri.rank == 0:
        print(json.dumps({"impl": "nccl_ring_baseline", "n_gpus": ri.world, "kv_bytes_per_rank": kv_bytes,
                          "ms_per_step": round(ms, 4), "GBps_per_rank": round(kv_bytes / ms / 1e6, 1),
                          "GBps_aggregate": round(ri.world * kv_bytes / ms / 1e6, 1),
                          "path": "index_select -> batch_isend_irecv (ncclSend/ncclRecv) -> index_copy_"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
