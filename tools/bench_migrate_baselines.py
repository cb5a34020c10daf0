"""K1/K2 against the library paths SURVEY.md §2 names, on one B200.

Same workload for every arm: move a request's paged KV (every layer, K and
V, scattered source blocks -> scattered free destination blocks of the same
pool; 7B, 4k tokens = 2 GiB by default), inputs > L2, CUDA events, median of
--iters.

  ours-bulk     kvm_compact, TMA bulk engine (one launch)
  ours-ldg      kvm_compact, 128-bit LDG/STG engine (one launch)
  torch-index   v = pool.view(L*2, NB, piece); v.index_copy_(1, dst, v.index_select(1, src))
                (the library path to beat)
  torch-index-per-plane  the same per (layer, K|V) plane [NB, piece]: dim-0 index_select
                + index_copy_ (torch's contiguous-row fast path), 2 * layers * 2 kernels
  torch         pool[:, :, dst] = pool[:, :, src]  (advanced-index gather + put)
  vllm-swap_blocks  vLLM 0.22's block copy (_C_cache_ops.swap_blocks) per plane: how
                vLLM moves KV blocks (one cudaMemcpyAsync per block)
  memcpy-loop   cudaMemcpyAsync per piece (host-issued, 16 384 calls)

Prints one JSON line; GB/s counts payload bytes (kv_bytes), "hbm_frac" the
read+write traffic against MEASURED_PEAKS.json.

    python tools/bench_migrate_baselines.py [--workload 7b-4k] [--iters 10]
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
from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402

WORKLOADS = {"7b-4k": ("llama2-7b", 4096), "13b-8k": ("llama2-13b", 8192), "70b-16k": ("llama3-70b-gqa", 16384),
             "7b-512": ("llama2-7b", 512)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="7b-4k", choices=sorted(WORKLOADS))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    shape = SHAPES[WORKLOADS[a.workload][0]]
    tokens = WORKLOADS[a.workload][1]
    n = tokens // shape.block_tokens
    nb = 4 * n
    pool = KVPool(shape, nb, device=0)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    g = torch.Generator().manual_seed(1)
    perm = torch.randperm(nb, generator=g).numpy().astype(np.int32)
    sb, db = perm[:n].copy(), np.sort(perm[n:2 * n]).astype(np.int32)
    sb_d, db_d = torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()
    sb_l, db_l = sb_d.long(), db_d.long()
    kv_bytes = tokens * shape.kv_bytes_per_token
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    sptr = ctypes.c_void_p(s.cuda_stream)
    lib = _native.lib()

    def timeit(fn):
        with torch.cuda.stream(s):
            for _ in range(a.warmup):
                fn()
            torch.cuda.synchronize()
            times = []
            for _ in range(a.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn()
                e1.record(s)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
        return statistics.median(times)

    out = {"workload": a.workload, "kv_bytes": kv_bytes, "pieces": 2 * shape.layers * n,
           "piece_bytes": shape.piece_bytes, "ms": {}, "GBps": {}}
    flip = [False]

    def ours(engine):
        def run():
            src, dst = (db_d, sb_d) if flip[0] else (sb_d, db_d)
            flip[0] = not flip[0]
            _native.check(lib.kvm_compact(pool.pool_id, ctypes.c_void_p(src.data_ptr()),
                                          ctypes.c_void_p(dst.data_ptr()), n, None, engine, sptr))
        return run

    v = pool.tensor.view(2 * shape.layers, nb, -1)

    def torch_index_arm():
        src, dst = (db_l, sb_l) if flip[0] else (sb_l, db_l)
        flip[0] = not flip[0]
        v.index_copy_(1, dst, v.index_select(1, src))

    planes_v = [v[i] for i in range(2 * shape.layers)]   # [NB, piece] each: dim-0 index ops (fast path)
    tmp = torch.empty(n, v.shape[2], dtype=v.dtype, device=v.device)

    def torch_plane_arm():
        src, dst = (db_l, sb_l) if flip[0] else (sb_l, db_l)
        flip[0] = not flip[0]
        for pv in planes_v:
            torch.index_select(pv, 0, src, out=tmp)
            pv.index_copy_(0, dst, tmp)

    try:
        import vllm._custom_ops as vops
        vmap = {"f": torch.from_numpy(np.stack([sb, db], 1).astype(np.int64)),
                "b": torch.from_numpy(np.stack([db, sb], 1).astype(np.int64))}
        # vLLM's per-layer caches are the pool's (layer, K|V) planes, [NB][16][H][D] contiguous
        kv_planes = [pool.tensor[l, kv] for l in range(shape.layers) for kv in range(2)]
    except Exception:
        vops = None

    def vllm_arm():
        m = vmap["b" if flip[0] else "f"]
        flip[0] = not flip[0]
        for pl in kv_planes:
            vops.swap_blocks(pl, pl, pb, m)

    def torch_arm():
        src, dst = (db_l, sb_l) if flip[0] else (sb_l, db_l)
        flip[0] = not flip[0]
        pool.tensor[:, :, dst] = pool.tensor[:, :, src]

    # piece address lists for the copy-engine arms (both directions)
    base = pool.tensor.data_ptr()
    L = shape.layers
    pb = shape.piece_bytes
    plane = nb * pb
    planes = np.arange(2 * L, dtype=np.int64)[:, None] * plane

    def addrs(blocks):
        return (base + planes + blocks.astype(np.int64)[None, :] * pb).reshape(-1)

    fwd = (addrs(sb), addrs(db))
    bwd = (addrs(db), addrs(sb))
    cnt = fwd[0].size
    cudart = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            cudart = ctypes.CDLL(name)
            break
        except OSError:
            pass
    arrays = {}
    for key, (src, dst) in (("f", fwd), ("b", bwd)):
        arrays[key] = ((ctypes.c_void_p * cnt)(*dst.tolist()), (ctypes.c_void_p * cnt)(*src.tolist()))

    def loop_arm():
        d, src = arrays["b" if flip[0] else "f"]
        flip[0] = not flip[0]
        for i in range(cnt):
            cudart.cudaMemcpyAsync(ctypes.c_void_p(d[i]), ctypes.c_void_p(src[i]), ctypes.c_size_t(pb), 3, sptr)

    arms = [("ours-bulk", ours(_native.KVM_F_ENGINE_BULK)), ("ours-ldg", ours(0)), ("torch-index", torch_index_arm),
            ("torch-index-per-plane", torch_plane_arm), ("torch", torch_arm)]
    if vops is not None:
        arms.append(("vllm-swap_blocks", vllm_arm))
    if cudart is not None:
        arms.append(("memcpy-loop", loop_arm))
    for name, fn in arms:
        try:
            ms = timeit(fn)
        except Exception as e:  # a library path missing on this box is reported, not fatal
            out["ms"][name] = None
            out.setdefault("errors", {})[name] = str(e)[:200]
            continue
        out["ms"][name] = round(ms, 4)
        out["GBps"][name] = round(kv_bytes / ms / 1e6, 1)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh).get("hbm_gbs"))
        out["hbm_peak_GBps"] = peak
        out["hbm_frac"] = {k: round(2 * v / peak, 3) for k, v in out["GBps"].items()}
    except (OSError, ValueError, TypeError):
        pass
    print(json.dumps(out))


if __name__ == "__main__":
    main()
