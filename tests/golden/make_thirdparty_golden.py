"""Generate tests/golden/thirdparty_vectors.json from the THIRD-PARTY libraries
the paper's prototype ran its data plane in (vLLM) and the
paged decode library installed beside it (flashinfer).  Needs a GPU (both
libraries' kernels are CUDA-only), so it runs on a gpurun box:

    gpurun -- 'python tests/golden/make_thirdparty_golden.py'

and the JSON it writes under gpurun_out/ is committed here.  The reference
(kvpack) moves no bytes (sim.py:221-223), so these vectors are what pins the
CPU oracle's byte path and decode restatement: tests/test_oracle_cpu.py
regenerates every input from its seed (numpy PCG64, stable across versions),
runs oracle/kvmig_oracle.c / oracle/attention_ref.py on the CPU and compares
with the library's recorded output.

Vectors
  swap_blocks   vLLM 0.22 `_C_cache_ops.swap_blocks(src, dst, block_bytes,
                mapping)` applied to every (layer, K|V) plane of a pool laid
                out [L][2][NB][16][H][D] (each plane IS a vLLM per-layer K or V
                cache).  Inputs: uint16 bit patterns from default_rng(seed)
                (NaN / inf payloads included), mapping from the same rng.
                Output: sha256 of the whole destination pool (and of the source,
                which must not change).  Cases cover src != dst pools and the
                in-place compaction (src pool == dst pool, disjoint block sets).
  placement     vLLM 0.22 `_C_cache_ops.reshape_and_cache_flash(key, value,
                key_cache, value_cache, slot_mapping, "auto", ...)`: token t of a
                re-prefilled suffix lands in slot (tok0 + t) of the request's
                block list; bf16 K = V = X from numpy, output sha256 of the
                key cache.  The CPU test reproduces it with the C oracle's
                re-prefill under identity projections (K = X exactly).
  decode        flashinfer 0.6 BatchDecodeWithPagedKVCacheWrapper (NHD layout)
                over one layer's K/V planes of such a pool, fp16, GQA ratios
                1/4/8, ragged lengths: output as float32 hex per element.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(HERE))), "gpurun_out",
                   "thirdparty_vectors.json")

SWAP_CASES = [   # (name, layers, kv_heads, head_dim, src_nb, dst_nb, n_moved, seed, in_place)
    ("small", 2, 2, 16, 24, 24, 7, 1, False),
    ("odd_head_dim", 3, 5, 40, 40, 33, 13, 2, False),
    ("one_block", 2, 4, 32, 16, 16, 1, 3, False),
    ("all_blocks", 2, 2, 64, 12, 12, 12, 4, False),
    ("compact_in_place", 3, 2, 32, 48, 48, 20, 5, True),
    ("llama_piece", 2, 8, 128, 32, 40, 17, 6, False),
]

PLACEMENT_CASES = [  # (name, kv_heads, rows, tok0, seed)
    ("one_row", 2, 1, 0, 21),
    ("ragged", 4, 77, 5, 22),
    ("deep_offset", 1, 300, 4000, 23),
    ("block_aligned", 8, 128, 16, 24),
]

DECODE_CASES = [  # (name, kv_heads, q_heads, seq_lens, seed)
    ("mha", 4, 4, [1, 17, 64], 11),
    ("gqa4", 2, 8, [33, 5, 128, 200], 12),
    ("gqa8", 1, 8, [16, 250], 13),
]


def swap_inputs(layers, kv_heads, head_dim, src_nb, dst_nb, n, seed, in_place):
    """Inputs regenerated bit-for-bit by the CPU test (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    per_block = 16 * kv_heads * head_dim
    src = rng.integers(0, 1 << 16, size=(layers, 2, src_nb, per_block), dtype=np.uint16)
    if in_place:
        perm = rng.permutation(src_nb)
        sb, db = perm[:n], perm[n:2 * n]
        return src, None, sb.astype(np.int32), db.astype(np.int32)
    dst = rng.integers(0, 1 << 16, size=(layers, 2, dst_nb, per_block), dtype=np.uint16)
    sb = rng.permutation(src_nb)[:n]
    db = rng.permutation(dst_nb)[:n]
    return src, dst, sb.astype(np.int32), db.astype(np.int32)


def decode_inputs(kv_heads, q_heads, seq_lens, seed, head_dim=128):
    """Pool plane K/V [NB][16][H][D] fp16 + per-request block lists + q [B][Hq][D] fp16 from numpy."""
    rng = np.random.default_rng(seed)
    nblk = [(s + 15) // 16 for s in seq_lens]
    nb = sum(nblk) + 5
    k = rng.standard_normal((nb, 16, kv_heads, head_dim)).astype(np.float16)
    v = rng.standard_normal((nb, 16, kv_heads, head_dim)).astype(np.float16)
    perm = rng.permutation(nb).astype(np.int32)
    tables, o = [], 0
    for c in nblk:
        tables.append(perm[o:o + c])
        o += c
    q = rng.standard_normal((len(seq_lens), q_heads, head_dim)).astype(np.float16)
    return k, v, tables, q


def placement_inputs(kv_heads, rows, tok0, seed, head_dim=128):
    """bf16 bits of X [rows][kv_heads * head_dim] and the request's block list."""
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((rows, kv_heads * head_dim)).astype(np.float32)
    x = (f.view(np.uint32) >> 16).astype(np.uint16)           # bf16 by truncation: exact bf16 values
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + 3
    blocks = rng.permutation(nb)[:nblk].astype(np.int32)
    return x, blocks, nb


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_swap():
    import vllm._custom_ops as vops
    out = []
    for name, L, H, D, snb, dnb, n, seed, in_place in SWAP_CASES:
        src, dst, sb, db = swap_inputs(L, H, D, snb, dnb, n, seed, in_place)
        s_t = torch.from_numpy(src.view(np.int16)).cuda()
        d_t = s_t if in_place else torch.from_numpy(dst.view(np.int16)).cuda()
        mapping = torch.from_numpy(np.stack([sb, db], 1).astype(np.int64))
        block_bytes = 16 * H * D * 2
        for l in range(L):
            for kv in range(2):
                vops.swap_blocks(s_t[l, kv], d_t[l, kv], block_bytes, mapping)
        torch.cuda.synchronize()
        res = d_t.cpu().numpy().view(np.uint16)
        out.append({"name": name, "layers": L, "kv_heads": H, "head_dim": D, "src_nb": snb, "dst_nb": dnb,
                    "n": n, "seed": seed, "in_place": in_place,
                    "dst_sha256": sha(res),
                    "src_sha256": sha(s_t.cpu().numpy().view(np.uint16)) if not in_place else None})
    return out


def gen_placement():
    import vllm._custom_ops as vops
    out = []
    for name, H, rows, tok0, seed in PLACEMENT_CASES:
        x, blocks, nb = placement_inputs(H, rows, tok0, seed)
        xt = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16).view(rows, H, 128).contiguous()
        kc = torch.zeros(nb, 16, H, 128, dtype=torch.bfloat16, device="cuda")
        vc = torch.zeros_like(kc)
        pos = np.arange(tok0, tok0 + rows)
        slots = torch.from_numpy((blocks[pos // 16].astype(np.int64) * 16 + pos % 16)).cuda()
        one = torch.ones((), dtype=torch.float32, device="cuda")
        vops.reshape_and_cache_flash(xt, xt, kc, vc, slots, "auto", one, one)
        torch.cuda.synchronize()
        out.append({"name": name, "kv_heads": H, "rows": rows, "tok0": tok0, "seed": seed,
                    "key_cache_sha256": sha(kc.view(torch.int16).cpu().numpy()),
                    "value_cache_sha256": sha(vc.view(torch.int16).cpu().numpy())})
    return out


def gen_decode():
    import flashinfer
    out = []
    for name, H, Hq, lens, seed in DECODE_CASES:
        k, v, tables, q = decode_inputs(H, Hq, lens, seed)
        kc = torch.from_numpy(k).cuda()
        vc = torch.from_numpy(v).cuda()
        indptr = torch.tensor(np.concatenate([[0], np.cumsum([len(t) for t in tables])]), dtype=torch.int32,
                              device="cuda")
        indices = torch.from_numpy(np.concatenate(tables)).cuda()
        last = torch.tensor([(s - 1) % 16 + 1 for s in lens], dtype=torch.int32, device="cuda")
        ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
        w.plan(indptr, indices, last, Hq, H, 128, 16, pos_encoding_mode="NONE", q_data_type=torch.float16,
               kv_data_type=torch.float16)
        o = w.run(torch.from_numpy(q).cuda(), (kc, vc))
        torch.cuda.synchronize()
        out.append({"name": name, "kv_heads": H, "q_heads": Hq, "seq_lens": lens, "seed": seed,
                    "out_f32_hex": [float(x).hex() for x in o.float().cpu().numpy().reshape(-1)]})
    return out


def main():
    import flashinfer
    import vllm
    res = {"generator": "tests/golden/make_thirdparty_golden.py",
           "libraries": {"vllm": vllm.__version__, "flashinfer": flashinfer.__version__,
                         "torch": torch.__version__, "device": torch.cuda.get_device_name(0)},
           "swap_blocks": gen_swap(), "placement": gen_placement(), "decode": gen_decode()}
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as fh:
        json.dump(res, fh, indent=1)
    print(f"wrote {OUT}: {len(res['swap_blocks'])} swap_blocks + {len(res['decode'])} decode vectors",
          file=sys.stderr)


if __name__ == "__main__":
    main()
