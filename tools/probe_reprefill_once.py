"""Launch the re-prefill GEMM once per engine (for ncu captures):
    ncu ... python tools/probe_reprefill_once.py [--rows 1360] [--shape llama2-13b]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200.kvcache import SHAPES, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=1360)
ap.add_argument("--shape", default="llama2-13b")
ap.add_argument("--engines", default="pair,single")
a = ap.parse_args()
shape = SHAPES[a.shape]
nblk = (a.rows + 15) // 16
pool = KVPool(shape, nblk + 4, dtype=torch.bfloat16)
blocks = torch.arange(nblk, dtype=torch.int32, device="cuda")
x = synthetic_hidden(shape, a.rows, 0)
w = synthetic_weights(shape, 0, with_q=True)
torch.cuda.synchronize()
for e in a.engines.split(","):
    reprefill(pool, x, w, blocks, single_cta=(e == "single"))
    torch.cuda.synchronize()
print("ok")
