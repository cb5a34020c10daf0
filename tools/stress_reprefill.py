"""Repeat small re-prefill launches and check every result (flakiness probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_06709_b200.kvcache import KVPool, ModelShape
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights
shape = ModelShape("sp", layers=6, kv_heads=4, head_dim=128, q_heads=8, d_model=512)
bad = 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for rows in (512, 77, 1, 300):
    nb = (rows + 15) // 16 + 20
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    db = torch.arange(nb, dtype=torch.int32, device="cuda")
    x = synthetic_hidden(shape, rows, 0, seed=4)
    w = synthetic_weights(shape, 0, with_q=True, seed=5)
    ref = torch.einsum("tk,lnk->ltn", x.float(), w.float())
    kvd, qc = shape.kv_cols, shape.q_cols
    toks = torch.arange(rows, device="cuda")
    s = torch.cuda.Stream()
    for it in range(n // 4):
        pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
        s.wait_stream(torch.cuda.current_stream())  # x, w and the pool fill come from the default stream
        reprefill(pool, x, w, db, tok0=0, stream=s)
        s.synchronize()
        k = pool.tensor[:, 0, db.long()[toks // 16], toks % 16].reshape(shape.layers, rows, kvd).float()
        if not torch.allclose(k, ref[:, :, qc:qc + kvd], atol=1e-2, rtol=1.6e-2):
            bad += 1
            print("BAD rows", rows, "iter", it, (k - ref[:, :, qc:qc + kvd]).abs().max().item())
print("stress done, bad =", bad)
