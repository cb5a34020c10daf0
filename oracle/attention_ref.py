"""ORACLE — TEST INFRASTRUCTURE ONLY: fp32 torch restatement of paged
decode attention (softmax(q.K^T * scale) . V per layer, request and query
head, grouped-query heads sharing their KV head), gathering K/V through the
block tables exactly as kvm_paged_decode addresses the pool.  Used by
tests/test_gpu_decode.py as the checker; the product never imports it.
Pinned by flashinfer 0.6's paged decode: tests/test_oracle_cpu.py reproduces
its outputs recorded on a B200 (tests/golden/thirdparty_vectors.json)."""
import math

def reference_decode(pool, q, block_tables, seq_lens, layer0: int = 0, scale: float = None):
    """fp32 torch reference (tests only): gather K/V through the tables."""
    import torch

    sh = pool.shape
    scale = scale if scale is not None else 1.0 / math.sqrt(sh.head_dim)
    L, B, Hq, D = q.shape
    G = Hq // sh.kv_heads
    out = torch.empty(L, B, Hq, D, dtype=torch.float32, device=q.device)
    for l in range(L):
        for b in range(B):
            n = int(seq_lens[b])
            t = torch.arange(n, device=q.device)
            blk = block_tables[b].long()[t // sh.block_tokens]
            K = pool.tensor[layer0 + l, 0, blk, t % sh.block_tokens].float()  # [n, Hkv, D]
            V = pool.tensor[layer0 + l, 1, blk, t % sh.block_tokens].float()
            Kq = K.repeat_interleave(G, dim=1)  # [n, Hq, D]
            Vq = V.repeat_interleave(G, dim=1)
            s = torch.einsum("hd,nhd->hn", q[l, b].float(), Kq) * scale
            p = torch.softmax(s, dim=-1)
            out[l, b] = torch.einsum("hn,nhd->hd", p, Vq)
    return out
