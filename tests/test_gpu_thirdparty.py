"""Data-plane parity pinned to third-party published implementations
(VERDICT r1 "what's missing" #5).  The reference moves no bytes and computes
no K/V; the paper's prototype did that inside vLLM
(PAPER.md:670).  So the re-prefill numerics, the token-slot placement and the
paged decode that consumes a migrated cache are checked here against the
libraries installed in the image — HF transformers 5.5 (Llama attention's
k_proj / v_proj / q_proj + apply_rotary_pos_emb), vLLM 0.22
(reshape_and_cache_flash slot mapping) and flashinfer 0.6 (paged decode) —
on the same inputs and, for vLLM/flashinfer, the same pool memory.

Tolerance for re-prefilled bf16 K/V/Q: |got - ref| <= 1e-2 + 1.6e-2 |ref|
(bf16 output of an fp32-accumulated bf16 GEMM; the HF side runs in fp32 on
the same bf16 operands).  Decode: atol 2e-3, rtol 2e-2 (fp16 softmax
attention, fp32 accumulation on both sides)."""
import numpy as np
import pytest
import torch

from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights

pytestmark = pytest.mark.gpu
ATOL, RTOL = 1e-2, 1.6e-2


def _hf_llama(shape, theta):
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaAttention, LlamaRotaryEmbedding

    cfg = LlamaConfig(hidden_size=shape.d_model, num_attention_heads=shape.q_heads,
                      num_key_value_heads=shape.kv_heads, head_dim=shape.head_dim, rope_theta=theta,
                      num_hidden_layers=shape.layers, intermediate_size=4 * shape.d_model, vocab_size=128)
    layers = [LlamaAttention(cfg, layer_idx=l).cuda().float() for l in range(shape.layers)]
    return cfg, layers, LlamaRotaryEmbedding(cfg).cuda()


@pytest.mark.parametrize("theta,tok0,rows", [(10000.0, 0, 200), (500000.0, 37, 333), (10000.0, 4000, 96)])
def test_reprefill_equals_hf_llama_qkv_and_rope(theta, tok0, rows):
    """K/V written into the pool (and Q out) by the tcgen05 re-prefill with the
    RoPE epilogue == HF LlamaAttention's k_proj / v_proj / q_proj of the same
    hidden states with the same bf16 weights, rotated by HF's
    LlamaRotaryEmbedding + apply_rotary_pos_emb at positions tok0 + t."""
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb

    shape = ModelShape("hf", layers=2, kv_heads=2, head_dim=128, q_heads=4, d_model=512)
    cfg, att, rot = _hf_llama(shape, theta)
    w = synthetic_weights(shape, 0, with_q=True, seed=21)          # [L][q + 2kv][d_model] bf16
    x = synthetic_hidden(shape, rows, 0, seed=22)                  # [rows][d_model] bf16
    qc, kc = shape.q_cols, shape.kv_cols
    with torch.no_grad():
        for l, a in enumerate(att):                                 # the same bf16 weights, nn.Linear layout
            a.q_proj.weight.copy_(w[l, :qc].float())
            a.k_proj.weight.copy_(w[l, qc:qc + kc].float())
            a.v_proj.weight.copy_(w[l, qc + kc:].float())
    nblk = (tok0 + rows + 15) // 16
    pool = KVPool(shape, nblk + 7, dtype=torch.bfloat16)
    pool.tensor.zero_()
    blocks = torch.randperm(nblk + 7, generator=torch.Generator().manual_seed(5))[:nblk].to(torch.int32).cuda()
    q_out = torch.empty(shape.layers, rows, qc, dtype=torch.bfloat16, device="cuda")
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q_out, rope_theta=theta)
    torch.cuda.synchronize()
    pos = torch.arange(tok0, tok0 + rows, device="cuda")
    blk, slot = blocks.long()[pos // 16], pos % 16
    xf = x.float()[None]                                            # [1, T, d_model]
    cos, sin = rot(xf, pos[None])
    with torch.no_grad():
        for l, a in enumerate(att):
            q = a.q_proj(xf).view(1, rows, shape.q_heads, 128).transpose(1, 2)
            k = a.k_proj(xf).view(1, rows, shape.kv_heads, 128).transpose(1, 2)
            v = a.v_proj(xf).view(1, rows, shape.kv_heads, 128)
            q_rot, k_rot = apply_rotary_pos_emb(q, k, cos, sin)
            got_k = pool.tensor[l, 0, blk, slot].float()            # [T, kv_heads, 128]
            got_v = pool.tensor[l, 1, blk, slot].float()
            torch.testing.assert_close(got_k, k_rot[0].transpose(0, 1), atol=ATOL, rtol=RTOL)
            torch.testing.assert_close(got_v, v[0], atol=ATOL, rtol=RTOL)
            torch.testing.assert_close(q_out[l].float().view(rows, shape.q_heads, 128), q_rot[0].transpose(0, 1),
                                       atol=ATOL, rtol=RTOL)


def test_reprefill_slot_placement_equals_vllm_reshape_and_cache():
    """Where token t's K/V lands: vLLM's reshape_and_cache_flash with the
    PagedAttention slot mapping (slot = block_table[p // 16] * 16 + p % 16)
    scatters the reference K/V into a flash-layout cache [blocks][16][H][D];
    our pool's per-layer planes have exactly that layout, and the re-prefill
    epilogue must fill the same slots (values within bf16 tolerance, every
    other slot untouched on both sides)."""
    vops = pytest.importorskip("vllm._custom_ops")
    shape = ModelShape("vl", layers=3, kv_heads=4, head_dim=128, q_heads=4, d_model=512)
    rows, tok0 = 250, 21
    w = synthetic_weights(shape, 0, with_q=False, seed=31)
    x = synthetic_hidden(shape, rows, 0, seed=32)
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + 9
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(8))[:nblk].to(torch.int32).cuda()
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.zero_()
    reprefill(pool, x, w, blocks, tok0=tok0)
    torch.cuda.synchronize()
    pos = torch.arange(tok0, tok0 + rows, device="cuda")
    slot_mapping = (blocks.long()[pos // 16] * 16 + pos % 16).contiguous()
    one = torch.ones((), dtype=torch.float32, device="cuda")
    kc = shape.kv_cols
    for l in range(shape.layers):
        ref = (x.float() @ w[l].float().t()).to(torch.bfloat16)
        key = ref[:, :kc].reshape(rows, shape.kv_heads, 128).contiguous()
        val = ref[:, kc:].reshape(rows, shape.kv_heads, 128).contiguous()
        kcache = torch.zeros(nb, 16, shape.kv_heads, 128, dtype=torch.bfloat16, device="cuda")
        vcache = torch.zeros_like(kcache)
        vops.reshape_and_cache_flash(key, val, kcache, vcache, slot_mapping, "auto", one, one)
        torch.cuda.synchronize()
        written = torch.zeros(nb, 16, dtype=torch.bool, device="cuda")
        written.view(-1)[slot_mapping] = True
        for plane, cache in ((0, kcache), (1, vcache)):
            ours = pool.tensor[l, plane]
            assert torch.equal(ours[~written].view(torch.int16), cache[~written].view(torch.int16))   # all zero
            torch.testing.assert_close(ours[written].float(), cache[written].float(), atol=ATOL, rtol=RTOL)


def _flashinfer_decode(fi, pool, q, table, seq, dtype):
    sh = pool.shape
    nblk = table.shape[1]
    batch = table.shape[0]
    ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    dec = fi.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
    indptr = torch.arange(0, (batch + 1) * nblk, nblk, dtype=torch.int32, device="cuda")
    last = torch.full((batch,), seq - (nblk - 1) * 16, dtype=torch.int32, device="cuda")
    dec.plan(indptr, table.reshape(-1).contiguous(), last, sh.q_heads, sh.kv_heads, 128, 16,
             pos_encoding_mode="NONE", q_data_type=dtype, kv_data_type=dtype)
    return torch.stack([dec.run(q[l], (pool.tensor[l, 0], pool.tensor[l, 1])) for l in range(sh.layers)])


@pytest.mark.parametrize("kv_heads,q_heads,seq,batch,dtype", [
    (8, 8, 1000, 2, torch.float16), (2, 16, 4096, 1, torch.float16), (8, 64, 777, 3, torch.bfloat16)])
def test_paged_decode_equals_flashinfer_on_the_same_pool(kv_heads, q_heads, seq, batch, dtype):
    """kvm_paged_decode vs flashinfer's BatchDecodeWithPagedKVCacheWrapper reading
    the same pool memory through the same page table (our per-layer K and V
    planes are flashinfer's NHD paged layout)."""
    fi = pytest.importorskip("flashinfer")
    from paper_2501_06709_b200.attention import paged_decode

    shape = ModelShape("fi", layers=3, kv_heads=kv_heads, head_dim=128, q_heads=q_heads, d_model=1024)
    nblk = (seq + 15) // 16
    nb = nblk * batch + 5
    pool = KVPool(shape, nb, dtype=dtype)
    pool.tensor.normal_()
    table = torch.randperm(nb, generator=torch.Generator().manual_seed(2))[:nblk * batch].to(torch.int32) \
        .view(batch, nblk).cuda()
    lens = torch.full((batch,), seq, dtype=torch.int32, device="cuda")
    q = torch.randn(shape.layers, batch, q_heads, 128, device="cuda").to(dtype)
    ours = paged_decode(pool, q, table, lens, max_seq_len=seq)
    theirs = _flashinfer_decode(fi, pool, q, table, seq, dtype)
    torch.cuda.synchronize()
    torch.testing.assert_close(ours.float(), theirs.float(), atol=2e-3 if dtype == torch.float16 else 1e-2,
                               rtol=2e-2)


def test_flashinfer_decodes_a_migrated_cache_like_the_source():
    """The consumer pin of the copy path: after kvm_migrate (block-table row
    rewritten by the kernel), flashinfer's decode through the destination's
    rewritten row equals flashinfer's decode of the source — bit for bit,
    since the bytes are identical."""
    fi = pytest.importorskip("flashinfer")
    from paper_2501_06709_b200.executor import MigrationExecutor
    from paper_2501_06709_b200.planner import KV_TRANSFER, PendingMove, PlannedMove

    shape = ModelShape("fim", layers=4, kv_heads=8, head_dim=128, q_heads=32, d_model=1024)
    pools = {0: KVPool(shape, 96), 1: KVPool(shape, 96)}
    tables = {0: BlockTable(4, 64), 1: BlockTable(4, 64)}
    for p in pools.values():
        p.tensor.normal_()
    ex = MigrationExecutor(pools, tables)
    seq = 37 * 16 - 5
    ex.admit(1, 0, seq)
    nblk = len(ex.where(1).blocks)
    q = torch.randn(shape.layers, 1, shape.q_heads, 128, device="cuda").half()
    src_table = torch.from_numpy(ex.where(1).blocks)[None].contiguous().cuda()
    before = _flashinfer_decode(fi, pools[0], q, src_table, seq, torch.float16)
    ex.execute([PlannedMove(PendingMove(1, 0, 1, 0, seq), KV_TRANSFER)])
    row = tables[1].rows[tables[1].slot(1), :nblk][None].contiguous()
    assert np.array_equal(row.cpu().numpy()[0], ex.where(1).blocks)
    after = _flashinfer_decode(fi, pools[1], q, row, seq, torch.float16)
    torch.cuda.synchronize()
    assert torch.equal(before.view(torch.int16), after.view(torch.int16))


# --- the byte path: kvm_migrate / kvm_compact == vLLM's own block copy --------------------------------------
# vLLM moves KV blocks with _C_cache_ops.swap_blocks(src, dst, block_bytes, mapping): per cache tensor, block
# mapping[i][0] of src -> block mapping[i][1] of dst.  The paper's prototype sits on vLLM, so
# this is the published byte semantics of a block move; the pool planes below ARE vLLM's per-layer caches
# ([NB][16][H][D] contiguous per (layer, K|V)), and the foreign-layout case hands kvm_migrate vLLM's own
# FlashAttention tensors.  Expectation: whole pools byte-identical after the same mapping.

def _vllm_ops():
    try:
        import vllm._custom_ops as vops
        torch.ops._C_cache_ops.swap_blocks   # noqa: B018  (raises when vLLM's CUDA ops are not loadable)
    except Exception as e:  # pragma: no cover - the image ships vLLM 0.22
        pytest.skip(f"vLLM cache ops unavailable: {e!r}")
    return vops


def _rand_fill(t, seed):
    g = torch.Generator(device=t.device).manual_seed(seed)
    v = t.view(torch.int16)
    v.copy_(torch.randint(-2 ** 15, 2 ** 15, v.shape, generator=g, device=t.device, dtype=torch.int16))


def _planes(pool):
    return [pool.tensor[l, kv] for l in range(pool.shape.layers) for kv in range(2)]


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
@pytest.mark.parametrize("host_blocks", [True, False])
@pytest.mark.parametrize("n", [1, 19, 64])
def test_migrate_equals_vllm_swap_blocks(engine, host_blocks, n):
    """kvm_migrate(src pool -> dst pool) leaves the destination pool byte-identical to vLLM's swap_blocks
    applied plane by plane with the same (src block, dst block) mapping, and the source untouched."""
    import ctypes

    from paper_2501_06709_b200 import _native
    vops = _vllm_ops()
    shape = ModelShape("v", layers=3, kv_heads=8, head_dim=128, q_heads=8, d_model=1024)   # 32 KiB pieces
    nb = 96
    src, dst = KVPool(shape, nb), KVPool(shape, nb)
    _rand_fill(src.tensor, 11 + n)
    _rand_fill(dst.tensor, 12 + n)
    rng = np.random.default_rng(n)
    sb = rng.permutation(nb)[:n].astype(np.int32)
    dst.allocator.take(rng.permutation(nb)[:nb // 3])
    db = dst.allocator.alloc(n)
    expect = dst.tensor.clone()
    src_before = src.tensor.clone()
    mapping = torch.from_numpy(np.stack([sb, db], 1).astype(np.int64))
    for ps, pd in zip(_planes(src), [expect[l, kv] for l in range(shape.layers) for kv in range(2)]):
        vops.swap_blocks(ps, pd, shape.piece_bytes, mapping)
    m = _native.Move()
    m.src_pool, m.dst_pool, m.n_blocks = src.pool_id, dst.pool_id, n
    keep = []
    if host_blocks:
        m.src_blocks, m.dst_blocks = sb.ctypes.data, db.ctypes.data
        flags = _native.KVM_F_BLOCKS_ON_HOST
    else:
        keep = [torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()]
        m.src_blocks, m.dst_blocks = keep[0].data_ptr(), keep[1].data_ptr()
        flags = 0
    flags |= _native.KVM_F_ENGINE_BULK if engine == "bulk" else 0
    arr = (_native.Move * 1)(m)
    _native.check(_native.lib().kvm_migrate(arr, 1, flags, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(dst.tensor.view(torch.int16), expect.view(torch.int16))
    assert torch.equal(src.tensor.view(torch.int16), src_before.view(torch.int16))


@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_compact_equals_vllm_swap_blocks_in_place(engine):
    """kvm_compact (src pool == dst pool, disjoint block sets) == vLLM swap_blocks with src == dst tensor."""
    import ctypes

    from paper_2501_06709_b200 import _native
    vops = _vllm_ops()
    shape = ModelShape("v", layers=4, kv_heads=4, head_dim=128, q_heads=4, d_model=512)     # 16 KiB pieces
    nb = 128
    pool = KVPool(shape, nb)
    _rand_fill(pool.tensor, 3)
    perm = np.random.default_rng(3).permutation(nb).astype(np.int32)
    sb, db = perm[:45], perm[45:90]
    expect = pool.tensor.clone()
    mapping = torch.from_numpy(np.stack([sb, db], 1).astype(np.int64))
    for l in range(shape.layers):
        for kv in range(2):
            vops.swap_blocks(expect[l, kv], expect[l, kv], shape.piece_bytes, mapping)
    flags = _native.KVM_F_BLOCKS_ON_HOST | (_native.KVM_F_ENGINE_BULK if engine == "bulk" else 0)
    _native.check(_native.lib().kvm_compact(pool.pool_id, sb.ctypes.data, db.ctypes.data, len(sb), None, flags,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(pool.tensor.view(torch.int16), expect.view(torch.int16))


@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer"])
@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_migrate_between_vllm_caches_equals_swap_blocks(layout, engine):
    """Two vLLM-shaped per-layer cache sets (vLLM's own get_kv_cache_shape), registered in place: kvm_migrate
    between them == vLLM swap_blocks on the same tensors' K and V blocks (FlashAttention layout: the K / V
    halves are block arrays; FlashInfer: blocks interleave K|V, so the mapping moves 2b and 2b+1 of the
    [NB*2][16][H][D] view)."""
    import ctypes

    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.foreign import StridedKVPool, vllm_cache_shape
    vops = _vllm_ops()
    L, nb, H, D = 3, 64, 8, 128
    shp = vllm_cache_shape(layout, nb, 16, H, D)
    srcs = [torch.empty(shp, dtype=torch.float16, device="cuda") for _ in range(L)]
    dsts = [torch.empty(shp, dtype=torch.float16, device="cuda") for _ in range(L)]
    for i, t in enumerate(srcs + dsts):
        _rand_fill(t, 40 + i)
    sp, dp = StridedKVPool.from_vllm(srcs, layout), StridedKVPool.from_vllm(dsts, layout)
    rng = np.random.default_rng(9)
    sb = rng.permutation(nb)[:23].astype(np.int32)
    db = rng.permutation(nb)[:23].astype(np.int32)
    expect = [t.clone() for t in dsts]
    piece = 16 * H * D * 2
    for s, e in zip(srcs, expect):
        if layout == "flash_attn":
            m = torch.from_numpy(np.stack([sb, db], 1).astype(np.int64))
            for kv in range(2):
                vops.swap_blocks(s[kv], e[kv], piece, m)
        else:
            m = torch.from_numpy(np.concatenate([np.stack([2 * sb + kv, 2 * db + kv], 1) for kv in range(2)])
                                 .astype(np.int64))
            vops.swap_blocks(s, e, piece, m)
    mv = _native.Move()
    mv.src_pool, mv.dst_pool, mv.n_blocks = sp.pool_id, dp.pool_id, len(sb)
    mv.src_blocks, mv.dst_blocks = sb.ctypes.data, db.ctypes.data
    flags = _native.KVM_F_BLOCKS_ON_HOST | (_native.KVM_F_ENGINE_BULK if engine == "bulk" else 0)
    _native.check(_native.lib().kvm_migrate((_native.Move * 1)(mv), 1, flags,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    for got, e in zip(dsts, expect):
        assert torch.equal(got.view(torch.int16), e.view(torch.int16))
    sp.close()
    dp.close()


@pytest.mark.parametrize("layout", ["native", "flash_attn", "flashinfer"])
@pytest.mark.parametrize("engine", ["ldg", "bulk"])
def test_fp8_kv_caches_migrate_like_vllm_swap_blocks(layout, engine):
    """vLLM's fp8 KV caches (kv_cache_dtype="fp8": one byte per element, stored as uint8 / float8_e4m3fn)
    are bytes to the copy path: a pool with elem_bytes = 1 (native layout, or vLLM's own per-layer caches
    registered in place) migrates byte-identically to vLLM swap_blocks with the same mapping."""
    import ctypes

    from paper_2501_06709_b200 import _native
    from paper_2501_06709_b200.foreign import StridedKVPool, vllm_cache_shape
    vops = _vllm_ops()
    L, nb, H, D = 3, 48, 8, 128
    shape = ModelShape("fp8", layers=L, kv_heads=H, head_dim=D, q_heads=H, d_model=H * D, elem_bytes=1)
    piece = shape.piece_bytes                                   # 16 KiB
    rng = np.random.default_rng(4)
    sb = rng.permutation(nb)[:19].astype(np.int32)
    db = rng.permutation(nb)[:19].astype(np.int32)

    def rand_u8(shp, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        return torch.randint(0, 256, shp, generator=g, device="cuda", dtype=torch.uint8)

    if layout == "native":
        src = KVPool(shape, nb, tensor=rand_u8((L, 2, nb, 16, H, D), 1).view(torch.float8_e4m3fn))
        dst = KVPool(shape, nb, tensor=rand_u8((L, 2, nb, 16, H, D), 2).view(torch.float8_e4m3fn))
        expect = dst.tensor.view(torch.uint8).clone()
        m = torch.from_numpy(np.stack([sb, db], 1).astype(np.int64))
        for l in range(L):
            for kv in range(2):
                vops.swap_blocks(src.tensor.view(torch.uint8)[l, kv], expect[l, kv], piece, m)
        got = lambda: dst.tensor.view(torch.uint8)           # noqa: E731
    else:
        shp = vllm_cache_shape(layout, nb, 16, H, D)
        srcs = [rand_u8(shp, 10 + l) for l in range(L)]
        dsts = [rand_u8(shp, 20 + l) for l in range(L)]
        src, dst = StridedKVPool.from_vllm(srcs, layout), StridedKVPool.from_vllm(dsts, layout)
        exp_l = [t.clone() for t in dsts]
        for s_, e in zip(srcs, exp_l):
            if layout == "flash_attn":
                m = torch.from_numpy(np.stack([sb, db], 1).astype(np.int64))
                for kv in range(2):
                    vops.swap_blocks(s_[kv], e[kv], piece, m)
            else:
                m = torch.from_numpy(np.concatenate([np.stack([2 * sb + kv, 2 * db + kv], 1) for kv in range(2)])
                                     .astype(np.int64))
                vops.swap_blocks(s_, e, piece, m)
        expect = torch.stack(exp_l)
        got = lambda: torch.stack(dsts)                       # noqa: E731
    mv = _native.Move()
    mv.src_pool, mv.dst_pool, mv.n_blocks = src.pool_id, dst.pool_id, len(sb)
    mv.src_blocks, mv.dst_blocks = sb.ctypes.data, db.ctypes.data
    flags = _native.KVM_F_BLOCKS_ON_HOST | (_native.KVM_F_ENGINE_BULK if engine == "bulk" else 0)
    _native.check(_native.lib().kvm_migrate((_native.Move * 1)(mv), 1, flags,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(got(), expect)
