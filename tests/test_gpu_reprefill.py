"""tcgen05 re-prefill vs an fp32 reference (torch fp32 on the GPU for speed,
and the C oracle on the smallest case).

Tolerance (stated, bf16 output of an fp32-accumulated bf16 GEMM):
    |got - ref| <= 1e-2 + 1.6e-2 * |ref|     (ref = fp32 product of the bf16 operands)
Only the pool slots of the recomputed tokens may change.
"""
import numpy as np
import pytest
import torch

from oracle import kvmig_oracle as orc
from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool, ModelShape
from paper_2501_06709_b200.reprefill import reprefill, synthetic_hidden, synthetic_weights

pytestmark = pytest.mark.gpu
ATOL, RTOL = 1e-2, 1.6e-2


def _ref(x, w):  # [L, rows, n_out] fp32
    return torch.einsum("tk,lnk->ltn", x.float(), w.float())


def _check(shape, pool, blocks, tok0, rows, ref, q_out, before):
    kvd = shape.kv_cols
    qc = ref.shape[2] - 2 * kvd
    t = pool.tensor
    for l in range(shape.layers):
        toks = torch.arange(tok0, tok0 + rows, device="cuda")
        blk = blocks.long()[toks // 16]
        slot = toks % 16
        k = t[l, 0, blk, slot].reshape(rows, kvd).float()
        v = t[l, 1, blk, slot].reshape(rows, kvd).float()
        torch.testing.assert_close(k, ref[l, :, qc:qc + kvd], atol=ATOL, rtol=RTOL)
        torch.testing.assert_close(v, ref[l, :, qc + kvd:], atol=ATOL, rtol=RTOL)
        if q_out is not None:
            torch.testing.assert_close(q_out[l].float(), ref[l, :, :qc], atol=ATOL, rtol=RTOL)
    # nothing outside the recomputed token slots changed
    after = t.view(torch.int16).clone()
    mask = torch.ones(t.shape[2], 16, dtype=torch.bool, device="cuda")
    toks = torch.arange(tok0, tok0 + rows, device="cuda")
    mask[blocks.long()[toks // 16], toks % 16] = False
    assert torch.equal(after[:, :, mask], before[:, :, mask])


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("rows,tok0,with_q", [(1, 0, True), (77, 5, True), (128, 0, False),
                                              (300, 21, True), (513, 16, False), (1000, 3, True)])
def test_reprefill_small_shapes(rows, tok0, with_q, single_cta):
    shape = ModelShape("rp", layers=3, kv_heads=4, head_dim=64, q_heads=8, d_model=256)
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + 10
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = pool.tensor.view(torch.int16).clone()
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(rows))[:nblk].to(torch.int32).cuda()
    x = synthetic_hidden(shape, rows, 0, seed=rows)
    w = synthetic_weights(shape, 0, with_q=with_q, seed=rows + 1)
    q = torch.zeros(shape.layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda") if with_q else None
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q, single_cta=single_cta)
    torch.cuda.synchronize()
    _check(shape, pool, blocks, tok0, rows, _ref(x, w), q, before)


@pytest.mark.parametrize("single_cta", [False, True])
def test_reprefill_matches_c_oracle(single_cta):
    shape = ModelShape("rp", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=128)
    rows, tok0, nb = 40, 3, 6
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.zero_()
    blocks = torch.tensor([4, 1, 5], dtype=torch.int32, device="cuda")
    x = synthetic_hidden(shape, rows, 0, seed=9)
    w = synthetic_weights(shape, 0, with_q=True, seed=10)
    q = torch.zeros(shape.layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda")
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q, single_cta=single_cta)
    torch.cuda.synchronize()
    exp = np.zeros(pool.view_shape, dtype=np.uint16)
    q_exp = np.zeros((shape.layers, rows, shape.q_cols), dtype=np.uint16)
    orc.reprefill(orc.desc(2, 2, 64, 16, nb), exp, blocks.cpu().numpy(), x.view(torch.int16).cpu().numpy().view(np.uint16),
                  w.view(torch.int16).cpu().numpy().view(np.uint16), rows, shape.d_model, shape.q_cols, tok0, q_exp)
    to_f = lambda b: torch.from_numpy(b.astype(np.int32) << 16).view(torch.float32)  # noqa: E731
    got = pool.tensor.float().cpu()
    exp_f = to_f(exp.reshape(-1)).view(pool.view_shape)
    torch.testing.assert_close(got, exp_f, atol=ATOL, rtol=RTOL)
    torch.testing.assert_close(q.float().cpu(), to_f(q_exp.reshape(-1)).view(q_exp.shape), atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("single_cta", [False, True])
def test_reprefill_13b_balanced_split(single_cta):
    """BASELINE configs[2]: 13B, suffix of s ~ 1.4k tokens of an 8k request."""
    shape = LLAMA2_13B
    rows, tok0 = 1360, 8192 - 1360
    nblk = 8192 // 16
    nb = nblk + 8
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(0))[:nblk].to(torch.int32).cuda()
    x = synthetic_hidden(shape, rows, 0, seed=2)
    w = synthetic_weights(shape, 0, with_q=True, seed=3)
    before = pool.tensor.view(torch.int16).clone()
    reprefill(pool, x, w, blocks, tok0=tok0, single_cta=single_cta)
    torch.cuda.synchronize()
    # check a sample of layers against fp32 (full einsum over 40 layers is 8.6 TFLOP)
    kvd, qc = shape.kv_cols, shape.q_cols
    for l in (0, 17, 39):
        ref = x.float() @ w[l].float().t()
        toks = torch.arange(tok0, tok0 + rows, device="cuda")
        blk, slot = blocks.long()[toks // 16], toks % 16
        torch.testing.assert_close(pool.tensor[l, 0, blk, slot].reshape(rows, kvd).float(), ref[:, qc:qc + kvd],
                                   atol=ATOL, rtol=RTOL)
        torch.testing.assert_close(pool.tensor[l, 1, blk, slot].reshape(rows, kvd).float(), ref[:, qc + kvd:],
                                   atol=ATOL, rtol=RTOL)
    after = pool.tensor.view(torch.int16)
    toks = torch.arange(tok0, tok0 + rows, device="cuda")
    mask = torch.ones(nb, 16, dtype=torch.bool, device="cuda")
    mask[blocks.long()[toks // 16], toks % 16] = False
    assert torch.equal(after[:, :, mask], before[:, :, mask])


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("kv_heads,head_dim,q_heads", [(3, 64, 1), (1, 32, 3), (5, 96, 0)])
def test_reprefill_n_not_multiple_of_tile(kv_heads, head_dim, q_heads, single_cta):
    """n_out = q_cols + 2*kv_cols not a multiple of the 256-column N tile."""
    shape = ModelShape("nt", layers=2, kv_heads=kv_heads, head_dim=head_dim, q_heads=max(q_heads, 1), d_model=128)
    rows, tok0 = 50, 7
    nb = (tok0 + rows + 15) // 16 + 3
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = pool.tensor.view(torch.int16).clone()
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:(tok0 + rows + 15) // 16]
    blocks = blocks.to(torch.int32).cuda()
    x = synthetic_hidden(shape, rows, 0, seed=3)
    w = synthetic_weights(shape, 0, with_q=q_heads > 0, seed=4)
    assert w.shape[1] % 256 != 0
    reprefill(pool, x, w, blocks, tok0=tok0, single_cta=single_cta)
    torch.cuda.synchronize()
    _check(shape, pool, blocks, tok0, rows, _ref(x, w), None, before)


@pytest.mark.parametrize("shape_name,rows,tok0", [("llama3-70b-gqa", 2000, 16384 - 2000), ("llama2-7b", 3000, 100)])
def test_reprefill_full_shapes_pair_kernel(shape_name, rows, tok0):
    """The default CTA-pair kernel at the other model shapes (70B GQA: d_model 8192,
    n_out 10240; 7B: 4096 / 12288), sampled layers against fp32, Q included."""
    from paper_2501_06709_b200.kvcache import SHAPES

    shape = SHAPES[shape_name]
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + 4
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(7))[:nblk].to(torch.int32).cuda()
    x = synthetic_hidden(shape, rows, 0, seed=11)
    w = synthetic_weights(shape, 0, with_q=True, seed=12)
    q = torch.zeros(shape.layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda")
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q)
    torch.cuda.synchronize()
    kvd, qc = shape.kv_cols, shape.q_cols
    toks = torch.arange(tok0, tok0 + rows, device="cuda")
    blk, slot = blocks.long()[toks // 16], toks % 16
    for l in (0, shape.layers // 2, shape.layers - 1):
        ref = x.float() @ w[l].float().t()
        torch.testing.assert_close(q[l].float(), ref[:, :qc], atol=ATOL, rtol=RTOL)
        torch.testing.assert_close(pool.tensor[l, 0, blk, slot].reshape(rows, kvd).float(), ref[:, qc:qc + kvd],
                                   atol=ATOL, rtol=RTOL)
        torch.testing.assert_close(pool.tensor[l, 1, blk, slot].reshape(rows, kvd).float(), ref[:, qc + kvd:],
                                   atol=ATOL, rtol=RTOL)


def _rope_ref(y, positions, theta, q_cols, kv_cols):
    """HF Llama rotate_half RoPE on the Q and K columns of y [L, rows, n_out] (fp32),
    angles in float64; V untouched."""
    y = y.clone()
    i = torch.arange(64, dtype=torch.float64, device=y.device)
    ang = positions.to(torch.float64)[:, None] * theta ** (-2.0 * i / 128.0)
    c, s = torch.cos(ang).float(), torch.sin(ang).float()          # [rows, 64]
    for lo, hi in ((0, q_cols), (q_cols, q_cols + kv_cols)):
        if hi <= lo:   # no Q columns
            continue
        seg = y[:, :, lo:hi].reshape(y.shape[0], y.shape[1], -1, 128).clone()   # (reshape may alias y)
        a, b = seg[..., :64].clone(), seg[..., 64:].clone()
        seg[..., :64] = a * c[None, :, None, :] - b * s[None, :, None, :]
        seg[..., 64:] = b * c[None, :, None, :] + a * s[None, :, None, :]
        y[:, :, lo:hi] = seg.reshape(y.shape[0], y.shape[1], -1)
    return y


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("rows,tok0", [(1, 0), (77, 5), (300, 4000), (513, 16)])
def test_reprefill_rope(rows, tok0, single_cta):
    """KVM_REPREFILL_ROPE: K in the pool and Q are post-RoPE (positions tok0 + t),
    V is not rotated; both engines."""
    shape = ModelShape("rope", layers=2, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + 6
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = pool.tensor.view(torch.int16).clone()
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(rows))[:nblk].to(torch.int32).cuda()
    x = synthetic_hidden(shape, rows, 0, seed=rows + 3)
    w = synthetic_weights(shape, 0, with_q=True, seed=rows + 4)
    q = torch.zeros(shape.layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda")
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q, single_cta=single_cta, rope_theta=10000.0)
    torch.cuda.synchronize()
    pos = torch.arange(tok0, tok0 + rows, device="cuda")
    ref = _rope_ref(_ref(x, w), pos, 10000.0, shape.q_cols, shape.kv_cols)
    _check(shape, pool, blocks, tok0, rows, ref, q, before)


def test_reprefill_rope_needs_head_dim_128():
    from paper_2501_06709_b200.errors import ConfigError

    shape = ModelShape("rope64", layers=1, kv_heads=2, head_dim=64, q_heads=2, d_model=128)
    pool = KVPool(shape, 4, dtype=torch.bfloat16)
    x = synthetic_hidden(shape, 16, 0)
    w = synthetic_weights(shape, 0, with_q=False)
    with pytest.raises(ConfigError):
        reprefill(pool, x, w, torch.arange(1, dtype=torch.int32, device="cuda"), rope_theta=10000.0)


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("rows,tok0,rope", [(1, 0, False), (300, 21, False), (1000, 3, True), (513, 4000, True)])
def test_reprefill_per_layer_hidden(rows, tok0, rope, single_cta):
    """KVM_REPREFILL_X_PER_LAYER: x is [layers][rows][d_model] and layer l's
    K/V/Q come from x[l] (a model forward's per-layer inputs)."""
    shape = ModelShape("xl", layers=4, kv_heads=2, head_dim=128, q_heads=4, d_model=256)
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + 5
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = pool.tensor.view(torch.int16).clone()
    blocks = torch.randperm(nb, generator=torch.Generator().manual_seed(rows + 1))[:nblk].to(torch.int32).cuda()
    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn(shape.layers, rows, shape.d_model, generator=g, device="cuda").to(torch.bfloat16)
    w = synthetic_weights(shape, 0, with_q=True, seed=rows + 2)
    q = torch.zeros(shape.layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda")
    theta = 10000.0 if rope else None
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q, single_cta=single_cta, rope_theta=theta)
    torch.cuda.synchronize()
    ref = torch.einsum("ltk,lnk->ltn", x.float(), w.float())
    if rope:
        ref = _rope_ref(ref, torch.arange(tok0, tok0 + rows, device="cuda"), theta, shape.q_cols, shape.kv_cols)
    _check(shape, pool, blocks, tok0, rows, ref, q, before)


def test_reprefill_per_layer_13b_sampled():
    """Per-layer x at the 13B balanced-split size (pair kernel), sampled layers."""
    shape = LLAMA2_13B
    rows, tok0 = 1360, 8192 - 1360
    nblk = 8192 // 16
    pool = KVPool(shape, nblk + 4, dtype=torch.bfloat16)
    blocks = torch.randperm(nblk + 4, generator=torch.Generator().manual_seed(5))[:nblk].to(torch.int32).cuda()
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(shape.layers, rows, shape.d_model, generator=g, device="cuda").to(torch.bfloat16)
    w = synthetic_weights(shape, 0, with_q=True, seed=7)
    reprefill(pool, x, w, blocks, tok0=tok0)
    torch.cuda.synchronize()
    kvd, qc = shape.kv_cols, shape.q_cols
    toks = torch.arange(tok0, tok0 + rows, device="cuda")
    blk, slot = blocks.long()[toks // 16], toks % 16
    for l in (0, 1, 22, 39):
        ref = x[l].float() @ w[l].float().t()
        torch.testing.assert_close(pool.tensor[l, 0, blk, slot].reshape(rows, kvd).float(), ref[:, qc:qc + kvd],
                                   atol=ATOL, rtol=RTOL)
        torch.testing.assert_close(pool.tensor[l, 1, blk, slot].reshape(rows, kvd).float(), ref[:, qc + kvd:],
                                   atol=ATOL, rtol=RTOL)


def test_reprefill_per_layer_wrong_layers():
    from paper_2501_06709_b200.errors import ConfigError

    shape = ModelShape("xl2", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=128)
    pool = KVPool(shape, 4, dtype=torch.bfloat16)
    x = torch.zeros(3, 16, 128, dtype=torch.bfloat16, device="cuda")
    w = synthetic_weights(shape, 0, with_q=False)
    with pytest.raises(ConfigError):
        reprefill(pool, x, w, torch.arange(1, dtype=torch.int32, device="cuda"))


def test_reprefill_many_launches_on_two_streams():
    """150 re-prefill launches alternating between two streams (more than the
    64 completion / tile counter slots, so slots are reused while the other
    stream may still hold them): every result matches fp32."""
    shape = ModelShape("two", layers=2, kv_heads=2, head_dim=64, q_heads=2, d_model=128)
    rows = 40
    nblk = (rows + 15) // 16
    pools = [KVPool(shape, nblk + 2, dtype=torch.bfloat16) for _ in range(2)]
    blocks = torch.arange(nblk, dtype=torch.int32, device="cuda")
    xs = [synthetic_hidden(shape, rows, 0, seed=30 + i) for i in range(2)]
    w = synthetic_weights(shape, 0, with_q=False, seed=32)
    streams = [torch.cuda.Stream() for _ in range(2)]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for k in range(150):
        i = k % 2
        reprefill(pools[i], xs[i], w, blocks, stream=streams[i], single_cta=(k % 3 == 0))
    torch.cuda.synchronize()
    kvd = shape.kv_cols
    toks = torch.arange(rows, device="cuda")
    for i in range(2):
        ref = _ref(xs[i], w)
        for l in range(shape.layers):
            t = pools[i].tensor
            k_ = t[l, 0, blocks.long()[toks // 16], toks % 16].reshape(rows, kvd).float()
            torch.testing.assert_close(k_, ref[l, :, :kvd], atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVM_FUZZ_SEEDS", "100"))))
def test_reprefill_randomized(seed):
    """Random geometry (layers, heads, head_dim, d_model, rows, tok0), Q on/off,
    RoPE on/off, per-layer X on/off, either GEMM engine, scattered blocks:
    every K/V slot and Q within tolerance of fp32, nothing else written."""
    rng = np.random.default_rng(5000 + seed)
    head_dim = int(rng.choice([64, 128]))
    kv_heads = int(rng.integers(1, 5))
    q_heads = kv_heads * int(rng.choice([1, 2, 4]))
    layers = int(rng.integers(1, 4))
    d_model = 64 * int(rng.integers(1, 9))
    shape = ModelShape(f"fz{seed}", layers=layers, kv_heads=kv_heads, head_dim=head_dim, q_heads=q_heads,
                       d_model=d_model)
    rows, tok0 = int(rng.integers(1, 700)), int(rng.integers(0, 300))
    with_q = bool(rng.integers(2))
    rope = head_dim == 128 and bool(rng.integers(2))
    per_layer = bool(rng.integers(2))
    single = bool(rng.integers(2))
    nblk = (tok0 + rows + 15) // 16
    nb = nblk + int(rng.integers(1, 9))
    pool = KVPool(shape, nb, dtype=torch.bfloat16)
    pool.tensor.view(torch.int16).random_(-2 ** 15, 2 ** 15 - 1)
    before = pool.tensor.view(torch.int16).clone()
    blocks = torch.from_numpy(rng.permutation(nb)[:nblk].astype(np.int32)).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    xs = (layers, rows, d_model) if per_layer else (rows, d_model)
    x = torch.randn(xs, generator=g, device="cuda").to(torch.bfloat16)
    w = synthetic_weights(shape, 0, with_q=with_q, seed=seed + 1)
    q = torch.zeros(layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda") if with_q else None
    reprefill(pool, x, w, blocks, tok0=tok0, q_out=q, single_cta=single, rope_theta=10000.0 if rope else None)
    torch.cuda.synchronize()
    ref = torch.einsum("ltk,lnk->ltn" if per_layer else "tk,lnk->ltn", x.float(), w.float())
    if rope:
        ref = _rope_ref(ref, torch.arange(tok0, tok0 + rows, device="cuda"), 10000.0,
                        shape.q_cols if with_q else 0, shape.kv_cols)
    _check(shape, pool, blocks, tok0, rows, ref, q, before)


@pytest.mark.parametrize("single_cta", [False, True])
@pytest.mark.parametrize("max_sms", [1, 2, 7, 40, 100, 255])
def test_reprefill_sm_budget_bit_identical(max_sms, single_cta):
    """KVM_REPREFILL_MAX_SMS(n): the re-prefill on at most n SMs writes exactly the bytes the uncapped
    launch writes (every output tile is the same contraction whichever CTA computes it), and Q too."""
    shape = ModelShape("b", layers=3, kv_heads=4, head_dim=128, q_heads=8, d_model=512)
    rows, tok0 = 700, 9
    nblk = (tok0 + rows + 15) // 16
    w = synthetic_weights(shape, 0, with_q=True, seed=5)
    x = synthetic_hidden(shape, rows, 0, seed=6)
    blocks = torch.randperm(nblk + 4, generator=torch.Generator().manual_seed(2))[:nblk].to(torch.int32).cuda()
    outs = []
    for cap in (0, max_sms):
        pool = KVPool(shape, nblk + 4, dtype=torch.bfloat16)
        pool.tensor.zero_()
        q = torch.zeros(shape.layers, rows, shape.q_cols, dtype=torch.bfloat16, device="cuda")
        reprefill(pool, x, w, blocks, tok0=tok0, q_out=q, single_cta=single_cta, max_sms=cap, rope_theta=10000.0)
        torch.cuda.synchronize()
        outs.append((pool.tensor.view(torch.int16).clone(), q.view(torch.int16).clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_reprefill_sm_budget_rejects_out_of_range():
    shape = ModelShape("b", layers=1, kv_heads=1, head_dim=128, q_heads=1, d_model=64)
    pool = KVPool(shape, 4, dtype=torch.bfloat16)
    w = synthetic_weights(shape, 0, with_q=False, seed=1)
    x = synthetic_hidden(shape, 16, 0, seed=1)
    with pytest.raises(ValueError):
        reprefill(pool, x, w, torch.arange(1, dtype=torch.int32, device="cuda"), max_sms=256)
