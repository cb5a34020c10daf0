"""CPU-only: the byte-path oracle's known answers, the host objects, and the
C ABI surface of libkvmig.so (load + exported symbols; no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import kvmig_oracle as orc
from paper_2501_06709_b200 import kvcache
from paper_2501_06709_b200.kvcache import (LLAMA2_7B, LLAMA2_13B, LLAMA3_70B, BlockAllocator,
                                           blocks_for_bytes)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pool(rng, L, H, D, nb):
    return rng.integers(-2 ** 15, 2 ** 15, size=(L, 2, nb, 16, H, D), dtype=np.int16)


def test_shapes_match_survey():
    assert LLAMA2_7B.kv_bytes_per_token == 524_288
    assert LLAMA2_13B.kv_bytes_per_token == 819_200
    assert LLAMA3_70B.kv_bytes_per_token == 327_680
    assert LLAMA2_7B.piece_bytes == 128 * 1024
    assert LLAMA2_13B.piece_bytes == 160 * 1024
    assert LLAMA3_70B.piece_bytes == 32 * 1024
    assert 4096 * LLAMA2_7B.kv_bytes_per_token == 2 ** 31
    assert blocks_for_bytes(4096 * LLAMA2_7B.kv_bytes_per_token, LLAMA2_7B) == 256
    with pytest.raises(ValueError):
        blocks_for_bytes(LLAMA2_7B.kv_bytes_per_token + 1, LLAMA2_7B)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_oracle_migrate_identity(threads):
    rng = np.random.default_rng(0)
    L, H, D, nb = 3, 4, 32, 40
    src, dst = _pool(rng, L, H, D, nb), _pool(rng, L, H, D, nb)
    before = dst.copy()
    sb = rng.permutation(nb)[:13].astype(np.int32)
    free = np.ones(nb, dtype=np.uint8)
    free[rng.permutation(nb)[:20]] = 0
    db = orc.alloc_ascending(free, 13)
    assert list(db) == sorted(db)
    sd = dd = orc.desc(L, H, D, 16, nb)
    row = orc.migrate(src, sd, dst, dd, sb, db, threads=threads)
    assert list(row) == list(db)
    for i in range(13):
        assert np.array_equal(dst[:, :, db[i]], src[:, :, sb[i]])
    untouched = np.setdiff1d(np.arange(nb), db)
    assert np.array_equal(dst[:, :, untouched], before[:, :, untouched])


def test_oracle_nan_payloads_bit_exact():
    L, H, D, nb = 1, 1, 8, 4
    src = np.full((L, 2, nb, 16, H, D), 0x7E01, dtype=np.uint16)  # fp16 NaN with payload
    src[..., 1] = 0xFC00  # -inf
    dst = np.zeros_like(src)
    d = orc.desc(L, H, D, 16, nb)
    orc.migrate(src, d, dst, d, [3, 0], [1, 2])
    assert np.array_equal(dst[:, :, 1], src[:, :, 3]) and np.array_equal(dst[:, :, 2], src[:, :, 0])


def test_oracle_rejects_out_of_range():
    d = orc.desc(1, 1, 8, 16, 4)
    a = np.zeros((1, 2, 4, 16, 1, 8), dtype=np.int16)
    with pytest.raises(ValueError):
        orc.migrate(a, d, a.copy(), d, [4], [0])


def test_allocator_matches_oracle():
    rng = np.random.default_rng(3)
    nb = 300
    a = BlockAllocator(nb)
    taken = rng.permutation(nb)[:150]
    a.take(taken)
    mask = np.ones(nb, dtype=np.uint8)
    mask[taken] = 0
    for n in (7, 1, 40, 0, 33):
        got = a.alloc(n)
        exp = orc.alloc_ascending(mask, n)
        assert np.array_equal(got, exp)
    a.free(got)
    with pytest.raises(ValueError):
        a.free(got)
    with pytest.raises(kvcache.RequestTooLarge):
        a.alloc(10 ** 6)


def test_oracle_reprefill_matches_numpy():
    rng = np.random.default_rng(5)
    L, H, D, nb, dm, qc, rows, tok0 = 2, 2, 16, 6, 64, 32, 21, 5
    kvd = H * D
    n_out = qc + 2 * kvd

    def bf16_bits(a):
        u = a.astype(np.float32).view(np.uint32)
        return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)

    def bits_to_f32(b):
        return (b.astype(np.uint32) << 16).view(np.float32)

    x = bf16_bits(rng.standard_normal((rows, dm)))
    w = bf16_bits(rng.standard_normal((L, n_out, dm)) / 8)
    pool = np.zeros((L, 2, nb, 16, H, D), dtype=np.uint16)
    blocks = np.array([4, 0, 2], dtype=np.int32)  # tokens 0..47
    q = np.zeros((L, rows, qc), dtype=np.uint16)
    orc.reprefill(orc.desc(L, H, D, 16, nb), pool, blocks, x, w, rows, dm, qc, tok0, q)
    ref = np.einsum("tk,lnk->ltn", bits_to_f32(x).astype(np.float64), bits_to_f32(w).astype(np.float64))
    for l in range(L):
        np.testing.assert_allclose(bits_to_f32(q[l]), ref[l, :, :qc], rtol=1e-2, atol=1e-2)
        for t in range(rows):
            tok = tok0 + t
            blk, slot = blocks[tok // 16], tok % 16
            k = bits_to_f32(pool[l, 0, blk, slot].reshape(-1))
            v = bits_to_f32(pool[l, 1, blk, slot].reshape(-1))
            np.testing.assert_allclose(k, ref[l, t, qc:qc + kvd], rtol=1e-2, atol=1e-2)
            np.testing.assert_allclose(v, ref[l, t, qc + kvd:], rtol=1e-2, atol=1e-2)


def test_oracle_reprefill_pinned_to_hf_llama_projections():
    """Pin the oracle to a third-party implementation: the C
    restatement's K/V for tokens [tok0, tok0 + rows) == HF transformers'
    LlamaAttention k_proj / v_proj / q_proj (nn.Linear, fp32 math on the same
    bf16 operands, rounded to bf16), scattered by the PagedAttention slot
    rule block_table[p // 16], p % 16.  RoPE is pinned on the GPU kernel
    (tests/test_gpu_thirdparty.py)."""
    import torch
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaAttention

    L, H, Hq, D, dm, rows, tok0, nb = 2, 2, 4, 64, 256, 45, 11, 8
    cfg = LlamaConfig(hidden_size=dm, num_attention_heads=Hq, num_key_value_heads=H, head_dim=D,
                      num_hidden_layers=L, intermediate_size=512, vocab_size=64)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(rows, dm, generator=g).to(torch.bfloat16)
    att = [LlamaAttention(cfg, layer_idx=l) for l in range(L)]
    ws = []
    with torch.no_grad():
        for a in att:
            for lin in (a.q_proj, a.k_proj, a.v_proj):
                lin.weight.copy_((torch.randn(lin.weight.shape, generator=g) / 8).to(torch.bfloat16).float())
            ws.append(torch.cat([a.q_proj.weight, a.k_proj.weight, a.v_proj.weight]).to(torch.bfloat16))
    w = torch.stack(ws)                                   # [L][q + 2kv][dm], our layout
    blocks = np.array([6, 1, 3, 0], dtype=np.int32)       # tokens 0..63
    pool = np.zeros((L, 2, nb, 16, H, D), dtype=np.uint16)
    q = np.zeros((L, rows, Hq * D), dtype=np.uint16)
    as_u16 = lambda t: t.contiguous().view(torch.int16).numpy().view(np.uint16)  # noqa: E731
    orc.reprefill(orc.desc(L, H, D, 16, nb), pool, blocks, as_u16(x), as_u16(w), rows, dm, Hq * D, tok0, q)
    pool_f = torch.from_numpy(pool.astype(np.int32) << 16).view(torch.float32)
    q_f = torch.from_numpy(q.astype(np.int32) << 16).view(torch.float32)
    pos = torch.arange(tok0, tok0 + rows)
    blk, slot = torch.from_numpy(blocks).long()[pos // 16], pos % 16
    with torch.no_grad():
        for l, a in enumerate(att):
            k = a.k_proj(x.float()).to(torch.bfloat16).float().view(rows, H, D)
            v = a.v_proj(x.float()).to(torch.bfloat16).float().view(rows, H, D)
            qq = a.q_proj(x.float()).to(torch.bfloat16).float()
            torch.testing.assert_close(pool_f[l, 0, blk, slot], k, atol=1e-2, rtol=1.6e-2)
            torch.testing.assert_close(pool_f[l, 1, blk, slot], v, atol=1e-2, rtol=1.6e-2)
            torch.testing.assert_close(q_f[l], qq, atol=1e-2, rtol=1.6e-2)
    # nothing outside the request's token slots was written
    mask = np.ones((nb, 16), dtype=bool)
    mask[blk.numpy(), slot.numpy()] = False
    assert not pool[:, :, mask].any()


# --- C ABI surface ----------------------------------------------------------------

def _header_symbols():
    with open(os.path.join(ROOT, "include", "kvmig.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(kvm_\w+)\(", text, re.M)))


def test_abi_library_exports_every_header_symbol():
    from paper_2501_06709_b200 import _native

    L = _native.lib()
    syms = _header_symbols()
    assert len(syms) >= 15
    assert set(syms) == set(_native.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    assert L.kvm_version() == _native.ABI_VERSION
    with open(os.path.join(ROOT, "include", "kvmig.h")) as fh:
        assert int(re.search(r"#define KVM_ABI_VERSION (\d+)", fh.read()).group(1)) == _native.ABI_VERSION


_STRUCTS = {  # ctypes mirror -> C struct in include/kvmig.h
    "PoolDesc": "kvm_pool_desc", "Move": "kvm_move", "ReprefillArgs": "kvm_reprefill_args",
    "SplitArgs": "kvm_split_args", "DecodeArgs": "kvm_decode_args", "Pending": "kvm_pending",
    "PlanParams": "kvm_plan_params", "Planned": "kvm_planned", "PlanLedgers": "kvm_plan_ledgers",
    "SchedParams": "kvm_sched_params",
}


def test_abi_struct_layouts_match_the_c_compiler(tmp_path):
    """Every ctypes mirror has the C compiler's size and field offsets for the
    header's struct (gcc on include/kvmig.h)."""
    import shutil
    import subprocess

    from paper_2501_06709_b200 import _native

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "kvmig.h"', "int main(void) {"]
    for py, c in _STRUCTS.items():
        lines.append(f'printf("{py} size %zu\\n", sizeof({c}));')
        for name, _ in getattr(_native, py)._fields_:
            lines.append(f'printf("{py} {name} %zu\\n", offsetof({c}, {name}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        py, field, val = line.split()
        got[(py, field)] = int(val)
    for py in _STRUCTS:
        cls = getattr(_native, py)
        assert got[(py, "size")] == ctypes.sizeof(cls), py
        for name, _ in cls._fields_:
            assert got[(py, name)] == getattr(cls, name).offset, (py, name)


def test_abi_error_mapping_without_gpu():
    from paper_2501_06709_b200 import ConfigError, _native

    d = _native.PoolDesc(0, 1, 1, 16, 1, 2)
    out = ctypes.c_int64()
    with pytest.raises(ConfigError):
        _native.check(_native.lib().kvm_pool_bytes(ctypes.byref(d), ctypes.byref(out)))
    d = _native.PoolDesc(32, 32, 128, 16, 256, 2)
    _native.check(_native.lib().kvm_pool_bytes(ctypes.byref(d), ctypes.byref(out)))
    assert out.value == 256 * 16 * LLAMA2_7B.kv_bytes_per_token
    with pytest.raises(ValueError):
        _native.check(_native.lib().kvm_migrate(None, -1, 0, None))
    assert _native.lib().kvm_migrate(None, 0, 0, None) == 0


def test_abi_struct_layout():
    from paper_2501_06709_b200 import _native

    assert ctypes.sizeof(_native.PoolDesc) == 24
    assert ctypes.sizeof(_native.Move) == 56
    assert _native.Move.src_blocks.offset == 16


# --- the oracle pinned to third-party outputs (vLLM swap_blocks, flashinfer decode) -------------------------
# tests/golden/thirdparty_vectors.json is written on a B200 by tests/golden/make_thirdparty_golden.py from the
# libraries the paper's prototype ran its data plane in; inputs are regenerated here from seeds.
_TP = os.path.join(ROOT, "tests", "golden", "thirdparty_vectors.json")


def _tp_vectors():
    import json
    with open(_TP) as fh:
        return json.load(fh)


def test_oracle_migrate_equals_vllm_swap_blocks_vectors():
    """oracle_migrate over whole pools == vLLM swap_blocks applied per (layer, K|V) plane (sha256 of the
    destination pool; the source unchanged), incl. in-place compaction and NaN/inf bit patterns."""
    import hashlib
    import importlib.util
    spec = importlib.util.spec_from_file_location("mk", os.path.join(ROOT, "tests", "golden",
                                                                    "make_thirdparty_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    vec = _tp_vectors()
    assert len(vec["swap_blocks"]) == len(mk.SWAP_CASES)
    for case in vec["swap_blocks"]:
        L, H, D = case["layers"], case["kv_heads"], case["head_dim"]
        src, dst, sb, db = mk.swap_inputs(L, H, D, case["src_nb"], case["dst_nb"], case["n"], case["seed"],
                                          case["in_place"])
        src = src.view(np.int16).reshape(L, 2, case["src_nb"], 16, H, D)
        sd = orc.desc(L, H, D, 16, case["src_nb"])
        if case["in_place"]:
            orc.migrate(src, sd, src, sd, sb, db)
            got = src
        else:
            dst = dst.view(np.int16).reshape(L, 2, case["dst_nb"], 16, H, D)
            before = hashlib.sha256(src.tobytes()).hexdigest()
            orc.migrate(src, sd, dst, orc.desc(L, H, D, 16, case["dst_nb"]), sb, db)
            got = dst
            assert hashlib.sha256(src.tobytes()).hexdigest() == before == case["src_sha256"], case["name"]
        assert hashlib.sha256(got.tobytes()).hexdigest() == case["dst_sha256"], case["name"]


def test_oracle_decode_equals_flashinfer_vectors():
    """oracle/attention_ref.reference_decode (fp32 torch on CPU) == flashinfer's paged decode output recorded
    on a B200 for the same pool / page table / queries (fp16; atol 2e-3, rtol 2e-2 as the GPU test)."""
    import importlib.util
    from types import SimpleNamespace

    import torch

    from oracle.attention_ref import reference_decode
    spec = importlib.util.spec_from_file_location("mk", os.path.join(ROOT, "tests", "golden",
                                                                    "make_thirdparty_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    for case in _tp_vectors()["decode"]:
        H, Hq, lens = case["kv_heads"], case["q_heads"], case["seq_lens"]
        k, v, tables, q = mk.decode_inputs(H, Hq, lens, case["seed"])
        pool = SimpleNamespace(shape=SimpleNamespace(head_dim=128, kv_heads=H, block_tokens=16),
                               tensor=torch.from_numpy(np.stack([k, v])[None]))
        got = reference_decode(pool, torch.from_numpy(q)[None], [torch.from_numpy(t) for t in tables], lens)
        want = torch.tensor([float.fromhex(x) for x in case["out_f32_hex"]]).view(len(lens), Hq, 128)
        torch.testing.assert_close(got[0], want, atol=2e-3, rtol=2e-2, msg=case["name"])


def test_python_flag_constants_mirror_the_header():
    """Every KVM_F_* / KVM_REPREFILL_* / KVM_DECODE_* / KVM_ERR_* value the Python side passes through
    the C ABI equals include/kvmig.h's #define, macros (KVM_F_CTAS_PER_SM, KVM_REPREFILL_MAX_SMS)
    evaluated for a few arguments."""
    from paper_2501_06709_b200 import _native
    with open(os.path.join(ROOT, "include", "kvmig.h")) as fh:
        hdr = fh.read()
    plain = dict(re.findall(r"#define (KVM_(?:F|REPREFILL|DECODE|ERR)_[A-Z_0-9]+) \(?(-?(?:0x)?[0-9a-fA-F]+)\)?", hdr))
    checked = 0
    for name, val in plain.items():
        if hasattr(_native, name) and not callable(getattr(_native, name)):
            assert getattr(_native, name) == int(val, 0), name
            checked += 1
    assert checked >= 16
    assert "#define KVM_F_CTAS_PER_SM(n) (((n)&0xff) << 8)" in hdr
    assert "#define KVM_REPREFILL_MAX_SMS(n) (((n)&0xff) << 8)" in hdr
    assert "#define KVM_F_MAX_SMS(n) (((n)&0xff) << 16)" in hdr
    for n in (0, 1, 64, 148, 255):
        assert _native.KVM_F_CTAS_PER_SM(n) == (n & 0xFF) << 8
        assert _native.KVM_F_MAX_SMS(n) == (n & 0xFF) << 16
        assert _native.KVM_REPREFILL_MAX_SMS(n) == (n & 0xFF) << 8
        assert _native.KVM_REPREFILL_MAX_SMS(n) & ~int(plain["KVM_REPREFILL_SMS_MASK"], 0) == 0


def test_sm_budget_maps_the_comp_budget_fraction():
    from paper_2501_06709_b200.reprefill import sm_budget
    assert sm_budget(0.2, 148) == 30          # the reference's default budget_fraction (config.py:70)
    assert sm_budget(1.0, 148) == 0 and sm_budget(3.0, 148) == 0     # every SM
    assert sm_budget(0.001, 148) == 2         # at least one CTA pair
    assert sm_budget(0.5, 1000) == 255        # the flag's 8-bit field
    with pytest.raises(ValueError):
        sm_budget(0.0, 148)


def test_oracle_reprefill_placement_equals_vllm_reshape_and_cache_vectors():
    """The C oracle's re-prefill places token t of the suffix in slot (tok0 + t) of the request's blocks
    exactly as vLLM's reshape_and_cache_flash does (recorded on a B200): with identity K / V projections
    (K = V = X, exact in fp32 accumulation) the oracle's K and V planes hash like vLLM's key / value caches."""
    import hashlib
    import importlib.util
    spec = importlib.util.spec_from_file_location("mk", os.path.join(ROOT, "tests", "golden",
                                                                    "make_thirdparty_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    cases = _tp_vectors()["placement"]
    assert len(cases) == len(mk.PLACEMENT_CASES)
    for case in cases:
        H, rows, tok0 = case["kv_heads"], case["rows"], case["tok0"]
        x, blocks, nb = mk.placement_inputs(H, rows, tok0, case["seed"])
        kvd = H * 128
        eye = np.zeros((kvd, kvd), dtype=np.uint16)
        eye[np.arange(kvd), np.arange(kvd)] = 0x3F80                       # bf16 1.0
        w = np.ascontiguousarray(np.concatenate([eye, eye])[None])          # [1][2 kvd][kvd]: K = V = X
        pool = np.zeros((1, 2, nb, 16, H, 128), dtype=np.uint16)
        orc.reprefill(orc.desc(1, H, 128, 16, nb), pool, blocks, np.ascontiguousarray(x), w, rows, kvd, 0, tok0)
        assert hashlib.sha256(pool[0, 0].tobytes()).hexdigest() == case["key_cache_sha256"], case["name"]
        assert hashlib.sha256(pool[0, 1].tobytes()).hexdigest() == case["value_cache_sha256"], case["name"]
