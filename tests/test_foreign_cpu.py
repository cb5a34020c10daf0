"""The foreign layouts StridedKVPool.from_vllm accepts are vLLM's own: the
per-layer cache shapes are checked against the installed vLLM backends'
get_kv_cache_shape (skipped when vLLM is not importable)."""
import pytest

from paper_2501_06709_b200.foreign import vllm_cache_shape


@pytest.mark.parametrize("layout,module,cls", [
    ("flash_attn", "vllm.v1.attention.backends.flash_attn", "FlashAttentionBackend"),
    ("flashinfer", "vllm.v1.attention.backends.flashinfer", "FlashInferBackend"),
])
def test_layouts_match_installed_vllm(layout, module, cls):
    import importlib

    try:
        backend = getattr(importlib.import_module(module), cls)
    except Exception as e:  # noqa: BLE001 - any import failure means "not available here"
        pytest.skip(f"vLLM backend not importable: {e}")
    for nb, bt, h, d in ((100, 16, 8, 128), (7, 16, 40, 128), (1, 16, 1, 64)):
        assert tuple(backend.get_kv_cache_shape(nb, bt, h, d)) == vllm_cache_shape(layout, nb, bt, h, d)
