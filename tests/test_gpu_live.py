"""Live migration (f2): the request keeps decoding on the source while full
blocks are pre-copied; the stop-and-copy moves only the tail.  The migrated
cache must equal what decode wrote, token for token, and the destination
block-table row must be the allocation (filled by the copy kernels)."""
import numpy as np
import pytest
import torch

from paper_2501_06709_b200.executor import MigrationExecutor
from paper_2501_06709_b200.kvcache import BlockTable, KVPool, ModelShape
from paper_2501_06709_b200.live import LiveMigration

pytestmark = pytest.mark.gpu
SHAPE = ModelShape("live", layers=4, kv_heads=4, head_dim=64, q_heads=4, d_model=256)


def _token_value(rid, tok, L):
    return ((rid * 131 + tok * 7) % 30000 + torch.arange(L, device="cuda")[:, None] * 2
            + torch.arange(2, device="cuda")[None, :]).to(torch.int16)


def _decode_write(ex, rid, tok, stream):
    """Mock decode step: write token `tok`'s K/V (all layers) at the source."""
    r = ex.where(rid)
    pool = ex.pool(r.gpu, r.model)
    blk, slot = int(r.blocks[tok // 16]), tok % 16
    with torch.cuda.stream(stream):
        v = _token_value(rid, tok, SHAPE.layers)
        pool.tensor.view(torch.int16)[:, :, blk, slot] = v[:, :, None, None]


@pytest.mark.parametrize("stream_ordered", [False, True])
@pytest.mark.parametrize("prompt,decode_steps,precopy_every", [(100, 200, 16), (33, 50, 5), (512, 0, 1)])
def test_live_migration_consistent(prompt, decode_steps, precopy_every, stream_ordered):
    pools = {0: KVPool(SHAPE, 128), 1: KVPool(SHAPE, 128)}
    tables = {0: BlockTable(4, 64), 1: BlockTable(4, 64)}
    ex = MigrationExecutor(pools, tables)
    dec = torch.cuda.Stream()
    rid = 5
    ex.admit(rid, 0, prompt)
    for t in range(prompt):
        _decode_write(ex, rid, t, dec)
    lm = LiveMigration(ex, rid, 1)
    tokens = prompt
    ev = torch.cuda.Event()
    for step in range(decode_steps):
        tokens += 1
        ex.grow(rid, tokens)
        _decode_write(ex, rid, tokens - 1, dec)
        if step % precopy_every == 0:
            ev.record(dec)
            lm.precopy(after=ev)
    ev.record(dec)
    lm.precopy(after=ev)
    ev.record(dec)
    st = lm.finish(after=ev, stream_ordered=stream_ordered)
    if stream_ordered:   # the destination's decode stream would wait on this event
        torch.cuda.current_stream().wait_event(st.done)
    assert ex.where(rid).gpu == 1
    assert st.blocks_stopcopied <= 2 or decode_steps == 0
    r = ex.where(rid)
    pool = pools[1]
    for t in range(tokens):
        got = pool.tensor.view(torch.int16)[:, :, int(r.blocks[t // 16]), t % 16]
        exp = _token_value(rid, t, SHAPE.layers)[:, :, None, None].expand_as(got)
        assert torch.equal(got, exp), f"token {t}"
    assert np.array_equal(tables[1].rows[tables[1].slot(rid), :len(r.blocks)].cpu().numpy(), r.blocks)
    assert pools[0].allocator.n_free == 128
