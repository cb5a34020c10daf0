"""Config 5 on one B200: replay the reference's recorded runs with real KV
bytes (8 logical GPUs = 8 pools on cuda:0, mini 7B shape), every resident
request's fingerprint verified periodically and at the end."""
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,max_slots", [("trace_7b_c48g_seed0.json", None),
                                            ("trace_7b_mixed_seed0.json", 900),
                                            ("trace_multillm_7b13b_seed0.json", None)])
def test_trace_replay_bit_exact(name, max_slots):
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from replay_trace import MINI, MINI_7B, build
    from paper_2501_06709_b200.replay import TraceReplay

    fx = load_golden(name)
    ex, _ = build(fx, MINI_7B, "bulk", [0], MINI)
    rp = TraceReplay(fx, ex, model_map={m: s.name for m, s in MINI.items()})
    rep = rp.run(max_slots=max_slots, verify_every=200)
    assert rep.executed > 0 and rep.verified_requests > 0
    if "mixed" in name:
        assert rep.recomputed_requests > 0 or rep.executed > 0
    else:
        assert rep.bytes_moved > 0
