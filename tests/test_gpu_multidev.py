"""Single-process multi-GPU path (tools/multidev_check.py): the executor with
pools on two devices, stream-ordered moves across devices with freed-block
reuse, the cross-device split (push + re-prefill) and the fused split pulling
over the peer mapping, and a layer-pipelined decode on the peer.  Byte-exact
for copies; re-prefilled suffix within the bf16 tolerance.

On a 1-GPU box the cross-device test skips and the same checks run with both
'devices' = cuda:0, which exercises the harness and the same-device code paths."""
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def _assert_ok(res):
    bad = {k: v for k, v in res.items() if isinstance(v, dict) and not v.get("ok", True)}
    assert res["all_ok"] and not bad, bad


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_cross_device_checks():
    from multidev_check import run_checks

    res = run_checks(0, 1)
    assert res["cross_device"] is True
    _assert_ok(res)


def test_same_device_harness():
    from multidev_check import run_checks

    res = run_checks(0, 0)
    _assert_ok(res)
