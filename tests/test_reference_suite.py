"""The REFERENCE's own planner tests, run against this repo's planner.

/root/reference/pkg/tests/test_migration.py (all cases), test_sim.py (the
slot loop, whose only data-plane call is plan_hybrid) and the acceptance
sweeps that exercise the planner (verification.budget_safety: 200 move sets
+ 10^4 consensus-order shuffles; determinism) are executed with
paper_2501_06709_b200.planner swapped into kvpack (tests/refsuite/patch_kvpack.py).
Skipped where the reference tree is not mounted (the GPU box)."""
import os
import subprocess
import sys

import pytest

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("test_file", ["test_migration.py", "test_sim.py",
                                       "test_acceptance.py::test_migration_budget_safety_and_consensus",
                                       "test_acceptance.py::test_simulation_is_deterministic"])
def test_reference_tests_pass_with_our_planner(test_file, tmp_path):
    if not os.path.isdir(REF):
        pytest.skip("reference tree not mounted")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), os.path.join(HERE, "refsuite"),
                                         env.get("PYTHONPATH", "")])
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "patch_kvpack", "-p", "no:cacheprovider",
                          "--rootdir", str(tmp_path), os.path.join(REF, "tests", test_file)],
                         capture_output=True, text=True, env=env, cwd=str(tmp_path), timeout=600)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and "failed" not in out.stdout


def test_entire_reference_suite_with_native_scheduler(tmp_path):
    """Every reference test (scheduler, model, sim, acceptance sweeps, oracle,
    baselines, CLI, ...) with BOTH the planner and the native C++ scheduler /
    cluster model (paper_2501_06709_b200.scheduler, .cluster) swapped into
    kvpack (KVPACK_PATCH_SCHEDULER=1 in tests/refsuite/patch_kvpack.py)."""
    if not os.path.isdir(REF):
        pytest.skip("reference tree not mounted")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), os.path.join(HERE, "refsuite"),
                                         env.get("PYTHONPATH", "")])
    env["KVPACK_PATCH_SCHEDULER"] = "1"
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "patch_kvpack", "-p", "no:cacheprovider",
                          "--rootdir", str(tmp_path), os.path.join(REF, "tests")],
                         capture_output=True, text=True, env=env, cwd=str(tmp_path), timeout=1200)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and "failed" not in out.stdout
