"""bench.py keeps the driver's JSON contract: the reference arm on CPU here,
the GPU arm under -m gpu (small test workload, no CPU-baseline sample)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--workload", "7b-512", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["unit"] == "GB/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"]


def test_reference_arm_under_torchrun_two_ranks():
    """The driver launches the reference arm like ours at N > 1 (torch.distributed.run, 2 ranks):
    rank 0 alone runs it and prints the one line, the other rank exits 0 without work."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--workload", "7b-512", "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0 and BASE_KEYS <= set(d)


def test_self_launch_runs_n_ranks_cpu():
    """`python bench.py --gpus 2` without torchrun re-launches itself under
    torch.distributed.run with 2 ranks (gloo here, no GPU): rank 0 prints the
    one line and it reports n_gpus == 2."""
    d = _run(["--launch-check", "--gpus", "2", "--steps", "3", "--warmup", "3"], timeout=300)
    assert d["launch_check"] is True and d["n_gpus"] == 2 and d["ranks"] == [0, 1] and d["max_rank"] == 1.0
    assert d["launcher"] == "self-launched torch.distributed.run"


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--launch-check", "--gpus", "1"],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr


def test_warmup_floor():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "2"], capture_output=True,
                         text=True, cwd=ROOT)
    assert out.returncode != 0


def test_ring_engine_choice_follows_the_peer_probe():
    """The N>1 A/B offers the TMA bulk engine only when the child-process probe
    pushed into a peer pool with it bit-exact; an explicit --engine wins."""
    sys.path.insert(0, ROOT)
    from bench import ring_engines

    ok = {"engine_push_over_peer": {"ok": True, "ldg": {"ok": True}, "bulk": {"ok": True}}}
    bad = {"engine_push_over_peer": {"ok": False, "error": "AssertionError: bulk: bytes differ on the peer"}}
    crashed = {"all_ok": False, "error": "rc=-6: illegal address"}
    assert ring_engines(None, None) == ["bulk", "ldg"]
    assert ring_engines(None, ok) == ["bulk", "ldg"]
    assert ring_engines(None, bad) == ["ldg"]
    assert ring_engines(None, crashed) == ["ldg"]
    assert ring_engines("bulk", bad) == ["bulk"]


def test_child_process_tools_report_instead_of_failing(tmp_path):
    """bench.py runs the cross-device probe, the 2-GPU split and config 5 in
    child processes: a result, a crash and a hang each come back as a dict
    (the rank that launched it stays alive and prints its line)."""
    sys.path.insert(0, ROOT)
    from bench import _tool_json

    ok = tmp_path / "ok.py"
    ok.write_text("import json, sys\nout = sys.argv[sys.argv.index('--out') + 1]\n"
                  "json.dump({'all_ok': True, 'x': int(sys.argv[1])}, open(out, 'w'))\n")
    crash = tmp_path / "crash.py"
    crash.write_text("raise SystemExit('illegal address')\n")
    hang = tmp_path / "hang.py"
    hang.write_text("import time\ntime.sleep(60)\n")
    r = _tool_json(str(ok), ["7"], timeout_s=60)
    assert r["all_ok"] is True and r["x"] == 7 and r["subprocess_s"] >= 0
    r = _tool_json(str(crash), [], timeout_s=60)
    assert r["all_ok"] is False and "illegal address" in r["error"]
    r = _tool_json(str(hang), [], timeout_s=2)
    assert r["all_ok"] is False and "timed out" in r["error"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--workload", "7b-512", "--steps", "5", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["bit_exact"] is True and d["value"] > 0 and d["n_gpus"] == 1
    assert d["gpu_launches"] == 5
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert r["peak"] > 1000
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * 32 * 4 and e["d2h_bytes_per_step"] == 32 * 4
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    k = d["kernels"]   # fresh re-prefill / decode measurements beside the headline
    assert k["reprefill_13b_s1360"]["unit"] == "TFLOP/s" and 0.3 < k["reprefill_13b_s1360"]["frac"] < 1.5
    assert k["reprefill_13b_s1360"]["cublas_same_shape"]["ms"] > 0
    assert k["decode_7b_4k_32l"]["unit"] == "GB/s" and 0.3 < k["decode_7b_4k_32l"]["frac"] < 1.5
    assert 0 < k["small_move_7b_1block"]["issue_to_landed_us_p50"] < 1000
    sp = k["split_13b_8k"]   # configs[2] on this GPU: parity first, then the timed arms
    assert sp["prefix_bit_exact"] is True and sp["suffix_within_tolerance"] is True, sp
    assert 0 < sp["ms"]["split_fused_one_kernel"] < sp["ms"]["split_two_kernels_serialized"]
    lib = d["library"]   # the library path on the same workload, timed in the same run
    assert lib["bit_exact"] is True and lib["value"] > 0 and lib["ours_over_library"] > 1


@pytest.mark.gpu
def test_gpu_arm_plain_python_two_ranks():
    """Plain `python bench.py --gpus 2` (no torchrun) measures two ranks: on a
    1-GPU box only with --shared-gpu (both ranks on the one GPU, IPC path, no
    NVLink), and it refuses without it."""
    import torch

    if torch.cuda.device_count() < 2:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "7b-512",
                              "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True,
                             timeout=600, cwd=ROOT)
        assert out.returncode != 0 and "--shared-gpu" in out.stderr
    d = _run(["--gpus", "2", "--workload", "7b-512", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
              "--shared-gpu"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 2 and d["bit_exact"] is True and d["value"] > 0
    assert d["config"]["launcher"] == "self-launched torch.distributed.run"
    assert d["e2e"]["value"] > 0 and d["e2e"]["row_ok"] is True
    assert d["config"]["engine"] in ("bulk", "ldg") and set(d["config"]["engine_ab"]) == {"bulk", "ldg"}
    assert "nvlink_counters" in d["roofline"] and d["gpu_launches"] > 0
    assert d["library"]["paper_transport"]["bit_exact"] is True and d["library"]["paper_transport"]["value"] > 0
    md = d["multi_device_checks"]   # the child-process probe ran (both 'devices' = cuda:0 on a 1-GPU box)
    assert md["all_ok"] is True and md["engine_push_over_peer"]["bulk"]["ok"] is True, md


@pytest.mark.gpu
def test_gpu_arm_four_ranks_shared():
    """Four ranks on the ring i -> (i+1) mod 4 (shared GPU on a 1-GPU box):
    every rank's received request bit-exact, one line with n_gpus == 4."""
    d = _run(["--gpus", "4", "--workload", "7b-512", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
              "--shared-gpu", "--no-multidev-checks"], timeout=900)
    assert d["n_gpus"] == 4 and d["bit_exact"] is True and d["value"] > 0 and d["e2e"]["row_ok"] is True


@pytest.mark.gpu
def test_gpu_arm_two_ranks_contract():
    """The N>1 launch (torchrun, one process per rank): on a 1-GPU box both ranks
    share the GPU (CUDA-IPC ring push, host-side receive); rank 0 prints one line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--workload", "7b-512", "--steps", "5", "--warmup", "3",
                          "--no-cpu-baseline", "--shared-gpu"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 2 and d["bit_exact"] is True and d["value"] > 0
    assert d["e2e"]["value"] > 0
