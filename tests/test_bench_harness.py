"""Host-side logic of bench.py's N-rank harness (no GPU): labels derive from the actual world size
and exchange, and --gpus N without enough devices refuses instead of timing one GPU."""
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _args(config="C3"):
    return types.SimpleNamespace(config=config)


def test_single_gpu_label():
    from paper_2503_10032_b200.configs import CONFIGS
    c = bench.workload_config(_args(), CONFIGS["C3"], 1)
    assert c["parallelism"] == "single GPU"
    assert c["subdomains"] == 64 and c["neurons_per_subdomain"] == 800


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_labels_follow_world_and_exchange(world):
    from paper_2503_10032_b200.configs import CONFIGS
    c = bench.workload_config(_args(), CONFIGS["C3"], world, "nccl")
    assert c["parallelism"].startswith(f"sharded x{world}") and "NCCL" in c["parallelism"]
    h = bench.workload_config(_args(), CONFIGS["C3"], world, "host-staged (NCCL unavailable or forced)")
    assert h["parallelism"].startswith(f"sharded x{world}") and "host-staged" in h["parallelism"]


def test_dist_env_reads_torchrun_variables(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("LOCAL_RANK", "3")
    monkeypatch.delenv("DDELM_BENCH_ONE_GPU", raising=False)
    assert bench.dist_env() == (4, 3, 3)
    monkeypatch.setenv("DDELM_BENCH_ONE_GPU", "1")  # harness self-test: every rank on device 0
    assert bench.dist_env() == (4, 3, 0)


def test_gpus_without_devices_refuses():
    """--gpus 2 with no torchrun environment and fewer than 2 visible devices exits 2 with a
    message instead of timing a single GPU under an N-GPU label."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "DDELM_BENCH_ONE_GPU")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "needs 2 visible CUDA devices" in r.stderr
