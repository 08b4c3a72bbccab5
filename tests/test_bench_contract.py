"""bench.py's reference arm (the oracle on host cores) prints one JSON line with the contract's keys,
for every workload, and the same `config` the GPU arm uses.  CPU only (no GPU needed)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


@pytest.mark.parametrize("workload", ["mlp", "moe", "attention"])
def test_reference_arm_json(workload):
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", workload, "--steps", "1",
                        "--warmup", "1", "--ref-rows", "8"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"]
    import bench
    import bench_workloads as BW   # the GPU arm's config for the same workload
    if workload == "mlp":
        assert d["config"] == bench.bench_config(1)
        assert d["config"]["workload"] == "llama70b_mlp_w1"   # the largest single-GPU config (MLP-5)
        assert d["cpu_baseline"]["cores"] >= 1 and "cpu_model" in d["cpu_baseline"]
    elif workload == "moe":
        assert d["config"] == BW.moe_config(1)
    elif workload == "attention":
        assert d["config"] == BW.attn_config(1)


@pytest.mark.parametrize("gpus", [2, 4])
def test_self_launch_dry_run(gpus):
    """`bench.py --gpus N` outside torchrun re-executes itself with N ranks (gloo in --dry-run): exactly one
    JSON line, from rank 0, for the W = N workload, with the max over ranks taken across all N."""
    import bench
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(gpus), "--dry-run", "--steps", "2"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["ranks_seen"] == gpus
    assert d["config"] == bench.bench_config(gpus) and d["config"]["workload"] == f"llama70b_mlp_w{gpus}"


def test_reference_arm_other_ranks_silent():
    """Under torchrun the reference arm runs on rank 0 only; other ranks exit 0 without output."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 0 and not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_roofline_terms():
    """Layer roofline of SURVEY §8(d): FLOPs and NVLink bytes per rank at the 7B and 70B shapes."""
    import bench
    f1, f2 = bench.layer_flops(8192, 4096, 11008, 8)
    assert (f1, f2) == (2 * 8192 * 4096 * 2752, 2 * 8192 * 1376 * 4096)
    assert bench.nvlink_bytes(8192, 4096, 8) == (7 * 1024 * 4096 * 2,) * 2      # 56 MiB per direction
    assert bench.nvlink_bytes(8192, 8192, 1) == (0, 0)
