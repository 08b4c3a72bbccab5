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
    elif workload == "moe":
        assert d["config"] == BW.moe_config(1)
    elif workload == "attention":
        assert d["config"] == BW.attn_config(1)
