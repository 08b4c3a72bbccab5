"""The N > 1 bench path on real GPU processes: `bench.py --gpus 2` self-launches two ranks (torchrun, NCCL),
both time-sharing the one test GPU (TL_BENCH_SHARED_GPU=1: a code-path check, not a measurement; the
process group is gloo, so the NCCL + cuBLAS baseline is skipped).  The driver's multi-GPU run executes the
same code with one GPU per rank: CUDA-IPC bootstrap, the fused layer's AG/RS protocol across processes,
max-over-ranks timing, e2e through the pipeline, and the sampled element-wise parity of every rank's block
against the fp64 oracle."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_shared_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["TL_BENCH_SHARED_GPU"] = "1"
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "llama7b", "--M", "2048", "--steps", "2",
                        "--warmup", "3", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["world"] == 2 and d["config"]["workload"] == "llama7b_mlp_w2_M2048"
    assert d["parity"]["status"] == 0 and d["parity"]["elements_over_bound"] == 0, d["parity"]
    assert d["e2e"]["output_matches_device_run"] is True
    base = d["baseline_nccl_cublas"]   # skipped when the ranks share one GPU (NCCL needs one device per rank)
    assert base is None or base["parity_rel_fro"] < 5e-3
    assert d["gpu_launches"] > 0 and "TL_BENCH_SHARED_GPU" in d["mode"]
