#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( for o in "n_sub=1" "n_sub=2"; do echo "== 7b_tp8 g1 $o"; python tools/tile_timeline.py 7b_tp8 g1 "$o"; echo "== 70b_tp8 g2 $o"; python tools/tile_timeline.py 70b_tp8 g2 "$o"; done ) > gpurun_out/timeline4.log 2>&1
( timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_moe.py -q -x 2>&1 | tail -5 ) > gpurun_out/pytest_mma.log 2>&1
export AB_ROUNDS=5
( AB_ITERS=200 python tools/ab.py 7b_tp8 mlp "" "n_sub=1" "n_sub=2" cublas
  AB_ITERS=100 python tools/ab.py 7b_tp4 mlp "" "n_sub=1" "n_sub=2" cublas
  AB_ITERS=60 python tools/ab.py 70b_tp8 mlp "" "n_sub=1" "n_sub=2" cublas
  AB_ITERS=10 python tools/ab.py 70b mlp "" "n_sub=1" "mlp_fused=0" cublas ) > gpurun_out/ab_mma.jsonl 2> gpurun_out/ab_mma.err
echo done
