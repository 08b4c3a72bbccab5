#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
true
export AB_ROUNDS=5
( AB_ITERS=200 python tools/ab.py 7b_tp8 mlp "mlp_fused=0" "mlp_fused=1" "mlp_fused=1,n_sub=1" "mlp_fused=1,n_sub=2"
  AB_ITERS=60 python tools/ab.py 70b_tp8 mlp "mlp_fused=0" "mlp_fused=1"
  AB_ITERS=100 python tools/ab.py 7b_tp4 mlp "mlp_fused=0" "mlp_fused=1"
  AB_ITERS=10 python tools/ab.py 70b mlp "mlp_fused=0" "mlp_fused=1" ) > gpurun_out/ab_fused.jsonl 2> gpurun_out/ab_fused.err
echo done
