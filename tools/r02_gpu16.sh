#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( AB_ROUNDS=10 AB_ITERS=8 python tools/ab.py 70b mlp "mlp_fused=0,n_sub=1" "mlp_fused=0,n_sub=2" "mlp_fused=0"
  AB_ROUNDS=8 AB_ITERS=30 python tools/ab.py 70b_tp2 mlp "n_sub=1" "n_sub=2" "mlp_fused=0,n_sub=1" "mlp_fused=0,n_sub=2"
  AB_ROUNDS=8 AB_ITERS=60 python tools/ab.py 70b_tp4 mlp "n_sub=1" "n_sub=2" "mlp_fused=0"
  AB_ROUNDS=8 AB_ITERS=20 python tools/ab.py mix mlp "mlp_fused=0,n_sub=1" "mlp_fused=0,n_sub=2" ) > gpurun_out/ab_nsub3.jsonl 2> gpurun_out/ab_nsub3.err
timeout 900 python bench.py --workload attention --no-loopback > gpurun_out/bench_attn_v2.json 2> gpurun_out/bench_attn_v2.err
echo done
