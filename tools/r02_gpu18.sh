#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( TL_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --config llama7b --M 2048 --steps 3 --warmup 3 --cpu-seconds 1 ) > gpurun_out/shared2.log 2>&1
( TL_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 4 --config llama7b --M 4096 --steps 3 --warmup 3 --cpu-seconds 1 ) > gpurun_out/shared4.log 2>&1
export AB_ROUNDS=6
( AB_ITERS=60 python tools/ab.py 70b_tp8 mlp "" "n_sub=1" "n_sub=2"
  AB_ITERS=200 python tools/ab.py 7b_tp8 mlp "" "n_sub=1"
  AB_ITERS=8 python tools/ab.py 70b mlp "" "n_sub=1" "n_sub=2" ) > gpurun_out/ab_nsub4.jsonl 2> gpurun_out/ab_nsub4.err
echo done
