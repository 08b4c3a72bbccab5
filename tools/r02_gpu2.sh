#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( time timeout 900 python bench.py ) > gpurun_out/b70.log 2>&1
timeout 600 python bench.py --config llama7b --no-loopback --cpu-seconds 3 > gpurun_out/b7.log 2>&1
timeout 600 python bench.py --config llama7b --rank-shape-of 8 --no-loopback --cpu-seconds 2 > gpurun_out/b7r8.log 2>&1
timeout 600 python bench.py --gpus 2 --steps 3 > gpurun_out/b_n2.log 2>&1
echo done
