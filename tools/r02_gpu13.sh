#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --no-loopback > gpurun_out/bench70_v2.json 2> gpurun_out/bench70_v2.err
timeout 900 python bench.py --workload moe --no-loopback > gpurun_out/bench_moe.json 2> gpurun_out/bench_moe.err
timeout 900 python bench.py --workload attention --no-loopback > gpurun_out/bench_attn.json 2> gpurun_out/bench_attn.err
echo done
