#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 ) > gpurun_out/pytest_gpu.log 2>&1
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench70_v3.json 2> gpurun_out/bench70_v3.err
timeout 900 python bench.py --config llama7b --no-loopback --cpu-seconds 3 > gpurun_out/bench7_v3.json 2> gpurun_out/bench7_v3.err
timeout 600 python bench.py --config llama70b --rank-shape-of 8 --no-loopback --cpu-seconds 2 > gpurun_out/bench70r8.json 2>&1
timeout 600 python bench.py --config llama7b --rank-shape-of 8 --no-loopback --cpu-seconds 2 > gpurun_out/bench7r8_v3.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-loopback > gpurun_out/ncu_launches.log 2>&1
echo done
