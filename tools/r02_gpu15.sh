#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_pull.py -q -x 2>&1 | tail -5 ) > gpurun_out/pytest_moe.log 2>&1
timeout 900 python bench.py --workload moe --no-loopback > gpurun_out/bench_moe_v2.json 2> gpurun_out/bench_moe_v2.err
TL_PROBE_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 5 -c 2 \
     -o gpurun_out/r02_70b_w1_v2 -f python tools/r02_probe.py 70b > gpurun_out/ncu70b_v2.log 2>&1
echo done
