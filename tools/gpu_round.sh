#!/bin/bash
# GPU session: parity suite, smoke, optional ncu captures, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
which nvidia-cuda-mps-control > gpurun_out/mps.txt 2>&1; nvidia-smi -q | grep -i -E "compute mode|MIG mode" -A1 >> gpurun_out/mps.txt 2>&1
( timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -30 ) > gpurun_out/pytest_gpu.log 2>&1
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > gpurun_out/smoke.log 2>&1
if [ -n "$NCU_GEMM" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 3 -c 1 \
     -o gpurun_out/prof_$NCU_NAME -f python tools/probe.py $NCU_GEMM > gpurun_out/ncu_gemm.log 2>&1
fi
if [ -n "$NCU_LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_launches.log 2>&1
fi
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
