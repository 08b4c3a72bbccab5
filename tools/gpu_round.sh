#!/bin/bash
# GPU session: parity suite, smoke, ncu capture of the GEMM core, quick bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 ) > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > gpurun_out/smoke.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 3 -c 1 \
     -o gpurun_out/prof_gemm1 -f python tools/probe.py gemm 2 8192 11008 4096 1 > gpurun_out/ncu_gemm.log 2>&1
fi
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
