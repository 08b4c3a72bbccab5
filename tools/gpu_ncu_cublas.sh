#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:nvjet -s 3 -c 1 -o gpurun_out/prof_cublas_gemm1 -f python tools/cublas_probe.py gemm1 > gpurun_out/ncu_cublas.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:nvjet -s 3 -c 1 -o gpurun_out/prof_cublas_gemm2 -f python tools/cublas_probe.py gemm2 >> gpurun_out/ncu_cublas.log 2>&1
NCU_GEMM="2 8192 4096 11008" NCU_NAME=gemm2 bash tools/gpu_round.sh
