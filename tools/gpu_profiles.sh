#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command, full capture of the dominant kernel,
# full capture of the fused AG kernel (loopback W=8, copy role + flags active).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 3 -c 1 \
   -o gpurun_out/prof_gemm1_final -f python tools/probe.py gemm 2 8192 11008 4096 1 > gpurun_out/ncu_gemm1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 3 -c 1 \
   -o gpurun_out/prof_gemm2_final -f python tools/probe.py gemm 2 8192 4096 11008 > gpurun_out/ncu_gemm2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -c 1 \
   -o gpurun_out/prof_loopback_ag8 -f python tools/probe.py ag 8 8192 1376 4096 1 > gpurun_out/ncu_ag8.log 2>&1
