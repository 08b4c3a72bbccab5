#!/bin/bash
# A/B of GEMM-core variants on the 7B layer shapes (one process per point).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
for ns in 1 2; do
  for shape in "2 8192 11008 4096 1" "2 8192 4096 11008" "2 8192 8192 8192" "2 8192 1376 4096 1" "2 8192 4096 1376"; do
    echo "n_sub=$ns"; TL_N_SUB=$ns timeout 120 python tools/probe.py gemm $shape 2>&1 | tail -1
  done
done
} 2>&1 | tee gpurun_out/perf_sweep.log
