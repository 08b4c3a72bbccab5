#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
for g in 4 8 16 32; do
  for shape in "2 8192 11008 4096 1" "2 8192 4096 11008"; do
    echo "raster_group=$g"; TL_RASTER_GROUP=$g timeout 120 python tools/probe.py gemm $shape 2>&1 | tail -1
  done
done
} 2>&1 | tee gpurun_out/raster_sweep.log
