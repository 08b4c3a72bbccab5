#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export AB_ROUNDS=5 AB_ITERS=30
( python tools/ab.py 70b g1 "" "n_sub=1" "raster_group=8" "raster_group=32" "raster_group=4" cublas
  python tools/ab.py 70b g2 "" "n_sub=1" "raster_group=8" "raster_group=32" "raster_group=4" cublas
  AB_ITERS=300 python tools/ab.py 7b_tp8 layer "" "n_sub=1" "n_sub=2" cublas
  AB_ITERS=100 python tools/ab.py 70b_tp8 layer "" "n_sub=1" "n_sub=2" cublas ) > gpurun_out/ab1.jsonl 2> gpurun_out/ab1.err
echo done
