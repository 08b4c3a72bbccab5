#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_2503_20313_b200/libtilelink_b200_old.so paper_2503_20313_b200/libtilelink_b200.so; do
  for i in 1 2; do
    echo "$lib"; TL_LIB_PATH=$PWD/$lib timeout 120 python tools/probe.py rs 8 8192 4096 1376 2>&1 | tail -1
    TL_LIB_PATH=$PWD/$lib timeout 120 python tools/lb_rs_time.py 2>&1 | tail -1
  done
done 2>&1 | tee gpurun_out/ab_rs.log
