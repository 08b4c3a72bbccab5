#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for s in 7b_tp8 70b_tp8; do
  TL_PROBE_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 5 -c 2 \
     -o gpurun_out/r02_$s -f python tools/r02_probe.py $s > gpurun_out/ncu_$s.log 2>&1
done
TL_PROBE_OPTS=n_sub=1 TL_PROBE_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 5 -c 2 \
     -o gpurun_out/r02_7b_tp8_nsub1 -f python tools/r02_probe.py 7b_tp8 > gpurun_out/ncu_7b_tp8_nsub1.log 2>&1
echo done
