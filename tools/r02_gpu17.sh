#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "corrupted or full_size" 2>&1 | tail -5 ) > gpurun_out/pytest_neg.log 2>&1
for s in 7b_tp8 7b_tp4 70b_tp8; do
  AB_ROUNDS=1 AB_ITERS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_mlp_kernel -s 2 -c 1 \
     -o gpurun_out/r02_fused_v2_$s -f python tools/ab.py $s mlp "" > gpurun_out/ncu_fused_v2_$s.log 2>&1
done
timeout 1200 python bench.py --msweep --config llama7b --no-loopback --no-baseline --steps 10 > gpurun_out/msweep7b.jsonl 2> gpurun_out/msweep7b.err
echo done
