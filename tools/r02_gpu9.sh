#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 ) > gpurun_out/pytest_gpu.log 2>&1
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench70.json 2> gpurun_out/bench70.err
timeout 600 python bench.py --config llama7b --rank-shape-of 8 --no-loopback --cpu-seconds 2 > gpurun_out/bench7r8.json 2>&1
timeout 600 python bench.py --config llama7b --rank-shape-of 4 --no-loopback --cpu-seconds 2 > gpurun_out/bench7r4.json 2>&1
for s in 7b_tp8 7b_tp4; do
  TL_PROBE_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_mlp_kernel -s 1 -c 1 \
     -o gpurun_out/r02_fused_$s -f python tools/ab.py $s mlp "" > gpurun_out/ncu_fused_$s.log 2>&1
done
echo done
