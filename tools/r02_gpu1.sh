#!/bin/bash
# round-2 first contact: per-GEMM probe of the BASELINE shapes + ncu of the 70B W=1 GEMMs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 600 python tools/r02_probe.py 70b mix 7b 7b_tp2 7b_tp4 7b_tp8 70b_tp2 70b_tp4 70b_tp8 mix_tp2 mix_tp4 mix_tp8 > gpurun_out/probe.jsonl 2> gpurun_out/probe.err
TL_PROBE_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 5 -c 2 \
   -o gpurun_out/r02_70b_w1 -f python tools/r02_probe.py 70b > gpurun_out/ncu70b.log 2>&1
echo done
