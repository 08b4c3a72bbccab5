#!/bin/bash
# One probe step per process, each under its own timeout, so a trap or hang in one step
# cannot take the others (or the box) with it.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() { echo "== $*"; timeout 120 python tools/probe.py "$@" 2>&1 | tail -5; echo "rc=$?"; }
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
run gemm 1 128 256 64
run gemm 1 256 512 256
run gemm 2 256 256 64
run gemm 2 1024 1024 1024
run gemm 1 1000 1000 1000
run gemm 2 1000 1000 1000
run gemm 2 512 384 512 1
run gemm 1 512 384 512 1
run gemm 2 8192 8192 8192
run gemm 2 8192 11008 4096 1
run ag 2 512 256 256
run ag 4 1024 512 256 1
run ag 8 8192 1376 4096 1
run rs 2 512 256 256
run rs 2 512 256 256 1
run rs 8 8192 4096 1376
run rs 8 8192 4096 1376 1
} 2>&1 | tee gpurun_out/probe.log
