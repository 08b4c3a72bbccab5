#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( python tools/moe_timeline.py; python tools/moe_timeline.py "n_sub=1" ) > gpurun_out/moe_timeline.log 2>&1
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_ops.py 2,4 > gpurun_out/r02_sanitizer_memcheck.log 2>&1
timeout 2400 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_ops.py 2 > gpurun_out/r02_sanitizer_synccheck.log 2>&1
echo done
