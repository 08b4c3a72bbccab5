#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( timeout 1500 python -m pytest tests/test_gpu_pull.py tests/test_gpu_multiproc.py tests/test_gpu_parity.py -q -x 2>&1 | tail -40 ) > gpurun_out/pytest_pull.log 2>&1
echo done
