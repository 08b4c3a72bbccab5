#!/bin/bash
# Cross-device evidence for a box with >= 2 B200s (SURVEY §7 risk R3): the data plane over real NVLink
# peers -- bulk / TMA tensor stores into IPC-mapped peer memory, pull-mode peer loads, sys-scope
# release/acquire flags across devices -- checked against the oracle, then bench.py at N = 2 .. n_gpus
# with NVML NVLink byte counters in each JSON line (nvlink_counters).  Never wraps a multi-rank command
# in ncu (B200_PROFILING.md); per-kernel NVLink traffic comes from the NVML counters instead.
#   usage: tools/two_gpu_check.sh [max_gpus]      (writes gpurun_out/xdev_*)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
N=${1:-$(nvidia-smi -L | wc -l)}
nvidia-smi topo -m > gpurun_out/xdev_topo.txt 2>&1
python -c "import torch; n=torch.cuda.device_count(); print({(a,b): torch.cuda.can_device_access_peer(a,b) for a in range(n) for b in range(n) if a!=b})" > gpurun_out/xdev_p2p.txt 2>&1
( timeout 1800 python -m pytest tests/test_gpu_multiproc.py -q 2>&1 | tail -20 ) > gpurun_out/xdev_pytest.log 2>&1
for n in 2 4 8; do
  [ "$n" -le "$N" ] || continue
  timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/xdev_bench_n$n.json 2> gpurun_out/xdev_bench_n$n.err
  timeout 900 python bench.py --gpus $n --config llama7b --steps 20 --warmup 5 --cpu-seconds 2 > gpurun_out/xdev_bench7b_n$n.json 2>> gpurun_out/xdev_bench_n$n.err
done
echo "done (N=$N)"
