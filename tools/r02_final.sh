#!/bin/bash
# Round-2 final evidence: ncu full capture of the default bench layer's two kernels (70B, W = 1), the launch
# list of the default bench command, and the bench lines of every workload on the final build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tl_gemm_kernel -s 4 -c 2 \
   -o gpurun_out/prof_70b_final -f python tools/mlp_probe.py llama70b 3 > gpurun_out/ncu_70b_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/r02_final_bench_launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_launches_final.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err
timeout 900 python bench.py --config llama7b > gpurun_out/r02_final_bench_7b.json 2>> gpurun_out/r02_final_bench.err
timeout 900 python bench.py --config mixtral > gpurun_out/r02_final_bench_mixtral.json 2>> gpurun_out/r02_final_bench.err
timeout 900 python bench.py --rank-shape-of 8 > gpurun_out/r02_final_bench_70b_rank_of_tp8.json 2>> gpurun_out/r02_final_bench.err
timeout 900 python bench.py --config llama7b --rank-shape-of 8 > gpurun_out/r02_final_bench_7b_rank_of_tp8.json 2>> gpurun_out/r02_final_bench.err
timeout 900 python bench.py --workload moe > gpurun_out/r02_final_bench_moe.json 2>> gpurun_out/r02_final_bench.err
timeout 900 python bench.py --workload attention > gpurun_out/r02_final_bench_attention.json 2>> gpurun_out/r02_final_bench.err
echo done
