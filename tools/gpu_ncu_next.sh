#!/bin/bash
# ncu evidence for the NEXT rows: full captures of the SP attention kernel (W=1, Attn-1 S=16k) and of
# the MoE kernels (MoE-4 first half, second half GEMM+scatter and owner reduce; MoE-1 TP-8 rank shape).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${NCU_TAG:-next}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tl_attn_kernel -s 2 -c 1 \
   -o gpurun_out/prof_attn_${N} -f python tools/attn_bench.py 1,16384,32 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tl_gemm_kernel|tl_moe" -s 6 -c 3 \
   -o gpurun_out/prof_moe4_${N} -f python tools/moe_bench.py MoE-4 > gpurun_out/ncu_moe4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tl_gemm_kernel|tl_moe" -s 6 -c 3 \
   -o gpurun_out/prof_moe1tp8_${N} -f python tools/moe_bench.py MoE-1_rank_of_tp8 > gpurun_out/ncu_moe1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/moe_launches.csv \
   python tools/moe_bench.py MoE-4 MoE-1_rank_of_tp8 > gpurun_out/ncu_moe_launches.log 2>&1
