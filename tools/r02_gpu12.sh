#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( AB_ROUNDS=8 AB_ITERS=8 python tools/ab.py 70b mlp "n_sub=1" "n_sub=2" "n_sub=1" "n_sub=2"
  AB_ROUNDS=8 AB_ITERS=8 python tools/ab.py 70b g1 "n_sub=1" "n_sub=2"
  AB_ROUNDS=8 AB_ITERS=16 python tools/ab.py 70b g2 "n_sub=1" "n_sub=2"
  AB_ROUNDS=6 AB_ITERS=20 python tools/ab.py mix mlp "n_sub=1" "n_sub=2"
  AB_ROUNDS=6 AB_ITERS=60 python tools/ab.py 70b_tp4 mlp "n_sub=1" "n_sub=2"
  AB_ROUNDS=6 AB_ITERS=60 python tools/ab.py mix_tp4 mlp "n_sub=1" "n_sub=2"
  AB_ROUNDS=6 AB_ITERS=30 python tools/ab.py 70b_tp2 mlp "n_sub=1" "n_sub=2"
  AB_ROUNDS=6 AB_ITERS=40 python tools/ab.py 7b mlp "n_sub=1" "n_sub=2"
  AB_ROUNDS=6 AB_ITERS=100 python tools/ab.py mix_tp8 mlp "n_sub=1" "n_sub=2" ) > gpurun_out/ab_nsub2.jsonl 2> gpurun_out/ab_nsub2.err
echo done
