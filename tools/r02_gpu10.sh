#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( for o in "n_sub=1" "n_sub=1,num_ctas=74" "n_sub=1,num_ctas=20" "n_sub=2" "n_sub=2,num_ctas=20"; do echo "== 7b_tp8 g1 $o"; python tools/tile_timeline.py 7b_tp8 g1 "$o"; done
  for o in "n_sub=1" "n_sub=2"; do echo "== 70b_tp8 g1 $o"; python tools/tile_timeline.py 70b_tp8 g1 "$o"; echo "== 70b_tp8 g2 $o"; python tools/tile_timeline.py 70b_tp8 g2 "$o"; done ) > gpurun_out/timeline3.log 2>&1
echo done
