#!/bin/bash
# K3 diagnostics: kernel time under the OZ_DEBUG_MODE bits (see PairParams.debug).
for mode in 0 1 2 3 4 5; do
  for tn in 128 192; do
    echo -n "mode=$mode tile_n=$tn: "
    OZ_TILE_N=$tn OZ_DEBUG_MODE=$mode timeout 120 python tools/run_once.py --reps 3 --pair-cutoff ${CUT:-11} 2>&1 | tail -1
  done
done
