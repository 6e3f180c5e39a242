#!/bin/bash
# Kernel-variant choice vs problem size (tile quantisation against MMA shape).
for n in 2048 3072 4096 6144; do
  for v in "OZ_X=0" "OZ_TILE_N=128" "OZ_CTA_GROUP=1"; do
    echo -n "n=$n $v: "; env $v timeout 120 python bench.py --no-extras --steps 5 --n=$n --pair-cutoff=11 2>/dev/null | python tools/summ.py
  done
done
