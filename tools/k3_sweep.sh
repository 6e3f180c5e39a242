#!/bin/bash
# K3 configuration sweep: kernel time, clocks and power per setting (bench.py --no-extras).

run() { echo -n "$1: "; env $1 timeout 200 python bench.py --no-extras --steps ${STEPS:-8} ${ARGS} 2>/dev/null | python tools/summ.py; }
for e in ${CONFIGS:-"OZ_X=0" "OZ_DEBUG_MODE=1" "OZ_PACE_SLACK=0" "OZ_PACE_SLACK=4" "OZ_TILE_N=128"}; do run "$e"; done
