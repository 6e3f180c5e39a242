#!/bin/bash
# Square-size sweep (BASELINE config 2): device-timed FP64-equiv TFLOPS per n.
for n in 1024 2048 4096 8192 16384; do
  for a in "" "--pair-cutoff 11"; do
    echo -n "n=$n $a: "; timeout 300 python bench.py --no-extras --n $n $a 2>/dev/null | python tools/summ.py
  done
done
