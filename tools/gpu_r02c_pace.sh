# A/B: cross-CTA pacing slack (scheduling only) for the fixed-step cutoff-11 mode and the headline.
for s in 2 1 4 8 0 2; do OZ_PACE_SLACK=$s timeout 300 python tools/pace_time.py; done > gpurun_out/pace_ab.txt 2>&1
cat gpurun_out/pace_ab.txt
