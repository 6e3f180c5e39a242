# A/B of MMA queue-depth builds liboz_d{0,2,3}.so (experiment patch, reverted: OZ_MMA_DEPTH no longer exists; see profiles/mma_depth_ab_r01.json).
L=paper_2508_00441_b200/liboz_b200.so
cp $L liboz_keep.so
for r in 1 2; do
for v in d0 d2 d3; do
  cp liboz_$v.so $L
  for c in "" "--pair-cutoff 11"; do
    o=gpurun_out/dp_${v}_${r}_${c// /}.json
    timeout 300 python bench.py --no-extras --no-variants --steps 5 --warmup 3 $c > $o 2>> gpurun_out/dp_err.txt
    python -c "import json;d=json.loads(open('$o').read().strip().splitlines()[-1]);print('$v','$c',round(d['roofline']['kernel_ms'],2),round(d['value'],3),d['clocks']['sm_mhz'])"
  done
done
done
for v in d2 d3; do
  cp liboz_$v.so $L
  echo "tests $v"; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
done
cp liboz_keep.so $L
