# A/B: liboz_base.so (HEAD) vs liboz_pre.so (experiment patch OZ_EPI_PRELOAD, reverted; see profiles/epi_preload_ab_r01.json).
L=paper_2508_00441_b200/liboz_b200.so
cp $L liboz_keep.so
for r in 1 2; do
for v in base pre; do
  cp liboz_$v.so $L
  for c in "" "--pair-cutoff 11"; do
    o=gpurun_out/pre_${v}_${r}_${c// /}.json
    timeout 300 python bench.py --no-extras --no-variants --steps 5 --warmup 3 $c > $o 2>> gpurun_out/pre_err.txt
    python -c "import json;d=json.loads(open('$o').read().strip().splitlines()[-1]);print('$v','$c',round(d['roofline']['kernel_ms'],2),round(d['value'],3),d['clocks']['sm_mhz'])"
  done
done
done
cp liboz_pre.so $L
echo "tests pre"; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
cp liboz_keep.so $L
