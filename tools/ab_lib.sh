set -x
L=paper_2508_00441_b200/liboz_b200.so
for r in 1 2; do
for v in int fma; do  # build liboz_int.so with -DOZ_TERM_FMA=0, liboz_fma.so with the default
  cp liboz_$v.so $L
  for c in "" "--pair-cutoff 11"; do
    timeout 300 python bench.py --no-extras --no-variants --steps 5 --warmup 3 $c > gpurun_out/ab_${v}_${r}_${c// /}.json 2> gpurun_out/ab_err.txt
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${v}_${r}_${c// /}.json').read().strip().splitlines()[-1]);print('$v','$c',d['roofline']['kernel_ms'],d['value'],d['clocks']['sm_mhz'],d['e2e']['value'])"
  done
done
done
cp liboz_fma.so $L
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
