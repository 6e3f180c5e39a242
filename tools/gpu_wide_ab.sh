L=paper_2508_00441_b200/liboz_b200.so
for v in g1 g2; do cp liboz_$v.so $L
for tn in 192 256; do
ncu --metrics sm__cycles_elapsed.max,lts__t_bytes.sum --clock-control none -k regex:pair_gemm -c 3 --csv python tools/run_once.py --pair-cutoff 11 --fixed --variant 2 $tn --reps 3 2>/dev/null | grep pair_gemm | grep cycles | awk -F'","' -v tn=$tn -v v=$v '{print v, "N=" tn, $(NF-2), $NF}'
done; done
cp liboz_g2.so $L; python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "wide or fixed_step_grouped" 2>&1 | tail -2
cp liboz_g1.so $L
