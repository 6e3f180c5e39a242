L=paper_2508_00441_b200/liboz_b200.so
for r in 1 2; do for v in r0 r1; do cp liboz_$v.so $L
ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:pair_gemm -c 2 --csv python tools/run_once.py --pair-cutoff 11 --fixed --reps 2 2>/dev/null | grep pair_gemm | awk -F'","' -v v=$v '{print v, "fixed11", $(NF-2), $NF}'
ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:pair_gemm -c 1 --csv python tools/run_once.py --reps 1 2>/dev/null | grep pair_gemm | awk -F'","' -v v=$v '{print v, "defaults", $(NF-2), $NF}'
done; done
cp liboz_r0.so $L
