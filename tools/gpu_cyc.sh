for e in "" "--emu"; do
ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:pair_gemm -c 3 --csv python tools/run_once.py --pair-cutoff 11 --fixed $e --reps 3 2>/dev/null | grep pair_gemm | awk -F'","' -v e="$e" '{print "fixed11" e, $5, $(NF-2), $NF}'
done
