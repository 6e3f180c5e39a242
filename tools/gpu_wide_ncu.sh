for tn in 192 256; do
ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:pair_gemm -c 3 --csv python tools/run_once.py --pair-cutoff 11 --fixed --variant 2 $tn --reps 3 2>/dev/null | grep pair_gemm | awk -F'","' -v tn=$tn '{print "N=" tn, $(NF-2), $(NF-1), $NF}'
done
