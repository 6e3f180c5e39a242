ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_64k_cut11.csv python bench.py --strong --n 65536 --steps 1 --warmup 0 --pair-cutoff 11 --no-extras > /dev/null 2>gpurun_out/ncu64k_err.txt
tail -3 gpurun_out/ncu64k_err.txt
