python bench.py > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err; tail -2 gpurun_out/bench_head.err
python bench.py --strong --n 65536 --steps 1 --warmup 1 --pair-cutoff 11 --slice-exponents fixed --no-extras > gpurun_out/b_s64k_fixed11.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02_head.csv python bench.py --steps 2 --warmup 1 --no-extras --no-variants > /dev/null 2>&1
