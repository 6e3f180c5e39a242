set -x
python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
for r in 1 2; do
python bench.py --no-extras --no-variants --steps 10 --warmup 3 --pair-cutoff 11 --slice-exponents fixed > gpurun_out/b_fixed11_$r.json 2>gpurun_out/b_err.txt
python -c "import json;d=json.loads(open('gpurun_out/b_fixed11_$r.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['split_ms'],d['clocks'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_fixed11.csv python bench.py --no-extras --no-variants --steps 2 --warmup 1 --pair-cutoff 11 --slice-exponents fixed > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"col_slice|split_fused" -c 2 -o gpurun_out/split_fixed_r02 python tools/run_once.py --pair-cutoff 11 --fixed > /dev/null 2>&1
cp paper_2508_00441_b200/liboz_b200.so /tmp/prod.so
cp liboz_diag.so paper_2508_00441_b200/liboz_b200.so
python tools/k3_trace_dump.py 11 1 gpurun_out/trace_fixed11.npy
python tools/k3_trace_dump.py -1 0 gpurun_out/trace_defaults.npy
cp /tmp/prod.so paper_2508_00441_b200/liboz_b200.so
