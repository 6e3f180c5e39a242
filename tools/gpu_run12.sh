python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split or fixed" > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
python tools/split_time.py 8192 8192
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fixed11b.csv python bench.py --no-extras --no-variants --steps 2 --warmup 1 --pair-cutoff 11 --slice-exponents fixed > /dev/null 2>&1
python bench.py --no-extras --no-variants --steps 10 --warmup 3 --pair-cutoff 11 --slice-exponents fixed > gpurun_out/b_f11.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b_f11.json').read().strip().splitlines()[-1]);print('fixed11',d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['split_ms'],d['clocks']['sm_mhz'])"
