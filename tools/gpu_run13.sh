python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
for r in 1 2; do
python bench.py --no-extras --no-variants --steps 10 --warmup 3 --pair-cutoff 11 --slice-exponents fixed > gpurun_out/b_f11.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b_f11.json').read().strip().splitlines()[-1]);print('fixed11',d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['split_ms'],d['clocks']['sm_mhz'])"
done
python bench.py --no-extras --no-variants --steps 5 --warmup 3 > gpurun_out/b_def.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b_def.json').read().strip().splitlines()[-1]);print('defaults',d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['split_ms'],d['clocks']['sm_mhz'])"
