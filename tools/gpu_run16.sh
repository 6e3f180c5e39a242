python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_acceptance.py -m gpu -x -q -k "fixed or emu or split" > gpurun_out/t_e.log 2>&1; tail -2 gpurun_out/t_e.log
for r in 1 2; do
python bench.py --no-extras --no-variants --steps 5 --warmup 3 --emu --pair-cutoff 11 --slice-exponents fixed > gpurun_out/b_e.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b_e.json').read().strip().splitlines()[-1]);print('emu fixed11',d['value'],d['roofline']['kernel_ms'],d['roofline']['split_ms'])"
done
