python -m pytest tests -m gpu -x -q -k "emu or fp64emu or Emu" > gpurun_out/t_emu.log 2>&1; tail -3 gpurun_out/t_emu.log
for r in 1 2; do
python bench.py --no-extras --no-variants --steps 3 --warmup 2 --emu > gpurun_out/b_emu.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b_emu.json').read().strip().splitlines()[-1]);print('emu',d['value'],d['roofline']['kernel_ms'],d['clocks']['sm_mhz'])"
python bench.py --no-extras --no-variants --steps 3 --warmup 2 --emu --pair-cutoff 11 --slice-exponents fixed > gpurun_out/b_emu.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b_emu.json').read().strip().splitlines()[-1]);print('emu fixed11',d['value'],d['roofline']['kernel_ms'],d['clocks']['sm_mhz'])"
done
