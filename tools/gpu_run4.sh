python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
python bench.py --strong --n 65536 --steps 1 --warmup 1 --pair-cutoff 11 --slice-exponents fixed --no-extras > gpurun_out/b_strong64k_fixed11.json 2>gpurun_out/b_strong_err2.txt; tail -3 gpurun_out/b_strong_err2.txt
python -c "import json;d=json.loads(open('gpurun_out/b_strong64k_fixed11.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms'],d['roofline']['split_ms'])"
python bench.py --strong --n 65536 --steps 1 --warmup 1 --pair-cutoff 11 --no-extras > gpurun_out/b_strong64k_cut11.json 2>gpurun_out/b_strong_err3.txt; tail -3 gpurun_out/b_strong_err3.txt
python -c "import json;d=json.loads(open('gpurun_out/b_strong64k_cut11.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms'],d['roofline']['split_ms'])"
