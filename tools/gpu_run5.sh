for extra in "--pair-cutoff 11" "" ; do
python bench.py --strong --n 65536 --steps 1 --warmup 1 $extra --no-extras > gpurun_out/b_s64k.json 2>gpurun_out/b_s64k_err.txt; tail -2 gpurun_out/b_s64k_err.txt
python -c "import json;d=json.loads(open('gpurun_out/b_s64k.json').read().strip().splitlines()[-1]);print('$extra',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms'],d['roofline']['split_ms'],d['clocks'])"
done
