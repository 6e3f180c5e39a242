# Session 3: emulated split on 512 x 16 — full GPU suite, split timings, config-3 bench line.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_t3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t3.log
tail -3 gpurun_out/pytest_t3.log
python tools/split_time_emu.py 8192 8192 > gpurun_out/split_time_t3.txt 2>&1; cat gpurun_out/split_time_t3.txt
timeout 900 python bench.py --emu --no-variants > gpurun_out/bench_emu_t3.json 2> gpurun_out/bench_emu_t3.err; echo "bench emu rc=$?"
head -c 300 gpurun_out/bench_emu_t3.json; echo
