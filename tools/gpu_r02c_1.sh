# Session 3: batched adaptive split + pair_trim — targeted parity, split timing, launch list, bench.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "split or trim or structured or fixed_step_sampled or oz_gemm_bitwise" > gpurun_out/pytest_t1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t1.log
tail -3 gpurun_out/pytest_t1.log
timeout 300 python tools/split_time.py 8192 8192 > gpurun_out/split_time.txt 2>&1
cat gpurun_out/split_time.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:split --csv --log-file gpurun_out/split_launches.csv python tools/split_time.py 8192 8192 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_t1.json 2> gpurun_out/bench_t1.err; echo "bench rc=$?"
