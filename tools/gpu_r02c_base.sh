# Round-2 (session 3) baseline at HEAD: GPU tests, then one bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log
