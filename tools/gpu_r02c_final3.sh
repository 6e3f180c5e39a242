# Session 3 final at HEAD: full GPU suite, smoke, bench line (both arms).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final3.log
tail -3 gpurun_out/pytest_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo "bench rc=$?"
head -c 300 gpurun_out/bench_final3.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref3.json 2> gpurun_out/bench_ref3.err; echo "ref rc=$?"
