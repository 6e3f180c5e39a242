# Session 3: device integer mul/lt for the CLI fp64emu suite; full GPU suite at HEAD.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_t5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t5.log
tail -3 gpurun_out/pytest_t5.log
python -m paper_2508_00441_b200.cli verify --trials 100000 > gpurun_out/cli_verify.json 2>&1; cat gpurun_out/cli_verify.json | head -c 600
