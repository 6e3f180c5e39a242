# Session 3: type3 = fp64 within the exact range; production-kernel accumulator ladder.
timeout 600 python -m pytest tests -m gpu -x -q -k "type3_fp64 or accumulator_is_exact or distributed" > gpurun_out/pytest_t6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t6.log
tail -5 gpurun_out/pytest_t6.log
