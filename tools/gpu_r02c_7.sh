timeout 600 python -m pytest tests -m gpu -x -q -k "structured or fixed_point_rows" > gpurun_out/pytest_t7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t7.log
tail -4 gpurun_out/pytest_t7.log
