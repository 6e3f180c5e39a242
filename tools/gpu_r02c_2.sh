# Session 3: fixed-point residuals in the adaptive emulated split + occupancy knob.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "split or structured or occupancy or emu or fixed_step" > gpurun_out/pytest_t2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t2.log
tail -3 gpurun_out/pytest_t2.log
timeout 300 python tools/split_time_emu.py 8192 8192 > gpurun_out/split_time_emu.txt 2>&1
cat gpurun_out/split_time_emu.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:split --csv --log-file gpurun_out/split_emu_launches.csv python tools/split_time_emu.py 8192 8192 > /dev/null 2>&1
