python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
python tools/sweep_config2.py gpurun_out/sweep_small.json 1024 2048 > gpurun_out/sweep_small.txt 2>&1; cat gpurun_out/sweep_small.txt
