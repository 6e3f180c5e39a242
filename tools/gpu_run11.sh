python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/t_p.log 2>&1; tail -2 gpurun_out/t_p.log
python tools/sweep_config2.py gpurun_out/sweep_small2.json 1024 2048 4096 > gpurun_out/sweep_small2.txt 2>&1; grep -A3 "cuBLAS" gpurun_out/sweep_small2.txt
