ncu --set full --clock-control none --import-source on -k regex:pair_gemm -c 1 -o gpurun_out/k3_emu_cut11 python tools/run_once.py --emu --pair-cutoff 11 > gpurun_out/ncu_emu.log 2>&1
tail -3 gpurun_out/ncu_emu.log
