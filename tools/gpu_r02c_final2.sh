# Session 3 final (re-run, small outputs): bench (both arms), launch list, ncu of the emulated split
# exported to CSV on the box, and the 512 x 16 adaptive-split A/B (alternative build in gpurun_alt/).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
head -c 400 gpurun_out/bench_final.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-extras --no-variants > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:split_fused_kernel -s 4 -c 1 -o /tmp/split_emu_full python tools/split_time_emu.py 8192 8192 > /tmp/ncu_split.log 2>&1; echo "ncu split rc=$?"
ncu -i /tmp/split_emu_full.ncu-rep --page raw --csv > gpurun_out/split_emu_full_raw.csv 2>/dev/null; ncu -i /tmp/split_emu_full.ncu-rep --page details --csv > gpurun_out/split_emu_full_details.csv 2>/dev/null
python tools/split_time_emu.py 8192 8192 > gpurun_out/split_time_head.txt 2>&1
python -c "import sys; sys.argv=['x','8192','8192']; sys.path.insert(0,'.'); import paper_2508_00441_b200._lib as L; L._lib=L.load('gpurun_alt/liboz_b200.so'); exec(open('tools/split_time_emu.py').read())" > gpurun_out/split_time_alt512.txt 2>&1
cat gpurun_out/split_time_head.txt gpurun_out/split_time_alt512.txt
du -sh gpurun_out
