# A/B: adaptive HW/emu row split at 512 x 16 (gpurun_alt/ build) vs HEAD's 256 x 32.
python tools/split_time_emu.py 8192 8192 > gpurun_out/split_time_head.txt 2>&1
python -c "import sys; sys.argv=['tools/split_time_emu.py','8192','8192']; sys.path.insert(0,'.'); import paper_2508_00441_b200._lib as L; L._lib=L.load('gpurun_alt/liboz_b200.so'); g={'__file__':'tools/split_time_emu.py','__name__':'__main__'}; exec(open('tools/split_time_emu.py').read(), g)" > gpurun_out/split_time_alt512.txt 2>&1
python tools/split_time_emu.py 8192 8192 >> gpurun_out/split_time_head.txt 2>&1
cat gpurun_out/split_time_head.txt gpurun_out/split_time_alt512.txt
