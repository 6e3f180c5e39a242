# A/B: 16 vs 8 epilogue warps in the emulated CTA-pair N = 128 pair GEMM (alternative build in gpurun_alt2/).
for lib in head gpurun_alt2/liboz_b200.so head gpurun_alt2/liboz_b200.so; do timeout 300 python tools/emu_epi_ab.py $lib; done > gpurun_out/emu_epi_ab.txt 2>&1
cat gpurun_out/emu_epi_ab.txt
