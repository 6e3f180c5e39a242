# Final round-2 captures at HEAD: K3 --set full (reference defaults; fixed-step cutoff 11 on 256x256 tiles),
# the launch list of the headline bench command, and the full bench line.
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02_final.csv python bench.py --steps 2 --warmup 1 --no-extras --no-variants > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_gemm -c 1 -o gpurun_out/k3_defaults_final python tools/run_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_gemm -c 1 -o gpurun_out/k3_fixed11_final python tools/run_once.py --pair-cutoff 11 --fixed > /dev/null 2>&1
for r in k3_defaults_final k3_fixed11_final; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; rm -f gpurun_out/$r.ncu-rep; done
