#!/bin/bash
# Round-2 profiles: K3 --set full (reference defaults and the fixed-step mode at
# pair_cutoff 11), the split kernel, and the bench launch list.  Run on the GPU box:
#   bash tools/profile_r02.sh [tag]
set -x
T=${1:-r02}
O=gpurun_out
NCU="ncu --clock-control none --import-source on"
$NCU --set full -k regex:pair_gemm_kernel -c 1 -o $O/k3_defaults_$T -f python tools/run_once.py > $O/k3_defaults_$T.log 2>&1
$NCU --set full -k regex:pair_gemm_kernel -c 1 -o $O/k3_fixed11_$T -f python tools/run_once.py --fixed --pair-cutoff 11 > $O/k3_fixed11_$T.log 2>&1
$NCU --set full -k regex:split_fused_kernel -c 2 -o $O/split_$T -f python tools/run_once.py > $O/split_$T.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-extras > $O/launches_bench_$T.log 2>&1
ls -la $O
# Summaries (the .ncu-rep files are ~35 MB each; gpurun brings back <= 64 MiB)
for r in k3_defaults_$T k3_fixed11_$T split_$T; do
  ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_source.csv 2>/dev/null
  gzip -f $O/${r}_raw.csv $O/${r}_source.csv
done
rm -f $O/k3_defaults_$T.ncu-rep $O/split_$T.ncu-rep
mv $O/k3_fixed11_$T.ncu-rep /tmp/ 2>/dev/null
ls -la $O
