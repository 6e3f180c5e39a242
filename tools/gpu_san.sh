export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/san
python tools/sanitize_case.py > gpurun_out/san/plain.txt 2>&1; cat gpurun_out/san/plain.txt
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name regex="pair_gemm|split_fused|col_slice|pad_planes" --print-limit 20 python tools/sanitize_case.py > gpurun_out/san/$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/san/$tool.txt
done
