set -e
mkdir -p build gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include profiles/gemm_clock_probe.cu -L paper_2111_06312_b200 -l:libisvd.so -Xlinker -rpath=$PWD/paper_2111_06312_b200 -o build/gemm_clock_probe
for v in 0 1; do
  echo "ISVD_GEMM_KRES=$v"
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/smi_$v.txt &
  SMI=$!
  ISVD_GEMM_KRES=$v build/gemm_clock_probe 800
  kill $SMI
  sort gpurun_out/smi_$v.txt | uniq -c | sort -rn | head -6
done > gpurun_out/r02h_gemm_clock_probe.txt 2>&1
cat gpurun_out/r02h_gemm_clock_probe.txt
