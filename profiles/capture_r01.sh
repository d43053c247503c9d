# Round-1 evidence capture on one B200 (run from the repo root under gpurun):
#   1. launch list of the default bench command (per-kernel time + DRAM bytes)
#   2. ncu --set full of the tensor-core product kernel (one launch)
set -e
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_bench.log 2>&1 || true
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_atb_kernel -s 2 -c 2 \
  -o gpurun_out/tc_atb_full -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1 || true
