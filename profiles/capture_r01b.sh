# Round-1 evidence (later pass): bench line, launch list, ncu --set full of spmm_kernel and the
# tensor-core kernels (one launch each).  Run from the repo root under gpurun.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-variants > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel|tc_atb_kernel|atb_dmma_kernel" \
  -c 3 -o gpurun_out/full_r01b -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants > gpurun_out/ncu_full.log 2>&1
