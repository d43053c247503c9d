mkdir -p gpurun_out
for c in 0 200 100 136 52; do
  ISVD_SPMM_COLS=$c timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err
done
