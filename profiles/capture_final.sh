# Final round-1 evidence: smoke, bench line (default N=1), launch list, ncu --set full of one
# spmm_kernel and one tc_atb_kernel launch.  Run from the repo root under gpurun.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-variants > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel" -c 1 \
  -o gpurun_out/spmm_final -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_atb_kernel" -c 1 \
  -o gpurun_out/tcatb_final -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants > gpurun_out/ncu_full2.log 2>&1
