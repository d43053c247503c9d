# ncu --set full of one launch each of the tensor-core Gram (tcgen05) and the exact fp64 Gram (DMMA)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_atb_kernel -c 1 \
  -o gpurun_out/tc_atb_r01 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants \
  > gpurun_out/ncu_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:atb_dmma_kernel -c 1 \
  -o gpurun_out/dmma_r01 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants \
  > gpurun_out/ncu_dmma.log 2>&1
