# ncu --set full of the two SIMT contractions on the default path (one launch each)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -c 1 \
  -o gpurun_out/gemm_tn_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants \
  > gpurun_out/ncu_gemm_tn.log 2>&1 || true
timeout 600 ncu --set full --clock-control none --import-source on -k regex:atb_f32_kernel -c 1 \
  -o gpurun_out/atb_f32_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-variants \
  > gpurun_out/ncu_atb.log 2>&1 || true
