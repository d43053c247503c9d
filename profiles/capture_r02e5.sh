#!/bin/bash
# Config-4 SpMM DRAM traffic vs the L2 persisting window size, warm L2 (--cache-control none).
set -u
OUT=gpurun_out
mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum"
CMD="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$CMD > $OUT/re5_plain.json 2>&1
for mb in 0 20 40 60 79; do
  ISVD_L2_PERSIST_MB=$mb ncu --metrics $M --clock-control none --cache-control none -k regex:spmm_kernel -s 20 -c 3 --csv \
    --log-file $OUT/re5_window_$mb.csv $CMD > $OUT/re5_ncu_$mb.log 2>&1
done
echo done
