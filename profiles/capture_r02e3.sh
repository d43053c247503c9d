#!/bin/bash
# Round 2 (session e) evidence, part 3: per-config SpMM L2 / DRAM traffic (ncu, the eager profiled pass
# of a one-step bench) for the BASELINE.md results table, and the config-4 SpMM with a WARM L2
# (--cache-control none: the hub window as the timed runs see it).
set -u
OUT=gpurun_out
mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct"
for c in 0 1 2 3; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
  $CMD > $OUT/re3_plain_c$c.json 2>&1 &&
    ncu --metrics $M --clock-control none -k regex:spmm_kernel -c 60 --csv --log-file $OUT/re3_spmm_c$c.csv $CMD \
      > $OUT/re3_ncu_c$c.log 2>&1
done
CMD="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$CMD > $OUT/re3_plain_c4.json 2>&1 &&
  ncu --metrics $M --clock-control none --cache-control none -k regex:spmm_kernel -s 20 -c 4 --csv \
    --log-file $OUT/re3_spmm_c4_warm.csv $CMD > $OUT/re3_ncu_c4.log 2>&1
echo done
