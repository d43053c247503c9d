#!/bin/bash
# Round 2 (session e) evidence: launch list of a short config-4 bench (graph replay, per-kernel device
# times) and one ncu --set full capture of the MN-major tcgen05 Gram and of one SpMM launch.
set -u
OUT=gpurun_out
mkdir -p $OUT
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$SHORT > $OUT/re_short_plain.json 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/re_launches_cfg4.csv $SHORT \
    > $OUT/re_ncu_launches.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"tc_atb_mn_kernel|spmm_kernel" -s 6 -c 3 \
    -o $OUT/re_full $SHORT > $OUT/re_ncu_full.log 2>&1
python profiles/summarize_launches.py $OUT/re_launches_cfg4.csv > $OUT/re_launches_cfg4.txt 2>&1
echo done
