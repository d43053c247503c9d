#!/bin/bash
# Round 2 final evidence on one B200 (from the repo root under gpurun):
#   1. the whole -m gpu suite
#   2. the default bench line (config 4) and lines for configs 0-3
#   3. the ncu launch list of a short config-4 bench, and one ncu --set full capture of two SpMM
#      launches in the graph-replayed solver (DRAM / L2 traffic per launch)
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2111_06312_b200 import _build; _build.build()"
python -m pytest tests -m gpu -q -rA --durations=25 -p no:cacheprovider > $OUT/rf_gputest.log 2>&1
tail -2 $OUT/rf_gputest.log
python bench.py > $OUT/rf_bench_cfg4.json 2> $OUT/rf_bench_cfg4.err
for c in 0 1 2 3; do
  python bench.py --config $c --steps 20 --no-variants > $OUT/rf_bench_cfg$c.json 2> $OUT/rf_bench_cfg$c.err
done
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$SHORT > $OUT/rf_short_plain.json 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/rf_launches_cfg4.csv $SHORT \
    > $OUT/rf_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 8 -c 2 -o $OUT/rf_spmm_full $SHORT \
    > $OUT/rf_ncu_full.log 2>&1
echo done
