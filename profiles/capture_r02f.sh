#!/bin/bash
# Round 2 final evidence (session e, end): whole -m gpu suite, bench lines for configs 0-4, the
# config-4 launch list, ncu full of the config-4 SpMM (eager profiled pass) and of X^T Z_j.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -m gpu -q -rA --durations=30 -p no:cacheprovider > $OUT/rf2_gputest.log 2>&1
tail -2 $OUT/rf2_gputest.log
python bench.py > $OUT/rf2_bench_cfg4.json 2> $OUT/rf2_bench_cfg4.err
for c in 0 1 2 3; do
  python bench.py --config $c --steps 20 > $OUT/rf2_bench_cfg$c.json 2> $OUT/rf2_bench_cfg$c.err
done
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$SHORT > $OUT/rf2_short_plain.json 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/rf2_launches_cfg4.csv $SHORT \
    > $OUT/rf2_ncu_launches.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel|atb_f32_kernel" -s 40 -c 4 \
    -o $OUT/rf2_full $SHORT > $OUT/rf2_ncu_full.log 2>&1
python profiles/summarize_launches.py $OUT/rf2_launches_cfg4.csv > $OUT/rf2_launches_cfg4.txt 2>&1
echo done
