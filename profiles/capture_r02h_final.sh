#!/bin/bash
# Round 2, last session (r02h): whole -m gpu suite, smoke, bench lines for configs 0-4 and the
# reference arm, the config-4 launch list, ncu full of the config-4 SpMM and of the K-resident GEMM.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider > $OUT/r02h_gputest.log 2>&1
tail -3 $OUT/r02h_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02h_smoke.txt 2>&1; tail -1 $OUT/r02h_smoke.txt
timeout 1200 python bench.py > $OUT/r02h_bench_cfg4.json 2> $OUT/r02h_bench_cfg4.err
for c in 0 1 2 3; do
  timeout 900 python bench.py --config $c --steps 20 > $OUT/r02h_bench_cfg$c.json 2> $OUT/r02h_bench_cfg$c.err
done
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$SHORT > $OUT/r02h_short_plain.json 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02h_launches_cfg4.csv $SHORT \
    > $OUT/r02h_ncu_launches.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"spmm_kernel|gemm_kres_kernel" -s 40 -c 4 \
    -o $OUT/r02h_full -f $SHORT > $OUT/r02h_ncu_full.log 2>&1
ncu -i $OUT/r02h_full.ncu-rep --page raw --csv > $OUT/r02h_spmm_kres_full_raw.csv 2>/dev/null
python profiles/summarize_launches.py $OUT/r02h_launches_cfg4.csv > $OUT/r02h_launches_cfg4.txt 2>&1
head -20 $OUT/r02h_launches_cfg4.txt
echo done
