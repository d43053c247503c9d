#!/bin/bash
# Round-2 evidence run on one B200 (run from the repo root under gpurun):
#   1. the default bench line (config 4: headline, roofline pass, e2e, full-oracle cpu_baseline)
#   2. bench lines for configs 0-3 (parity configs; L2 flushed between timed isvds)
#   3. the random-gather microbenchmark (L2 / DRAM gather ceilings, profiles/l2_gather_bench2.cu)
#   4. ncu launch list of a short config-4 bench (each launch's device time, cold, serialised)
#   5. one ncu --set full capture of two SpMM launches (DRAM / L2 traffic per launch)
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2111_06312_b200 import _build; _build.build()"
python bench.py > $OUT/r02_bench_cfg4.json 2> $OUT/r02_bench_cfg4.err
for c in 0 1 2 3; do
  python bench.py --config $c --steps 20 --no-variants > $OUT/r02_bench_cfg$c.json 2> $OUT/r02_bench_cfg$c.err
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o $OUT/l2_gather_bench2 profiles/l2_gather_bench2.cu &&
  $OUT/l2_gather_bench2 > $OUT/r02_l2_gather_bench2.jsonl 2>&1
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$SHORT > $OUT/r02_short_plain.json 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_launches_cfg4.csv $SHORT \
    > $OUT/r02_ncu_launches.log 2>&1
$SHORT > $OUT/r02_short_plain2.json 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 8 -c 2 -o $OUT/r02_spmm_full $SHORT \
    > $OUT/r02_ncu_full.log 2>&1
echo done
