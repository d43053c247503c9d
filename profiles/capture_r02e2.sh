#!/bin/bash
# Round 2 (session e) evidence, part 2: the whole -m gpu suite; ncu --set full of the MN-major
# tcgen05 Gram (graph replay) and of two SpMM launches of the bench's eager profiled pass (the pass
# its roofline.avg_launch_ms is measured on).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -m gpu -q -rA --durations=30 -p no:cacheprovider > $OUT/re_gputest.log 2>&1
tail -2 $OUT/re_gputest.log
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants --e2e-steps 0"
$SHORT > $OUT/re_short_plain2.json 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:tc_atb_mn_kernel -s 2 -c 2 \
    -o $OUT/re_gram_full $SHORT > $OUT/re_ncu_gram.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 40 -c 2 \
    -o $OUT/re_spmm_eager_full $SHORT > $OUT/re_ncu_spmm.log 2>&1
echo done
