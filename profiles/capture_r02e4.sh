#!/bin/bash
# Round 2 (session e) bench lines: the default (config 4) line and configs 0-3, plus the sticky probe test.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "probe" -p no:cacheprovider > $OUT/re4_probe_test.log 2>&1
tail -1 $OUT/re4_probe_test.log
python bench.py > $OUT/re4_bench_cfg4.json 2> $OUT/re4_bench_cfg4.err
for c in 0 1 2 3; do
  python bench.py --config $c --steps 20 > $OUT/re4_bench_cfg$c.json 2> $OUT/re4_bench_cfg$c.err
done
echo done
