set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2111_06312_b200 import _build; _build.build()" > $OUT/v_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider > $OUT/v_gputest.log 2>&1
tail -3 $OUT/v_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/v_smoke.log 2>&1; tail -1 $OUT/v_smoke.log
timeout 900 python bench.py > $OUT/v_bench_cfg4.json 2> $OUT/v_bench_cfg4.err; tail -c 600 $OUT/v_bench_cfg4.json
