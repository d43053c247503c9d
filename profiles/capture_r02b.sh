#!/bin/bash
# Round 2, call 3: new parity tests (row subset, distributed split path), the GEMM register-tile
# experiment (dense_check at config-4 shapes), the L2 window sweep and graph-replay timing.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2111_06312_b200 import _build; _build.build()"
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "multirank or subset" > $OUT/r02b_tests.log 2>&1
tail -3 $OUT/r02b_tests.log
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include \
  profiles/dense_check.cu -L paper_2111_06312_b200 -l:libisvd.so -Xlinker -rpath=$PWD/paper_2111_06312_b200 \
  -o $OUT/dense_check && for v in 0 1 3; do echo "ISVD_GEMM_TM16=$v"; ISVD_GEMM_TM16=$v $OUT/dense_check; done \
  > $OUT/r02b_dense_check.txt 2>&1
python profiles/spmm_window_sweep.py > $OUT/r02b_window_sweep.jsonl 2> $OUT/r02b_window_sweep.err
echo done
