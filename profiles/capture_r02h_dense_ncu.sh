set -e
mkdir -p build gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include profiles/dense_check.cu -L paper_2111_06312_b200 -l:libisvd.so -Xlinker -rpath=$PWD/paper_2111_06312_b200 -o build/dense_check
ncu --set full --clock-control none --import-source on -k regex:gemm_kchunk -c 1 -o gpurun_out/r02h_kch -f build/dense_check > gpurun_out/r02h_kch_ncu.log 2>&1 || tail -5 gpurun_out/r02h_kch_ncu.log
ncu -i gpurun_out/r02h_kch.ncu-rep --page raw --csv > gpurun_out/r02h_kch_raw.csv
ncu -i gpurun_out/r02h_kch.ncu-rep --page source --csv > gpurun_out/r02h_kch_source.csv 2>/dev/null || true
ls -la gpurun_out | tail -5
