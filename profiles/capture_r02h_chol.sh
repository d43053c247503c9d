set -e
mkdir -p build gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include profiles/chol_check.cu -L paper_2111_06312_b200 -l:libisvd.so -Xlinker -rpath=$PWD/paper_2111_06312_b200 -o build/chol_check
timeout 300 build/chol_check > gpurun_out/r02h_chol_check.txt 2>&1
cat gpurun_out/r02h_chol_check.txt
