set -e
mkdir -p build gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include profiles/dense_check.cu -L paper_2111_06312_b200 -l:libisvd.so -Xlinker -rpath=$PWD/paper_2111_06312_b200 -o build/dense_check
for v in "ISVD_GEMM_KRES=0 ISVD_GEMM_KCHUNK=0 ISVD_ATB_TN16=0" "ISVD_GEMM_KRES=1"; do echo "$v"; env $v timeout 300 build/dense_check; done > gpurun_out/r02h_dense_check.txt 2>&1
cat gpurun_out/r02h_dense_check.txt
