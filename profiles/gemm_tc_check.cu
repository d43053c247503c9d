// Stand-alone check + timing of the tcgen05 3xTF32 tall GEMM (gemm_tc.cu) against fp64 on the host:
//   C[map(i), :] = s_i A[i, :] B   for (K, N) = (l, l) [Y R^-1] and (d, l) [X G_j, row-scaled, row map]
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include \
//        profiles/gemm_tc_check.cu -L paper_2111_06312_b200 -l:libisvd.so \
//        -Xlinker -rpath='$ORIGIN/../paper_2111_06312_b200' -o build/gemm_tc_check
//   build/gemm_tc_check [rows] [l] [d]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "common.cuh"

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 1000000;
  const int64_t l = argc > 2 ? atoll(argv[2]) : 400;
  const int64_t d = argc > 3 ? atoll(argv[3]) : 100;
  const int sms = 148;
  int rc = 0;
  std::mt19937 rng(3);
  std::normal_distribution<float> nd;
  for (int which = 0; which < 2; ++which) {
    const int64_t K = which == 0 ? l : d, N = l, lda = (K + 3) / 4 * 4, ldc = (N + 3) / 4 * 4;
    std::vector<float> A(rows * lda, 0.f), B(K * N), s(rows), C(rows * ldc, 0.f);
    std::vector<int32_t> map(rows);
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t k = 0; k < K; ++k) A[i * lda + k] = nd(rng);
    for (auto& v : B) v = nd(rng) / std::sqrt((float)K);
    for (auto& v : s) v = 0.1f + std::fabs(nd(rng));
    std::iota(map.begin(), map.end(), 0);
    std::shuffle(map.begin(), map.end(), rng);
    float *dA, *dB, *dC, *ds, *ws;
    int32_t* dmap;
    cudaMalloc(&dA, 4 * rows * lda);
    cudaMalloc(&dB, 4 * K * N);
    cudaMalloc(&dC, 4 * rows * ldc);
    cudaMalloc(&ds, 4 * rows);
    cudaMalloc(&dmap, 4 * rows);
    cudaMalloc(&ws, 4 * isvd::tc_gemm_ws_floats(N, K));
    cudaMemcpy(dA, A.data(), 4 * rows * lda, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), 4 * K * N, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, s.data(), 4 * rows, cudaMemcpyHostToDevice);
    cudaMemcpy(dmap, map.data(), 4 * rows, cudaMemcpyHostToDevice);
    const bool scaled = which == 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 6; ++it) {
      if (it == 1) cudaEventRecord(e0);
      cudaError_t e = isvd::launch_tc_gemm(dA, lda, dB, N, dC, ldc, rows, N, K, scaled ? ds : nullptr, 1.f, nullptr, 0,
                                           scaled ? dmap : nullptr, ws, sms);
      if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%s: %s  %.3f ms/launch  (%.1f GB/s of A read + C write, %.1f TFLOP/s 3xTF32)\n",
           which == 0 ? "Y Rinv (K=l)" : "X G (K=d, scaled, mapped)", cudaGetErrorString(e), ms,
           (double)rows * (K + N) * 4 / (ms * 1e-3) / 1e9, 3.0 * 2.0 * rows * K * N / (ms * 1e-3) / 1e12);
    if (e != cudaSuccess) return 1;
    cudaMemcpy(C.data(), dC, 4 * rows * ldc, cudaMemcpyDeviceToHost);
    double num = 0, den = 0, maxrel = 0;
    for (int t = 0; t < 2000; ++t) {
      const int64_t i = (int64_t)(rng() % rows);
      const int64_t oi = scaled ? map[i] : i;
      double rn = 0;
      for (int64_t k = 0; k < K; ++k) rn += (double)A[i * lda + k] * A[i * lda + k];
      for (int64_t j = 0; j < N; ++j) {
        double ref = 0, cn = 0;
        for (int64_t k = 0; k < K; ++k) {
          ref += (double)A[i * lda + k] * B[k * N + j];
          cn += (double)B[k * N + j] * B[k * N + j];
        }
        if (scaled) ref *= (double)s[i];
        const double got = C[oi * ldc + j];
        num += (got - ref) * (got - ref);
        den += ref * ref;
        maxrel = std::fmax(maxrel, std::fabs(got - ref) / (std::sqrt(rn * cn) * (scaled ? s[i] : 1.0)));
      }
    }
    const double fro = std::sqrt(num / den);
    printf("   sampled rel-fro %.3e   max |C - C64| / (|a_i| |b_j|) %.3e\n", fro, maxrel);
    if (fro > 3e-6) rc = 2;
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(ds); cudaFree(dmap); cudaFree(ws);
  }
  return rc;
}
