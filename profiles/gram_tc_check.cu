// Stand-alone check of the tcgen05 Gram (gram_tc.cu) against an fp64 CPU Gram.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc \
//        profiles/gram_tc_check.cu -L paper_2111_06312_b200 -l:libisvd.so -Xlinker -rpath=... -o build/gram_tc_check
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "common.cuh"

namespace isvd {
thread_local int64_t g_launches_unused = 0;
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 70000;
  const int64_t l = argc > 2 ? atoll(argv[2]) : 256;
  const int64_t ld = (l + 3) / 4 * 4;
  std::vector<float> Y(rows * ld, 0.f);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < l; ++j) Y[i * ld + j] = nd(rng);
  float *dY, *ws;
  double* dG;
  cudaMalloc(&dY, sizeof(float) * rows * ld);
  cudaMemcpy(dY, Y.data(), sizeof(float) * rows * ld, cudaMemcpyHostToDevice);
  int64_t chunks = 0, cr = 0;
  int64_t wsf = isvd::gram_tc_ws_floats(rows, l, &chunks, &cr);
  cudaMalloc(&ws, sizeof(float) * wsf);
  cudaMalloc(&dG, sizeof(double) * l * l);
  int64_t lda = 0, ldw = 0;
  cudaError_t e = isvd::launch_gram_tc(dY, ld, rows, l, ws, &lda, &ldw, &chunks, nullptr, 0);
  printf("launch: %s (chunks %lld, ws %lld x %lld)\n", cudaGetErrorString(e), (long long)chunks, (long long)lda,
         (long long)ldw);
  e = isvd::launch_atb_f32_reduce(ws, lda, ldw, chunks, l, l, true, dG, l, nullptr, 0, 148, nullptr, 0);
  e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<double> G(l * l);
  cudaMemcpy(G.data(), dG, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  {
    std::vector<float> w0(lda * ldw);
    cudaMemcpy(w0.data(), ws, sizeof(float) * lda * ldw, cudaMemcpyDeviceToHost);
    const int64_t r1 = cr < rows ? cr : rows;
    int pairs[6][2] = {{0, 0}, {1, 1}, {0, 1}, {1, 0}, {5, 9}, {130, 200}};
    for (auto& pq : pairs) {
      int a = pq[0], b = pq[1];
      if (a >= l || b >= l) continue;
      double s = 0.0;
      for (int64_t i = 0; i < r1; ++i) s += (double)Y[i * ld + a] * (double)Y[i * ld + b];
      printf("chunk0 (%d,%d): tc %.6e  cpu %.6e   G %.6e\n", a, b, w0[a * ldw + b], s, G[a * l + b]);
    }
  }
  double maxrel = 0.0;
  for (int64_t a = 0; a < l; a += 7)
    for (int64_t b = a; b < l; b += 5) {
      double s = 0.0;
      for (int64_t i = 0; i < rows; ++i) s += (double)Y[i * ld + a] * (double)Y[i * ld + b];
      double den = std::sqrt(G[a * l + a] * G[b * l + b]);
      maxrel = std::fmax(maxrel, std::fabs(G[a * l + b] - s) / den);
    }
  printf("max |G_tc - G_fp64| / sqrt(G_aa G_bb) = %.3e\n", maxrel);
  return maxrel < 3e-5 ? 0 : 2;
}
