// Timing of the blocked cluster Cholesky + inverse (smallmat.cu) at l = 256 / 400 for 8- and
// 16-CTA clusters (ISVD_CHOL_CLUSTER), with the residual |R^T R - G| / |G| of each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include \
//        profiles/chol_check.cu -L paper_2111_06312_b200 -l:libisvd.so \
//        -Xlinker -rpath='$ORIGIN/../paper_2111_06312_b200' -o build/chol_check
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "common.cuh"

int main() {
  for (int l : {100, 250, 256, 400}) {
    const int ld = (l + 3) / 4 * 4;
    std::mt19937 rng(l);
    std::normal_distribution<double> nd;
    // SPD Gram of a random tall matrix
    const int rows = 3 * l;
    std::vector<double> Y((size_t)rows * l), G((size_t)l * l, 0.0);
    for (auto& v : Y) v = nd(rng);
    for (int i = 0; i < l; ++i)
      for (int j = i; j < l; ++j) {
        double s = 0;
        for (int r = 0; r < rows; ++r) s += Y[(size_t)r * l + i] * Y[(size_t)r * l + j];
        G[(size_t)i * l + j] = G[(size_t)j * l + i] = s;
      }
    double *dG, *R64, *ws;
    float* Rinv;
    isvd::DevStatus* st;
    cudaMalloc(&dG, 8 * l * l);
    cudaMalloc(&R64, 8 * l * l);
    cudaMalloc(&ws, 8 * l * l);
    cudaMalloc(&Rinv, 4 * ld * ld);
    cudaMalloc(&st, sizeof(isvd::DevStatus));
    cudaMemset(st, 0, sizeof(isvd::DevStatus));
    cudaMemcpy(dG, G.data(), 8 * l * l, cudaMemcpyHostToDevice);
    for (int cs : {8, 16}) {
      char buf[8];
      snprintf(buf, sizeof(buf), "%d", cs);
      setenv("ISVD_CHOL_CLUSTER", buf, 1);
      isvd::launch_chol_inv(dG, l, l, ld, Rinv, R64, ws, st, false, nullptr, 0);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) isvd::launch_chol_inv(dG, l, l, ld, Rinv, R64, ws, st, false, nullptr, 0);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<double> R((size_t)l * l);
      cudaMemcpy(R.data(), R64, 8 * l * l, cudaMemcpyDeviceToHost);
      double num = 0, den = 0;
      for (int i = 0; i < l; i += 7)
        for (int j = i; j < l; j += 5) {
          double s = 0;
          for (int k = 0; k <= i; ++k) s += R[(size_t)k * l + i] * R[(size_t)k * l + j];
          num += (s - G[(size_t)i * l + j]) * (s - G[(size_t)i * l + j]);
          den += G[(size_t)i * l + j] * G[(size_t)i * l + j];
        }
      // the fp32 inverse: |R Rinv - I|_max over sampled rows (fp32 storage of Rinv: ~1e-7 kappa(R))
      std::vector<float> Ri((size_t)ld * ld);
      cudaMemcpy(Ri.data(), Rinv, 4 * (size_t)ld * ld, cudaMemcpyDeviceToHost);
      double worst = 0;
      for (int i = 0; i < l; i += 3)
        for (int j = 0; j < l; ++j) {
          double s = 0;
          for (int k = i; k < l; ++k) s += R[(size_t)i * l + k] * (double)Ri[(size_t)k * ld + j];
          worst = std::max(worst, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
      printf("l=%d cluster %2d: %s %.3f ms  |R^T R - G| / |G| = %.2e  max|R Rinv - I| = %.2e\n", l, cs,
             cudaGetErrorString(e), ms / 10, std::sqrt(num / den), worst);
    }
  }
  return 0;
}
