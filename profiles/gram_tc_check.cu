// Stand-alone check + timing of the tcgen05 3xTF32 tall product (gram_tc.cu) against fp64 on the host:
//   (a) symmetric Gram  Y^T Y          (rows x l)
//   (b) NC block        X^T diag(s) Z  (rows x d, rows x l), row-scaled
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc \
//        profiles/gram_tc_check.cu -L paper_2111_06312_b200 -l:libisvd.so \
//        -Xlinker -rpath=$PWD/paper_2111_06312_b200 -o build/gram_tc_check
//   build/gram_tc_check [rows] [l] [d]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "common.cuh"

static double check(const char* name, const std::vector<float>& A, int64_t lda, int64_t Ka, const float* rs,
                    const std::vector<float>& B, int64_t ldb, int64_t Kb, int64_t rows, const std::vector<double>& G,
                    bool sym) {
  // sampled entries, error relative to sqrt(sum A_i^2 sum B_j^2) (the Cauchy-Schwarz scale)
  std::mt19937 rng(7);
  double maxrel = 0.0, maxrel_fro = 0.0;
  double num = 0.0, den = 0.0;
  for (int t = 0; t < 300; ++t) {
    int64_t i = rng() % Ka, j = rng() % Kb;
    if (sym && i > j) std::swap(i, j);
    double s = 0.0, na = 0.0, nb = 0.0;
    for (int64_t r = 0; r < rows; ++r) {
      const double af = (double)(float)(A[r * lda + i] * (rs ? rs[r] : 1.f));  // row scale applied in fp32
      const double b = B[r * ldb + j];
      s += af * b;
      na += af * af;
      nb += b * b;
    }
    const double g = G[i * Kb + j];
    maxrel = std::fmax(maxrel, std::fabs(g - s) / std::sqrt(na * nb));
    num += (g - s) * (g - s);
    den += s * s;
  }
  maxrel_fro = std::sqrt(num / den);
  printf("%s: max |C - C64| / (|a_i| |b_j|) = %.3e   sampled rel-fro = %.3e\n", name, maxrel, maxrel_fro);
  return maxrel_fro;
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 1000000;
  const int64_t l = argc > 2 ? atoll(argv[2]) : 400;
  const int64_t d = argc > 3 ? atoll(argv[3]) : 100;
  const int64_t ld = (l + 3) / 4 * 4, ldx = (d + 3) / 4 * 4;
  const int sms = 148;
  std::vector<float> Y(rows * ld, 0.f), X(rows * ldx, 0.f), s(rows);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ud(0.05f, 1.f);
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t j = 0; j < l; ++j) Y[i * ld + j] = nd(rng) + (j % 7 == 0 ? 2.f : 0.f);
    for (int64_t j = 0; j < d; ++j) X[i * ldx + j] = nd(rng);
    s[i] = ud(rng);
  }
  float *dY, *dX, *ds, *ws;
  double* dG;
  cudaMalloc(&dY, sizeof(float) * rows * ld);
  cudaMalloc(&dX, sizeof(float) * rows * ldx);
  cudaMalloc(&ds, sizeof(float) * rows);
  cudaMemcpy(dY, Y.data(), sizeof(float) * rows * ld, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), sizeof(float) * rows * ldx, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), sizeof(float) * rows, cudaMemcpyHostToDevice);
  int64_t wsf = std::max(isvd::tc_atb_ws_floats(rows, l, l, true, sms), isvd::tc_atb_ws_floats(rows, d, l, false, sms));
  cudaMalloc(&ws, sizeof(float) * wsf);
  cudaMalloc(&dG, sizeof(double) * l * l);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int rc = 0;
  for (int which = 0; which < 2; ++which) {
    const bool sym = which == 0;
    const float* A = sym ? dY : dX;
    const int64_t lda = sym ? ld : ldx, Ka = sym ? l : d;
    const float* rsd = sym ? nullptr : ds;
    int64_t wlda = 0, wld = 0, parts = 0;
    float ms = 0.f;
    for (int it = 0; it < 6; ++it) {
      if (it == 1) cudaEventRecord(e0);
      cudaError_t e = isvd::launch_tc_atb(A, lda, Ka, rsd, dY, ld, l, rows, sym, ws, &wlda, &wld, &parts, sms, nullptr,
                                          0);
      if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    e = isvd::launch_atb_f32_reduce(ws, wlda, wld, parts, Ka, l, sym, dG, l, nullptr, 0, sms, nullptr, 0);
    e = cudaDeviceSynchronize();
    printf("%s: %s  parts %lld ws %lld x %lld  %.3f ms/launch  (%.1f GB/s of operand reads, %.1f TFLOP/s 3xTF32)\n",
           sym ? "gram" : "xtz", cudaGetErrorString(e), (long long)parts, (long long)wlda, (long long)wld, ms,
           (double)rows * (sym ? l : (l + d)) * 4 / (ms * 1e-3) / 1e9,
           3.0 * 2.0 * rows * Ka * l / (ms * 1e-3) / 1e12);
    if (e != cudaSuccess) return 1;
    std::vector<double> G(Ka * l);
    cudaMemcpy(G.data(), dG, sizeof(double) * Ka * l, cudaMemcpyDeviceToHost);
    double rel = check(sym ? "gram" : "xtz", sym ? Y : X, lda, Ka, sym ? nullptr : s.data(), Y, ld, l, rows, G, sym);
    if (rel > 1e-5) rc = 2;
  }
  return rc;
}
