// Timing + sampled fp64 check of the SIMT dense kernels at config-4 shapes (dense.cu):
//   X^T diag(s) Z  (n x 100, n x 400)        launch_atb(f32_stage)
//   Y^T Y exact    (n x 400)                 launch_atb (fp64 / DMMA)
//   X G            (n x 100) (100 x 400)     launch_gemm_tn
//   Y R^-1         (n x 400) (400 x 400 upper) launch_gemm_tn(upper_tri_b)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include \
//        profiles/dense_check.cu -L paper_2111_06312_b200 -l:libisvd.so \
//        -Xlinker -rpath='$ORIGIN/../paper_2111_06312_b200' -o build/dense_check
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "common.cuh"

template <class F>
static float time_ms(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 2449029;
  const int64_t l = 400, d = 100, sms = 148;
  std::mt19937 rng(5);
  std::normal_distribution<float> nd;
  std::vector<float> X(n * d), Z(n * l), s(n), R(l * l, 0.f), G(d * l);
  for (auto& v : X) v = nd(rng);
  for (auto& v : Z) v = nd(rng);
  for (auto& v : s) v = 0.2f + std::fabs(nd(rng));
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = i; j < l; ++j) R[i * l + j] = (i == j ? 1.f : 0.f) + 0.01f * nd(rng);
  for (auto& v : G) v = nd(rng) / 10.f;
  float *dX, *dZ, *ds, *dR, *dG, *dC;
  double *ws, *dOut;
  cudaMalloc(&dX, 4 * n * d);
  cudaMalloc(&dZ, 4 * n * l);
  cudaMalloc(&ds, 4 * n);
  cudaMalloc(&dR, 4 * l * l);
  cudaMalloc(&dG, 4 * d * l);
  cudaMalloc(&dC, 4 * n * l);
  const int64_t wsd = std::max(isvd::atb_ws_doubles(n, l, l, sms), isvd::atb_ws_doubles(n, d, l, sms));
  cudaMalloc(&ws, 8 * wsd);
  cudaMalloc(&dOut, 8 * l * l);
  cudaMemcpy(dX, X.data(), 4 * n * d, cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), 4 * n * l, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, R.data(), 4 * l * l, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, G.data(), 4 * d * l, cudaMemcpyHostToDevice);
  const double gf = 2.0 * n * d * l / 1e9;
  float t;
  // X^T diag(s) Z
  t = time_ms([&] { isvd::launch_atb(dX, d, dZ, l, n, d, l, ds, false, ws, dOut, l, nullptr, 0, sms, nullptr, 0, true); });
  {
    std::vector<double> out(d * l);
    cudaMemcpy(out.data(), dOut, 8 * d * l, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (int t2 = 0; t2 < 40; ++t2) {
      const int64_t i = rng() % d, j = rng() % l;
      double ref = 0;
      for (int64_t r = 0; r < n; ++r) ref += (double)X[r * d + i] * ((double)(float)(s[r] * Z[r * l + j]));
      num += (out[i * l + j] - ref) * (out[i * l + j] - ref);
      den += ref * ref;
    }
    printf("X^T s Z   : %7.3f ms  %6.1f TFLOP/s   sampled rel err %.2e\n", t, gf / t, std::sqrt(num / den));
    // the solver's form: X pre-scaled once per op, no per-element row scale in the kernel
    const float tn = time_ms([&] { isvd::launch_atb(dX, d, dZ, l, n, d, l, nullptr, false, ws, dOut, l, nullptr, 0, sms,
                                                     nullptr, 0, true); });
    printf("X^T Z     : %7.3f ms  %6.1f TFLOP/s   (pre-scaled X)\n", tn, gf / tn);
  }
  t = time_ms([&] { isvd::launch_atb(dZ, l, dZ, l, n, l, l, nullptr, true, ws, dOut, l, nullptr, 0, sms, nullptr, 0, false); });
  printf("Z^T Z fp64: %7.3f ms  %6.1f TFLOP/s (symmetric half)\n", t, 2.0 * n * l * l / 2 / 1e9 / t);
  {
    cudaError_t le = isvd::launch_gemm_tn(dX, d, dG, l, dC, l, n, l, d, nullptr, 1.f, false, nullptr, 0);
    cudaError_t se = cudaDeviceSynchronize();
    if (le != cudaSuccess || se != cudaSuccess) printf("X G launch: %s / %s\n", cudaGetErrorString(le), cudaGetErrorString(se));
  }
  t = time_ms([&] { isvd::launch_gemm_tn(dX, d, dG, l, dC, l, n, l, d, nullptr, 1.f, false, nullptr, 0); });
  {
    // sampled fp64 check: rows from the first, a middle and the ragged last tile, every column
    std::vector<float> Cs(l);
    double worst = 0;
    const int64_t rows[6] = {0, 63, 64, n / 2 + 7, n - 2, n - 1};
    for (int64_t r : rows) {
      cudaMemcpy(Cs.data(), dC + r * l, 4 * l, cudaMemcpyDeviceToHost);
      for (int64_t j = 0; j < l; ++j) {
        double ref = 0, mag = 0;
        for (int64_t k = 0; k < d; ++k) {
          ref += (double)X[r * d + k] * G[k * l + j];
          mag += std::fabs((double)X[r * d + k] * G[k * l + j]);
        }
        worst = std::max(worst, std::fabs(Cs[j] - ref) / mag);
      }
    }
    printf("X G       : %7.3f ms  %6.1f TFLOP/s   sampled worst err / sum|terms| %.2e\n", t, gf / t, worst);
  }
  t = time_ms([&] { isvd::launch_gemm_tn(dX, d, dG, l, dC, l, n, l, d, ds, 1.f, false, nullptr, 0); });
  printf("s X G     : %7.3f ms  %6.1f TFLOP/s   (row scale in the epilogue)\n", t, gf / t);
  t = time_ms([&] { isvd::launch_gemm_tn(dZ, l, dR, l, dC, l, n, l, l, nullptr, 1.f, true, nullptr, 0); });
  {
    std::vector<float> Cs(l);
    double worst = 0;
    const int64_t rows[6] = {0, 63, 64, n / 2 + 7, n - 2, n - 1};
    for (int64_t r : rows) {
      cudaMemcpy(Cs.data(), dC + r * l, 4 * l, cudaMemcpyDeviceToHost);
      for (int64_t j = 0; j < l; ++j) {
        double ref = 0, mag = 0;
        for (int64_t k = 0; k <= j; ++k) {
          ref += (double)Z[r * l + k] * R[k * l + j];
          mag += std::fabs((double)Z[r * l + k] * R[k * l + j]);
        }
        worst = std::max(worst, std::fabs(Cs[j] - ref) / mag);
      }
    }
    printf("Y R^-1    : %7.3f ms  %6.1f TFLOP/s (triangular half)   sampled worst err / sum|terms| %.2e\n", t,
           2.0 * n * l * l / 2 / 1e9 / t, worst);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
