// Does the SIMT tall GEMM run power-capped?  Repeats X G (n x 100 by 100 x 400) for ~3 s while
// nvidia-smi samples clocks and power (profiles/capture_r02h_clock.sh), and reports ms per launch
// for the first 5 launches (cool) and the last 50 (sustained).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

int main(int argc, char** argv) {
  const int64_t n = 2449029, l = 400, d = 100;
  const int reps = argc > 1 ? atoi(argv[1]) : 600;
  float *dX, *dG, *dC;
  cudaMalloc(&dX, 4 * n * d);
  cudaMalloc(&dG, 4 * d * l);
  cudaMalloc(&dC, 4 * n * l);
  cudaMemset(dX, 0x3c, 4 * n * d);
  cudaMemset(dG, 0x3c, 4 * d * l);
  std::vector<cudaEvent_t> ev(reps + 1);
  for (auto& e : ev) cudaEventCreate(&e);
  isvd::launch_gemm_tn(dX, d, dG, l, dC, l, n, l, d, nullptr, 1.f, false, nullptr, 0);
  cudaDeviceSynchronize();
  cudaEventRecord(ev[0]);
  for (int i = 0; i < reps; ++i) {
    isvd::launch_gemm_tn(dX, d, dG, l, dC, l, n, l, d, nullptr, 1.f, false, nullptr, 0);
    cudaEventRecord(ev[i + 1]);
  }
  cudaDeviceSynchronize();
  auto span = [&](int a, int b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return ms / (b - a);
  };
  printf("first 5: %.3f ms   launches 50-100: %.3f ms   last 50: %.3f ms   (%d launches)\n", span(0, 5), span(50, 100),
         span(reps - 50, reps), reps);
  return 0;
}
