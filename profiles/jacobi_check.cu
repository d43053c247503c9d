// Timing of the on-device one-sided Jacobi SVD (smallmat.cu) at l = 160 / 256 / 400: block variant
// (default) vs pairwise cooperative variant (ISVD_JACOBI_PAIRWISE=1); singular values compared.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc -I include \
//        profiles/jacobi_check.cu -L paper_2111_06312_b200 -l:libisvd.so \
//        -Xlinker -rpath='$ORIGIN/../paper_2111_06312_b200' -o build/jacobi_check
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "common.cuh"

int main() {
  int rc = 0;
  for (int l : {160, 256, 400}) {
    const int k = l * 5 / 8, ldk = (k + 3) / 4 * 4;
    std::mt19937 rng(l);
    std::normal_distribution<double> nd;
    // R upper triangular with a decaying spectrum (like the R of W = M^T Q)
    std::vector<double> R((size_t)l * l, 0.0);
    for (int i = 0; i < l; ++i)
      for (int j = i; j < l; ++j) R[(size_t)i * l + j] = (i == j ? 10.0 * std::exp(-i / 60.0) : 0.3 * nd(rng));
    double *dR, *ws, *sig;
    float *Ub, *Vb;
    isvd::DevStatus* st;
    cudaMalloc(&dR, 8 * l * l);
    cudaMalloc(&ws, 8 * isvd::jacobi_ws_doubles(l));
    cudaMalloc(&sig, 8 * l);
    cudaMalloc(&Ub, 4 * l * ldk);
    cudaMalloc(&Vb, 4 * l * ldk);
    cudaMalloc(&st, sizeof(isvd::DevStatus));
    cudaMemcpy(dR, R.data(), 8 * l * l, cudaMemcpyHostToDevice);
    std::vector<double> s_mode[2];
    for (int mode = 0; mode < 2; ++mode) {
      if (mode == 1) setenv("ISVD_JACOBI_PAIRWISE", "1", 1);
      else unsetenv("ISVD_JACOBI_PAIRWISE");
      cudaMemset(st, 0, sizeof(isvd::DevStatus));
      isvd::launch_jacobi_svd(dR, l, k, ldk, sig, Ub, Vb, ws, st, 148, 0);  // warm-up
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int reps = 3;
      for (int r = 0; r < reps; ++r) isvd::launch_jacobi_svd(dR, l, k, ldk, sig, Ub, Vb, ws, st, 148, 0);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      isvd::DevStatus h;
      cudaMemcpy(&h, st, sizeof(h), cudaMemcpyDeviceToHost);
      s_mode[mode].resize(k);
      cudaMemcpy(s_mode[mode].data(), sig, 8 * k, cudaMemcpyDeviceToHost);
      printf("l=%d %-9s: %s %8.3f ms  sweeps %d  sigma0 %.6f\n", l, mode ? "pairwise" : "block", cudaGetErrorString(e),
             ms / reps, h.jacobi_sweeps, s_mode[mode][0]);
      if (e != cudaSuccess) return 1;
    }
    double md = 0;
    for (int i = 0; i < k; ++i) md = std::fmax(md, std::fabs(s_mode[0][i] - s_mode[1][i]) / s_mode[1][0]);
    printf("l=%d max |s_block - s_pairwise| / s_max = %.2e\n", l, md);
    if (md > 1e-12) rc = 2;
  }
  return rc;
}
