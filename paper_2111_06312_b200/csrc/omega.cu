// Omega generator (Alg. 1 line 4: Q ~ N(0,1)^{c x 2k}).
//
// The paper only says "standard normal".  The stream is fixed by DESIGN.md
// reading O11 so that it depends on (seed, global row, column) only and is
// identical for every row partition:
//   Philox4x32-10 (Salmon et al. SC'11), key = (seed lo, seed hi),
//   counter of block b = (b lo, b hi, 0x4F4D4547, 0);
//   element (i, j) -> e = i*l + j, block b = e >> 2, word t = e & 3;
//   u_t = (x_t + 0.5) 2^-32;  z0,z1 = sqrt(-2 ln u0) (cos, sin)(2 pi u1),
//   z2,z3 = sqrt(-2 ln u2) (cos, sin)(2 pi u3), in fp64, rounded to fp32.
// This file is compiled with --fmad=false so each fp64 operation rounds once.
#include "common.cuh"

namespace isvd {
namespace {

struct U4 { uint32_t x, y, z, w; };

ISVD_DEVICE U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    U4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Box-Muller output t of Philox block b (the pair (u0,u1) feeds words 0,1; (u2,u3) words 2,3).
ISVD_DEVICE void gauss4(int64_t b, uint32_t k0, uint32_t k1, double z[4]) {
  const double two_pi = 6.283185307179586;  // nearest double to 2 pi
  const double two_m32 = 2.3283064365386963e-10;  // 2^-32
  U4 c{(uint32_t)(b & 0xFFFFFFFFu), (uint32_t)((uint64_t)b >> 32), 0x4F4D4547u, 0u};
  U4 x = philox4x32_10(c, k0, k1);
  double u0 = ((double)x.x + 0.5) * two_m32;
  double u1 = ((double)x.y + 0.5) * two_m32;
  double u2 = ((double)x.z + 0.5) * two_m32;
  double u3 = ((double)x.w + 0.5) * two_m32;
  double r01 = sqrt(-2.0 * log(u0));
  double r23 = sqrt(-2.0 * log(u2));
  double t1 = two_pi * u1, t3 = two_pi * u3;
  z[0] = r01 * cos(t1);
  z[1] = r01 * sin(t1);
  z[2] = r23 * cos(t3);
  z[3] = r23 * sin(t3);
}

// Contiguous global rows [row0, row0 + rows): one thread per Philox block.
__global__ void omega_kernel(uint32_t k0, uint32_t k1, int64_t row0, int64_t rows, int l, int64_t ld,
                             float* __restrict__ out) {
  const int64_t e0 = row0 * (int64_t)l;
  const int64_t e1 = (row0 + rows) * (int64_t)l;
  const int64_t b0 = e0 >> 2, b1 = (e1 + 3) >> 2;
  for (int64_t b = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < b1;
       b += (int64_t)gridDim.x * blockDim.x) {
    double z[4];
    gauss4(b, k0, k1, z);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int64_t e = 4 * b + t;
      if (e < e0 || e >= e1) continue;
      int64_t i = e / l - row0;
      int64_t j = e - (e / l) * l;
      out[i * ld + j] = (float)z[t];
    }
  }
}

// Relabelled rows: internal row i is global row row_map[i]; one thread per element.
__global__ void omega_mapped_kernel(uint32_t k0, uint32_t k1, const int32_t* __restrict__ row_map, int64_t rows,
                                    int l, int64_t ld, float* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * l; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / l, j = t - i * l;
    int64_t e = (int64_t)row_map[i] * l + j;
    double z[4];
    gauss4(e >> 2, k0, k1, z);
    out[i * ld + j] = (float)z[e & 3];
  }
}

__global__ void zero_pad_kernel(float* out, int64_t rows, int l, int64_t ld) {
  int64_t np = ld - l;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * np; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / np;
    out[i * ld + l + (t - i * np)] = 0.f;
  }
}

}  // namespace

cudaError_t launch_omega(uint64_t seed, int64_t row0, int64_t rows, int l, int64_t ld, float* out,
                         const int32_t* row_map, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const uint32_t k0 = (uint32_t)(seed & 0xFFFFFFFFu), k1 = (uint32_t)(seed >> 32);
  const int threads = 256;
  if (row_map) {
    int64_t blocks = (rows * l + threads - 1) / threads;
    if (blocks > 148 * 32) blocks = 148 * 32;
    ++g_launches;
    omega_mapped_kernel<<<(int)blocks, threads, 0, st>>>(k0, k1, row_map, rows, l, ld, out);
  } else {
    int64_t nb = ((row0 + rows) * l + 3) / 4 - (row0 * l) / 4;
    int64_t blocks = (nb + threads - 1) / threads;
    if (blocks > 148 * 32) blocks = 148 * 32;
    ++g_launches;
    omega_kernel<<<(int)blocks, threads, 0, st>>>(k0, k1, row0, rows, l, ld, out);
  }
  if (ld > l) {
    int64_t tot = rows * (ld - l);
    int64_t zb = (tot + 255) / 256;
    if (zb > 148 * 8) zb = 148 * 8;
    ++g_launches; zero_pad_kernel<<<(int)zb, 256, 0, st>>>(out, rows, l, ld);
  }
  return cudaGetLastError();
}

}  // namespace isvd
