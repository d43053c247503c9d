// FP32 FMA issue/throughput probe on sm_100a: FFMA (scalar) vs FFMA2 (fma.rn.f32x2) with 8
// independent accumulator chains per thread, 4 warps x 8 CTAs per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 profiles/ffma2_rate.cu -o build/ffma2_rate
#include <cstdio>

__global__ void ffma(float* out, int iters, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2(float* out, int iters, float a, float b) {
  unsigned long long acc[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  const unsigned long long ad = *reinterpret_cast<unsigned long long*>(&av), bd = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
    acc[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(ad), "l"(bd));
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 v = *reinterpret_cast<float2*>(&acc[i]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  const int iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) ffma<<<148 * 8, 256>>>(d, iters, 0.999f, 1e-3f);
      else ffma2<<<148 * 8, 256>>>(d, iters, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 16 * (double)iters * 148 * 8 * 256;
      if (rep) printf("%s: %.3f ms  %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA ", ms, flops / ms / 1e9);
    }
  }
  return 0;
}
