// Microbenchmark: per-SM throughput of MUFU.EX2 vs FMA-pipe polynomial exp2 on this part.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2_poly3(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(5.500872061e-02f, f, 2.422104627e-01f), f, 6.932829022e-01f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
template <int MODE>
__global__ void k(float* out, int iters, float seed) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = -0.001f * (threadIdx.x + j) - seed;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float e;
      if (MODE == 0) e = ex2(a[j]);
      else if (MODE == 1) e = ex2_poly3(a[j]);
      else e = fmaf(a[j], 1.0001f, -0.5f);
      acc += e;
      a[j] = a[j] * 0.999f - 1e-3f;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    for (int mode = 0; mode < 3; ++mode) {
      dim3 grid(sms * 2048 / threads);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&]() {
        if (mode == 0) k<0><<<grid, threads>>>(d, iters, 0.1f);
        else if (mode == 1) k<1><<<grid, threads>>>(d, iters, 0.1f);
        else k<2><<<grid, threads>>>(d, iters, 0.1f);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double n = (double)grid.x * threads * iters * 8;
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("threads %4d mode %s: %.3f ms  %.3e exp/s  %.2f per SM per clk(@max %d MHz)\n", threads,
             mode == 0 ? "MUFU.EX2 " : mode == 1 ? "poly3    " : "FFMA+FADD", ms, n / ms * 1e3,
             n / (ms * 1e-3) / sms / (1965e6), clk / 1000);
    }
  }
  return 0;
}
