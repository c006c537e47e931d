// Microbenchmark: MUFU ex2 and FFMA throughput per SM on this GPU (calibrates the "alu" roofline).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ex2_kernel(float* out, int iters, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-6f + i * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y * -0.5f; }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void ffma_kernel(float* out, int iters, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-6f + i * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void ffma2_kernel(float* out, int iters, float seed) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(seed + threadIdx.x * 1e-6f + i * 1e-3f, seed); a[i] = *reinterpret_cast<unsigned long long*>(&v); }
  float2 m2 = make_float2(0.999f, 0.999f), c2 = make_float2(0.001f, 0.001f);
  unsigned long long m = *reinterpret_cast<unsigned long long*>(&m2), c = *reinterpret_cast<unsigned long long*>(&c2);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(m), "l"(c));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += reinterpret_cast<float2*>(&a[i])->x;
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, blocks = sms * 4, threads = 512;
  for (int k = 0; k < 3; ++k) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0);
      if (k == 0) ex2_kernel<<<blocks, threads>>>(d, iters, 0.1f);
      else if (k == 1) ffma_kernel<<<blocks, threads>>>(d, iters, 0.1f);
      else ffma2_kernel<<<blocks, threads>>>(d, iters, 0.1f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8 * (k == 2 ? 2 : 1);
      if (w == 1) printf("%s: %.3f ms, %.3f Tops/s, %.2f ops/clk/SM at max clock %d MHz\n", k == 0 ? "ex2" : (k == 1 ? "ffma" : "ffma2 (per fp32 fma)"), ms, ops / ms / 1e9,
             ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
