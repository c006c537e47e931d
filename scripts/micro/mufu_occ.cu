// Microbenchmark: MUFU ex2 throughput vs warps per SM and independent chains per thread (ILP),
// plus the same with a dependent FFMA2 consumer (the implicit kernel's dot pattern).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void ex2_ilp(float* out, int iters, float seed) {
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = seed + threadIdx.x * 1e-6f + i * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y * -0.5f; }
  }
  float s = 0; for (int i = 0; i < ILP; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
// pattern: e = fma(w, x, b) (x2), ex2, dot += f * s  -- 32 entries per "tile", independent across tiles
__global__ void pattern(float* out, int iters, float seed) {
  float w[32], b[32], sv[32];
  for (int i = 0; i < 32; ++i) { w[i] = 0.01f * i + seed; b[i] = -0.02f * i; sv[i] = 1.0f + i * 1e-3f; }
  float x = seed + threadIdx.x * 1e-6f, acc = 0.f, dot = 0.f;
  for (int it = 0; it < iters; ++it) {
    float f[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) { float e = fmaf(w[i], x, b[i]); asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(f[i]) : "f"(e)); }
    float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; i += 4) { d0 = fmaf(f[i], sv[i], d0); d1 = fmaf(f[i+1], sv[i+1], d1); d2 = fmaf(f[i+2], sv[i+2], d2); d3 = fmaf(f[i+3], sv[i+3], d3); }
    dot = (d0 + d1) + (d2 + d3);
    x = x * 0.999f + dot * 1e-9f;
    acc += dot;
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  int warps_list[] = {4, 8, 12, 16, 32};
  for (int wi = 0; wi < 5; ++wi) {
    int threads = warps_list[wi] * 32;
    for (int k = 0; k < 4; ++k) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (k == 0) ex2_ilp<8><<<sms, threads>>>(d, iters * 4, 0.1f);
        else if (k == 1) ex2_ilp<16><<<sms, threads>>>(d, iters * 2, 0.1f);
        else if (k == 2) ex2_ilp<32><<<sms, threads>>>(d, iters, 0.1f);
        else pattern<<<sms, threads>>>(d, iters, 0.1f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      double ops = (double)sms * threads * iters * 32;
      printf("warps/SM %2d %-10s ex2/clk/SM %.2f\n", warps_list[wi], k == 0 ? "ilp8" : k == 1 ? "ilp16" : k == 2 ? "ilp32" : "pattern",
             ops / (best * 1e-3) / sms / (clk * 1e3));
    }
  }
  return 0;
}
