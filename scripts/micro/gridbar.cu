// Microbenchmark: latency of the persistent kernels' grid barrier (one monotone counter, one
// red.release per CTA, thread 0 polls with ld.acquire) against K sub-counters (CTA c adds to
// counter c % K, lanes 0..K-1 poll one counter each), 148 CTAs x 256 threads, 4000 barriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar gridbar.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void red_release_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int K>
__global__ void bar_kernel(unsigned int* ctr, int nbar, unsigned long long* out) {
  const int tid = threadIdx.x, cta = blockIdx.x, G = gridDim.x;
  unsigned long long t0 = clock64();
  for (int b = 1; b <= nbar; ++b) {
    __syncthreads();
    if (K == 1) {
      if (tid == 0) {
        red_release_add(ctr, 1u);
        while (ld_acquire(ctr) < (unsigned)(b * G)) {
        }
      }
    } else {
      if (tid == 0) red_release_add(ctr + (cta % K) * 32, 1u);
      if (tid < K) {
        const unsigned cnt = (unsigned)((G - tid + K - 1) / K);
        while (ld_acquire(ctr + tid * 32) < (unsigned)b * cnt) {
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) out[cta] = clock64() - t0;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned int* ctr;
  unsigned long long* out;
  cudaMalloc(&ctr, 64 * 32 * 4);
  cudaMalloc(&out, sms * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nbar = 4000;
  for (int rep = 0; rep < 2; ++rep)
    for (int K : {1, 4, 8, 16, 32}) {
      cudaMemset(ctr, 0, 64 * 32 * 4);
      void* args[] = {&ctr, (void*)&nbar, &out};
      const void* f = K == 1 ? (const void*)bar_kernel<1> : K == 4 ? (const void*)bar_kernel<4>
                    : K == 8 ? (const void*)bar_kernel<8> : K == 16 ? (const void*)bar_kernel<16>
                    : (const void*)bar_kernel<32>;
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel(f, dim3(sms), dim3(256), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("K = %2d: %.3f us per grid barrier (%d CTAs)\n", K, 1e3 * ms / nbar, sms);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
