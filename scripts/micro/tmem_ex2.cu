// Microbenchmark for the tensor-core exponent idea (DESIGN.md §6 K5, round 2):
//  (1) TMEM read bandwidth (tcgen05.ld 32x32b.x16) per SM, alone and feeding MUFU ex2;
//  (2) ex2 fed from registers (the current kernel) for comparison;
//  (3) accuracy of the exponent E_kj = beta_k + W_k . p_j from ONE kind::tf32 MMA with K = 8
//      (3xTF32 packed into K: [Wh1 Wh2 Wl1 Wl2 Wh1 Wh2 bh bl] x [ph1 ph2 ph1 ph2 pl1 pl2 1 1])
//      against fp64 on the host, for two SWIZZLE_NONE descriptor readings.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ex2 tmem_ex2.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#define LDTM16(r, taddr)                                                                      \
  asm volatile(                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15}, [%16];"                                                                      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),   \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),            \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                                                 \
      : "r"(taddr))

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t t, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(ncols)
               : "memory");
}

#define STTM16(r, taddr)                                                                      \
  asm volatile(                                                                               \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16};" ::"r"(taddr),                                                            \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),            \
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),                  \
        "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory")
// mode 0: LDTM only (sum); 1: LDTM -> ex2 -> sum; 2: registers -> ex2 -> sum (no TMEM)
// 3: 8 LDTMs in flight then one wait (sum); 4: per block LDTM E -> ex2 -> STTM G, then per block
// LDTM G -> FFMA (the phase-split tile: E and G both through TMEM)
template <int MODE>
__global__ void bw_kernel(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const int q = warp & 3;
  const int per_q = nw / 4;                      // warps per lane quarter
  const int ncol = 512 / per_q;                  // columns per warp
  const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((warp >> 2) * ncol);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float rv[16];
  for (int i = 0; i < 16; ++i) rv[i] = -1.f + 0.001f * (lane + i);
  for (int it = 0; it < iters; ++it) {
    const uint32_t c0 = (uint32_t)((it * 128) % ncol);
#pragma unroll
    if (MODE == 3) {
      uint32_t r[8][16];
#pragma unroll
      for (int b = 0; b < 8; ++b) LDTM16(r[b], base + ((c0 + b * 16) % ncol));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i & 7] += __uint_as_float(r[b][i] & 0x3effffffu);
      continue;
    }
    if (MODE == 4) {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        uint32_t r[16];
        const uint32_t ta = base + ((c0 + b * 16) % ncol);
        LDTM16(r, ta);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float g = ex2f(__uint_as_float(r[i] & 0x3effffffu));
          acc[i & 7] += g;
          r[i] = __float_as_uint(g);
        }
        STTM16(r, ta);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        uint32_t r[16];
        LDTM16(r, base + ((c0 + b * 16) % ncol));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i & 7] = fmaf(__uint_as_float(r[i]), 0.5f, acc[i & 7]);
      }
      continue;
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      uint32_t r[16];
      if (MODE != 2) {
        LDTM16(r, base + ((c0 + b * 16) % ncol));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float v = MODE == 2 ? rv[i] + acc[i & 7] * 1e-30f : __uint_as_float(r[i] & 0x3effffffu);
        if (MODE != 0) v = ex2f(v);
        acc[i & 7] += v;
      }
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// ---- accuracy of the packed 3xTF32 exponent MMA ----------------------------------------
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// element (row, k) of a K-major SWIZZLE_NONE image with K = 8 tf32 (two 16-byte core columns)
__host__ __device__ inline uint32_t off_none(int row, int k, int kstride_bytes, int rstride_bytes) {
  return (uint32_t)((row >> 3) * rstride_bytes + (k >> 2) * kstride_bytes + (row & 7) * 16 + (k & 3) * 4);
}

__global__ void acc_kernel(const float* Aimg, const float* Bimg, int N, float* D, int variant) {
  // Aimg: 128 x 8 (row-major logical), Bimg: N x 8; D: 128 x N
  __shared__ __align__(1024) unsigned char sm[128 * 32 + 256 * 32];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* sa = sm;
  unsigned char* sb = sm + 128 * 32;
  // variant 0: LBO (K direction) = 128, SBO (8-row groups) = 256
  // variant 1: LBO = 256-ish swapped reading: K direction stride = 8*16*(rows/8) (K-halves as planes)
  const int rowsA = 128, rowsB = N;
  for (int i = tid; i < rowsA * 8; i += blockDim.x) {
    const int row = i / 8, k = i % 8;
    uint32_t o = variant == 0 ? off_none(row, k, 128, 256) : off_none(row, k, rowsA * 16, 128);
    *reinterpret_cast<float*>(sa + o) = Aimg[i];
  }
  for (int i = tid; i < rowsB * 8; i += blockDim.x) {
    const int row = i / 8, k = i % 8;
    uint32_t o = variant == 0 ? off_none(row, k, 128, 256) : off_none(row, k, rowsB * 16, 128);
    *reinterpret_cast<float*>(sb + o) = Bimg[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(&slot, 32);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint64_t ad = variant == 0 ? desc_none(smem_u32(sa), 128, 256) : desc_none(smem_u32(sa), rowsA * 16, 128);
    const uint64_t bd = variant == 0 ? desc_none(smem_u32(sb), 128, 256) : desc_none(smem_u32(sb), rowsB * 16, 128);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar)) : "memory");
  }
  // wait
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  LDTM16(r, tmem + ((uint32_t)(warp * 32) << 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int m = warp * 32 + lane;
  for (int j = 0; j < 16 && j < N; ++j) D[m * N + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 32);
}

static float tf32_rna_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x1000u;   // round to nearest (ties away) at bit 13
  u &= 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sms * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double clk = 1.965e9;
  for (int threads : {256, 512}) {
    const int iters = 4000;
    for (int mode = 0; mode < 5; ++mode) {
      auto launch = [&]() {
        if (mode == 0) bw_kernel<0><<<sms, threads>>>(out, iters);
        if (mode == 1) bw_kernel<1><<<sms, threads>>>(out, iters);
        if (mode == 2) bw_kernel<2><<<sms, threads>>>(out, iters);
        if (mode == 3) bw_kernel<3><<<sms, threads>>>(out, iters);
        if (mode == 4) bw_kernel<4><<<sms, threads>>>(out, iters);
      };
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double vals = (double)sms * threads * iters * 128.0;
      const double per_clk_sm = vals / (ms * 1e-3) / clk / sms;
      printf("threads %d mode %d (%s): %.3f ms, %.2f values/clk/SM (%.1f B/clk/SM of TMEM)\n",
             threads, mode, mode == 0 ? "LDTM only" : mode == 1 ? "LDTM->ex2" : mode == 2 ? "reg->ex2" : mode == 3 ? "LDTM x8 pipelined" : "E->ex2->STTM->LDTM->FFMA", ms,
             per_clk_sm, mode == 2 ? 0.0 : per_clk_sm * (mode == 4 ? 8 : 4));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));

  // accuracy test
  const int N = 16;
  srand(1);
  auto nrm = [&]() {
    double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0);
    return sqrt(-2 * log(u1)) * cos(2 * M_PI * u2);
  };
  std::vector<double> W(128 * 2), beta(128), P(N * 2);
  std::vector<float> Wf(128 * 2), bf(128), Pf(N * 2);
  for (int k = 0; k < 128; ++k) {
    for (int c = 0; c < 2; ++c) { Wf[k * 2 + c] = (float)(57.7 * 0.3 * nrm()); W[k * 2 + c] = Wf[k * 2 + c]; }
    bf[k] = (float)(-20.0 + 3 * nrm());
    beta[k] = bf[k];
  }
  for (int j = 0; j < N; ++j)
    for (int c = 0; c < 2; ++c) { Pf[j * 2 + c] = (float)(0.5 * nrm()); P[j * 2 + c] = Pf[j * 2 + c]; }
  std::vector<float> A(128 * 8), B(N * 8);
  for (int k = 0; k < 128; ++k) {
    float wh[2], wl[2];
    for (int c = 0; c < 2; ++c) { wh[c] = tf32_rna_host(Wf[k * 2 + c]); wl[c] = tf32_rna_host(Wf[k * 2 + c] - wh[c]); }
    const float bh = tf32_rna_host(bf[k]), bl = tf32_rna_host(bf[k] - bh);
    float row[8] = {wh[0], wh[1], wl[0], wl[1], wh[0], wh[1], bh, bl};
    for (int i = 0; i < 8; ++i) A[k * 8 + i] = row[i];
  }
  for (int j = 0; j < N; ++j) {
    float ph[2], pl[2];
    for (int c = 0; c < 2; ++c) { ph[c] = tf32_rna_host(Pf[j * 2 + c]); pl[c] = tf32_rna_host(Pf[j * 2 + c] - ph[c]); }
    float row[8] = {ph[0], ph[1], ph[0], ph[1], pl[0], pl[1], 1.f, 1.f};
    for (int i = 0; i < 8; ++i) B[j * 8 + i] = row[i];
  }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dD, 0, 128 * N * 4);
    acc_kernel<<<1, 128>>>(dA, dB, N, dD, variant);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(128 * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxabs = 0, maxfma = 0, maxE = 0;
    for (int k = 0; k < 128; ++k)
      for (int j = 0; j < N; ++j) {
        const double ex = beta[k] + W[k * 2] * P[j * 2] + W[k * 2 + 1] * P[j * 2 + 1];
        float f = bf[k];
        f = fmaf(Wf[k * 2], Pf[j * 2], f);
        f = fmaf(Wf[k * 2 + 1], Pf[j * 2 + 1], f);
        maxabs = fmax(maxabs, fabs(D[k * N + j] - ex));
        maxfma = fmax(maxfma, fabs(f - ex));
        maxE = fmax(maxE, fabs(ex));
      }
    printf("variant %d (%s): max |E_tc - E| = %.3e, fp32 FMA chain max err = %.3e, max |E| = %.2f; D[0]=%g\n",
           variant, cudaGetErrorString(e), maxabs, maxfma, maxE, D[0]);
  }
  return 0;
}
