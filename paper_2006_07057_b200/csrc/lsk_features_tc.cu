// lsk_features_tc.cu — a3 for large d: the Gaussian positive feature map with
// the x.u contraction on the 5th-generation tensor cores (tcgen05.mma, kind::tf32, fp32
// accumulators in TMEM), in 3xTF32 (reading C14: plain TF32 misses the 1e-4 scaling parity):
//     G = X W^T,  W = (4 log2e / eps) U,  G ~= Xhi Whi^T + Xhi Wlo^T + Xlo Whi^T
//     xi_ik = 2^( alpha2_i + beta2_k + G_ik ),  alpha2_i = -(2 log2e/eps)|x_i|^2,
//     beta2_k = log2e (-(2/eps)|u_k|^2 + |u_k|^2/(eps q) + log_scale)
// hi = cvt.rna.tf32(v), lo = cvt.rna.tf32(v - hi) are formed explicitly, so the MMA sees exactly
// representable operands.
//
// CTA tile 128 rows x 256 anchors, K in chunks of 32 (one 128-byte swizzle row).  Operands
// live in shared memory in the canonical K-major SWIZZLE_128B layout (8-row x 128 B atoms,
// SBO = 1024 B): W hi/lo images are pre-built once per call in global memory and brought in
// with one bulk async copy per chunk (TMA engine, mbarrier complete_tx); X chunks are loaded,
// split and swizzled by the threads.  One elected thread issues 3 x 4 MMAs (128x256x8) per
// chunk; tcgen05.commit signals an mbarrier that releases the buffers and, after the last
// chunk, the epilogue: 8 warps read the accumulator with tcgen05.ld (warp w: TMEM lanes
// 32(w%4).., columns 128(w/4)..), add alpha2 + beta2, MUFU ex2, store fp32.
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"

namespace lsk {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 32;
constexpr int kThreads = 256;
constexpr int kXBytes = BM * BK * 4;   // 16 KB per hi / lo image
constexpr int kWBytes = BN * BK * 4;   // 32 KB per hi / lo image
constexpr double kLog2e = 1.4426950408889634074;
// smem: xhi | xlo | whi | wlo | beta2[BN] | alpha[BM] | barriers
constexpr int kOffXhi = 0, kOffXlo = kXBytes, kOffWhi = 2 * kXBytes, kOffWlo = 2 * kXBytes + kWBytes;
constexpr int kOffBeta = 2 * kXBytes + 2 * kWBytes;
constexpr int kOffAlpha = kOffBeta + BN * 4;
constexpr int kOffBar = kOffAlpha + BM * 4;
constexpr int kSmemBytes = kOffBar + 64 + 1024;   // + alignment slack

// byte offset of element (row, k) inside a K-major SWIZZLE_128B image (rows of 128 B)
__host__ __device__ __forceinline__ uint32_t swz128(int row, int k) {
  const uint32_t chunk = (uint32_t)(k >> 2) ^ (uint32_t)(row & 7);
  return (uint32_t)row * 128u + chunk * 16u + (uint32_t)(k & 3) * 4u;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, cta_group::1
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// W hi/lo images: [ntile][kchunk][2][BN rows x 128 B swizzled]; rows >= r and k >= d are 0.
__global__ void w_images_kernel(const float* __restrict__ U, int r, int d, double sc,
                                float* __restrict__ img) {
  const int nt = blockIdx.x, kc = blockIdx.y;
  const int nkc = gridDim.y;
  char* base = reinterpret_cast<char*>(img) + ((size_t)nt * nkc + kc) * 2 * kWBytes;
  for (int i = threadIdx.x; i < BN * BK; i += blockDim.x) {
    const int row = i / BK, k = i % BK;
    const int n = nt * BN + row, c = kc * BK + k;
    const float w = (n < r && c < d) ? (float)(sc * (double)U[(int64_t)n * d + c]) : 0.f;
    const float hi = tf32_rna(w);
    const float lo = tf32_rna(w - hi);
    *reinterpret_cast<float*>(base + swz128(row, k)) = hi;
    *reinterpret_cast<float*>(base + kWBytes + swz128(row, k)) = lo;
  }
}

// mode 0 (Gaussian): out = 2^(alpha2 + beta2_k + acc); mode 1 (arc-cosine): out =
// beta2_k relu(acc)^sdeg with beta2 = the per-anchor coefficient.  Output row stride ld.
__global__ void __launch_bounds__(kThreads, 2) feature_map_tc_kernel(
    const float* __restrict__ X, int64_t M, int d, const float* __restrict__ wimg,
    const float* __restrict__ beta2, int r, float c2, float* __restrict__ Xi, int ld, int mode,
    int sdeg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array itself: an integer round
  // trip would drop the address space and turn every smem access below into a generic LD/ST
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* beta_s = reinterpret_cast<float*>(smem + kOffBeta);
  float* alpha_s = reinterpret_cast<float*>(smem + kOffAlpha);
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* mbar = wbar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wbar + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int nkc = (d + BK - 1) / BK;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(wbar, 1);
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < BN; i += kThreads) beta_s[i] = (n0 + i < r) ? beta2[n0 + i] : 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  // idesc: D=f32, A=B=tf32, K-major both, N = 256, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(BM >> 4) << 24);

  // X chunk loader: thread t -> row t/2, k-half t%2 (16 consecutive k)
  const int xrow = tid >> 1, xk0 = (tid & 1) * 16;
  const int64_t grow = m0 + xrow;
  float xx = 0.f;

  for (int kc = 0; kc < nkc; ++kc) {
    // global loads for this chunk (overlap the previous chunk's MMAs)
    float v[16];
    const int cb = kc * BK + xk0;
    if ((d & 3) == 0 && grow < M && cb + 16 <= d) {   // 16-byte vector loads
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 t4 = __ldg(reinterpret_cast<const float4*>(X + grow * d + cb) + q);
        v[4 * q] = t4.x; v[4 * q + 1] = t4.y; v[4 * q + 2] = t4.z; v[4 * q + 3] = t4.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = (grow < M && cb + i < d) ? __ldg(X + grow * d + cb + i) : 0.f;
    }
    if (kc > 0) mbar_wait(mbar, (uint32_t)((kc - 1) & 1));   // previous MMAs done: buffers free
    if (tid == 0) {
      mbar_arrive_expect_tx(wbar, 2 * kWBytes);
      const char* src = reinterpret_cast<const char*>(wimg) +
                        ((size_t)blockIdx.y * nkc + kc) * 2 * kWBytes;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sbase + kOffWhi),
          "l"(src), "r"(2 * kWBytes), "r"(smem_u32(wbar))
          : "memory");
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 hi, lo;
      float* h = &hi.x;
      float* l = &lo.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = v[q * 4 + e];
        xx = fmaf(x, x, xx);
        h[e] = tf32_rna(x);
        l[e] = tf32_rna(x - h[e]);
      }
      const uint32_t off = swz128(xrow, xk0 + q * 4);
      *reinterpret_cast<float4*>(smem + kOffXhi + off) = hi;
      *reinterpret_cast<float4*>(smem + kOffXlo + off) = lo;
    }
    fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
    __syncthreads();
    if (tid == 0) {
      mbar_wait(wbar, (uint32_t)(kc & 1));
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t axh = umma_desc_sw128(sbase + kOffXhi + kk * 32);
        const uint64_t axl = umma_desc_sw128(sbase + kOffXlo + kk * 32);
        const uint64_t bwh = umma_desc_sw128(sbase + kOffWhi + kk * 32);
        const uint64_t bwl = umma_desc_sw128(sbase + kOffWlo + kk * 32);
        const uint32_t acc0 = (kc > 0 || kk > 0) ? 1u : 0u;
        mma_tf32(tmem, axh, bwh, idesc, acc0);
        mma_tf32(tmem, axh, bwl, idesc, 1u);
        mma_tf32(tmem, axl, bwh, idesc, 1u);
      }
      mma_commit(mbar);
    }
  }
  // alpha2 of each row: the two half-row partials of |x|^2
  xx += __shfl_xor_sync(0xffffffffu, xx, 1);
  if ((tid & 1) == 0) alpha_s[xrow] = c2 * xx;
  mbar_wait(mbar, (uint32_t)((nkc - 1) & 1));
  tc_fence_after();
  __syncthreads();

  // epilogue: warp w -> TMEM lanes 32(w%4).., columns 128(w/4) .. +128
  const int q4 = warp & 3, half = warp >> 2;
  const int row = q4 * 32 + lane;
  const int64_t orow = m0 + row;
  const float al = alpha_s[row];
  // two 32-column TMEM loads in flight per wait (the epilogue was TMEM-latency bound)
#pragma unroll 1
  for (int cp = 0; cp < 4; cp += 2) {
    uint32_t a[2][32];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int col = half * 128 + (cp + h2) * 32;
      const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)col;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(a[h2][0]), "=r"(a[h2][1]), "=r"(a[h2][2]), "=r"(a[h2][3]), "=r"(a[h2][4]),
            "=r"(a[h2][5]), "=r"(a[h2][6]), "=r"(a[h2][7]), "=r"(a[h2][8]), "=r"(a[h2][9]),
            "=r"(a[h2][10]), "=r"(a[h2][11]), "=r"(a[h2][12]), "=r"(a[h2][13]), "=r"(a[h2][14]),
            "=r"(a[h2][15]), "=r"(a[h2][16]), "=r"(a[h2][17]), "=r"(a[h2][18]), "=r"(a[h2][19]),
            "=r"(a[h2][20]), "=r"(a[h2][21]), "=r"(a[h2][22]), "=r"(a[h2][23]), "=r"(a[h2][24]),
            "=r"(a[h2][25]), "=r"(a[h2][26]), "=r"(a[h2][27]), "=r"(a[h2][28]), "=r"(a[h2][29]),
            "=r"(a[h2][30]), "=r"(a[h2][31])
          : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (orow < M) {
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int col = half * 128 + (cp + h2) * 32;
        float* dst = Xi + orow * ld + n0 + col;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          if (n0 + col + j < r) {
            float o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float acc = __uint_as_float(a[h2][j + e]);
              if (mode == 0) {
                o[e] = ex2(al + beta_s[col + j + e] + acc);
              } else {
                const float rl = fmaxf(acc, 0.f);
                o[e] = beta_s[col + j + e] * (sdeg == 0 ? (acc > 0.f ? 1.f : 0.f) : (sdeg == 1 ? rl : rl * rl));
              }
            }
            st_global_cs(reinterpret_cast<float4*>(dst + j), make_float4(o[0], o[1], o[2], o[3]));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN)
                 : "memory");
  }
}

}  // namespace tc

// ============================================================================================
// Persistent, warp-specialised version (round 2; d <= 128): the CTA keeps ONE 128-anchor block
// of the W hi/lo images resident in shared memory (the A operand, loaded once) and streams
// 128-row tiles of X through a 2-slot ring (the B operand):
//   warps 0-3  (loaders)  X chunk (128 rows x 32 k) -> hi/lo split -> SW128 images, |x|^2;
//   warp 4..7  (epilogue) TMEM accumulator -> 2^(alpha_i + beta2_k + G) (or the arc-cosine
//                          form) -> fp32 stores, one per register across the 32 lanes = 128
//                          contiguous bytes of a row (the anchors are the MMA's M, on the TMEM
//                          lanes; the rows are its N, on the columns);
//   warp 8     (MMA)      one elected thread: 3 x 4 tcgen05.mma (128 x 128 x 8) per chunk into a
//                          double-buffered TMEM accumulator; tcgen05.commit frees the X slot
//                          and, after the last chunk, hands the buffer to the epilogue.
// CTA c serves anchor block c % NTN and row tiles c / NTN, c / NTN + G, ... (G = grid / NTN):
// the NTN CTAs of a row tile run side by side, so X comes from HBM once and from L2 after.
namespace tc2 {
using tc::swz128;
using tc::tf32_rna;
using tc::umma_desc_sw128;
using tc::mma_tf32;
using tc::mma_commit;
using tc::tc_fence_after;
using tc::tc_fence_before;


constexpr int BM = 128;             // anchors per CTA (MMA M)
constexpr int BNR = 128;            // rows per tile (MMA N)
constexpr int BK = 32;              // k per loader sub-chunk (the tf32 chunk)
constexpr int kImg = 128 * 128;     // bytes of one 128-row x 128-byte image (16 KB)
constexpr int LW = 8;               // loader warps
constexpr int NL = LW * 32;         // loader threads
constexpr int JR = 1024 / NL;       // 16-byte quads per loader thread per sub-chunk

// Operand precision: H = false: 3xTF32 (hi/lo = cvt.rna.tf32), 32 k per 128-byte chunk row;
// H = true: 3xFP16 on kind::f16 (twice the tf32 MMA rate, the same 11-bit significands), 64 k
// per chunk row, operands pre-scaled by powers of two (x 2^sx from R, W 2^sw from max |W|) so
// that they stay inside the fp16 range and the lo parts stay normal; the epilogue multiplies
// the fp32 accumulator by 2^-(sx+sw) (exact).  The fp16 W images are half the size, so an fp16
// CTA keeps TWO 128-anchor blocks resident (MB = 2: 256 anchors, two MMAs per k-step, all 512
// TMEM columns): every X tile it loads feeds twice the MMA work, and half as many CTAs load
// each X tile.
template <bool H>
struct Cfg {
  static constexpr int MB = H ? 2 : 1;            // 128-anchor blocks per CTA
  static constexpr int SUB = H ? 2 : 1;           // loader sub-chunks per MMA chunk
  static constexpr int kMaxChunks = H ? 2 : 4;    // d <= 128
  static constexpr int kSlots = H ? 3 : 2;
  static constexpr int kAlphaRing = H ? 3 : 4;
  // smem: W images [MB][nkc][2][kImg] | X slots [kSlots][2][kImg] | alpha [kAlphaRing][BNR] | bars
  static constexpr int kOffW = 0;
  static constexpr int kOffX = kOffW + MB * kMaxChunks * 2 * kImg;
  static constexpr int kOffAlpha = kOffX + kSlots * 2 * kImg;
  static constexpr int kOffBar = kOffAlpha + kAlphaRing * BNR * 4;
  static constexpr int kSmemBytes = kOffBar + 256 + 1024;   // + alignment slack
  // D = f32; A = B = tf32 (2) or f16 (0); both K-major; N = BNR, M = BM
  static constexpr uint32_t kIdesc = (1u << 4) | ((H ? 0u : 2u) << 7) | ((H ? 0u : 2u) << 10) |
                                     ((uint32_t)(BNR >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static constexpr int EW = 4 * MB;                // epilogue warps: one per (lane quarter, block)
  static constexpr int kThreads = (LW + EW + 1) * 32;   // loaders, epilogue, 1 MMA warp
};
static_assert(Cfg<true>::kSmemBytes <= 232448 && Cfg<false>::kSmemBytes <= 232448, "smem");

// byte offset of fp16 element (row, k) inside a K-major SWIZZLE_128B image (64 k per row)
__host__ __device__ __forceinline__ uint32_t swz128h(int row, int k) {
  const uint32_t chunk = (uint32_t)(k >> 3) ^ (uint32_t)(row & 7);
  return (uint32_t)row * 128u + chunk * 16u + (uint32_t)(k & 7) * 2u;
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// max |v| over n floats (non-negative float bits order as unsigned integers)
__global__ void absmax_kernel(const float* __restrict__ v, int64_t n, unsigned int* out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(v[i]));
  for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// fp16 W hi/lo images: [nt][kc][2][128 rows x 64 k x 2 B swizzled], W' = sc U 2^sw with
// max |W'| ~ 2^14; block (0, 0) publishes the epilogue factor 2^-(sx + sw)
__global__ void w_images_h_kernel(const float* __restrict__ U, int r, int d, double sc,
                                  const unsigned int* __restrict__ amax, int sx,
                                  float* __restrict__ img, float* __restrict__ fscale) {
  const int nt = blockIdx.x, kc = blockIdx.y;
  const int nkc = gridDim.y;
  const double wmax = sc * (double)__uint_as_float(*amax);
  const int sw = wmax > 0.0 ? max(-60, min(60, 14 - (int)ceil(log2(wmax)))) : 0;
  const double s2 = sc * ldexp(1.0, sw);
  char* base = reinterpret_cast<char*>(img) + ((size_t)nt * nkc + kc) * 2 * kImg;
  for (int i = threadIdx.x; i < BM * 64; i += blockDim.x) {
    const int row = i / 64, k = i % 64;
    const int n = nt * BM + row, c = kc * 64 + k;
    const float w = (n < r && c < d) ? (float)(s2 * (double)U[(int64_t)n * d + c]) : 0.f;
    const __half hi = __float2half_rn(w);
    const __half lo = __float2half_rn(w - __half2float(hi));
    *reinterpret_cast<__half*>(base + swz128h(row, k)) = hi;
    *reinterpret_cast<__half*>(base + kImg + swz128h(row, k)) = lo;
  }
  if (nt == 0 && kc == 0 && threadIdx.x == 0) *fscale = (float)ldexp(1.0, -(sx + sw));
}

// W hi/lo images for 128-anchor blocks: [nt][kc][2][128 rows x 128 B swizzled]
__global__ void w_images_kernel(const float* __restrict__ U, int r, int d, double sc,
                                float* __restrict__ img) {
  const int nt = blockIdx.x, kc = blockIdx.y;
  const int nkc = gridDim.y;
  char* base = reinterpret_cast<char*>(img) + ((size_t)nt * nkc + kc) * 2 * kImg;
  for (int i = threadIdx.x; i < BM * BK; i += blockDim.x) {
    const int row = i / BK, k = i % BK;
    const int n = nt * BM + row, c = kc * BK + k;
    const float w = (n < r && c < d) ? (float)(sc * (double)U[(int64_t)n * d + c]) : 0.f;
    const float hi = tf32_rna(w);
    const float lo = tf32_rna(w - hi);
    *reinterpret_cast<float*>(base + swz128(row, k)) = hi;
    *reinterpret_cast<float*>(base + kImg + swz128(row, k)) = lo;
  }
}

template <int MODE, bool H>   // MODE 0: Gaussian 2^(alpha + beta2 + G); 1: arc-cosine beta2 relu(G)^sdeg
__global__ void __launch_bounds__(Cfg<H>::kThreads, 1) feature_map_kernel(
    const float* __restrict__ X, int64_t M, int d, const float* __restrict__ wimg,
    const float* __restrict__ beta2, int r, float c2, float* __restrict__ Xi, int ld, int sdeg,
    const float* __restrict__ fscale, float xscale) {
  using C = Cfg<H>;
  constexpr int kSlots = C::kSlots, kOffW = C::kOffW, kOffX = C::kOffX;
  constexpr int kOffAlpha = C::kOffAlpha, kOffBar = C::kOffBar;
  constexpr int MB = C::MB, kAlphaRing = C::kAlphaRing, EW = C::EW;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* alpha_s = reinterpret_cast<float*>(smem + kOffAlpha);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wbar = bars;                  // W images landed
  uint64_t* xfull = bars + 1;             // [kSlots] X chunk written (128 loader arrivals)
  uint64_t* xempty = bars + 1 + kSlots;   // [kSlots] X chunk consumed (tcgen05.commit)
  uint64_t* tfull = bars + 1 + 2 * kSlots;       // [2] accumulator ready (tcgen05.commit)
  uint64_t* tempty = bars + 3 + 2 * kSlots;      // [2] accumulator drained (128 epilogue arrivals)
  uint64_t* abar = bars + 5 + 2 * kSlots;        // [kAlphaRing] alpha of a tile written (128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5 + 2 * kSlots + kAlphaRing);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntn = (r + MB * BM - 1) / (MB * BM);
  const int groups = gridDim.x / ntn;
  const int nt = blockIdx.x % ntn, grp = blockIdx.x / ntn;
  const int nkc = (d + BK * C::SUB - 1) / (BK * C::SUB);   // MMA chunks (128-byte rows)
  const int nsc = nkc * C::SUB;                             // loader sub-chunks per tile
  const int64_t mtiles = (M + BNR - 1) / BNR;
  const int n0 = nt * MB * BM;

  if (warp == LW + EW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(2 * MB * BNR)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(wbar, 1);
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(xfull + i, NL);
      mbar_init(xempty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 32 * EW);
    }
    for (int i = 0; i < kAlphaRing; ++i) mbar_init(abar + i, NL);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);

  if (warp < LW) {
    // ------------------------------ loaders ---------------------------------------------
    if (tid == 0) {   // this CTA's anchor block of the W images, once
      const uint32_t bytes = (uint32_t)(MB * nkc) * 2u * kImg;
      mbar_arrive_expect_tx(wbar, bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sbase + kOffW),
          "l"(reinterpret_cast<const char*>(wimg) + (size_t)nt * MB * nkc * 2 * kImg), "r"(bytes),
          "r"(smem_u32(wbar))
          : "memory");
    }
    // thread t: 16-byte k-quad q = t % 8 of rows t / 8 + (NL / 8) j (j < JR) of the chunk
    const int q = tid & 7, rb = tid >> 3;
    constexpr int RS = NL / 8;   // row stride between a thread's quads
    const bool vec = (d & 3) == 0;
    // the chunks of this CTA's tiles as one sequence; the next chunk's global loads are in
    // flight (registers) while the current one is split and stored
    auto load_chunk = [&](int64_t mt, int kc, float4 (&v)[JR]) {
      const int64_t m0 = mt * BNR;
      const int c0 = kc * BK + 4 * q;
#pragma unroll
      for (int j = 0; j < JR; ++j) {
        const int64_t row = m0 + rb + RS * j;
        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < M) {
          const float* src = X + row * d + c0;
          if (vec && c0 + 4 <= d) {
            v[j] = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            float* e = &v[j].x;
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = (c0 + u < d) ? __ldg(src + u) : 0.f;
          }
        }
      }
    };
    uint32_t it = 0;   // chunks so far (slot it % kSlots)
    int ti = 0;        // tiles so far (alpha ring)
    int64_t mt = grp;
    int kc = 0;
    float xx[JR];
#pragma unroll
    for (int j = 0; j < JR; ++j) xx[j] = 0.f;
    // a 4-deep register queue: sub-chunks it+1 .. it+3 are in flight while sub-chunk it is split
    // (two cursors: the sub-chunk being split, and the next one to load)
    float4 q0[JR], q1[JR], q2[JR], q3[JR];
    auto advance = [&](int64_t& m, int& c) {
      if (++c == nsc) {
        c = 0;
        m += groups;
      }
    };
    int64_t mL = mt;
    int kL = kc;
    if (mL < mtiles) load_chunk(mL, kL, q0);
    advance(mL, kL);
    if (mL < mtiles) load_chunk(mL, kL, q1);
    advance(mL, kL);
    if (mL < mtiles) load_chunk(mL, kL, q2);
    advance(mL, kL);
    // the loop body rotates the queue's roles (no register copies, which would wait for the
    // loads just issued): step(split this, load into that)
    auto step = [&](float4 (&cu)[JR], float4 (&ld2)[JR]) {
      if (mL < mtiles) load_chunk(mL, kL, ld2);
      advance(mL, kL);
      const int slot = (int)(it % kSlots);
      const int sub = H ? (kc & 1) : 0;
      if (sub == 0 && it >= (uint32_t)kSlots) mbar_wait(xempty + slot, ((it / kSlots) - 1) & 1u);
      unsigned char* xs = smem + kOffX + slot * 2 * kImg;
#pragma unroll
      for (int j = 0; j < JR; ++j) {
        const float* e = &cu[j].x;
#pragma unroll
        for (int u = 0; u < 4; ++u) xx[j] = fmaf(e[u], e[u], xx[j]);
        if constexpr (H) {
          const float x0 = e[0] * xscale, x1 = e[1] * xscale, x2 = e[2] * xscale, x3 = e[3] * xscale;
          const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          const __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y);
          const __half2 l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
          const uint32_t off = swz128h(rb + RS * j, 32 * sub + 4 * q);
          *reinterpret_cast<uint2*>(xs + off) =
              make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
          *reinterpret_cast<uint2*>(xs + kImg + off) =
              make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
        } else {
          float4 hi, lo;
          float* h = &hi.x;
          float* l = &lo.x;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            h[u] = tf32_rna(e[u]);
            l[u] = tf32_rna(e[u] - h[u]);
          }
          const uint32_t off = swz128(rb + RS * j, 4 * q);
          *reinterpret_cast<float4*>(xs + off) = hi;
          *reinterpret_cast<float4*>(xs + kImg + off) = lo;
        }
      }
      if (sub == C::SUB - 1) {
        fence_proxy_async_smem();
        mbar_arrive(xfull + slot);
        ++it;
      }
      if (kc == nsc - 1) {
        // alpha_i = c2 |x_i|^2: the 8 k-quads of a row are 8 consecutive lanes
#pragma unroll
        for (int j = 0; j < JR; ++j) {
          float t = xx[j];
          t += __shfl_xor_sync(0xffffffffu, t, 1);
          t += __shfl_xor_sync(0xffffffffu, t, 2);
          t += __shfl_xor_sync(0xffffffffu, t, 4);
          if (q == 0) alpha_s[(ti % kAlphaRing) * BNR + rb + RS * j] = c2 * t;
          xx[j] = 0.f;
        }
        // ring entry ti % kAlphaRing is rewritten at tile ti + kAlphaRing; the loader finishes
        // that tile only after the MMAs of tile ti + kAlphaRing - 1 started, which follow the
        // epilogue's release of tile ti (issued after its last read of alpha)
        mbar_arrive(abar + (ti % kAlphaRing));
        ++ti;
      }
      advance(mt, kc);
    };
    while (mt < mtiles) {
      step(q0, q3);
      if (mt >= mtiles) break;
      step(q1, q0);
      if (mt >= mtiles) break;
      step(q2, q1);
      if (mt >= mtiles) break;
      step(q3, q2);
    }
  } else if (warp < LW + EW) {
    // ------------------------------ epilogue --------------------------------------------
    const int qd = warp & 3;                    // TMEM lane quarter = anchors 32 qd ..
    const int mb = (warp - LW) >> 2;            // this warp's 128-anchor block
    const int k = n0 + mb * BM + 32 * qd + lane;   // this thread's anchor
    const bool kvm = k < r;
    const float bkm = kvm ? beta2[k] : 0.f;
    const float fs = H ? __ldg(fscale) : 1.f;   // 2^-(sx + sw): the operands' pre-scaling
    int ti = 0;
    for (int64_t mt = grp; mt < mtiles; mt += groups, ++ti) {
      const int64_t m0 = mt * BNR;
      const int buf = ti & 1;
      mbar_wait(abar + (ti % kAlphaRing), (uint32_t)(ti / kAlphaRing) & 1u);   // alpha written
      mbar_wait(tfull + buf, (uint32_t)(ti >> 1) & 1u);
      tc_fence_after();
      const float* al = alpha_s + (ti % kAlphaRing) * BNR;
#pragma unroll 1
      for (int g = 0; g < BNR / 32; ++g) {
        uint32_t a[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)((buf * MB + mb) * BNR + 32 * g);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
              "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]),
              "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]),
              "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]),
              "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]),
              "=r"(a[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int64_t rg = m0 + 32 * g;
        float o[32];
        if (kvm) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 a4 = *reinterpret_cast<const float4*>(al + 32 * g + j);
            const float* ap = &a4.x;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float acc = H ? __uint_as_float(a[j + u]) * fs : __uint_as_float(a[j + u]);
              if (MODE == 0) {
                o[j + u] = ex2((ap[u] + bkm) + acc);
              } else {
                const float rl = fmaxf(acc, 0.f);
                o[j + u] = bkm * (sdeg == 0 ? (acc > 0.f ? 1.f : 0.f) : (sdeg == 1 ? rl : rl * rl));
              }
            }
          }
        }
        // the tile's accumulator and alpha have been read: the next tile's MMAs may start (and,
        // with them, the loader's reuse of this alpha entry)
        if (g == BNR / 32 - 1) {
          tc_fence_before();
          mbar_arrive(tempty + buf);
        }
        if (kvm) {
          // one 64-bit base per 32-row group; rows as 32-bit offsets (32 ld < 2^31); a lane's
          // store j and its neighbours' form 128 contiguous bytes of row rg + j
          float* dst = Xi + rg * ld + k;
          const int nrow = (M - rg) < 32 ? (int)(M - rg) : 32;
          if (nrow == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcs(dst + j * ld, o[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nrow) __stcs(dst + j * ld, o[j]);
          }
        }
      }
    }
  } else {
    // ------------------------------ MMA issuer ------------------------------------------
    if (lane == 0) {
      mbar_wait(wbar, 0);
      uint32_t it = 0;
      int ti = 0;
      for (int64_t mt = grp; mt < mtiles; mt += groups, ++ti) {
        const int buf = ti & 1;
        if (ti >= 2) mbar_wait(tempty + buf, (uint32_t)((ti >> 1) - 1) & 1u);
        tc_fence_after();
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int slot = (int)(it % kSlots);
          mbar_wait(xfull + slot, (it / kSlots) & 1u);
          tc_fence_after();
          const uint32_t xa = sbase + kOffX + slot * 2 * kImg;
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) {
            const uint32_t dcol = tmem + (uint32_t)((buf * MB + mb) * BNR);
            const uint32_t wa = sbase + kOffW + (mb * nkc + kc) * 2 * kImg;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {   // 4 MMA k-steps of 32 bytes per 128-byte row
              const uint64_t awh = umma_desc_sw128(wa + kk * 32);
              const uint64_t awl = umma_desc_sw128(wa + kImg + kk * 32);
              const uint64_t bxh = umma_desc_sw128(xa + kk * 32);
              const uint64_t bxl = umma_desc_sw128(xa + kImg + kk * 32);
              const uint32_t acc0 = (kc > 0 || kk > 0) ? 1u : 0u;
              if constexpr (H) {
                mma_f16(dcol, awh, bxh, C::kIdesc, acc0);
                mma_f16(dcol, awl, bxh, C::kIdesc, 1u);
                mma_f16(dcol, awh, bxl, C::kIdesc, 1u);
              } else {
                mma_tf32(dcol, awh, bxh, C::kIdesc, acc0);
                mma_tf32(dcol, awl, bxh, C::kIdesc, 1u);
                mma_tf32(dcol, awh, bxl, C::kIdesc, 1u);
              }
            }
          }
          mma_commit(xempty + slot);   // the slot is free once these MMAs have read it
        }
        mma_commit(tfull + buf);
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == LW + EW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * MB * BNR)
                 : "memory");
  }
}

}  // namespace tc2

size_t feature_map_tc_image_bytes(int r, int d) {
  const int nt = (r + tc::BN - 1) / tc::BN, nkc = (d + tc::BK - 1) / tc::BK;
  const int nt2 = (r + tc2::BM - 1) / tc2::BM + 1;   // + 1: the fp16 path pads to pairs of blocks
  // + 256 bytes: the fp16 path's max |U| and epilogue factor
  return std::max((size_t)nt * nkc * 2 * tc::kWBytes, (size_t)nt2 * nkc * 2 * tc2::kImg) + 256;
}

static int g_tc2_grid = 0;   // persistent grid (SM count), queried once

template <int MODE, bool H>
static cudaError_t launch_tc2(const float* X, int64_t n, int d, const float* wimg,
                              const float* beta2, int r, float c2, float* Xi, int ld, int sdeg,
                              const float* fscale, float xscale, cudaStream_t s) {
  auto kern = tc2::feature_map_kernel<MODE, H>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tc2::Cfg<H>::kSmemBytes);
  if (e != cudaSuccess) return e;
  if (g_tc2_grid == 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_tc2_grid = sms;
  }
  const int ntn = (r + tc2::Cfg<H>::MB * tc2::BM - 1) / (tc2::Cfg<H>::MB * tc2::BM);
  const int64_t mtiles = (n + tc2::BNR - 1) / tc2::BNR;
  int groups = std::max(1, g_tc2_grid / ntn);
  groups = (int)std::min<int64_t>(groups, mtiles);
  kern<<<groups * ntn, tc2::Cfg<H>::kThreads, tc2::Cfg<H>::kSmemBytes, s>>>(X, n, d, wimg, beta2, r, c2, Xi,
                                                                     ld, sdeg, fscale, xscale);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_feature_map_tc(const float* X, int64_t n, int d, const float* U,
                                  const float* beta2, int r, double eps, float* wimg, float* Xi,
                                  cudaStream_t s, int mode, int sdeg, int ld, double R) {
  if (n <= 0) return cudaSuccess;
  if (ld <= 0) ld = r;
  const int nt = (r + tc::BN - 1) / tc::BN, nkc = (d + tc::BK - 1) / tc::BK;
  const double wscale = mode == 0 ? 4.0 * tc::kLog2e / eps : 1.0;
  const float c2 = (float)(-2.0 * tc::kLog2e / eps);
  const int nt2 = (r + tc2::BM - 1) / tc2::BM;
  if (mode == 0 && R > 0.0 && d <= 64 * tc2::Cfg<true>::kMaxChunks) {
    // 3xFP16 (kind::f16): x scaled by 2^sx so that |x'| <= 2^12 for |x| <= 16 R
    const int sx = std::max(-60, std::min(60, 12 - (int)std::ceil(std::log2(R))));
    const int nkh = (d + 63) / 64;
    const int nt2p = (nt2 + 1) & ~1;   // pairs of 128-anchor blocks (the pad block is zero)
    char* scal = reinterpret_cast<char*>(wimg) + (size_t)nt2p * nkh * 2 * tc2::kImg;
    unsigned int* amax = reinterpret_cast<unsigned int*>(scal);
    float* fscale = reinterpret_cast<float*>(scal + 128);
    cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    tc2::absmax_kernel<<<64, 256, 0, s>>>(U, (int64_t)r * d, amax);
    count_launch();
    tc2::w_images_h_kernel<<<dim3(nt2p, nkh), 256, 0, s>>>(U, r, d, wscale, amax, sx, wimg, fscale);
    count_launch();
    return launch_tc2<0, true>(X, n, d, wimg, beta2, r, c2, Xi, ld, sdeg, fscale,
                               (float)std::ldexp(1.0, sx), s);
  }
  if (nkc <= tc2::Cfg<false>::kMaxChunks) {   // 3xTF32, W block resident
    tc2::w_images_kernel<<<dim3(nt2, nkc), 256, 0, s>>>(U, r, d, wscale, wimg);
    count_launch();
    return mode == 0 ? launch_tc2<0, false>(X, n, d, wimg, beta2, r, c2, Xi, ld, sdeg, nullptr, 1.f, s)
                     : launch_tc2<1, false>(X, n, d, wimg, beta2, r, c2, Xi, ld, sdeg, nullptr, 1.f, s);
  }
  tc::w_images_kernel<<<dim3(nt, nkc), 256, 0, s>>>(U, r, d, wscale, wimg);
  count_launch();
  cudaError_t e = cudaFuncSetAttribute(tc::feature_map_tc_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((n + tc::BM - 1) / tc::BM), (unsigned)nt);
  tc::feature_map_tc_kernel<<<grid, tc::kThreads, tc::kSmemBytes, s>>>(X, n, d, wimg, beta2, r, c2, Xi,
                                                                        ld, mode, sdeg);
  count_launch();
  return cudaGetLastError();
}

}  // namespace lsk
