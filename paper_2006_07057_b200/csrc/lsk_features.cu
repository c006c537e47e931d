// lsk_features.cu — steps a1 (auto R), a2 (anchors), a3 (feature map) and a9 (read-out).
//
//  a1  R = max(|x_i|, |y_j|) in fp64 (reading C3)                      — max_sqnorm_kernel
//  a2  u_k ~ N(0, sigma^2 I): Philox4x32-10 + fp64 Box-Muller (C5)        — anchors_kernel
//  a3  xi_ik = exp(-(2/eps)|x_i-u_k|^2 + |u_k|^2/(eps q) + log_scale)     — feature_map_*
//      (Lemma decomp-RBF appendix form, 1/sqrt(r) of PAPER.md:297 folded into
//      log_scale).  Computed in base 2 with one MUFU ex2 per entry.  d <= 16: direct
//      difference form on FFMA (no cancellation); d > 16: expanded form
//      |x|^2 + |u|^2 - 2 x.u with the x.u contraction register-tiled through shared memory.
//  a9  a^T log u and b^T log v in fp64, fixed-order two-stage reduction   — rot_partial_kernel
#include <cmath>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"

namespace lsk {

constexpr double kLog2e = 1.4426950408889634074;

// ---------------------------------------------------------------- a1: max squared norm ---
__global__ void max_sqnorm_kernel(const float* __restrict__ X, int64_t n, int d,
                                  unsigned long long* out) {
  double best = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
      const double v = (double)X[i * d + c];
      s += v * v;
    }
    best = fmax(best, s);
  }
  for (int off = 16; off >= 1; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

cudaError_t launch_max_sqnorm(const float* X, int64_t n, int d, unsigned long long* out,
                              cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  max_sqnorm_kernel<<<blocks, 256, 0, s>>>(X, n, d, out);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- a2: anchors ------------
__device__ __forceinline__ uint4 philox_round(uint4 c, uint2 k) {
  const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
  const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
  return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
}
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    if (i > 0) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    c = philox_round(c, k);
  }
  return c;
}

// one thread per (anchor k, block p of 4 coordinates)
__global__ void anchors_kernel(uint64_t seed, int r, int d, double sigma, float* U,
                               uint32_t* words) {
  const int P = (d + 3) / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= r * P) return;
  const int k = idx / P, p = idx - k * P;
  const uint2 key = make_uint2((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  const uint4 w = philox4x32_10(make_uint4((uint32_t)k, (uint32_t)p, 0u, 0u), key);
  if (words) {
    uint32_t* o = words + (int64_t)idx * 4;
    o[0] = w.x; o[1] = w.y; o[2] = w.z; o[3] = w.w;
  }
  if (U) {
    const double two32 = 4294967296.0;
    const double u1a = ((double)w.x + 1.0) / two32, u2a = (double)w.y / two32;
    const double u1b = ((double)w.z + 1.0) / two32, u2b = (double)w.w / two32;
    const double ra = sqrt(-2.0 * log(u1a)), rb = sqrt(-2.0 * log(u1b));
    const double twopi = 2.0 * 3.14159265358979323846;
    const double z[4] = {ra * cos(twopi * u2a), ra * sin(twopi * u2a), rb * cos(twopi * u2b),
                         rb * sin(twopi * u2b)};
    for (int j = 0; j < 4; ++j) {
      const int c = 4 * p + j;
      if (c < d) U[(int64_t)k * d + c] = (float)(sigma * z[j]);
    }
  }
}

cudaError_t launch_anchors(uint64_t seed, int r, int d, double sigma, float* U, uint32_t* words,
                           cudaStream_t s) {
  const int P = (d + 3) / 4;
  const int total = r * P;
  anchors_kernel<<<(total + 127) / 128, 128, 0, s>>>(seed, r, d, sigma, U, words);
  count_launch();
  return cudaGetLastError();
}

// Per-anchor constants (fp64 from the stored fp32 anchors, rounded once to fp32):
//   Wt[c][k]  = (4 log2e / eps) U_kc                               (expanded cross term)
//   beta2[k]  = log2e (-(2/eps)|U_k|^2 + |U_k|^2/(eps q) + log_scale) (expanded form)
//   betaD[k]  = log2e (|U_k|^2/(eps q) + log_scale)                   (direct form)
__global__ void anchor_prep_kernel(const float* __restrict__ U, int r, int d, double eps,
                                   double q, double log_scale, float* Wt, float* beta2,
                                   float* betaD) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= r) return;
  double uu = 0.0;
  for (int c = 0; c < d; ++c) {
    const double v = (double)U[(int64_t)k * d + c];
    uu += v * v;
    if (Wt) Wt[(int64_t)c * r + k] = (float)(4.0 * kLog2e / eps * v);
  }
  if (beta2) beta2[k] = (float)(kLog2e * (-2.0 / eps * uu + uu / (eps * q) + log_scale));
  if (betaD) betaD[k] = (float)(kLog2e * (uu / (eps * q) + log_scale));
}

cudaError_t launch_anchor_prep(const float* U, int r, int d, double eps, double q,
                               double log_scale, float* Wt, float* beta2, float* betaD,
                               cudaStream_t s) {
  anchor_prep_kernel<<<(r + 127) / 128, 128, 0, s>>>(U, r, d, eps, q, log_scale, Wt, beta2, betaD);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- a3: feature map --------
// d <= 16, direct form: e2 = betaD_k + c2 * sum_c (x_ic - U_kc)^2, xi = 2^e2.
// Block = 256 threads x RB rows (32 for d < 8, where the kernel is write-bound; 128 for d >= 8,
// where the anchor loads per column group are amortised over more rows); thread t owns float4
// column groups t, t+256, ...  The next row's coordinates are read from shared memory while
// the current row is computed (one row ahead, in registers).
#ifndef LSK_DIRECT_RB
#define LSK_DIRECT_RB 128
#endif
#ifndef LSK_DIRECT_UNROLL
#define LSK_DIRECT_UNROLL 1
#endif
template <int D> struct DirectRows { static constexpr int value = D >= 8 ? LSK_DIRECT_RB : 32; };

template <int D>
__global__ void __launch_bounds__(256) feature_map_direct_kernel(
    const float* __restrict__ X, int64_t n, const float* __restrict__ U,
    const float* __restrict__ betaD, int r, float c2, float* __restrict__ Xi) {
  constexpr int RB = DirectRows<D>::value;
  __shared__ __align__(16) float xs[RB + 1][D];   // row RB: zero pad read by the look-ahead
  const int64_t row0 = (int64_t)blockIdx.x * RB;
  const int rows = (int)min((int64_t)RB, n - row0);
  for (int i = threadIdx.x; i < (RB + 1) * D; i += blockDim.x)
    xs[i / D][i % D] = i < rows * D ? X[row0 * D + i] : 0.f;
  __syncthreads();
  const int R4 = r >> 2;
  for (int g = threadIdx.x; g < R4; g += blockDim.x) {
    float u[4][D];
    if constexpr (D % 4 == 0) {
      const float4* U4 = reinterpret_cast<const float4*>(U + (int64_t)4 * g * D);   // 4 rows of U
#pragma unroll
      for (int j = 0; j < D; ++j) {   // 4 * D floats = D float4
        const float4 t = U4[j];
        u[(4 * j) / D][(4 * j) % D] = t.x;
        u[(4 * j) / D][(4 * j) % D + 1] = t.y;
        u[(4 * j) / D][(4 * j) % D + 2] = t.z;
        u[(4 * j) / D][(4 * j) % D + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < D; ++c) u[q][c] = U[(int64_t)(4 * g + q) * D + c];
    }
    const float4 bd = *reinterpret_cast<const float4*>(betaD + 4 * g);
    const float bq[4] = {bd.x, bd.y, bd.z, bd.w};
    float xc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) xc[c] = xs[0][c];
    constexpr int kUnroll = LSK_DIRECT_UNROLL;
#pragma unroll kUnroll
    for (int i = 0; i < rows; ++i) {
      float xn[D];
#pragma unroll
      for (int c = 0; c < D; ++c) xn[c] = xs[i + 1][c];
      float o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float sq = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float df = xc[c] - u[q][c];
          sq = fmaf(df, df, sq);
        }
        o[q] = ex2(fmaf(c2, sq, bq[q]));
      }
      st_global_cs(reinterpret_cast<float4*>(Xi + (row0 + i) * r) + g, make_float4(o[0], o[1], o[2], o[3]));
#pragma unroll
      for (int c = 0; c < D; ++c) xc[c] = xn[c];
    }
  }
}

// d > 16, expanded form: e2 = alpha2_i + beta2_k + sum_c Wt[c][k] x_ic with alpha2_i =
// c2 |x_i|^2.  Tile 64 rows x 128 columns, K-chunks of 32, thread tile 8 rows x 4 columns.
__global__ void __launch_bounds__(256) feature_map_tiled_kernel(
    const float* __restrict__ X, int64_t n, int d, const float* __restrict__ Wt,
    const float* __restrict__ beta2, int r, float c2, float* __restrict__ Xi) {
  constexpr int BM = 64, BN = 128, BK = 32;
  __shared__ __align__(16) float xs[BK][BM];
  __shared__ __align__(16) float ws[BK][BN];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int col0 = blockIdx.y * BN;
  float acc[8][4] = {};
  float xx[8] = {};
  for (int c0 = 0; c0 < d; c0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      const int rr = i / BK, cc = i % BK;
      const int64_t row = row0 + rr;
      xs[cc][rr] = (row < n && c0 + cc < d) ? X[row * d + c0 + cc] : 0.f;
    }
    for (int i = threadIdx.x; i < BK * BN; i += 256) {
      const int cc = i / BN, kk = i % BN;
      ws[cc][kk] = (c0 + cc < d && col0 + kk < r) ? Wt[(int64_t)(c0 + cc) * r + col0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < BK; ++cc) {
      const float4 xa = *reinterpret_cast<const float4*>(&xs[cc][ty * 8]);
      const float4 xb = *reinterpret_cast<const float4*>(&xs[cc][ty * 8 + 4]);
      const float4 w = *reinterpret_cast<const float4*>(&ws[cc][tx * 4]);
      const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[i][0] = fmaf(xv[i], w.x, acc[i][0]);
        acc[i][1] = fmaf(xv[i], w.y, acc[i][1]);
        acc[i][2] = fmaf(xv[i], w.z, acc[i][2]);
        acc[i][3] = fmaf(xv[i], w.w, acc[i][3]);
        xx[i] = fmaf(xv[i], xv[i], xx[i]);
      }
    }
    __syncthreads();
  }
  const int col = col0 + tx * 4;
  if (col >= r) return;
  const float4 b = *reinterpret_cast<const float4*>(beta2 + col);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = row0 + ty * 8 + i;
    if (row >= n) break;
    const float al = c2 * xx[i];
    const float4 o = make_float4(ex2(al + b.x + acc[i][0]), ex2(al + b.y + acc[i][1]),
                                 ex2(al + b.z + acc[i][2]), ex2(al + b.w + acc[i][3]));
    st_global_cs(reinterpret_cast<float4*>(Xi + row * r + col), o);
  }
}

cudaError_t launch_feature_map(const float* X, int64_t n, int d, const float* U,
                               const float* Wt, const float* beta2, const float* betaD, int r,
                               double eps, float* Xi, cudaStream_t s) {
  const float c2 = (float)(-2.0 * kLog2e / eps);
  if (n <= 0) return cudaSuccess;
  if (d <= 16) {
    switch (d) {
#define CASE(DD) case DD: feature_map_direct_kernel<DD><<<(unsigned)((n + DirectRows<DD>::value - 1) / DirectRows<DD>::value), 256, 0, s>>>(X, n, U, betaD, r, c2, Xi); break;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
      CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
      default: return cudaErrorInvalidValue;
    }
  } else {
    dim3 grid((unsigned)((n + 63) / 64), (unsigned)((r + 127) / 128));
    feature_map_tiled_kernel<<<grid, 256, 0, s>>>(X, n, d, Wt, beta2, r, c2, Xi);
  }
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- NEXT f4: stabilised ---
// Row-normalised features (reading C30): with e2_ik = betaD_k + c2 |x_i - U_k|^2 (log2 of
// phi/sqrt(r)), M_i = max_k e2_ik, write xi_tilde_ik = 2^(e2_ik - M_i) (every row's largest
// entry is 1: no row can underflow) and the natural-log offset A_i = M_i ln 2 (fp64).
// Block = 256 threads x 32 rows: pass 1 finds the 32 row maxima (registers, warp butterfly,
// then 8 warp values in smem), pass 2 recomputes the exponents and writes.
template <int D>
__global__ void __launch_bounds__(256) feature_map_stab_kernel(
    const float* __restrict__ X, int64_t n, const float* __restrict__ U,
    const float* __restrict__ betaD, int r, float c2, float* __restrict__ Xi,
    double* __restrict__ logoff) {
  constexpr int RB = 32;
  __shared__ float xs[RB][D];
  __shared__ float wmax[8][RB];
  __shared__ float rmax[RB];
  const int64_t row0 = (int64_t)blockIdx.x * RB;
  const int rows = (int)min((int64_t)RB, n - row0);
  for (int i = threadIdx.x; i < rows * D; i += blockDim.x) xs[i / D][i % D] = X[row0 * D + i];
  __syncthreads();
  const int R4 = r >> 2;
  float mx[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) mx[i] = -INFINITY;
  for (int g = threadIdx.x; g < R4; g += blockDim.x) {
    float u[4][D];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < D; ++c) u[q][c] = U[(int64_t)(4 * g + q) * D + c];
    const float4 bd = *reinterpret_cast<const float4*>(betaD + 4 * g);
    const float bq[4] = {bd.x, bd.y, bd.z, bd.w};
#pragma unroll
    for (int i = 0; i < RB; ++i) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float sq = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float df = xs[i][c] - u[q][c];
          sq = fmaf(df, df, sq);
        }
        mx[i] = fmaxf(mx[i], fmaf(c2, sq, bq[q]));
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    float v = mx[i];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) wmax[warp][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < RB) {
    float v = wmax[0][threadIdx.x];
    for (int w = 1; w < 8; ++w) v = fmaxf(v, wmax[w][threadIdx.x]);
    rmax[threadIdx.x] = v;
    if (threadIdx.x < rows) logoff[row0 + threadIdx.x] = (double)v * 0.69314718055994530942;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < R4; g += blockDim.x) {
    float u[4][D];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < D; ++c) u[q][c] = U[(int64_t)(4 * g + q) * D + c];
    const float4 bd = *reinterpret_cast<const float4*>(betaD + 4 * g);
    const float bq[4] = {bd.x, bd.y, bd.z, bd.w};
    for (int i = 0; i < rows; ++i) {
      float o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float sq = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float df = xs[i][c] - u[q][c];
          sq = fmaf(df, df, sq);
        }
        o[q] = ex2(fmaf(c2, sq, bq[q]) - rmax[i]);
      }
      st_global_cs(reinterpret_cast<float4*>(Xi + (row0 + i) * r) + g, make_float4(o[0], o[1], o[2], o[3]));
    }
  }
}

cudaError_t launch_feature_map_stab(const float* X, int64_t n, int d, const float* U,
                                    const float* betaD, int r, double eps, float* Xi,
                                    double* logoff, cudaStream_t s) {
  const float c2 = (float)(-2.0 * kLog2e / eps);
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)((n + 31) / 32);
  switch (d) {
#define CASE(DD) case DD: feature_map_stab_kernel<DD><<<blocks, 256, 0, s>>>(X, n, U, betaD, r, c2, Xi, logoff); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- NEXT f3: arc-cosine ---
// Xi[i][k] = coef_k relu(u_k . x_i)^s (k < r), Xi[i][r] = sqrt(kappa), Xi[i][r+1..r+3] = 0,
// coef_k = sigma^{d/2} sqrt(2) exp(-|u_k|^2/4 (1 - 1/sigma^2)) / sqrt(r).
__global__ void arccos_coef_kernel(const float* __restrict__ U, int r, int d, double sigma,
                                   float* coef) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= r) return;
  double uu = 0.0;
  for (int c = 0; c < d; ++c) {
    const double v = (double)U[(int64_t)k * d + c];
    uu += v * v;
  }
  coef[k] = (float)(pow(sigma, 0.5 * d) * sqrt(2.0) * exp(-uu / 4.0 * (1.0 - 1.0 / (sigma * sigma))) /
                    sqrt((double)r));
}

__device__ __forceinline__ float relu_pow(float t, int sdeg) {
  if (sdeg == 0) return t > 0.f ? 1.f : 0.f;
  const float rl = fmaxf(t, 0.f);
  return sdeg == 1 ? rl : rl * rl;
}

template <int D>
__global__ void __launch_bounds__(256) arccos_direct_kernel(
    const float* __restrict__ X, int64_t n, const float* __restrict__ U,
    const float* __restrict__ coef, int r, int sdeg, float sqrt_kappa, float* __restrict__ Xi) {
  constexpr int RB = 32;
  __shared__ float xs[RB][D];
  const int64_t row0 = (int64_t)blockIdx.x * RB;
  const int rows = (int)min((int64_t)RB, n - row0);
  for (int i = threadIdx.x; i < rows * D; i += blockDim.x) xs[i / D][i % D] = X[row0 * D + i];
  __syncthreads();
  const int ld = r + 4, R4 = r >> 2;
  for (int g = threadIdx.x; g <= R4; g += blockDim.x) {
    if (g == R4) {   // the collapsed kappa slot + zero padding
      for (int i = 0; i < rows; ++i)
        st_global_cs(reinterpret_cast<float4*>(Xi + (row0 + i) * ld) + g, make_float4(sqrt_kappa, 0.f, 0.f, 0.f));
      continue;
    }
    float u[4][D];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < D; ++c) u[q][c] = U[(int64_t)(4 * g + q) * D + c];
    const float4 cf = *reinterpret_cast<const float4*>(coef + 4 * g);
    const float cq[4] = {cf.x, cf.y, cf.z, cf.w};
    for (int i = 0; i < rows; ++i) {
      float o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float t = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) t = fmaf(u[q][c], xs[i][c], t);
        o[q] = cq[q] * relu_pow(t, sdeg);
      }
      st_global_cs(reinterpret_cast<float4*>(Xi + (row0 + i) * ld) + g, make_float4(o[0], o[1], o[2], o[3]));
    }
  }
}

__global__ void const_cols_kernel(float* Xi, int64_t n, int ld, int col, float val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n)
    *reinterpret_cast<float4*>(Xi + i * ld + col) = make_float4(val, 0.f, 0.f, 0.f);
}

cudaError_t launch_arccos_coef(const float* U, int r, int d, double sigma, float* coef,
                               cudaStream_t s) {
  arccos_coef_kernel<<<(r + 127) / 128, 128, 0, s>>>(U, r, d, sigma, coef);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_feature_map_arccos(const float* X, int64_t n, int d, const float* U,
                                      const float* coef, int r, int sdeg, double kappa,
                                      float* Xi, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)((n + 31) / 32);
  const float sk = (float)sqrt(kappa);
  switch (d) {
#define CASE(DD) case DD: arccos_direct_kernel<DD><<<blocks, 256, 0, s>>>(X, n, U, coef, r, sdeg, sk, Xi); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_const_cols(float* Xi, int64_t n, int ld, int col, float val, cudaStream_t s) {
  const_cols_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(Xi, n, ld, col, val);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- a9: read-out -----------
// partials[(prob * 2 + side) * B + blk] = sum over the block's fixed range of c ln w
constexpr int kRotBlocks = 64;
__global__ void rot_partial_kernel(const float* __restrict__ u, const float* __restrict__ v,
                                   const float* __restrict__ a, const float* __restrict__ b,
                                   int64_t n, int64_t m, double* partials,
                                   const double* __restrict__ offA,
                                   const double* __restrict__ offB) {
  const int prob = blockIdx.z, side = blockIdx.y, blk = blockIdx.x;
  const int64_t len = side == 0 ? n : m;
  const float* w = side == 0 ? u + prob * n : v + prob * m;
  const float* c = side == 0 ? a + prob * n : b + prob * m;
  const double* off = side == 0 ? offA : offB;   // stabilised read-out (C30): log u = log u~ - A
  const int64_t lo = len * blk / kRotBlocks, hi = len * (blk + 1) / kRotBlocks;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    acc += (double)c[i] * (log((double)w[i]) - (off ? off[prob * len + i] : 0.0));
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[((int64_t)prob * 2 + side) * kRotBlocks + blk] = sh[0];
}

__global__ void rot_final_kernel(const double* partials, int batch, double* out2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= batch * 2) return;
  double s = 0.0;
  for (int k = 0; k < kRotBlocks; ++k) s += partials[(int64_t)i * kRotBlocks + k];
  out2[i] = s;   // out2[prob*2 + side]
}

cudaError_t launch_rot_value(const float* u, const float* v, const float* a, const float* b,
                             int64_t n, int64_t m, int batch, double* partials, double* out2,
                             cudaStream_t s, const double* offA, const double* offB) {
  rot_partial_kernel<<<dim3(kRotBlocks, 2, batch), 256, 0, s>>>(u, v, a, b, n, m, partials,
                                                                 offA, offB);
  rot_final_kernel<<<(batch * 2 + 127) / 128, 128, 0, s>>>(partials, batch, out2);
  count_launch(2);
  return cudaGetLastError();
}

}  // namespace lsk
