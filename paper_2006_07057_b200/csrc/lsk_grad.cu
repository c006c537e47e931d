// lsk_grad.cu — NEXT row f2: envelope gradients of W_{eps,c_theta} (Prop. diff-gene,
// PAPER.md:402-412; chain rule PAPER.md:414-420) for the Gaussian positive features, at the
// scalings (u, v) returned by the solver, with the anchors theta = U and q held fixed.
//
//   dW/dK = -eps u v^T  =>  dW/dxi_ik = -eps u_i s_u,k,  dW/dzeta_jk = -eps v_j s_v,k,
//   s_u = zeta^T v, s_v = xi^T u (r-vectors, fp64), and with the map of PAPER.md:934:
//   grad_x_i = 4 u_i sum_k xi_ik s_u,k (x_i - U_k)                    (one row pass over xi)
//   grad_y_j = 4 v_j sum_k zeta_jk s_v,k (y_j - U_k)                  (one row pass over zeta)
//   grad_U_k = -4 (s_u,k B_x,k + s_v,k B_y,k) - (4/q) s_u,k s_v,k U_k,
//   B_x,k = sum_i u_i xi_ik (x_i - U_k),  B_y,k = sum_j v_j zeta_jk (y_j - U_k)
// The differences (x - U) are formed directly (no |x|^2 - 2x.U cancellation).  Every sum over
// rows is fp64 with fixed-order CTA partials (deterministic).  Linear in n+m; d <= 16.
#include <cmath>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"

namespace lsk {

constexpr int kGradMaxD = 16;
constexpr int kAccCtas = 296;   // two CTAs per SM

// Per-CTA partials over a row range: out[cta][k][0] = sum_i w_i F_ik,
// out[cta][k][1+c] = sum_i w_i F_ik (P_ic - U_kc) = sum_i w_i F_ik P_ic - U_kc out[cta][k][0].
// One warp per 4 rows; lane l holds float4 column groups {l, l+32, ...} of a chunk of JC
// groups (coalesced 512-byte loads, four rows in flight); fp32 sums per lane over <= 32 rows,
// flushed into per-warp fp64 sums in shared memory, then the 8 warps are added in a fixed
// order (deterministic).
template <int D, int JC>
__global__ void __launch_bounds__(256) grad_accum_kernel(const float* __restrict__ F, int64_t rows,
                                                         int r, const float* __restrict__ w,
                                                         const float* __restrict__ P,
                                                         const float* __restrict__ U,
                                                         double* __restrict__ part) {
  constexpr int NWP = 8;
  extern __shared__ double wsum[];   // [NWP][D + 1][JC * 4][32] fp64 warp partials of a chunk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = rows * blockIdx.x / gridDim.x, i1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int R4 = r >> 2;
  double* my = wsum + (int64_t)warp * (D + 1) * JC * 4 * 32;
  for (int g0 = 0; g0 < R4; g0 += 32 * JC) {
    float acc[D + 1][JC][4];
#pragma unroll
    for (int c = 0; c <= D; ++c)
#pragma unroll
      for (int j = 0; j < JC; ++j) acc[c][j][0] = acc[c][j][1] = acc[c][j][2] = acc[c][j][3] = 0.f;
    for (int e = lane; e < (D + 1) * JC * 4 * 32; e += 32) my[e] = 0.0;
    auto flush = [&]() {
#pragma unroll
      for (int c = 0; c <= D; ++c)
#pragma unroll
        for (int j = 0; j < JC; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            my[((c * JC + j) * 4 + e) * 32 + lane] += (double)acc[c][j][e];
            acc[c][j][e] = 0.f;
          }
    };
    int nit = 0;
    constexpr int RW = 4;   // rows in flight per warp
    for (int64_t i = i0 + RW * warp; i < i1; i += RW * NWP) {
      float4 f[RW][JC];
      float wp[RW][D + 1];
#pragma unroll
      for (int q = 0; q < RW; ++q) {
        const bool rv = i + q < i1;
        const float4* Fi = reinterpret_cast<const float4*>(F + (i + q) * r);
#pragma unroll
        for (int j = 0; j < JC; ++j) {
          const int gidx = g0 + lane + 32 * j;
          f[q][j] = (rv && gidx < R4) ? __ldcs(Fi + gidx) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const float wi = rv ? w[i + q] : 0.f;
        wp[q][0] = wi;
#pragma unroll
        for (int c = 0; c < D; ++c) wp[q][c + 1] = rv ? wi * P[(i + q) * D + c] : 0.f;
      }
#pragma unroll
      for (int q = 0; q < RW; ++q)
#pragma unroll
        for (int c = 0; c <= D; ++c)
#pragma unroll
          for (int j = 0; j < JC; ++j) {
            acc[c][j][0] = fmaf(f[q][j].x, wp[q][c], acc[c][j][0]);
            acc[c][j][1] = fmaf(f[q][j].y, wp[q][c], acc[c][j][1]);
            acc[c][j][2] = fmaf(f[q][j].z, wp[q][c], acc[c][j][2]);
            acc[c][j][3] = fmaf(f[q][j].w, wp[q][c], acc[c][j][3]);
          }
      if (++nit == 8) {   // <= 32 rows in fp32
        nit = 0;
        flush();
      }
    }
    flush();
    __syncthreads();
    // element (c, j, e, l) <-> column k = 4 (g0 + l + 32 j) + e
    for (int t = threadIdx.x; t < JC * 4 * 32; t += blockDim.x) {
      const int l = t & 31, je = t >> 5, j = je >> 2, e = je & 3;
      const int k = 4 * (g0 + l + 32 * j) + e;
      if (k >= r) continue;
      double sc[D + 1];
#pragma unroll
      for (int c = 0; c <= D; ++c) {
        double x = 0.0;
#pragma unroll
        for (int ww = 0; ww < NWP; ++ww)
          x += wsum[(int64_t)ww * (D + 1) * JC * 4 * 32 + ((c * JC + j) * 4 + e) * 32 + l];
        sc[c] = x;
      }
      double* o = part + ((int64_t)blockIdx.x * r + k) * (D + 1);
      o[0] = sc[0];
#pragma unroll
      for (int c = 0; c < D; ++c) o[1 + c] = sc[1 + c] - (double)U[(int64_t)k * D + c] * sc[0];
    }
    __syncthreads();
  }
}

// fixed-order reduction of the CTA partials: acc[k][j] = sum_cta part[cta][k][j]
// (block of 32 elements x 8 warps: warp w adds parts w, w+8, ... in order, then the 8 warp
// sums in order — deterministic and 8x the loads in flight of a thread-per-element loop).
// blockIdx.y selects the factor: the partial arrays of xi and zeta are contiguous, and so are
// their sums (one launch for both).
__global__ void __launch_bounds__(256) grad_reduce_kernel(const double* __restrict__ part,
                                                          int nparts, int64_t len,
                                                          double* __restrict__ acc) {
  part += (int64_t)blockIdx.y * nparts * len;
  acc += (int64_t)blockIdx.y * len;
  __shared__ double red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < len)
    for (int p = warp; p < nparts; p += 8) s += part[(int64_t)p * len + e];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < len) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    acc[e] = t;
  }
}

// grad_p_i = 4 w_i sum_k F_ik s_k (p_i - U_k) = 4 w_i (p_i t_i - sum_k F_ik s_k U_k) with
// t_i = F_i . s: d+1 dots of the row with fixed r-vectors (s and s o U_c), staged once per CTA
// in shared memory as fp32 (k-major float4 groups).  One warp per 4 rows: lane l reads the
// float4 column groups {l, l+32, ...} of all four (coalesced), then a warp butterfly.
template <int D, int NV>
__global__ void __launch_bounds__(256) grad_rows_kernel(const float* __restrict__ F, int64_t rows,
                                                        int r, const float* __restrict__ w,
                                                        const float* __restrict__ P,
                                                        const float* __restrict__ U,
                                                        const double* __restrict__ sacc,
                                                        float* __restrict__ g) {
  extern __shared__ float4 vsm[];   // [D + 1][NV * 32]: s, then s o U_c
  const int R4 = r >> 2;
  for (int e = threadIdx.x; e < NV * 32; e += blockDim.x) {
    float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f);
    float vc[D][4] = {};
    float* pv0 = &v0.x;
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * e + q;
      if (e < R4) {
        const double sk = sacc[(int64_t)k * (D + 1)];
        pv0[q] = (float)sk;
#pragma unroll
        for (int c = 0; c < D; ++c) vc[c][q] = (float)(sk * (double)U[(int64_t)k * D + c]);
      }
    }
    vsm[e] = v0;
#pragma unroll
    for (int c = 0; c < D; ++c) vsm[(c + 1) * NV * 32 + e] = make_float4(vc[c][0], vc[c][1], vc[c][2], vc[c][3]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  constexpr int JC = NV < 4 ? NV : 4;   // column groups in registers at a time (per row)
  constexpr int RW = 4;                  // rows in flight per warp
  for (int64_t i = RW * warp; i < rows; i += RW * nwarps) {
    float acc2[RW][D + 1];
#pragma unroll
    for (int q = 0; q < RW; ++q)
#pragma unroll
      for (int c = 0; c <= D; ++c) acc2[q][c] = 0.f;
#pragma unroll 1
    for (int j0 = 0; j0 < NV; j0 += JC) {
      float4 f[RW][JC];
#pragma unroll
      for (int q = 0; q < RW; ++q) {
        const float4* Fi = reinterpret_cast<const float4*>(F + (i + q) * r);
#pragma unroll
        for (int j = 0; j < JC; ++j) {
          const int gidx = lane + 32 * (j0 + j);
          f[q][j] = (i + q < rows && gidx < R4) ? __ldcs(Fi + gidx) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int c = 0; c <= D; ++c) {
#pragma unroll
        for (int j = 0; j < JC; ++j) {
          const float4 v = vsm[c * NV * 32 + lane + 32 * (j0 + j)];
#pragma unroll
          for (int q = 0; q < RW; ++q) {
            acc2[q][c] = fmaf(f[q][j].x, v.x, acc2[q][c]);
            acc2[q][c] = fmaf(f[q][j].y, v.y, acc2[q][c]);
            acc2[q][c] = fmaf(f[q][j].z, v.z, acc2[q][c]);
            acc2[q][c] = fmaf(f[q][j].w, v.w, acc2[q][c]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      float acc[D + 1];
#pragma unroll
      for (int c = 0; c <= D; ++c) {
        float a = acc2[q][c];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        acc[c] = a;
      }
      if (lane == 0 && i + q < rows) {
        const float wi = 4.f * w[i + q];
#pragma unroll
        for (int c = 0; c < D; ++c) g[(i + q) * D + c] = wi * fmaf(P[(i + q) * D + c], acc[0], -acc[c + 1]);
      }
    }
  }
}

// grad_U_k = -4 (s_u,k B_x,k + s_v,k B_y,k) - (4/q) s_u,k s_v,k U_k
__global__ void grad_anchor_kernel(const double* __restrict__ accx, const double* __restrict__ accy,
                                   const float* __restrict__ U, int r, int d, double q,
                                   float* __restrict__ gU) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= r) return;
  const double sv = accx[(int64_t)k * (d + 1)];   // xi^T u
  const double su = accy[(int64_t)k * (d + 1)];   // zeta^T v
  for (int c = 0; c < d; ++c) {
    const double bx = accx[(int64_t)k * (d + 1) + 1 + c], by = accy[(int64_t)k * (d + 1) + 1 + c];
    gU[(int64_t)k * d + c] =
        (float)(-4.0 * (su * bx + sv * by) - (4.0 / q) * su * sv * (double)U[(int64_t)k * d + c]);
  }
}

size_t grad_workspace_bytes(int r, int d) {
  return sizeof(double) * (size_t)r * (d + 1) * (2 * kAccCtas + 2) + 1024;
}

cudaError_t launch_gradients(const float* X, int64_t n, const float* Y, int64_t m, int d,
                             const float* U, int r, double q, const float* Xi, const float* Zeta,
                             const float* u, const float* v, float* gX, float* gY, float* gU,
                             double* ws, cudaStream_t s) {
  const int64_t len = (int64_t)r * (d + 1);
  double* partx = ws;
  double* party = partx + len * kAccCtas;
  double* accx = party + len * kAccCtas;   // [k][0] = s_v = xi^T u, [k][1+c] = B_x
  double* accy = accx + len;               // [k][0] = s_u = zeta^T v, [k][1+c] = B_y
  const int red_blocks = (int)((len + 31) / 32);
  const int nv = r <= 128 ? 1 : r <= 256 ? 2 : r <= 512 ? 4 : r <= 1024 ? 8 : r <= 2048 ? 16 : 32;
  if (sizeof(float4) * (size_t)(d + 1) * nv * 32 > 200 * 1024) return cudaErrorInvalidValue;
  switch (d) {
#define ROWS(DD, NV_, FF, RR, WW, PP, SS, GG)                                                      \
  {                                                                                              \
    const size_t dyn = sizeof(float4) * (DD + 1) * NV_ * 32;                                     \
    cudaFuncSetAttribute(grad_rows_kernel<DD, NV_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn); \
    grad_rows_kernel<DD, NV_><<<148 * 2, 256, dyn, s>>>(FF, RR, r, WW, PP, U, SS, GG);             \
  }
#define ROWS_NV(DD, FF, RR, WW, PP, SS, GG)                                                        \
  if (nv == 1) ROWS(DD, 1, FF, RR, WW, PP, SS, GG) else if (nv == 2) ROWS(DD, 2, FF, RR, WW, PP, SS, GG) \
  else if (nv == 4) ROWS(DD, 4, FF, RR, WW, PP, SS, GG) else if (nv == 8) ROWS(DD, 8, FF, RR, WW, PP, SS, GG) \
  else if (nv == 16) ROWS(DD, 16, FF, RR, WW, PP, SS, GG) else ROWS(DD, 32, FF, RR, WW, PP, SS, GG)
#define ACCUM(DD, FF, RR, WW, PP, OUT)                                                           \
  {                                                                                              \
    constexpr int JC = (DD + 1) <= 2 ? 4 : (DD + 1) <= 4 ? 2 : 1;                                 \
    const size_t dyn = sizeof(double) * 8 * (DD + 1) * JC * 4 * 32;                              \
    cudaFuncSetAttribute(grad_accum_kernel<DD, JC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn); \
    grad_accum_kernel<DD, JC><<<kAccCtas, 256, dyn, s>>>(FF, RR, r, WW, PP, U, OUT);             \
  }
#define CASE(DD)                                                                                 \
  case DD:                                                                                       \
    ACCUM(DD, Xi, n, u, X, partx)                                                                \
    ACCUM(DD, Zeta, m, v, Y, party)                                                              \
    grad_reduce_kernel<<<dim3(red_blocks, 2), 256, 0, s>>>(partx, kAccCtas, len, accx);          \
    if (gX) ROWS_NV(DD, Xi, n, u, X, accy, gX)                                                   \
    if (gY) ROWS_NV(DD, Zeta, m, v, Y, accx, gY)                                                 \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
#undef ACCUM
#undef ROWS_NV
#undef ROWS
    default:
      return cudaErrorInvalidValue;
  }
  count_launch(3 + (gX ? 1 : 0) + (gY ? 1 : 0));
  if (gU) {
    grad_anchor_kernel<<<(r + 127) / 128, 128, 0, s>>>(accx, accy, U, r, d, q, gU);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace lsk
