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
constexpr int kAccCtas = 148;

// Per-CTA partials over a row range: out[cta][k][0] = sum_i w_i F_ik,
// out[cta][k][1+c] = sum_i w_i F_ik (P_ic - U_kc).  Thread t owns columns k = t, t+256, ...
template <int D>
__global__ void __launch_bounds__(256) grad_accum_kernel(const float* __restrict__ F, int64_t rows,
                                                         int r, const float* __restrict__ w,
                                                         const float* __restrict__ P,
                                                         const float* __restrict__ U,
                                                         double* __restrict__ part) {
  const int64_t i0 = rows * blockIdx.x / gridDim.x, i1 = rows * (blockIdx.x + 1) / gridDim.x;
  __shared__ float ps[64][D + 1];   // staged (w_i, P_i) for 64 rows
  for (int k0 = 0; k0 < r; k0 += 256) {
    const int k = k0 + threadIdx.x;
    float uk[D];
#pragma unroll
    for (int c = 0; c < D; ++c) uk[c] = (k < r) ? U[(int64_t)k * D + c] : 0.f;
    double s = 0.0, bsum[D];
#pragma unroll
    for (int c = 0; c < D; ++c) bsum[c] = 0.0;
    for (int64_t ib = i0; ib < i1; ib += 64) {
      const int nb = (int)min((int64_t)64, i1 - ib);
      __syncthreads();
      for (int e = threadIdx.x; e < nb * (D + 1); e += blockDim.x) {
        const int row = e / (D + 1), c = e % (D + 1);
        ps[row][c] = (c == 0) ? w[ib + row] : P[(ib + row) * D + (c - 1)];
      }
      __syncthreads();
      if (k < r) {
        for (int rr = 0; rr < nb; ++rr) {
          const float fw = F[(ib + rr) * r + k] * ps[rr][0];
          s += (double)fw;
#pragma unroll
          for (int c = 0; c < D; ++c) bsum[c] += (double)(fw * (ps[rr][c + 1] - uk[c]));
        }
      }
    }
    if (k < r) {
      double* o = part + ((int64_t)blockIdx.x * r + k) * (D + 1);
      o[0] = s;
#pragma unroll
      for (int c = 0; c < D; ++c) o[1 + c] = bsum[c];
    }
  }
}

// fixed-order reduction of the CTA partials: acc[k][j] = sum_cta part[cta][k][j]
__global__ void grad_reduce_kernel(const double* __restrict__ part, int nparts, int64_t len,
                                   double* __restrict__ acc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * len + e];
  acc[e] = s;
}

// grad_p_i = 4 w_i sum_k F_ik s_k (p_i - U_k): one warp per row, lanes stride over k.
template <int D>
__global__ void __launch_bounds__(256) grad_rows_kernel(const float* __restrict__ F, int64_t rows,
                                                        int r, const float* __restrict__ w,
                                                        const float* __restrict__ P,
                                                        const float* __restrict__ U,
                                                        const double* __restrict__ sacc,
                                                        float* __restrict__ g) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int nwarps = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
  for (int64_t i = warp; i < rows; i += nwarps) {
    float p[D], acc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      p[c] = P[i * D + c];
      acc[c] = 0.f;
    }
    const float* Fi = F + i * r;
    for (int k = lane; k < r; k += 32) {
      const float fs = Fi[k] * (float)sacc[(int64_t)k * (D + 1)];
#pragma unroll
      for (int c = 0; c < D; ++c) acc[c] = fmaf(fs, p[c] - U[(int64_t)k * D + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      float x = acc[c];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      acc[c] = x;
    }
    if (lane == 0) {
      const float wi = 4.f * w[i];
#pragma unroll
      for (int c = 0; c < D; ++c) g[i * D + c] = wi * acc[c];
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
  const int red_blocks = (int)((len + 255) / 256);
  switch (d) {
#define CASE(DD)                                                                                 \
  case DD:                                                                                       \
    grad_accum_kernel<DD><<<kAccCtas, 256, 0, s>>>(Xi, n, r, u, X, U, partx);                    \
    grad_accum_kernel<DD><<<kAccCtas, 256, 0, s>>>(Zeta, m, r, v, Y, U, party);                  \
    grad_reduce_kernel<<<red_blocks, 256, 0, s>>>(partx, kAccCtas, len, accx);                   \
    grad_reduce_kernel<<<red_blocks, 256, 0, s>>>(party, kAccCtas, len, accy);                   \
    if (gX) grad_rows_kernel<DD><<<148 * 8, 256, 0, s>>>(Xi, n, r, u, X, U, accy, gX);           \
    if (gY) grad_rows_kernel<DD><<<148 * 8, 256, 0, s>>>(Zeta, m, r, v, Y, U, accx, gY);         \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default:
      return cudaErrorInvalidValue;
  }
  count_launch(4 + (gX ? 1 : 0) + (gY ? 1 : 0));
  if (gU) {
    grad_anchor_kernel<<<(r + 127) / 128, 128, 0, s>>>(accx, accy, U, r, d, q, gU);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace lsk
