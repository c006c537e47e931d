// lsk_accel.cu — kernels of the accelerated Sinkhorn algorithm (Alg. 2, PAPER.md:697-730;
// NEXT f4) on K_theta = Xi Zeta^T streamed from HBM.  The host loop (lsk_api.cu) drives the
// adaptive line search; per trial it launches
//   lam_kernel      lambda = tau zeta + (1 - tau) eta (fp64); block maxima M1, M2
//   pass(Zeta)      s2 = Zeta^T e^{l2 - M2}                         (accumulate)
//   pass(Xi)        t1 = Xi s2,  s1 = Xi^T e^{l1 - M1}              (dot + accumulate, one read)
//   pass(Zeta)      t2 = Zeta s1                                     (dot)
//   stat1..3        S1 = sum e^{l1-M1} t1, S2, <l1,a>, <l2,b>; |grad_1|^2, |grad_2|^2 and the
//                   block i_k; the block minimiser eta_new and phi(eta_new)'s two sums
// and reads the scalar block (one synchronisation) to take the accept / double-L decision;
// accept_kernel then moves zeta, the averaged plan's marginals and eta.
//
// K e^{l2} = e^{M2} Xi (Zeta^T e^{l2 - M2}) = e^{M2} t1: every e^{lambda} entering a pass is
// shifted by its block maximum (fp32 weights in (0, 1]; the fp64 exponents carry the scale),
// and c = <e^{l1}, K e^{l2}> = e^{M1 + M2} S1 (= e^{M1 + M2} S2 in exact arithmetic).
// Grid-wide sums use the last-CTA pattern: every CTA writes its partial, the last to arrive
// (atomic ticket) adds all partials in a fixed order into the scalar block — deterministic,
// and later kernels read one value instead of G partials.
#include <cmath>
#include <cstdint>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {

namespace accel {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum_f64(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) t += red[i];   // fixed order
  __syncthreads();
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = -INFINITY;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) t = fmax(t, red[i]);
  __syncthreads();
  return t;
}

// Last-CTA finish: thread 0 of every CTA has written its partials; returns true in the CTA
// that arrived last (its thread 0 may then read every partial).
__device__ __forceinline__ bool last_cta(unsigned int* ticket, int nblk) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    last = (t == (unsigned int)nblk - 1);
    if (last) {
      *ticket = 0;   // re-armed for the next launch (stream order)
      __threadfence();
    }
  }
  __syncthreads();
  return last;
}

// Sum of nblk partials by one warp (call with all 32 lanes): lane l adds c = l, l+32, ... in
// order, then a fixed xor butterfly — the same bits on every run; every lane returns the sum.
__device__ __forceinline__ double fixed_sum(const double* p, int nblk) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int c = lane; c < nblk; c += 32) s += __ldcg(p + c);
  return warp_sum_f64(s);
}
__device__ __forceinline__ double fixed_max(const double* p, int nblk) {
  const int lane = threadIdx.x & 31;
  double s = -INFINITY;
  for (int c = lane; c < nblk; c += 32) s = fmax(s, __ldcg(p + c));
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, off));
  return s;
}

// lambda = tau zeta + (1 - tau) eta for block blockIdx.y (0: n rows, 1: m rows);
// scal[SC_M1], scal[SC_M2] = block maxima
__global__ void __launch_bounds__(kThreads) lam_kernel(double tau, AccelVecs v) {
  __shared__ double red[kWarps];
  if (v.ctl) tau = v.ctl[CT_TAU];   // graph-driven solve: this trial's tau
  const int side = blockIdx.y;
  const double* z = side ? v.zet2 : v.zet1;
  const double* e = side ? v.eta2 : v.eta1;
  double* l = side ? v.lam2 : v.lam1;
  const int64_t len = side ? v.m : v.n;
  double mx = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * kThreads) {
    const double x = tau * z[i] + (1.0 - tau) * e[i];
    l[i] = x;
    mx = fmax(mx, x);
  }
  mx = block_max(mx, red);
  const int nblk = gridDim.x * 2, cta = side * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) v.part[cta] = mx;
  if (last_cta(v.ticket, nblk) && threadIdx.x < 32) {
    const double a = fixed_max(v.part, gridDim.x), b = fixed_max(v.part + gridDim.x, gridDim.x);
    if (threadIdx.x == 0) {
      v.scal[SC_M1] = a;
      v.scal[SC_M2] = b;
    }
  }
}

// One read of the factor F (rows x r, fp32 row-major): optionally t_out[row] = F_row . s_in
// (fp32 dot, stored fp64) and part_out[cta][k] = sum_rows F_row,k e^{lam_row - M} (fp32 over
// <= 32 rows per warp, then fp64; warps combined in a fixed order).  One warp per row pair:
// lane l holds float4 column groups {l, l+32, ...} (coalesced 512-byte loads per group).
template <int NV, int ROWS>
__global__ void __launch_bounds__(kThreads, 1) pass_kernel(const float* __restrict__ F,
                                                        int64_t rows, int r,
                                                        const double* __restrict__ s_in,
                                                        const double* __restrict__ lam,
                                                        const double* __restrict__ Mp,
                                                        double* __restrict__ t_out,
                                                        double* __restrict__ part_out) {
  __shared__ __align__(16) float s_sm[128 * NV];
  extern __shared__ double accw[];   // [kWarps][NV * 4][32] when lam != NULL
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int R4 = r >> 2;
  const double M = lam ? *Mp : 0.0;
  if (s_in)
    for (int k = tid; k < 128 * NV; k += kThreads) s_sm[k] = k < r ? (float)s_in[k] : 0.f;
  double* myacc = accw + warp * NV * 4 * 32;
  if (lam)
    for (int e = lane; e < NV * 4 * 32; e += 32) myacc[e] = 0.0;
  __syncthreads();

  const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  float4 acc32[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  int nflush = 0;
  const float4* s4 = reinterpret_cast<const float4*>(s_sm);
  for (int64_t row0 = r0 + (int64_t)warp * ROWS; row0 < r1; row0 += (int64_t)kWarps * ROWS) {
    float4 f[ROWS][NV];
    double lr[ROWS];
    float w[ROWS];
#pragma unroll
    for (int q = 0; q < ROWS; ++q) lr[q] = (lam && row0 + q < r1) ? __ldg(lam + row0 + q) : -INFINITY;
#pragma unroll
    for (int q = 0; q < ROWS; ++q) {
      const int64_t row = row0 + q;
      const float4* Fr = reinterpret_cast<const float4*>(F + row * r);
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int g = lane + 32 * j;
        f[q][j] = (row < r1 && g < R4) ? __ldcs(Fr + g) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int q = 0; q < ROWS; ++q) w[q] = lam ? (float)exp(lr[q] - M) : 0.f;
#pragma unroll
    for (int q = 0; q < ROWS; ++q) {
      const int64_t row = row0 + q;
      if (s_in) {
        float d = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const float4 sv = s4[lane + 32 * j];
          d = fmaf(f[q][j].x, sv.x, d);
          d = fmaf(f[q][j].y, sv.y, d);
          d = fmaf(f[q][j].z, sv.z, d);
          d = fmaf(f[q][j].w, sv.w, d);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        if (lane == 0 && row < r1) t_out[row] = (double)d;
      }
      if (lam) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          acc32[j].x = fmaf(f[q][j].x, w[q], acc32[j].x);
          acc32[j].y = fmaf(f[q][j].y, w[q], acc32[j].y);
          acc32[j].z = fmaf(f[q][j].z, w[q], acc32[j].z);
          acc32[j].w = fmaf(f[q][j].w, w[q], acc32[j].w);
        }
      }
    }
    if (lam && ++nflush * ROWS >= 32) {
      nflush = 0;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        myacc[(4 * j + 0) * 32 + lane] += (double)acc32[j].x;
        myacc[(4 * j + 1) * 32 + lane] += (double)acc32[j].y;
        myacc[(4 * j + 2) * 32 + lane] += (double)acc32[j].z;
        myacc[(4 * j + 3) * 32 + lane] += (double)acc32[j].w;
        acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  if (!lam) return;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    myacc[(4 * j + 0) * 32 + lane] += (double)acc32[j].x;
    myacc[(4 * j + 1) * 32 + lane] += (double)acc32[j].y;
    myacc[(4 * j + 2) * 32 + lane] += (double)acc32[j].z;
    myacc[(4 * j + 3) * 32 + lane] += (double)acc32[j].w;
  }
  __syncthreads();
  // element e = (4 j + q) * 32 + l holds column 4 (l + 32 j) + q
  for (int e = tid; e < NV * 4 * 32; e += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += accw[ww * NV * 4 * 32 + e];
    const int l = e & 31, jq = e >> 5;
    const int col = 4 * (l + 32 * (jq >> 2)) + (jq & 3);
    if (col < r) part_out[(int64_t)blockIdx.x * r + col] = s;
  }
}

// s_out[k] = sum_c part[c][k] over c = 0..G-1: block of 32 columns x 8 warps; warp w adds the
// rows c = w, w+8, ... in order, then the 8 warp sums are added in order (deterministic)
__global__ void __launch_bounds__(kThreads) reduce_kernel(const double* __restrict__ part, int G,
                                                          int r, double* s_out) {
  __shared__ double red[kWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (k < r)
    for (int c = warp; c < G; c += kWarps) s += part[(int64_t)c * r + k];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && k < r) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += red[w][lane];
    s_out[k] = t;
  }
}

// stat 1 (grid G x 2): S_side = sum e^{l-M} t, <l, w>, bad-count(t) -> scal
__global__ void __launch_bounds__(kThreads) stat1_kernel(AccelVecs v) {
  __shared__ double red[kWarps];
  const int side = blockIdx.y;
  const double M = v.scal[side ? SC_M2 : SC_M1];
  const double* l = side ? v.lam2 : v.lam1;
  const double* t = side ? v.t2 : v.t1;
  const double* w = side ? v.bn : v.an;
  const int64_t len = side ? v.m : v.n;
  double S = 0.0, lw = 0.0, bad = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * kThreads) {
    S += exp(l[i] - M) * t[i];
    lw += l[i] * w[i];
    if (!(t[i] > 0.0) || !isfinite(t[i])) bad += 1.0;
  }
  S = block_sum(S, red);
  lw = block_sum(lw, red);
  bad = block_sum(bad, red);
  const int G = gridDim.x, nblk = 2 * G, cta = side * G + blockIdx.x;
  if (threadIdx.x == 0) {
    v.part[cta] = S;
    v.part[nblk + cta] = lw;
    v.part[2 * nblk + cta] = bad;
  }
  if (last_cta(v.ticket, nblk) && threadIdx.x < 32) {
    const double S1 = fixed_sum(v.part, G), S2 = fixed_sum(v.part + G, G);
    const double la = fixed_sum(v.part + nblk, G), lb = fixed_sum(v.part + nblk + G, G);
    const double bad = fixed_sum(v.part + 2 * nblk, nblk);
    if (threadIdx.x == 0) {
      v.scal[SC_S1] = S1;
      v.scal[SC_S2] = S2;
      v.scal[SC_LA] = la;
      v.scal[SC_LB] = lb;
      v.scal[SC_BAD] = bad;
    }
  }
}

// grad_1 phi = e^{l1-M1} t1 / S1 - a,  grad_2 phi = e^{l2-M2} t2 / S1 - b  (c = e^{M1+M2} S1)
__device__ __forceinline__ double grad_entry(const AccelVecs& v, int side, int64_t i, double M1,
                                             double M2, double S1) {
  return side ? exp(v.lam2[i] - M2) * v.t2[i] / S1 - v.bn[i]
              : exp(v.lam1[i] - M1) * v.t1[i] / S1 - v.an[i];
}

// stat 2: |grad_1|^2, |grad_2|^2 and the block i_k = argmax (ties: 1, reading C27) -> scal
__global__ void __launch_bounds__(kThreads) stat2_kernel(AccelVecs v) {
  __shared__ double red[kWarps];
  const double M1 = v.scal[SC_M1], M2 = v.scal[SC_M2], S1 = v.scal[SC_S1];
  const int side = blockIdx.y;
  const int64_t len = side ? v.m : v.n;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * kThreads) {
    const double g = grad_entry(v, side, i, M1, M2, S1);
    s += g * g;
  }
  s = block_sum(s, red);
  const int G = gridDim.x, nblk = 2 * G;
  if (threadIdx.x == 0) v.part[side * G + blockIdx.x] = s;
  if (last_cta(v.ticket, nblk) && threadIdx.x < 32) {
    const double n1 = fixed_sum(v.part, G), n2 = fixed_sum(v.part + G, G);
    if (threadIdx.x == 0) {
      v.scal[SC_N1] = n1;
      v.scal[SC_N2] = n2;
      v.scal[SC_BLK] = n1 >= n2 ? 1.0 : 2.0;
    }
  }
}

// stat 3 (grid G over the chosen block's rows): the block minimiser
//   blk 1: eta1_new = log a - M2 - log t1   (= l1 + log a - log(e^{l1} o K e^{l2}))
//   blk 2: eta2_new = log b - M1 - log t2
// into etan; scal: E = sum e^{eta_new + M_other} t, <eta_new, w>
__global__ void __launch_bounds__(kThreads) stat3_kernel(AccelVecs v) {
  __shared__ double red[kWarps];
  const int blk = v.scal[SC_BLK] == 1.0 ? 1 : 2;
  const double Mo = blk == 1 ? v.scal[SC_M2] : v.scal[SC_M1];
  const int64_t len = blk == 1 ? v.n : v.m;
  const double* t = blk == 1 ? v.t1 : v.t2;
  const double* w = blk == 1 ? v.an : v.bn;
  double E = 0.0, ew = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * kThreads) {
    const double e = log(w[i]) - Mo - log(t[i]);
    v.etan[i] = e;
    E += exp(e + Mo) * t[i];
    ew += e * w[i];
  }
  E = block_sum(E, red);
  ew = block_sum(ew, red);
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    v.part[blockIdx.x] = E;
    v.part[G + blockIdx.x] = ew;
  }
  if (last_cta(v.ticket, G) && threadIdx.x < 32) {
    const double E = fixed_sum(v.part, G), ew = fixed_sum(v.part + G, G);
    if (threadIdx.x == 0) {
      v.scal[SC_E] = E;
      v.scal[SC_EW] = ew;
    }
  }
}

// accepted step: zeta -= a1 grad; p = (a1 (grad + w) + A_k p) / A_{k+1}; eta_blk <- eta_new;
// scal[SC_PERR] = |p1 - a|_1 + |p2 - b|_1
__global__ void __launch_bounds__(kThreads) accept_kernel(AccelVecs v, double a1, double Ak,
                                                          double Ak1) {
  __shared__ double red[kWarps];
  if (v.ctl) {   // graph-driven solve: runs after every trial, moves only on acceptance
    if (v.ctl[CT_ACC] == 0.0) return;   // uniform over the grid: no CTA takes a ticket
    a1 = v.ctl[CT_A1];
    Ak = v.ctl[CT_AKP];
    Ak1 = v.ctl[CT_AK1];
  }
  const double M1 = v.scal[SC_M1], M2 = v.scal[SC_M2], S1 = v.scal[SC_S1];
  const int blk = v.scal[SC_BLK] == 1.0 ? 1 : 2;
  const int side = blockIdx.y;
  const int64_t len = side ? v.m : v.n;
  double* z = side ? v.zet2 : v.zet1;
  double* p = side ? v.p2 : v.p1;
  double* e = side ? v.eta2 : v.eta1;
  const double* lam = side ? v.lam2 : v.lam1;
  const double* w = side ? v.bn : v.an;
  const bool moved = (blk == 1 && side == 0) || (blk == 2 && side == 1);
  double err = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * kThreads) {
    const double g = grad_entry(v, side, i, M1, M2, S1);
    z[i] -= a1 * g;
    const double pn = (a1 * (g + w[i]) + Ak * p[i]) / Ak1;
    p[i] = pn;
    err += fabs(pn - w[i]);
    e[i] = moved ? v.etan[i] : lam[i];
  }
  err = block_sum(err, red);
  const int G = gridDim.x, nblk = 2 * G;
  if (threadIdx.x == 0) v.part[side * G + blockIdx.x] = err;
  if (last_cta(v.ticket, nblk) && threadIdx.x < 32) {
    const double e = fixed_sum(v.part, nblk);
    if (threadIdx.x == 0) v.scal[SC_PERR] = e;
  }
}

// fp64 simplex weights an = a / sum a (reading C28); sums by one CTA in a fixed order
__global__ void __launch_bounds__(kThreads) normalise_kernel(const float* a, const float* b,
                                                             AccelVecs v) {
  __shared__ double red[kWarps];
  __shared__ double tot;
  const float* x = blockIdx.x ? b : a;
  double* out = blockIdx.x ? v.bn : v.an;
  const int64_t len = blockIdx.x ? v.m : v.n;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += kThreads) s += (double)x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) tot = s;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < len; i += kThreads) out[i] = (double)x[i] / tot;
}

// ---- device-driven line search (graph-driven solve; the host loop's arithmetic, C24-C29) ----
// iteration start: L_{k+1} = L_k / 2 (C24), trials re-armed
__global__ void ls_begin_kernel(AccelVecs v, cudaGraphConditionalHandle trial) {
  if (threadIdx.x != 0) return;
  v.ctl[CT_L1] = v.ctl[CT_LK] / 2.0;
  cudaGraphSetConditional(trial, 1u);
}
// trial start: a_{k+1} from L_{k+1} a_{k+1}^2 = A_k + a_{k+1}, tau = a_{k+1} / A_{k+1}
__global__ void ls_prepare_kernel(AccelVecs v) {
  if (threadIdx.x != 0) return;
  double* c = v.ctl;
  const double L1 = c[CT_L1], ak = c[CT_AK], Lk = c[CT_LK];
  const double a1 = 1.0 / (2.0 * L1) + sqrt(1.0 / (4.0 * L1 * L1) + ak * ak * Lk / L1);
  c[CT_A1] = a1;
  c[CT_TAU] = 1.0 / (a1 * L1);
  c[CT_TRIALS] += 1.0;
  c[CT_ACC] = 0.0;
}
// accept (phi(eta_new) <= phi(lambda) - |grad|^2 / (2 L) + the C29 allowance) or double L
__global__ void ls_decide_kernel(AccelVecs v, cudaGraphConditionalHandle trial,
                                 cudaGraphConditionalHandle iter) {
  if (threadIdx.x != 0) return;
  const double* sc = v.scal;
  double* c = v.ctl;
  const double M1 = sc[SC_M1], M2 = sc[SC_M2], S1 = sc[SC_S1], S2 = sc[SC_S2];
  const double la = sc[SC_LA], lb = sc[SC_LB], n1 = sc[SC_N1], n2 = sc[SC_N2];
  if (sc[SC_BAD] > 0.0 || !(S1 > 0.0) || !isfinite(S1) || !(S2 > 0.0)) {
    c[CT_ERR] = 1.0;   // breakdown: both loops end
    cudaGraphSetConditional(trial, 0u);
    cudaGraphSetConditional(iter, 0u);
    return;
  }
  const int blk = sc[SC_BLK] == 1.0 ? 1 : 2;   // argmax, ties -> 1 (C27)
  const double phi_lam = M1 + M2 + log(blk == 1 ? S1 : S2) - la - lb;
  const double phi_new = log(sc[SC_E]) - (blk == 1 ? sc[SC_EW] + lb : la + sc[SC_EW]);
  const double L1 = c[CT_L1], a1 = c[CT_A1];
  if (phi_new <= phi_lam - (n1 + n2) / (2.0 * L1) + 1e-13 * fmax(1.0, fabs(phi_lam))) {
    c[CT_ACC] = 1.0;
    c[CT_AKP] = c[CT_LK] * c[CT_AK] * c[CT_AK];   // A_k = L_k a_k^2
    c[CT_AK1] = L1 * a1 * a1;                     // A_{k+1}
    c[CT_AK] = a1;
    c[CT_LK] = L1;
    c[CT_PHI] = phi_new;
    c[CT_BLK] = (double)blk;
    cudaGraphSetConditional(trial, 0u);
  } else {
    c[CT_L1] = 2.0 * L1;
    if (!(2.0 * L1 < 1e300)) {
      c[CT_ERR] = 2.0;   // the line search diverged
      cudaGraphSetConditional(trial, 0u);
      cudaGraphSetConditional(iter, 0u);
    }
  }
}
// iteration end: traces, the iteration count and the stopping test (tol on the averaged plan)
__global__ void ls_end_kernel(AccelVecs v, cudaGraphConditionalHandle iter, double eps,
                              int max_iters, double tol, double* Ftr, double* Ltr, int* Btr) {
  if (threadIdx.x != 0) return;
  double* c = v.ctl;
  if (c[CT_ERR] != 0.0) {
    cudaGraphSetConditional(iter, 0u);
    return;
  }
  const int it = (int)c[CT_IT];
  const double F = -eps * c[CT_PHI];
  c[CT_F] = F;
  if (Ftr) Ftr[it] = F;
  if (Ltr) Ltr[it] = c[CT_LK];
  if (Btr) Btr[it] = (int)c[CT_BLK];
  c[CT_IT] = (double)(it + 1);
  const double perr = v.scal[SC_PERR];
  c[CT_PERR] = perr;
  bool stop = it + 1 >= max_iters;
  if (tol > 0.0 && perr < tol) {
    c[CT_CONV] = 1.0;
    stop = true;
  }
  cudaGraphSetConditional(iter, stop ? 0u : 1u);
}

}  // namespace accel

// ------------------------------------------------------------------------------ launchers
// vector kernels: one CTA per SM per block side; factor passes: one CTA per SM with up to
// 255 registers (four rows of 4 KB in flight per warp at r = 1000), partials reduced by
// reduce_kernel
int accel_grid() { return 148; }
int accel_pass_grid() { return 148; }

cudaError_t launch_accel_normalise(const float* a, const float* b, const AccelVecs& v,
                                   cudaStream_t s) {
  accel::normalise_kernel<<<2, accel::kThreads, 0, s>>>(a, b, v);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_accel_lambda(double tau, const AccelVecs& v, cudaStream_t s) {
  accel::lam_kernel<<<dim3(accel_grid(), 2), accel::kThreads, 0, s>>>(tau, v);
  count_launch();
  return cudaGetLastError();
}

template <int NV>
static cudaError_t pass_nv(const float* F, int64_t rows, int r, const double* s_in,
                           const double* lam, const double* Mp, double* t_out, double* part,
                           cudaStream_t s) {
  constexpr int ROWS = NV <= 4 ? 8 : NV <= 8 ? 4 : 1;   // rows in flight per warp
  const int G = accel_pass_grid();
  auto kern = accel::pass_kernel<NV, ROWS>;
  const size_t dyn = lam ? sizeof(double) * accel::kWarps * NV * 4 * 32 : 0;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  kern<<<G, accel::kThreads, dyn, s>>>(F, rows, r, s_in, lam, Mp, t_out, part);
  count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess || !lam) return e;
  accel::reduce_kernel<<<(r + 31) / 32, accel::kThreads, 0, s>>>(part, G, r, part + (int64_t)G * r);
  count_launch();
  return cudaGetLastError();
}

// part must hold (accel_pass_grid() + 1) * r doubles; the reduced r-vector lands in part + G r
cudaError_t launch_accel_pass(const float* F, int64_t rows, int r, const double* s_in,
                              const double* lam, const double* Mp, double* t_out, double* part,
                              cudaStream_t s) {
  if (r <= 128) return pass_nv<1>(F, rows, r, s_in, lam, Mp, t_out, part, s);
  if (r <= 256) return pass_nv<2>(F, rows, r, s_in, lam, Mp, t_out, part, s);
  if (r <= 512) return pass_nv<4>(F, rows, r, s_in, lam, Mp, t_out, part, s);
  if (r <= 1024) return pass_nv<8>(F, rows, r, s_in, lam, Mp, t_out, part, s);
  if (r <= 2048) return pass_nv<16>(F, rows, r, s_in, lam, Mp, t_out, part, s);
  return cudaErrorInvalidValue;
}

static cudaError_t add_kernel_node(cudaGraph_t g, const cudaGraphNode_t* dep, size_t ndep,
                                   void* func, void** args, cudaGraphNode_t* out) {
  cudaKernelNodeParams kp = {};
  kp.func = func;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  kp.extra = nullptr;
  return cudaGraphAddKernelNode(out, g, dep, ndep, &kp);
}

cudaError_t accel_solve_graph(const AccelVecs& v, const float* Xi, int64_t n, const float* Zeta,
                              int64_t m, int r, double* partA, double* partB, double eps,
                              int max_iters, double tol, double* Ftr, double* Ltr, int* Btr,
                              cudaStream_t s) {
  const int Gp = accel_pass_grid();
  cudaGraph_t g = nullptr, body1, body2;
  cudaGraphExec_t ge = nullptr;
  cudaStream_t cs = nullptr;
  cudaError_t e;
#define GT(x)                \
  do {                       \
    e = (x);                 \
    if (e != cudaSuccess) goto done; \
  } while (0)
  {
    GT(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hIter, hTrial;
    GT(cudaGraphConditionalHandleCreate(&hIter, g, 1u, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hIter;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t nIter;
    GT(cudaGraphAddNode(&nIter, g, nullptr, 0, &cp));
    body1 = cp.conditional.phGraph_out[0];
    // iteration body: begin -> while(trial) -> end
    GT(cudaGraphConditionalHandleCreate(&hTrial, body1, 1u, cudaGraphCondAssignDefault));
    AccelVecs va = v;
    cudaGraphNode_t nBegin, nTrial, nEnd;
    {
      void* args[] = {&va, &hTrial};
      GT(add_kernel_node(body1, nullptr, 0, (void*)accel::ls_begin_kernel, args, &nBegin));
    }
    cudaGraphNodeParams tp = {};
    tp.type = cudaGraphNodeTypeConditional;
    tp.conditional.handle = hTrial;
    tp.conditional.type = cudaGraphCondTypeWhile;
    tp.conditional.size = 1;
    GT(cudaGraphAddNode(&nTrial, body1, &nBegin, 1, &tp));
    body2 = tp.conditional.phGraph_out[0];
    {
      double eps_ = eps, tol_ = tol;
      int mi = max_iters;
      void* args[] = {&va, &hIter, &eps_, &mi, &tol_, &Ftr, &Ltr, &Btr};
      GT(add_kernel_node(body1, &nTrial, 1, (void*)accel::ls_end_kernel, args, &nEnd));
    }
    // trial body, captured from the same launchers the host-driven loop uses
    GT(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    GT(cudaStreamBeginCaptureToGraph(cs, body2, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    accel::ls_prepare_kernel<<<1, 32, 0, cs>>>(va);
    launch_accel_lambda(0.0, va, cs);
    launch_accel_pass(Zeta, m, r, nullptr, va.lam2, va.scal + SC_M2, nullptr, partA, cs);
    launch_accel_pass(Xi, n, r, partA + (size_t)Gp * r, va.lam1, va.scal + SC_M1, va.t1, partB, cs);
    launch_accel_pass(Zeta, m, r, partB + (size_t)Gp * r, nullptr, nullptr, va.t2, nullptr, cs);
    launch_accel_stats(1, va, 0, 0, 0, cs);
    launch_accel_stats(2, va, 0, 0, 0, cs);
    launch_accel_stats(3, va, 0, 0, 0, cs);
    accel::ls_decide_kernel<<<1, 32, 0, cs>>>(va, hTrial, hIter);
    launch_accel_stats(4, va, 0, 0, 0, cs);
    {
      cudaGraph_t cap = nullptr;
      GT(cudaStreamEndCapture(cs, &cap));
    }
    GT(cudaGraphInstantiate(&ge, g, 0));
    GT(cudaGraphLaunch(ge, s));
    count_launch(2);
  }
done:
#undef GT
  if (ge) cudaGraphExecDestroy(ge);   // destruction waits for nothing: the launch is enqueued
  if (g) cudaGraphDestroy(g);
  if (cs) cudaStreamDestroy(cs);
  return e;
}

cudaError_t launch_accel_stats(int phase, const AccelVecs& v, double a1, double Ak, double Ak1,
                               cudaStream_t s) {
  const int G = accel_grid();
  if (phase == 1) accel::stat1_kernel<<<dim3(G, 2), accel::kThreads, 0, s>>>(v);
  else if (phase == 2) accel::stat2_kernel<<<dim3(G, 2), accel::kThreads, 0, s>>>(v);
  else if (phase == 3) accel::stat3_kernel<<<G, accel::kThreads, 0, s>>>(v);
  else accel::accept_kernel<<<dim3(G, 2), accel::kThreads, 0, s>>>(v, a1, Ak, Ak1);
  count_launch();
  return cudaGetLastError();
}

}  // namespace lsk
