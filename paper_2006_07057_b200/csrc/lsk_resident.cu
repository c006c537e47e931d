// lsk_resident.cu — Alg. 1 for small problems with BOTH factors resident in
// shared memory: each problem is one thread-block cluster of G <= 8 CTAs; CTA c holds its rows of
// xi and zeta (the row partition of lsk_shard_range) for the whole solve, so a pass reads no
// global memory at all, and the pass boundary is one cluster barrier plus G DSMEM reads per
// r-vector entry.  The persistent grid kernels pay ~6 us per pass of boundary machinery (named
// barriers, svec sentinels, the team exchange chain) whatever the problem size; here a pass of
// config 1 (n = m = 500, r = 100) is a few hundred cycles of shared-memory GEMV plus one cluster
// round trip (DESIGN.md §6 K10).
//
// Per pass (side f, r-vector s from the previous pass):
//   t_j = F_j . s (fp32, fixed order), w_j = c_j / t_j (u or v), s'_k = sum_j F_jk w_j,
// with the same pass schedule, lagged stopping test and fp64 read-out W = eps (a^T log u +
// b^T log v) as the grid kernels (lsk_sinkhorn.cu / lsk_implicit.cu).
//
// Layout: 8 warps per CTA; a warp takes batches of 8 rows (rows w*8, w*8 + 64, ...); lane l owns
// the float4 column groups l + 32 i (i < NG).  Row dots: lane partials + a warp transpose-reduce
// (lanes 4k..4k+3 end with row k's total; fixed shuffle order).  Accumulation: fp32 over <= 64
// rows, then fp64 per lane; warp partials -> CTA partial in fixed warp order (fp64, shared
// memory) -> pushed with st.async into slot [p & 1][cta] of EVERY CTA's receive buffer,
// completing bytes on the receiver's parity-(p & 1) mbarrier -> every CTA waits on its own
// mbarrier and sums the G slots in CTA order (identical bits in every CTA, so every CTA takes
// the same stopping decision without a broadcast).  No cluster barrier per pass: the sender of
// pass p + 2's partial has received every CTA's pass p + 1 partial, so every CTA had finished
// reading its pass-p slots.  Breakdown and bad-weight counts only matter for the report: they
// stay per thread until the end; only the marginal error is summed every pass.
#include <algorithm>
#include <cmath>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {

namespace res {

constexpr int kW = 8;          // warps per CTA
constexpr int kT = 32 * kW;    // threads per CTA
constexpr int kTR = 8;         // rows per warp batch

__host__ __device__ inline size_t up16(size_t x) { return (x + 15) & ~size_t(15); }

// dynamic shared memory layout (bytes), identical on host and device
struct Lay {
  size_t F0, F1, c0, c1, u, v, s32, wp, rb, tot, xs, rdo, bar, total;
  __host__ __device__ Lay(int r, int n0, int n1, int G) {
    size_t o = 0;
    F0 = o; o += up16(sizeof(float) * (size_t)n0 * r);
    F1 = o; o += up16(sizeof(float) * (size_t)n1 * r);
    c0 = o; o += up16(sizeof(float) * n0);
    c1 = o; o += up16(sizeof(float) * n1);
    u = o;  o += up16(sizeof(float) * n0);
    v = o;  o += up16(sizeof(float) * 2 * (size_t)n1);        // v by iteration parity
    s32 = o; o += up16(sizeof(float) * r);
    wp = o; o += up16(sizeof(double) * kW * (size_t)r);        // warp partials
    rb = o; o += up16(sizeof(double) * 2 * (size_t)G * (r + 1));   // received [parity][cta][r+1]
    tot = o; o += up16(sizeof(double) * (r + 1));              // cluster totals (+ the error)
    xs = o; o += up16(sizeof(double) * kW * 4);                // warp extras
    rdo = o; o += up16(sizeof(double) * 4);                    // read-out partials
    bar = o; o += up16(sizeof(uint64_t) * 2);                  // receive mbarriers [parity]
    total = o;
  }
};

template <int NG>
__global__ void __launch_bounds__(kT, 1) resident_kernel(const SinkArgs A, int G, int nmax0, int nmax1) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Lay L(A.r, nmax0, nmax1, G);
  float* F0 = reinterpret_cast<float*>(smem + L.F0);
  float* F1 = reinterpret_cast<float*>(smem + L.F1);
  float* cw0 = reinterpret_cast<float*>(smem + L.c0);
  float* cw1 = reinterpret_cast<float*>(smem + L.c1);
  float* us = reinterpret_cast<float*>(smem + L.u);
  float* vs = reinterpret_cast<float*>(smem + L.v);
  float* s32 = reinterpret_cast<float*>(smem + L.s32);
  double* wp = reinterpret_cast<double*>(smem + L.wp);
  double* rbuf = reinterpret_cast<double*>(smem + L.rb);
  double* tot = reinterpret_cast<double*>(smem + L.tot);
  double* xs = reinterpret_cast<double*>(smem + L.xs);
  double* rdo = reinterpret_cast<double*>(smem + L.rdo);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(smem + L.bar);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int prob = blockIdx.x / G;
  const int cta = (int)cluster_ctarank();
  const int r = A.r, R4 = r >> 2, RX = r + 1;   // r-vector + the marginal error
  int64_t b0, e0, b1, e1;
  cta_rows(A.rows[0], G, cta, &b0, &e0);
  cta_rows(A.rows[1], G, cta, &b1, &e1);
  const int n0 = (int)(e0 - b0), n1 = (int)(e1 - b1);

  // the CTA's factor rows and weights, once per solve
  {
    const float4* g0 = reinterpret_cast<const float4*>(A.F[0] + (int64_t)prob * A.fstride[0] + b0 * r);
    const float4* g1 = reinterpret_cast<const float4*>(A.F[1] + (int64_t)prob * A.fstride[1] + b1 * r);
    float4* d0 = reinterpret_cast<float4*>(F0);
    float4* d1 = reinterpret_cast<float4*>(F1);
    for (int i = tid; i < n0 * R4; i += kT) d0[i] = __ldg(g0 + i);
    for (int i = tid; i < n1 * R4; i += kT) d1[i] = __ldg(g1 + i);
    const float* a = A.w[0] + (int64_t)prob * A.wstride[0] + b0;
    const float* b = A.w[1] + (int64_t)prob * A.wstride[1] + b1;
    for (int i = tid; i < n0; i += kT) cw0[i] = __ldg(a + i);
    for (int i = tid; i < n1; i += kT) cw1[i] = __ldg(b + i);
  }
  if (tid == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    fence_mbar_init();
  }
  cluster_sync_all();   // every CTA's receive mbarriers are initialised before any push

  double stErr = 0.0, ferr = -1.0;
  double brkT = 0.0, wbT = 0.0;   // this thread's breakdown / bad-weight counts (summed at the end)
  int final_t = -1, conv = 0;
  for (int p = 0; p < A.num_passes; ++p) {
    const int kind = pass_kind(p, A);
    const bool kDot = kind != PK_INIT, kAcc = kind != PK_ERR, kOut = kind == PK_U || kind == PK_V;
    const int f = (kind == PK_V || kind == PK_ERR) ? 1 : 0;
    const int nr = f ? n1 : n0;
    const float* Fs = f ? F1 : F0;
    const float* cw = f ? cw1 : cw0;
    const int it = (p + 1) / 2;   // iteration of a v-pass
    float* outp = kind == PK_U ? us : (kind == PK_V ? vs + (it & 1) * nmax1 : nullptr);
    const float* vold = (kind == PK_ERR) ? vs + (A.T & 1) * nmax1
                        : (kind == PK_V && it >= 2) ? vs + ((it - 1) & 1) * nmax1 : nullptr;
    float4 s4[NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int g = lane + 32 * i;
      s4[i] = (kDot && g < R4) ? reinterpret_cast<const float4*>(s32)[g] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 acc[NG];
    double acc64[NG][4];
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      acc64[i][0] = acc64[i][1] = acc64[i][2] = acc64[i][3] = 0.0;
    }
    auto flush = [&]() {
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        acc64[i][0] += (double)acc[i].x;
        acc64[i][1] += (double)acc[i].y;
        acc64[i][2] += (double)acc[i].z;
        acc64[i][3] += (double)acc[i].w;
        acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    double errw = 0.0;
    int nb = 0;
    for (int rb = warp * kTR; rb < nr; rb += kW * kTR) {
      float4 fr[kTR][NG];
#pragma unroll
      for (int k = 0; k < kTR; ++k)
#pragma unroll
        for (int i = 0; i < NG; ++i) {
          const int g = lane + 32 * i;
          fr[k][i] = (rb + k < nr && g < R4) ? lds128(Fs + (size_t)(rb + k) * r + 4 * g)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      const int krow = lane >> 2;          // the row whose total this lane holds
      const int row = rb + krow;
      float wl = 0.f;
      if (kDot) {
        float pr[kTR];
#pragma unroll
        for (int k = 0; k < kTR; ++k) {
          float d = 0.f;
#pragma unroll
          for (int i = 0; i < NG; ++i) {
            d = fmaf(fr[k][i].x, s4[i].x, d);
            d = fmaf(fr[k][i].y, s4[i].y, d);
            d = fmaf(fr[k][i].z, s4[i].z, d);
            d = fmaf(fr[k][i].w, s4[i].w, d);
          }
          pr[k] = d;
        }
        const float t = warp_transpose_reduce<kTR>(pr, lane);   // t_j = F_j . s
        if (row < nr) {
          const float c = cw[row];
          const float w = c * rcp_approx(t);                    // w_j = c_j / t_j
          if ((lane & 3) == 0) {
            if (bad_weight(c)) wbT += 1.0;
            if (vold) errw += fabs((double)vold[row] * (double)t - (double)c);
            if (kOut) {
              if (!(w > 0.f) || !isfinite(w)) brkT += 1.0;
              outp[row] = w;
            }
          }
          wl = kAcc ? w : 0.f;
        }
      } else {
        wl = row < nr ? 1.f : 0.f;   // u^0 = 1 (reading C6)
      }
      if (kAcc) {
#pragma unroll
        for (int k = 0; k < kTR; ++k) {
          const float wk = __shfl_sync(0xffffffffu, wl, 4 * k);
#pragma unroll
          for (int i = 0; i < NG; ++i) {
            acc[i].x = fmaf(fr[k][i].x, wk, acc[i].x);
            acc[i].y = fmaf(fr[k][i].y, wk, acc[i].y);
            acc[i].z = fmaf(fr[k][i].z, wk, acc[i].z);
            acc[i].w = fmaf(fr[k][i].w, wk, acc[i].w);
          }
        }
        if (++nb == 8) {   // fp32 partials over <= 64 rows, then fp64 (as the grid kernels)
          nb = 0;
          flush();
        }
      }
    }
    flush();
    // warp partials -> shared memory; warp extras
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int g = lane + 32 * i;
      if (g < R4) {
        double* w4 = wp + (size_t)warp * r + 4 * g;
        w4[0] = acc64[i][0];
        w4[1] = acc64[i][1];
        w4[2] = acc64[i][2];
        w4[3] = acc64[i][3];
      }
    }
    const bool kErr = vold != nullptr;   // uniform: this pass evaluates the marginal error
    if (kErr) {
      errw = warp_sum_f64(errw);
      if (lane == 0) xs[warp * 4] = errw;
    }
    __syncthreads();
    // CTA partial (fixed warp order), pushed into slot [p & 1][cta] of every CTA of the cluster
    const uint32_t slot = smem_u32(rbuf + ((size_t)(p & 1) * G + cta) * RX);
    const uint32_t mb = smem_u32(&rbar[p & 1]);
    for (int k = tid; k < RX; k += kT) {
      double x = 0.0;
      if (k < r) {
        if (kAcc) {
#pragma unroll
          for (int w = 0; w < kW; ++w) x += wp[(size_t)w * r + k];
        }
      } else if (kErr) {
#pragma unroll
        for (int w = 0; w < kW; ++w) x += xs[w * 4];
      }
      for (int c = 0; c < G; ++c)
        st_async_f64(mapa_shared(slot + 8u * (uint32_t)k, (uint32_t)c), x, mapa_shared(mb, (uint32_t)c));
    }
    if (tid == 0) mbar_arrive_expect_tx(&rbar[p & 1], (uint32_t)(G * RX * 8));
    while (!mbar_try_wait_cluster(&rbar[p & 1], (uint32_t)((p >> 1) & 1))) {
    }
    // cluster totals, CTA order 0..G-1 (the same bits in every CTA)
    const double* rp = rbuf + (size_t)(p & 1) * G * RX;
    for (int k = tid; k < RX; k += kT) {
      double x = 0.0;
      for (int c = 0; c < G; ++c) x += rp[(size_t)c * RX + k];
      tot[k] = x;
      if (k < r) s32[k] = (float)x;
    }
    __syncthreads();
    // stopping test on pass p's error (every thread: the same value, the same decision)
    {
      const double e_err = tot[r];
      if (kind == PK_V) {
        if (it >= 2) {
          stErr = e_err;
          if (A.tol_mode && e_err < A.tol) {
            final_t = it - 1;
            ferr = e_err;
            conv = 1;
          }
        }
      } else if (kind == PK_ERR) {
        stErr = e_err;
      }
      if (final_t < 0 && p == A.num_passes - 1) {
        final_t = A.T;
        ferr = A.want_err ? stErr : -1.0;
        conv = A.tol_mode ? (stErr < A.tol ? 1 : 0) : 0;
      }
    }
    if (final_t >= 0) break;
  }

  // returned scalings (u of the returned iterate; v of iteration final_t) and the read-out
  const float* vfin = vs + (final_t & 1) * nmax1;
  float* ug = A.out[0] + (int64_t)prob * A.wstride[0] + b0;
  float* vg = A.out[1] + (int64_t)prob * A.wstride[1] + b1;
  double la = 0.0, lb = 0.0;
  for (int i = tid; i < n0; i += kT) {
    ug[i] = us[i];
    la += (double)cw0[i] * log((double)us[i]);
  }
  for (int i = tid; i < n1; i += kT) {
    vg[i] = vfin[i];
    lb += (double)cw1[i] * log((double)vfin[i]);
  }
  la = warp_sum_f64(la);
  lb = warp_sum_f64(lb);
  const double bk = warp_sum_f64(brkT), wb = warp_sum_f64(wbT);
  __syncthreads();   // the last pass's readers of xs are done
  if (lane == 0) {
    xs[warp * 4 + 0] = la;
    xs[warp * 4 + 1] = lb;
    xs[warp * 4 + 2] = bk;
    xs[warp * 4 + 3] = wb;
  }
  __syncthreads();
  if (tid < 4) {
    double x = 0.0;
    for (int w = 0; w < kW; ++w) x += xs[w * 4 + tid];
    rdo[tid] = x;
  }
  cluster_sync_all();
  if (cta == 0 && tid == 0) {
    double x = 0.0, y = 0.0, stBrk = 0.0, stWb = 0.0;
    for (int c = 0; c < G; ++c) {
      x += ld_dsmem_f64(mapa_shared(smem_u32(rdo), (uint32_t)c));
      y += ld_dsmem_f64(mapa_shared(smem_u32(rdo + 1), (uint32_t)c));
      stBrk += ld_dsmem_f64(mapa_shared(smem_u32(rdo + 2), (uint32_t)c));
      stWb += ld_dsmem_f64(mapa_shared(smem_u32(rdo + 3), (uint32_t)c));
    }
    double* st = A.state + (int64_t)prob * kStateDoubles;
    st[ST_ITERS] = (double)final_t;
    st[ST_FINAL_A] = x;
    st[ST_FINAL_B] = y;
    st[ST_ROT] = A.eps * (x + y);
    st[ST_ERR] = ferr;
    st[ST_CONV] = (double)conv;
    st[ST_BRK] = stBrk;
    st[ST_WBAD] = stWb;
    sticky_flags(A, stBrk, stWb);
    __threadfence();
    st[ST_STOP] = 1.0;
  }
  cluster_sync_all();   // no CTA exits while CTA 0 reads its read-out partials
}

}  // namespace res

size_t resident_smem_bytes(int r, int64_t n, int64_t m, int G) {
  const int64_t n0 = (n + G - 1) / G, n1 = (m + G - 1) / G;
  return res::Lay(r, (int)n0, (int)n1, G).total;
}

// smallest cluster that holds the factors (<= 227 KB per CTA), then more CTAs while half the
// warps of every CTA still get a row batch (rows / G >= 4 warps x 8 rows).  Config 1 (500 rows,
// r = 100), us per pass for G = 4 / 8: 2.10 / 1.73 (grid kernels: 6.36)
int resident_cluster(int r, int64_t n, int64_t m) {
  if (r > 512 || (r & 3)) return 0;
  const size_t cap = 227 * 1024;
  const int64_t rows = std::max(n, m);
  int G = 0;
  for (int g = 1; g <= 8; g *= 2)
    if (rows >= g && resident_smem_bytes(r, n, m, g) <= cap) {
      G = g;
      break;
    }
  if (!G) return 0;
  while (G < 8 && rows / (2 * G) >= (int64_t)(res::kW / 2) * res::kTR &&
         resident_smem_bytes(r, n, m, 2 * G) <= cap)
    G *= 2;
  return G;
}

cudaError_t launch_resident(const SinkArgs& a, int G, int batch, cudaStream_t s) {
  const int n0 = (int)((a.rows[0] + G - 1) / G), n1 = (int)((a.rows[1] + G - 1) / G);
  const size_t dyn = res::Lay(a.r, n0, n1, G).total;
  const int ng = (a.r / 4 + 31) / 32;
  void (*kern)(const SinkArgs, int, int, int) = nullptr;
  if (ng <= 1) kern = res::resident_kernel<1>;
  else if (ng <= 2) kern = res::resident_kernel<2>;
  else if (ng <= 4) kern = res::resident_kernel<4>;
  else return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(G * batch));
  cfg.blockDim = dim3(res::kT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a, G, n0, n1);
  count_launch();
  return e;
}

}  // namespace lsk
