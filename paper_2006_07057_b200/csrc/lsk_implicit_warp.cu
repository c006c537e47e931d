// lsk_implicit_warp.cu — the recompute (implicit) Sinkhorn pass for r <= 1024 with WARP-PRIVATE
// rows: Alg. 1 on K_theta = xi zeta^T, F_jk regenerated in registers
// (Lemma decomp-RBF, base 2; factored form as in lsk_implicit.cu):
//     F_jk = h_j G_jk,  G_jk = 2^(beta2_k + abar + sum_c W_kc p_jc),  h_j = 2^(alpha2_j - abar)
// (FACT; h = 1, abar = 0 and alpha2_j added per entry otherwise).
//
// Each warp owns ALL r columns (lane l owns float4 column groups {l, l+32, ...}: 4*NV columns)
// and processes its own tiles of TR rows (tiles warp, warp+NWARP, ... of the CTA's rows).  A
// row dot t_j = F_j . s is therefore complete after a warp transpose-reduce: the tile loop has
// no shared-memory exchange, no named barrier and no mbarrier — every warp runs independently
// and the scheduler interleaves one warp's shuffle/rcp chain with another warp's MUFU work.
// Each warp stages its tiles (c_j, h_j, v_old_j, point rows) kAhead tiles ahead with cp.async
// into a private smem ring (cp.async.wait_group + __syncwarp: no cross-warp ordering).  The
// fp32 accumulators (<= 32 rows) flush into per-warp fp64 accumulators in shared memory; the
// warps' accumulators are added in a fixed order at the end of the pass (deterministic).  Pass
// boundary (R1 / group barrier / R2), stopping test and fp64 read-out follow lsk_sinkhorn.cu.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {

namespace implw {

constexpr int kAhead = 6;           // tiles staged ahead of the one being computed
constexpr int kRing = kAhead + 2;   // slots per warp

template <int TR, int D>
struct Geo {
  static constexpr int XS = D <= 4 ? 4 : 8;                   // floats per staged point row
  static constexpr int SLOT = ((3 * TR + 3) / 4) * 4 + TR * XS;   // c[TR] h[TR] vold[TR] | x[TR][XS]
  static constexpr int XOFF = ((3 * TR + 3) / 4) * 4;
};

template <int NWARP>
struct Smem {
  double xs[2][NWARP];
  double ext[kExtra];
  double errL[NWARP][32];   // per-lane marginal-error sums (lanes that own a row)
  double brkL[NWARP][32];   // per-lane breakdown counts
  double st[3];             // running solve state: err, breakdowns, final err
  int ist[2];               // final_t, conv
};

template <int NWARP, int NV, int TR, int D, bool FACT>
__global__ void __launch_bounds__(NWARP * 32, 1) implicit_warp_kernel(const SinkArgs A) {
  constexpr int NT = NWARP * 32;
  constexpr int NE = NV * 4;                      // columns per lane
  constexpr int XS = Geo<TR, D>::XS, SLOT = Geo<TR, D>::SLOT, XOFF = Geo<TR, D>::XOFF;
  constexpr int kFlushTiles = (32 / TR) > 0 ? (32 / TR) : 1;
  constexpr int LPR = 32 / TR;                    // lanes per row after the transpose-reduce
  __shared__ __align__(16) Smem<NWARP> S;
  // dynamic: per-warp fp64 accumulators [NWARP][NE][32] (lane-consecutive), then the rings
  extern __shared__ double dyn[];
  double* accw = dyn;
  float* rings = reinterpret_cast<float*>(dyn + NWARP * NE * 32);
  float4* s_sm = reinterpret_cast<float4*>(rings + NWARP * kRing * SLOT);   // [NV * 32] s in fp32

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int prob = blockIdx.x / A.gpp;
  const int cta = blockIdx.x - prob * A.gpp;
  const int r = A.r;
  double* stg_state = A.state + (int64_t)prob * kStateDoubles;
  if (__ldcg(stg_state + ST_STOP) != 0.0) return;   // finished (multi-launch mode)

  double* myacc = accw + warp * NE * 32;
  float* ring = rings + warp * kRing * SLOT;
  for (int i = lane; i < kRing * SLOT; i += 32) ring[i] = 0.f;   // tail rows: finite data
  for (int e = 0; e < NE; ++e) myacc[e * 32 + lane] = 0.0;

  // per-lane anchor constants (float pairs for FFMA2)
  const int R4 = r >> 2;
  float2 W2[NV][D][2];
  float2 B2[NV][2];
  const float boff = FACT ? A.abar : 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int g = lane + 32 * j;
    if (g < R4) {
      const float4 b = *reinterpret_cast<const float4*>(A.beta2 + 4 * g);
      B2[j][0] = make_float2(b.x + boff, b.y + boff);
      B2[j][1] = make_float2(b.z + boff, b.w + boff);
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const float4 w = *reinterpret_cast<const float4*>(A.Wt + (int64_t)c * r + 4 * g);
        W2[j][c][0] = make_float2(w.x, w.y);
        W2[j][c][1] = make_float2(w.z, w.w);
      }
    } else {   // padding groups produce exact zeros: ex2(-inf) = 0
      B2[j][0] = B2[j][1] = make_float2(-INFINITY, -INFINITY);
#pragma unroll
      for (int c = 0; c < D; ++c) W2[j][c][0] = W2[j][c][1] = make_float2(0.f, 0.f);
    }
  }

  double& stErr = S.st[0];
  double& stBrk = S.st[1];
  double& ferr = S.st[2];
  int& final_t = S.ist[0];
  int& conv = S.ist[1];
  if (tid == 0) {
    stErr = __ldcg(stg_state + ST_ERR);
    stBrk = __ldcg(stg_state + ST_BRK);
    ferr = -1.0;
    final_t = -1;
    conv = 0;
  }
  S.errL[warp][lane] = 0.0;
  S.brkL[warp][lane] = 0.0;
  __syncthreads();

  float4 s[NV];
  const int64_t rstride = r + kExtra;
  double* part = A.part + prob * part_per_problem(r, A.gpp);   // [blk][gpp][4]
  const bool multi = A.multi_launch != 0;
  unsigned int nbar = 0;

  for (int p = A.pass_begin;; ++p) {
    // ---------------- results of pass q = p-1: stopping test (see lsk_sinkhorn.cu) -------
    const bool have_prev = multi ? (p == A.pass_begin && p > 0) : (p > A.pass_begin);
    if (have_prev) {
      if (tid == 0) {
        const int q = p - 1;
        const int qk = pass_kind(q, A);
        double e_err, e_brk;
        if (A.gpp > 1) {
          e_err = sv_load(sv_of(A, prob, q) + r, multi);
          e_brk = sv_load(sv_of(A, prob, q) + r + 1, multi);
        } else {
          e_err = S.ext[0];
          e_brk = S.ext[1];
        }
        stBrk += e_brk;
        if (qk == PK_V) {
          const int t = (q + 1) / 2;
          if (t >= 2) {
            stErr = e_err;
            if (A.tol_mode && e_err < A.tol) {
              final_t = t - 1;
              ferr = e_err;
              conv = 1;
            }
          }
        } else if (qk == PK_ERR) {
          stErr = e_err;
        }
        if (final_t < 0 && q == A.num_passes - 1) {
          final_t = A.T;
          ferr = A.want_err ? stErr : -1.0;
          conv = A.tol_mode ? (stErr < A.tol ? 1 : 0) : 0;
        }
      }
      named_bar(1, NT);
      if (final_t >= 0) break;
    }
    if (p >= A.pass_end) break;

    // ---------------- pass p ---------------------------------------------------------------
    const int kind = pass_kind(p, A);
    if (kind == PK_NONE) continue;
    const int f = (kind == PK_V || kind == PK_ERR) ? 1 : 0;
    if (kind != PK_INIT) {
      // s (fp64 in L2 or in warp 0's accumulators) -> fp32 in shared memory ONCE per CTA: the
      // warps then read it from smem (148 CTAs x every warp reading the same 8 KB of L2 would
      // hot-spot the L2 slices holding it)
      for (int g = tid; g < NV * 32; g += NT) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g < R4) {
          if (A.gpp > 1) {
            double2 lo, hi;
            sv_load4(sv_of(A, prob, p - 1) + 4 * g, multi, lo, hi);
            v = make_float4((float)lo.x, (float)lo.y, (float)hi.x, (float)hi.y);
          } else {   // element (4 j + q) * 32 + l holds column 4 (l + 32 j) + q
            const int l = g & 31, j = g >> 5;
            v = make_float4((float)accw[(4 * j + 0) * 32 + l], (float)accw[(4 * j + 1) * 32 + l],
                            (float)accw[(4 * j + 2) * 32 + l], (float)accw[(4 * j + 3) * 32 + l]);
          }
        }
        s_sm[g] = v;
      }
      named_bar(1, NT);   // s staged; every warp is done with warp 0's accumulators
#pragma unroll
      for (int j = 0; j < NV; ++j) s[j] = s_sm[lane + 32 * j];
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) myacc[e * 32 + lane] = 0.0;

    int64_t r0, r1;
    cta_rows(A.rows[f], A.gpp, cta, &r0, &r1);
    const int nrows = (int)(r1 - r0);
    const int ntiles_cta = (nrows + TR - 1) / TR;
    const int ntiles = (ntiles_cta - warp + NWARP - 1) / NWARP;   // tiles warp, warp+NWARP, ...
    const float* wp0 = A.w[f] + (int64_t)prob * A.wstride[f] + r0;
    const float* Xp0 = A.X[f] + (int64_t)prob * A.fstride[f] + r0 * D;
    const float* hp0 = FACT ? A.hrow[f] + (int64_t)prob * A.wstride[f] + r0 : nullptr;
    const bool need_vold = (kind == PK_ERR) || (kind == PK_V && p >= 3);
    const float* vold0 =
        need_vold ? vbuf_ptr(A, prob, (kind == PK_ERR) ? A.T : (p + 1) / 2 - 1) + r0 : nullptr;
    float* outp0 = nullptr;
    if (kind == PK_U) outp0 = A.out[0] + (int64_t)prob * A.wstride[0] + r0;
    if (kind == PK_V) outp0 = vbuf_ptr(A, prob, (p + 1) / 2) + r0;
    float4 acc32[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);

    auto run_tiles = [&](auto kind_tag) {
      constexpr int KIND = decltype(kind_tag)::value;
      constexpr bool kDot = KIND != PK_INIT;
      constexpr bool kAcc = KIND != PK_ERR;
      constexpr bool kOut = KIND == PK_U || KIND == PK_V;
      // stage tile t of this warp (slot t % kRing); one commit group per tile, even if empty
      auto issue = [&](int t) {
        if (t < ntiles) {
          const int lr = (warp + t * NWARP) * TR;
          float* sl = ring + (t % kRing) * SLOT;
          const int rows = min(TR, nrows - lr);
          if (lane < rows) {
            cp_async4(sl + lane, wp0 + lr + lane);
            if (FACT) cp_async4(sl + TR + lane, hp0 + lr + lane);
            if (need_vold) cp_async4(sl + 2 * TR + lane, vold0 + lr + lane);
          }
          if (lane < rows * D) {
            const int i = lane / D, c = lane - i * D;
            cp_async4(sl + XOFF + i * XS + c, Xp0 + (lr + i) * D + c);
          }
          if constexpr (TR * D > 32) {
            for (int e = lane + 32; e < rows * D; e += 32) {
              const int i = e / D, c = e - i * D;
              cp_async4(sl + XOFF + i * XS + c, Xp0 + (lr + i) * D + c);
            }
          }
        }
        cp_async_commit();
      };
#pragma unroll
      for (int t = 0; t < kAhead; ++t) issue(t);
      int nfin = 0;
      for (int t = 0; t < ntiles; ++t) {
        issue(t + kAhead);
        cp_async_wait<kAhead>();
        __syncwarp();
        const int lr = (warp + t * NWARP) * TR;
        const int rows = min(TR, nrows - lr);
        const float* sl = ring + (t % kRing) * SLOT;
        float2 fr[TR][NV][2];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
          float x[XS];
          {
            const float4 x0 = lds128(sl + XOFF + i * XS);
            x[0] = x0.x; if (XS > 1) x[1] = x0.y;
            if (XS > 2) x[2] = x0.z;
            if (XS > 3) x[3] = x0.w;
            if constexpr (XS > 4) {
              const float4 x1 = lds128(sl + XOFF + i * XS + 4);
              x[4] = x1.x; x[5] = x1.y; x[6] = x1.z; x[7] = x1.w;
            }
          }
          float2 al2 = make_float2(0.f, 0.f);
          if constexpr (!FACT) {
            float al = 0.f;
#pragma unroll
            for (int c = 0; c < D; ++c) al = fmaf(x[c], x[c], al);
            al *= A.c2;
            al2 = make_float2(al, al);
          }
#pragma unroll
          for (int j = 0; j < NV; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float2 e = FACT ? B2[j][h] : add2(al2, B2[j][h]);
#pragma unroll
              for (int c = 0; c < D; ++c) e = fma2(W2[j][c][h], make_float2(x[c], x[c]), e);
              fr[i][j][h] = make_float2(ex2(e.x), ex2(e.y));
            }
          }
        }
        const int row = lane / LPR;
        const bool valid = row < rows;
        float wt = 0.f;
        if constexpr (kDot) {
          float pr[TR];
#pragma unroll
          for (int i = 0; i < TR; ++i) {
            float2 pp = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              pp = fma2(fr[i][j][0], make_float2(s[j].x, s[j].y), pp);
              pp = fma2(fr[i][j][1], make_float2(s[j].z, s[j].w), pp);
            }
            pr[i] = pp.x + pp.y;
          }
          const float tot = warp_transpose_reduce<TR>(pr, lane);   // row `row`, every lane of it
          if (valid) {
            const float c = sl[row];
            const float h = FACT ? sl[TR + row] : 1.f;
            const float tj = FACT ? h * tot : tot;     // t_j = F_j . s
            const float w = c * rcp_approx(tj);        // w_j = c_j / t_j
            wt = FACT ? w * h : w;
            if ((lane & (LPR - 1)) == 0) {             // outputs: one lane per row
              if (need_vold) S.errL[warp][lane] += fabs((double)sl[2 * TR + row] * (double)tj - (double)c);
              if constexpr (kOut) {
                if (!(w > 0.f) || !isfinite(w)) S.brkL[warp][lane] += 1.0;
                outp0[lr + row] = w;
              }
            }
          }
          if constexpr (!kAcc) wt = 0.f;
        } else {
          if (valid) wt = FACT ? sl[TR + row] : 1.f;   // u^0 = 1 (reading C6): w~ = h
        }
        if constexpr (kAcc) {
#pragma unroll
          for (int i = 0; i < TR; ++i) {
            const float vi = __shfl_sync(0xffffffffu, wt, i * LPR);
            const float2 v2 = make_float2(vi, vi);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              const float2 lo = fma2(fr[i][j][0], v2, make_float2(acc32[j].x, acc32[j].y));
              const float2 hi = fma2(fr[i][j][1], v2, make_float2(acc32[j].z, acc32[j].w));
              acc32[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
            }
          }
          if (++nfin == kFlushTiles) {
            nfin = 0;
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
        __syncwarp();   // slot t is read before it is restaged (t + kRing)
      }
    };
    switch (kind) {
      case PK_INIT: run_tiles(std::integral_constant<int, PK_INIT>{}); break;
      case PK_V: run_tiles(std::integral_constant<int, PK_V>{}); break;
      case PK_U: run_tiles(std::integral_constant<int, PK_U>{}); break;
      default: run_tiles(std::integral_constant<int, PK_ERR>{}); break;
    }
    cp_async_wait<0>();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      myacc[(4 * j + 0) * 32 + lane] += (double)acc32[j].x;
      myacc[(4 * j + 1) * 32 + lane] += (double)acc32[j].y;
      myacc[(4 * j + 2) * 32 + lane] += (double)acc32[j].z;
      myacc[(4 * j + 3) * 32 + lane] += (double)acc32[j].w;
    }

    // ---------------- end of pass: warps combined (fixed order), cross-CTA fp64 reduction ---
    {
      const double e0w = warp_sum_f64(S.errL[warp][lane]);
      const double e1w = warp_sum_f64(S.brkL[warp][lane]);
      S.errL[warp][lane] = 0.0;
      S.brkL[warp][lane] = 0.0;
      if (lane == 0) {
        S.xs[0][warp] = e0w;
        S.xs[1][warp] = e1w;
      }
    }
    named_bar(1, NT);
    for (int e = tid; e < NE * 32; e += NT) {   // warp 0 + warp 1 + ... (deterministic)
      double acc = accw[e];
#pragma unroll
      for (int w = 1; w < NWARP; ++w) acc += accw[w * NE * 32 + e];
      accw[e] = acc;
    }
    double e0 = 0.0, e1 = 0.0;
    if (tid == 0) {
      for (int w = 0; w < NWARP; ++w) {
        e0 += S.xs[0][w];
        e1 += S.xs[1][w];
      }
    }
    named_bar(1, NT);
    unsigned long long* trc = (A.trace && tid == 0) ? A.trace + ((int64_t)p * A.gpp + cta) * 4 : nullptr;
    if (trc) trc[0] = globaltimer();
    if (A.gpp > 1) {
      for (int e = tid; e < NE * 32; e += NT) {   // element e = (4 j + q) * 32 + l: column 4(l + 32 j) + q
        const int l = e & 31, jq = e >> 5;
        const int col = 4 * (l + 32 * (jq >> 2)) + (jq & 3);
        if (col < r) *part_at(part, A.gpp, col, cta) = accw[e];
      }
      if (tid == 0) part_store4(part, A.gpp, r >> 2, cta, e0, e1, 0.0, 0.0);
      group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
      if (trc) trc[1] = globaltimer();
      // R2: this CTA reduces column blocks kb = cta, cta+gpp, ... (block r/4: the extras)
      r2_cta(A, prob, p, part, cta, warp, NWARP, lane);
      if (trc) trc[2] = globaltimer();
      if (trc) trc[3] = globaltimer();
    } else {
      if (tid == 0) {
        S.ext[0] = e0;
        S.ext[1] = e1;
      }
      named_bar(1, NT);
    }
  }

  if (final_t >= 0) {
    // returned v into the user buffer, then W_hat = eps (a^T log u + b^T log v) in fp64
    int64_t u0, u1, v0, v1;
    cta_rows(A.rows[0], A.gpp, cta, &u0, &u1);
    cta_rows(A.rows[1], A.gpp, cta, &v0, &v1);
    float* vdst = A.out[1] + (int64_t)prob * A.wstride[1];
    const float* udst = A.out[0] + (int64_t)prob * A.wstride[0];
    if ((final_t ^ A.T) & 1) {
      const float* src = A.vbuf1 + (int64_t)prob * A.wstride[1];
      for (int64_t i = v0 + tid; i < v1; i += NT) vdst[i] = __ldcg(src + i);
    }
    named_bar(1, NT);
    const float* ap = A.w[0] + (int64_t)prob * A.wstride[0];
    const float* bp = A.w[1] + (int64_t)prob * A.wstride[1];
    double la = 0.0, lb = 0.0;
    for (int64_t i = u0 + tid; i < u1; i += NT) la += (double)ap[i] * log((double)__ldcg(udst + i));
    for (int64_t i = v0 + tid; i < v1; i += NT) lb += (double)bp[i] * log((double)__ldcg(vdst + i));
    la = warp_sum_f64(la);
    lb = warp_sum_f64(lb);
    if (lane == 0) {
      S.xs[0][warp] = la;
      S.xs[1][warp] = lb;
    }
    named_bar(1, NT);
    if (tid == 0) {
      la = 0.0;
      lb = 0.0;
      for (int w = 0; w < NWARP; ++w) {
        la += S.xs[0][w];
        lb += S.xs[1][w];
      }
    }
    if (A.gpp > 1) {
      if (tid == 0) {
        *part_at(part, A.gpp, (int)rstride, cta) = la;       // columns r+kExtra, r+kExtra+1:
        *part_at(part, A.gpp, (int)rstride + 1, cta) = lb;   // never read by R2 (no race with it)
      }
      group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
      if (cta == 0 && tid == 0) {
        la = 0.0;
        lb = 0.0;
        for (int c = 0; c < A.gpp; ++c) {
          la += __ldcg(part_at(part, A.gpp, (int)rstride, c));
          lb += __ldcg(part_at(part, A.gpp, (int)rstride + 1, c));
        }
      }
    }
    if (cta == 0 && tid == 0) {
      if (A.nranks > 1) {   // all-rank read-out: columns r+kExtra, r+kExtra+1 of parity 0
        la = xrank_total(A, prob, 0, (int)rstride, la);
        lb = xrank_total(A, prob, 0, (int)rstride + 1, lb);
      }
      stg_state[ST_ITERS] = (double)final_t;
      stg_state[ST_FINAL_A] = la;
      stg_state[ST_FINAL_B] = lb;
      stg_state[ST_ROT] = A.eps * (la + lb);
      stg_state[ST_ERR] = ferr;
      stg_state[ST_CONV] = (double)conv;
      stg_state[ST_BRK] = stBrk;
      __threadfence();
      stg_state[ST_STOP] = 1.0;
    }
  } else if (multi && cta == 0 && tid == 0) {
    stg_state[ST_ERR] = stErr;
    stg_state[ST_BRK] = stBrk;
  }
}

template <int NWARP, int NV, int TR, int D>
constexpr size_t dyn_smem() {
  return sizeof(double) * NWARP * NV * 4 * 32 + sizeof(float) * NWARP * kRing * Geo<TR, D>::SLOT +
         sizeof(float4) * NV * 32;
}

}  // namespace implw

// Warp-private configurations: (NWARP, NV, TR) by r and d.  32 columns per lane (r <= 1024)
// needs 255 registers at d <= 2 (W, beta2, s and accumulators all per lane), so larger d
// there uses the team kernel (lsk_implicit.cu).  LSK_IWCFG="nwarp,nv,tr" selects another
// instantiated configuration (tuning knob).
bool implicit_warp_config(int r, int d, int* nwarp, int* nv, int* tr) {
  const int r4 = (r + 3) / 4;
  if (r4 > 256 || (r4 > 128 && d > 2)) return false;
  if (r4 <= 32) { *nwarp = 16; *nv = 1; *tr = 4; }
  else if (r4 <= 64) { *nwarp = 16; *nv = 2; *tr = 4; }
  else if (r4 <= 128) { *nwarp = 8; *nv = 4; *tr = 2; }
  else { *nwarp = 8; *nv = 8; *tr = 1; }
  if (const char* e = getenv("LSK_IWCFG")) {
    int a, b, c;
    if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && b * 128 >= r) { *nwarp = a; *nv = b; *tr = c; }
  }
  return true;
}

#define LSK_IW_D(X, NW, NV, TR) X(NW, NV, TR, 1) X(NW, NV, TR, 2) X(NW, NV, TR, 3) X(NW, NV, TR, 4) \
  X(NW, NV, TR, 5) X(NW, NV, TR, 6) X(NW, NV, TR, 7) X(NW, NV, TR, 8)
#define LSK_IW_D12(X, NW, NV, TR) X(NW, NV, TR, 1) X(NW, NV, TR, 2)
#define LSK_IW_ALL(X) LSK_IW_D(X, 16, 1, 4) LSK_IW_D(X, 16, 2, 4) LSK_IW_D(X, 8, 4, 2) \
  LSK_IW_D12(X, 8, 8, 1) X(8, 8, 2, 2) X(16, 4, 2, 2) X(8, 4, 4, 2)

template <int NW, int NV, int TR, int D, bool FACT>
static cudaError_t launch_w(const SinkArgs& a, bool coop, int grid, cudaStream_t s, int* occ) {
  auto kern = implw::implicit_warp_kernel<NW, NV, TR, D, FACT>;
  constexpr size_t dyn = implw::dyn_smem<NW, NV, TR, D>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  if (occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, NW * 32, dyn);
    return cudaSuccess;
  }
  if (coop) {
    void* args[] = {(void*)&a};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(NW * 32), args, dyn, s);
  } else {
    kern<<<grid, NW * 32, dyn, s>>>(a);
    e = cudaGetLastError();
  }
  count_launch();
  return e;
}

// occ != NULL: report CTAs per SM instead of launching
cudaError_t launch_implicit_warp(const SinkArgs& a, bool coop, int grid, cudaStream_t s, int* occ) {
  int nw, nv, tr;
  if (!implicit_warp_config(a.r, a.d, &nw, &nv, &tr)) return cudaErrorInvalidConfiguration;
  const bool fact = a.hrow[0] != nullptr;
#define X(NW_, NV_, TR_, D_)                                                      \
  if (nw == NW_ && nv == NV_ && tr == TR_ && a.d == D_)                           \
    return fact ? launch_w<NW_, NV_, TR_, D_, true>(a, coop, grid, s, occ)        \
                : launch_w<NW_, NV_, TR_, D_, false>(a, coop, grid, s, occ);
  LSK_IW_ALL(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

}  // namespace lsk
