// lsk_implicit.cu — Alg. 1 on K_theta = xi zeta^T WITHOUT materialising
// the factors: every pass regenerates F_jk = phi(p_j, u_k)/sqrt(r) in registers from the
// point rows and the anchors (Lemma decomp-RBF, expanded in base 2):
//     F_jk = 2^( alpha2_j + beta2_k + sum_c W_kc p_jc ),
//     alpha2_j = -(2 log2e/eps)|p_j|^2, W_kc = (4 log2e/eps) U_kc,
//     beta2_k = log2e (-(2/eps)|U_k|^2 + |U_k|^2/(eps q) + log_scale)
// so a pass costs one MUFU ex2 + (d+3) FFMA-pipe ops per entry and ~(4d+12) bytes per row.
//
// Layout: one CTA per SM made of TEAMS independent teams of TS threads (all consumers, no
// producer warp: 512 threads x 128 registers).  A team owns every column: thread t of a
// team owns float4 column groups {t, t+TS, ...} (its W, beta2, slice of s and accumulators
// live in registers).  The teams take alternate tiles of the CTA's rows, each with its own
// loader warp (cp.async two tiles ahead into a 4-slot ring) and its own named barrier, so
// while one team waits on its per-tile row-dot exchange the other team issues MUFU work.
// The two teams' fp64 partials are added in a fixed order at the end of the pass.  Pass
// boundary, stopping test and the fp64 read-out are those of the streaming kernel.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {

namespace impl {

constexpr int kRing = 4;            // tile slots (two tiles in flight ahead of the current)
constexpr int kSlot = 64 + 32 * 8;  // floats per slot: c[32], vold[32], x[32][8]

template <int TS, int TEAMS>
struct Smem {
  float slot[TEAMS][kRing][kSlot];
  float red[TEAMS][2][TS / 32][32];
  double xs[2][TS * TEAMS / 32];
  double ext[kExtra];
};

template <int TS, int TEAMS, int NV, int TR, int D>
__global__ void __launch_bounds__(TS * TEAMS, 1) implicit_kernel(const SinkArgs A) {
  constexpr int NT = TS * TEAMS;       // CTA threads
  constexpr int NWT = TS / 32;         // warps per team
  constexpr int NW = NT / 32;
  constexpr int kFlushTiles = (32 / TR) > 0 ? (32 / TR) : 1;
  static_assert(TEAMS == 1 || TEAMS == 2 || TEAMS == 4, "1, 2 or 4 teams");
  __shared__ __align__(16) Smem<TS, TEAMS> S;
  // fp64 accumulators of every thread in shared memory (touched once per kFlushTiles tiles):
  // element-major so consecutive threads hit consecutive words
  extern __shared__ double acc_dyn[];   // dynamic: [NV * 4][NT]
  double (*acc_s)[NT] = reinterpret_cast<double (*)[NT]>(acc_dyn);

  const int tid = threadIdx.x;
  const int team = tid / TS, ttid = tid - team * TS;
  const int warp = tid >> 5, lane = tid & 31;
  const int twarp = ttid >> 5;          // warp index within the team
  const uint32_t team_bar = 2u + (uint32_t)team;   // ids 2..5 (1 = whole CTA)
  const int prob = blockIdx.x / A.gpp;
  const int cta = blockIdx.x - prob * A.gpp;
  const int r = A.r;
  double* stg_state = A.state + (int64_t)prob * kStateDoubles;
  if (__ldcg(stg_state + ST_STOP) != 0.0) return;   // finished (multi-launch mode)

  // per-thread anchor constants for the owned column groups
  const int R4 = r >> 2;
  int g[NV];
  bool gv[NV];
  float4 Wr[NV][D];
  float4 b2[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    g[j] = ttid + j * TS;
    gv[j] = g[j] < R4;
    if (gv[j]) {
      b2[j] = *reinterpret_cast<const float4*>(A.beta2 + 4 * g[j]);
#pragma unroll
      for (int c = 0; c < D; ++c) Wr[j][c] = *reinterpret_cast<const float4*>(A.Wt + (int64_t)c * r + 4 * g[j]);
    } else {   // padding groups produce exact zeros: ex2(-inf) = 0
      b2[j] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
      for (int c = 0; c < D; ++c) Wr[j][c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  for (int i = tid; i < TEAMS * kRing * kSlot; i += NT) (&S.slot[0][0][0])[i] = 0.f;
  __syncthreads();

  float4 s[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc_s[j * 4 + q][tid] = 0.0;
  }

  double stErr = __ldcg(stg_state + ST_ERR);
  double stBrk = __ldcg(stg_state + ST_BRK);
  const int64_t rstride = r + kExtra;
  double* part = A.part + (int64_t)prob * rstride * A.gpp;
  double* svec = A.svec + (int64_t)prob * rstride;
  const bool multi = A.multi_launch != 0;
  unsigned int nbar = 0;
  int final_t = -1, conv = 0;
  double ferr = -1.0;

  for (int p = A.pass_begin;; ++p) {
    // ---------------- results of pass q = p-1: stopping test (see lsk_sinkhorn.cu) -------
    const bool have_prev = multi ? (p == A.pass_begin && p > 0) : (p > A.pass_begin);
    if (have_prev) {
      const int q = p - 1;
      const int qk = pass_kind(q, A);
      double e_err, e_brk;
      if (A.gpp > 1) {
        e_err = __ldcg(svec + r);
        e_brk = __ldcg(svec + r + 1);
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
      if (final_t >= 0) break;
    }
    if (p >= A.pass_end) break;

    // ---------------- pass p ---------------------------------------------------------------
    const int kind = pass_kind(p, A);
    if (kind == PK_NONE) continue;
    const int f = (kind == PK_V || kind == PK_ERR) ? 1 : 0;
    if (kind != PK_INIT) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if (!gv[j]) {
          s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (A.gpp > 1) {
          const double2 lo = __ldcg(reinterpret_cast<const double2*>(svec + 4 * g[j]));
          const double2 hi = __ldcg(reinterpret_cast<const double2*>(svec + 4 * g[j] + 2));
          s[j] = make_float4((float)lo.x, (float)lo.y, (float)hi.x, (float)hi.y);
        } else {   // gpp == 1: the combined accumulator sits in team 0's slots
          s[j] = make_float4((float)acc_s[j * 4][ttid], (float)acc_s[j * 4 + 1][ttid],
                             (float)acc_s[j * 4 + 2][ttid], (float)acc_s[j * 4 + 3][ttid]);
        }
      }
      named_bar(1, NT);   // every team has read team 0's slots before they are cleared
    }
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc_s[j * 4 + q][tid] = 0.0;

    int64_t r0, r1;
    cta_rows(A.rows[f], A.gpp, cta, &r0, &r1);
    const int ntiles_cta = (int)((r1 - r0 + TR - 1) / TR);
    const int ntiles = (ntiles_cta - team + TEAMS - 1) / TEAMS;   // this team: tiles team, team+TEAMS, ...
    const float* wp = A.w[f] + (int64_t)prob * A.wstride[f];
    const float* Xp = A.X[f] + (int64_t)prob * A.fstride[f];
    const bool need_vold = (kind == PK_ERR) || (kind == PK_V && p >= 3);
    const bool err_here = need_vold;
    const float* vold = need_vold ? vbuf_ptr(A, prob, (kind == PK_ERR) ? A.T : (p + 1) / 2 - 1) : nullptr;
    float* outp = nullptr;
    if (kind == PK_U) outp = A.out[0] + (int64_t)prob * A.wstride[0];
    if (kind == PK_V) outp = vbuf_ptr(A, prob, (p + 1) / 2);
    double errsum = 0.0, brksum = 0.0;
    float4 acc32[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);

    // The tile loop is instantiated per pass kind (compile-time KIND: no per-tile kind
    // branches) with 32-bit row offsets relative to this CTA's first row.
    const int nrows = (int)(r1 - r0);
    const float* wp0 = wp + r0;
    const float* vold0 = need_vold ? vold + r0 : nullptr;
    const float* Xp0 = Xp + r0 * D;
    float* outp0 = outp ? outp + r0 : nullptr;

    auto run_tiles = [&](auto kind_tag) {
      constexpr int KIND = decltype(kind_tag)::value;
      constexpr bool kDot = KIND != PK_INIT;
      constexpr bool kAcc = KIND != PK_ERR;
      constexpr bool kOut = KIND == PK_U || KIND == PK_V;
      // warp 0 stages tile t (point rows + c_j + v_old_j) into slot t % kRing.  v_old_j was
      // written by this same lane two passes earlier (same tiling), so no extra ordering.
      auto issue = [&](int t) {
        if (t < ntiles) {
          const int lr = (team + t * TEAMS) * TR;
          float* sl = S.slot[team][t & (kRing - 1)];
          if (lane < nrows - lr && lane < TR) {
            cp_async4(sl + lane, wp0 + lr + lane);
            if (need_vold) cp_async4(sl + 32 + lane, vold0 + lr + lane);
#pragma unroll
            for (int c = 0; c < D; ++c) cp_async4(sl + 64 + lane * 8 + c, Xp0 + (lr + lane) * D + c);
          }
        }
        cp_async_commit();
      };
      if (twarp == 0) {
        issue(0);
        issue(1);
        cp_async_wait<1>();
      }
      named_bar(team_bar, TS);

      for (int t = 0; t < ntiles; ++t) {
        const int lr = (team + t * TEAMS) * TR;
        const int rows = min(TR, nrows - lr);
        const float* sl = S.slot[team][t & (kRing - 1)];
        if (twarp == 0) issue(t + 2);   // slot (t+2)%4 was last read in tile t-2

        // regenerate the TR x 4NV features of this thread (tail rows: finite stale/zero
        // data); packed fp32x2 arithmetic (FFMA2/FADD2): two columns per instruction
        float2 fr[TR][NV][2];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
          float x[D];
#pragma unroll
          for (int c = 0; c < D; ++c) x[c] = sl[64 + i * 8 + c];
          float al = 0.f;
#pragma unroll
          for (int c = 0; c < D; ++c) al = fmaf(x[c], x[c], al);
          al *= A.c2;
          const float2 al2 = make_float2(al, al);
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            float2 e01 = add2(al2, make_float2(b2[j].x, b2[j].y));
            float2 e23 = add2(al2, make_float2(b2[j].z, b2[j].w));
#pragma unroll
            for (int c = 0; c < D; ++c) {
              const float2 xc = make_float2(x[c], x[c]);
              e01 = fma2(make_float2(Wr[j][c].x, Wr[j][c].y), xc, e01);
              e23 = fma2(make_float2(Wr[j][c].z, Wr[j][c].w), xc, e23);
            }
            fr[i][j][0] = make_float2(ex2(e01.x), ex2(e01.y));
            fr[i][j][1] = make_float2(ex2(e23.x), ex2(e23.y));
          }
        }
        const int rb = t & 1;
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
          const float tot = warp_transpose_reduce<TR>(pr, lane);
          constexpr int kLanesPerRow = 32 / TR;
          if ((lane & (kLanesPerRow - 1)) == 0) S.red[team][rb][twarp][lane / kLanesPerRow] = tot;
        }
        if (twarp == 0) cp_async_wait<1>();   // tile t+1 has landed (only t+2 may be pending)
        named_bar(team_bar, TS);               // publishes red[rb] and slot (t+1) to the team

        float vr_l = 0.f;
        if constexpr (!kDot) {
          vr_l = (lane < rows) ? 1.f : 0.f;   // u^0 = 1 (reading C6)
        } else {
          if (lane < rows) {
            float tt = 0.f;
#pragma unroll
            for (int w = 0; w < NWT; ++w) tt += S.red[team][rb][w][lane];   // fixed order
            const float c = sl[lane];
            if constexpr (kAcc) vr_l = __fdiv_rn(c, tt);
            if (twarp == NWT - 1) {   // the loader is warp 0: outputs go to the last warp
              if (err_here) errsum += fabs((double)sl[32 + lane] * (double)tt - (double)c);
              if constexpr (kOut) {
                if (!(vr_l > 0.f) || !isfinite(vr_l)) brksum += 1.0;
                outp0[lr + lane] = vr_l;
              }
            }
          }
        }
        if constexpr (kAcc) {
#pragma unroll
          for (int i = 0; i < TR; ++i) {
            const float vi = __shfl_sync(0xffffffffu, vr_l, i);
            const float2 v2 = make_float2(vi, vi);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              const float2 lo = fma2(fr[i][j][0], v2, make_float2(acc32[j].x, acc32[j].y));
              const float2 hi = fma2(fr[i][j][1], v2, make_float2(acc32[j].z, acc32[j].w));
              acc32[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
            }
          }
          if ((t & (kFlushTiles - 1)) == kFlushTiles - 1) {
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              acc_s[j * 4 + 0][tid] += (double)acc32[j].x;
              acc_s[j * 4 + 1][tid] += (double)acc32[j].y;
              acc_s[j * 4 + 2][tid] += (double)acc32[j].z;
              acc_s[j * 4 + 3][tid] += (double)acc32[j].w;
              acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
        }
      }
    };
    switch (kind) {
      case PK_INIT: run_tiles(std::integral_constant<int, PK_INIT>{}); break;
      case PK_V: run_tiles(std::integral_constant<int, PK_V>{}); break;
      case PK_U: run_tiles(std::integral_constant<int, PK_U>{}); break;
      default: run_tiles(std::integral_constant<int, PK_ERR>{}); break;
    }
    if (twarp == 0) cp_async_wait<0>();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      acc_s[j * 4 + 0][tid] += (double)acc32[j].x;
      acc_s[j * 4 + 1][tid] += (double)acc32[j].y;
      acc_s[j * 4 + 2][tid] += (double)acc32[j].z;
      acc_s[j * 4 + 3][tid] += (double)acc32[j].w;
    }

    // ---------------- end of pass: teams combined (fixed order), cross-CTA fp64 reduction ---
    double e0 = 0.0, e1 = 0.0;
    if (twarp == NWT - 1) {
      e0 = warp_sum_f64(errsum);
      e1 = warp_sum_f64(brksum);
    }
    if (twarp == NWT - 1 && lane == 0) {   // hand the team's extras to its thread 0
      S.xs[0][NW - 1 - team] = e0;
      S.xs[1][NW - 1 - team] = e1;
    }
    named_bar(1, NT);
    if (ttid == 0) {
      e0 = S.xs[0][NW - 1 - team];
      e1 = S.xs[1][NW - 1 - team];
    }
    named_bar(1, NT);
    if constexpr (TEAMS > 1) {
      if (team > 0 && ttid == 0) {
        S.xs[0][team] = e0;
        S.xs[1][team] = e1;
      }
      named_bar(1, NT);
      if (team == 0) {   // fixed order: team 0 + team 1 + ... (deterministic)
#pragma unroll
        for (int tm = 1; tm < TEAMS; ++tm) {
#pragma unroll
          for (int e = 0; e < NV * 4; ++e) acc_s[e][ttid] += acc_s[e][ttid + tm * TS];
          if (ttid == 0) {
            e0 += S.xs[0][tm];
            e1 += S.xs[1][tm];
          }
        }
      }
      named_bar(1, NT);
    }
    unsigned long long* trc = (A.trace && tid == 0) ? A.trace + ((int64_t)p * A.gpp + cta) * 4 : nullptr;
    if (trc) trc[0] = globaltimer();
    if (A.gpp > 1) {
      if (team == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (gv[j]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) part[(int64_t)(4 * g[j] + q) * A.gpp + cta] = acc_s[j * 4 + q][ttid];
          }
        }
      }
      if (tid == 0) {
        part[(int64_t)(r + 0) * A.gpp + cta] = e0;
        part[(int64_t)(r + 1) * A.gpp + cta] = e1;
        part[(int64_t)(r + 2) * A.gpp + cta] = 0.0;
        part[(int64_t)(r + 3) * A.gpp + cta] = 0.0;
      }
      group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
      if (trc) trc[1] = globaltimer();
      for (int k = cta + A.gpp * warp; k < r + kExtra; k += A.gpp * NW) {
        const double* col = part + (int64_t)k * A.gpp;
        double acc = 0.0;
#pragma unroll 4
        for (int i = lane; i < A.gpp; i += 32) acc += __ldcg(col + i);
        acc = warp_sum_f64(acc);
        if (lane == 0) svec[k] = acc;
      }
      if (trc) trc[2] = globaltimer();
      if (!multi) group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
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
      for (int w = 0; w < NW; ++w) {
        la += S.xs[0][w];
        lb += S.xs[1][w];
      }
    }
    if (A.gpp > 1) {
      if (tid == 0) {
        part[cta] = la;
        part[A.gpp + cta] = lb;
      }
      group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
      if (cta == 0 && tid == 0) {
        la = 0.0;
        lb = 0.0;
        for (int c = 0; c < A.gpp; ++c) {
          la += __ldcg(part + c);
          lb += __ldcg(part + A.gpp + c);
        }
      }
    }
    if (cta == 0 && tid == 0) {
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

}  // namespace impl

// (TS, TEAMS, NV, TR) per r: r <= 1024 -> (256, 2, 1, 8); r <= 2048 -> (512, 1, 1, 8);
// r <= 4096 -> (512, 1, 2, 2).  Always 512 threads, one CTA per SM.
void implicit_config(int r, int* nt, int* nv, int* tr) {
  const int r4 = (r + 3) / 4;
  if (r4 <= 256) {
    // four 128-thread teams, 8 columns per thread (halves the per-entry exchange overhead)
    *nt = 128; *nv = 2; *tr = 4;
    if (const char* e = getenv("LSK_ITEAM")) {   // tuning knob: 2 = two 256-thread teams
      if (atoi(e) == 2) { *nt = 256; *nv = 1; *tr = 8; }
    }
  }
  else if (r4 <= 512) { *nt = 512; *nv = 1; *tr = 8; }
  else {
    *nt = 512; *nv = 2; *tr = 4;
    if (const char* e = getenv("LSK_ITR")) *tr = atoi(e) == 2 ? 2 : 4;   // tuning knob
  }
}

#define LSK_IMPL2(X, TS, TM, NV, TR) X(TS, TM, NV, TR, 1) X(TS, TM, NV, TR, 2) \
  X(TS, TM, NV, TR, 3) X(TS, TM, NV, TR, 4) X(TS, TM, NV, TR, 5) X(TS, TM, NV, TR, 6)     \
  X(TS, TM, NV, TR, 7) X(TS, TM, NV, TR, 8)
#define LSK_IMPL2_ALL(X) LSK_IMPL2(X, 256, 2, 1, 8) LSK_IMPL2(X, 128, 4, 2, 4) LSK_IMPL2(X, 512, 1, 1, 8) \
  LSK_IMPL2(X, 512, 1, 2, 2) LSK_IMPL2(X, 512, 1, 2, 4)

cudaError_t launch_implicit(const SinkArgs& a, bool coop, int grid, cudaStream_t s) {
  int ts, nv, tr;
  implicit_config(a.r, &ts, &nv, &tr);
#define X(TS_, TM_, NV_, TR_, D_)                                                              \
  if (ts == TS_ && nv == NV_ && tr == TR_ && a.d == D_) {                                      \
    auto kern = impl::implicit_kernel<TS_, TM_, NV_, TR_, D_>;                                 \
    const size_t dyn = sizeof(double) * NV_ * 4 * TS_ * TM_;                                   \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn); \
    if (e != cudaSuccess) return e;                                                            \
    if (coop) {                                                                                \
      void* args[] = {(void*)&a};                                                              \
      e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(TS_ * TM_), args, dyn, s); \
    } else {                                                                                   \
      kern<<<grid, TS_ * TM_, dyn, s>>>(a);                                                    \
      e = cudaGetLastError();                                                                  \
    }                                                                                          \
    count_launch();                                                                            \
    return e;                                                                                  \
  }
  LSK_IMPL2_ALL(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

int implicit_max_ctas_per_sm(int r, int d) {
  int ts, nv, tr;
  implicit_config(r, &ts, &nv, &tr);
#define X(TS_, TM_, NV_, TR_, D_)                                                              \
  if (ts == TS_ && nv == NV_ && tr == TR_ && d == D_) {                                        \
    int nb = 0;                                                                                \
    const size_t dyn = sizeof(double) * NV_ * 4 * TS_ * TM_;                                   \
    cudaFuncSetAttribute(impl::implicit_kernel<TS_, TM_, NV_, TR_, D_>,                        \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);               \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, impl::implicit_kernel<TS_, TM_, NV_, TR_, D_>, TS_ * TM_, dyn); \
    return nb;                                                                                 \
  }
  LSK_IMPL2_ALL(X)
#undef X
  return 0;
}

}  // namespace lsk
