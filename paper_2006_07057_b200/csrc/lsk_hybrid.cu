// lsk_hybrid.cu — Alg. 1 on K_theta = xi zeta^T with BOTH the MUFU and the
// HBM working in one persistent launch (warp-specialised hybrid, DESIGN.md §6 K8).
//
// The recompute kernel (lsk_implicit.cu) regenerates every entry F_jk with one MUFU ex2 and
// leaves HBM idle; the factor stream (lsk_sinkhorn.cu) reads every entry from HBM and leaves
// the MUFU idle.  Here the first phi n rows of xi (phi m of zeta) are materialised once per
// solve (the FFMA feature map) and, in every pass, streamed from HBM by a third team of the
// CTA, while two recompute teams regenerate the remaining rows.  The two row sets are disjoint,
// so every pass still computes exactly t_j = F_j . s, w_j = c_j / t_j and s' = sum_j F_j w_j
// over all rows; the three teams' fp64 partials are added in a fixed
// order (team 0 + team 1 + stream team: deterministic) before the usual cross-CTA reduction.
// phi balances the two rates: rows / (recompute rate) = rows / (HBM rate).
//
// Roles (384 threads, one CTA per SM):
//   warps 0-7   two recompute teams of 128 threads — the (128, 2, 2, 16) tile loop of
//               implicit_kernel (8 columns per thread, 16-row tiles);
//   warps 8-11  the stream team: 128 threads, the same column ownership (groups t, t + 128),
//               8-row tiles of materialised rows brought in by 1-D bulk copies (TMA engine,
//               mbarrier complete_tx) into a 4-stage shared-memory ring.
// Registers: the launch gives 384 x 168; the recompute teams raise theirs to 216
// (setmaxnreg.inc; their tile loop measured spill-free at 216) and the stream team lowers its
// own to 72 (setmaxnreg.dec): 256 x 216 + 128 x 72 = 384 x 168.  ptxas applies a raised
// limit only to code that runs after it, so each role runs its own copy of the whole pass loop
// (a role-templated body); the two copies meet only at the CTA-wide named barrier 1 with the
// same sequence of arrivals per pass.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {
namespace hyb {

constexpr int TS = 128;            // threads per team
constexpr int TEAMS = 2;           // recompute teams
constexpr int NV = 2;              // float4 column groups per thread (r <= 1024)
constexpr int TR = 16;             // recompute rows per tile
constexpr int TRS = 8;             // streamed rows per tile
constexpr int NSTG = 4;            // stream ring stages
constexpr int HDR = 64;            // stage header floats: c[32], v_old[32]
constexpr int NT = TS * (TEAMS + 1);
constexpr int NW = NT / 32;
constexpr int NWT = TS / 32;
constexpr int kRing = 8;           // recompute tile slots per team
constexpr int kAhead = 2;
constexpr int kRegCompute = 216;
constexpr int kRegStream = 72;

static_assert(TEAMS * TS * kRegCompute + TS * kRegStream <= NT * 168, "register split");

template <int D>
struct Geo {
  static constexpr int XS = D <= 4 ? 4 : 8;
  static constexpr int SLOT = 96 + 32 * XS;   // c[32] h[32] vold[32] x[32][XS]
};

__host__ __device__ constexpr int exchange_lanes(int nwt, int lpr) {
  int g = nwt < lpr ? nwt : lpr;
  while (nwt % g) --g;
  return g;
}

struct Smem {
  uint64_t full[TEAMS][kRing];     // recompute tile slots landed (32 cp.async arrivals)
  uint64_t sfull[NSTG];            // stream stages landed (tx bytes + 32 cp.async arrivals)

  float red[TEAMS + 1][3][TR][NWT];
  double xs[3][NW];
  double errL[TEAMS + 1][32];
  double brkL[TEAMS + 1][32];
  double wbL[TEAMS + 1][32];
  double st[4];                    // err, breakdowns, final err, bad weights
  int ist[2];                      // final_t, conv
};

__device__ __forceinline__ void reg_raise() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegCompute));
}
__device__ __forceinline__ void reg_lower() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegStream));
}

template <int D>
constexpr size_t dyn_smem_fixed() {
  return sizeof(double) * NV * 4 * NT + sizeof(float) * TEAMS * kRing * Geo<D>::SLOT +
         sizeof(float4) * NV * TS;
}
__host__ __device__ inline size_t stage_floats(int r) { return (size_t)HDR + (size_t)TRS * r; }

// MODE 0: expanded exponent; 1: factored (row factor h_j) — as implicit_kernel
template <int D, int MODE>
__global__ void __launch_bounds__(NT, 1) hybrid_kernel(const SinkArgs A) {
  constexpr bool FACT = MODE == 1;
  constexpr int XS = Geo<D>::XS, SLOT = Geo<D>::SLOT;
  constexpr int kFlushTiles = 64 / TR;
  constexpr int kFlushTilesS = 64 / TRS;
  constexpr int LPR = 32 / TR, G = exchange_lanes(NWT, LPR), PER = NWT / G;
  constexpr int LPRS = 32 / TRS, GS = exchange_lanes(NWT, LPRS), PERS = NWT / GS;
  __shared__ __align__(16) Smem S;
  extern __shared__ double acc_dyn[];
  double (*acc_s)[NT] = reinterpret_cast<double (*)[NT]>(acc_dyn);
  float* slots = reinterpret_cast<float*>(acc_dyn + NV * 4 * NT);
  float4* s_sm = reinterpret_cast<float4*>(slots + TEAMS * kRing * SLOT);
  float* ring = reinterpret_cast<float*>(s_sm + NV * TS);   // [NSTG][HDR + TRS r], 16B aligned

  const int tid = threadIdx.x;
  const int team = tid / TS, ttid = tid - team * TS;
  const int warp = tid >> 5, lane = tid & 31, twarp = ttid >> 5;
  const int cta = blockIdx.x;
  const int r = A.r;
  const int R4 = r >> 2;
  const int64_t STG = (int64_t)stage_floats(r);
  double* stg_state = A.state;

  if (tid == 0) {
    for (int tm = 0; tm < TEAMS; ++tm)
      for (int i = 0; i < kRing; ++i) mbar_init(&S.full[tm][i], 32);
    for (int i = 0; i < NSTG; ++i) mbar_init(&S.sfull[i], 33);   // tx arrive + 32 cp.async
    fence_mbar_init();
  }
  for (int i = tid; i < TEAMS * kRing * SLOT; i += NT) slots[i] = 0.f;
  for (int64_t i = tid; i < (int64_t)NSTG * STG / 4; i += NT)
    reinterpret_cast<float4*>(ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_proxy_async_smem();
  if (tid == 0) {
    S.st[0] = __ldcg(stg_state + ST_ERR);
    S.st[1] = __ldcg(stg_state + ST_BRK);
    S.st[2] = -1.0;
    S.st[3] = __ldcg(stg_state + ST_WBAD);
    S.ist[0] = -1;
    S.ist[1] = 0;
  }
  if (tid < 32)
    for (int tm = 0; tm <= TEAMS; ++tm) S.errL[tm][tid] = S.brkL[tm][tid] = S.wbL[tm][tid] = 0.0;
  __syncthreads();

  // rows of this CTA: the stream team takes its share of the materialised prefix [0, ns), the
  // recompute teams their share of [ns, rows)
  int64_t rbeg[2], sbeg[2];
  int rcnt[2], scnt[2];
#pragma unroll
  for (int fs = 0; fs < 2; ++fs) {
    const int64_t ns = A.nstream[fs];
    int64_t q1;
    cta_rows(A.rows[fs] - ns, A.gpp, cta, &rbeg[fs], &q1);
    rcnt[fs] = (int)(q1 - rbeg[fs]);
    rbeg[fs] += ns;
    cta_rows(ns, A.gpp, cta, &sbeg[fs], &q1);
    scnt[fs] = (int)(q1 - sbeg[fs]);
  }
  double* part = A.part;
  const int64_t rstride = r + kExtra;

  // ================================ one role's whole solve =================================
  auto body = [&](auto strm_tag) {
    constexpr bool STRM = decltype(strm_tag)::value;
    const uint32_t team_bar = 2u + (uint32_t)team;
    int g[NV];
    bool gv[NV];
    float2 W2[NV][D][2];
    float2 B2[NV][2];
    const float boff = FACT ? A.abar : 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      g[j] = ttid + j * TS;
      gv[j] = g[j] < R4;
      if constexpr (!STRM) {
        if (gv[j]) {
          const float4 b = *reinterpret_cast<const float4*>(A.beta2 + 4 * g[j]);
          B2[j][0] = make_float2(b.x + boff, b.y + boff);
          B2[j][1] = make_float2(b.z + boff, b.w + boff);
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float4 w = *reinterpret_cast<const float4*>(A.Wt + (int64_t)c * r + 4 * g[j]);
            W2[j][c][0] = make_float2(w.x, w.y);
            W2[j][c][1] = make_float2(w.z, w.w);
          }
        } else {   // padding groups produce exact zeros: ex2(-inf) = 0
          B2[j][0] = B2[j][1] = make_float2(-INFINITY, -INFINITY);
#pragma unroll
          for (int c = 0; c < D; ++c) W2[j][c][0] = W2[j][c][1] = make_float2(0.f, 0.f);
        }
      }
    }
    float4 s[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc_s[j * 4 + q][tid] = 0.0;
    }
    unsigned int nbar = 0;
    uint32_t gt = 0;    // recompute tiles of this team so far (slot gt % kRing, red gt % 3)
    uint32_t gs = 0;    // stream tiles so far (stage gs % NSTG, red gs % 3)
    float* tslots = slots + (STRM ? 0 : team) * kRing * SLOT;
    bool prefetched = false;

    // ---- recompute feed (team warp 0 loads tile slots with cp.async) ----
    struct Feed {
      const float *w, *X, *h, *vold;
      int nrows, ntiles;
    };
    auto make_feed = [&](int q) {
      const int kq = pass_kind(q, A);
      const int fq = (kq == PK_V || kq == PK_ERR) ? 1 : 0;
      const int64_t q0 = rbeg[fq];
      Feed fd;
      fd.nrows = rcnt[fq];
      fd.ntiles = ((fd.nrows + TR - 1) / TR - team + TEAMS - 1) / TEAMS;
      fd.w = A.w[fq] + q0;
      fd.X = A.X[fq] + q0 * D;
      fd.h = FACT ? A.hrow[fq] + q0 : nullptr;
      const bool nv = (kq == PK_ERR) || (kq == PK_V && q >= 3);
      fd.vold = nv ? vbuf_ptr(A, 0, (kq == PK_ERR) ? A.T : (q + 1) / 2 - 1) + q0 : nullptr;
      return fd;
    };
    auto issue_tile = [&](const Feed& fd, uint32_t g0, int t) {
      if (t >= fd.ntiles) {
        cp_async_commit();
        return;
      }
      const int lr = (team + t * TEAMS) * TR;
      float* sl = tslots + ((g0 + (uint32_t)t) % kRing) * SLOT;
      if (lane < TR && lane < fd.nrows - lr) {
        cp_async4(sl + lane, fd.w + lr + lane);
        if (FACT) cp_async4(sl + 32 + lane, fd.h + lr + lane);
        if (fd.vold) cp_async4(sl + 64 + lane, fd.vold + lr + lane);
#pragma unroll
        for (int c = 0; c < D; ++c) cp_async4(sl + 96 + lane * XS + c, fd.X + (lr + lane) * D + c);
      }
      cp_async_commit();
    };
    // ---- stream feed (stream warp 0: bulk copies of 8 contiguous rows + cp.async scalars) ----
    struct SFeed {
      const float *F, *w, *vold;
      int nrows, ntiles;
    };
    auto make_sfeed = [&](int q) {
      const int kq = pass_kind(q, A);
      const int fq = (kq == PK_V || kq == PK_ERR) ? 1 : 0;
      const int64_t q0 = sbeg[fq];
      SFeed fd;
      fd.nrows = scnt[fq];
      fd.ntiles = (fd.nrows + TRS - 1) / TRS;
      fd.F = A.F[fq] + q0 * r;
      fd.w = A.w[fq] + q0;
      const bool nv = (kq == PK_ERR) || (kq == PK_V && q >= 3);
      fd.vold = nv ? vbuf_ptr(A, 0, (kq == PK_ERR) ? A.T : (q + 1) / 2 - 1) + q0 : nullptr;
      return fd;
    };
    auto issue_stage = [&](const SFeed& fd, uint32_t g0, int t) {   // stream warp 0, all lanes
      if (t >= fd.ntiles) return;
      const uint32_t gi = g0 + (uint32_t)t;
      float* st = ring + (int64_t)(gi % NSTG) * STG;
      const int lr = t * TRS;
      const int rows = min(TRS, fd.nrows - lr);
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)rows * (uint32_t)r * 4u;
        mbar_arrive_expect_tx(&S.sfull[gi % NSTG], bytes);
        bulk_g2s(st + HDR, fd.F + (int64_t)lr * r, bytes, &S.sfull[gi % NSTG], policy_evict_first());
      }
      if (lane < rows) {
        cp_async4(st + lane, fd.w + lr + lane);
        if (fd.vold) cp_async4(st + 32 + lane, fd.vold + lr + lane);
      }
      cp_async_mbar_arrive_noinc(&S.sfull[gi % NSTG]);
    };

    for (int p = A.pass_begin;; ++p) {
      // ---------------- results of pass p-1: stopping test (as implicit_kernel) ----------
      if (p > A.pass_begin) {
        if (tid == 0) {
          const int q = p - 1;
          const int qk = pass_kind(q, A);
          double e_err, e_brk, e_wb;
          sv_load_extras(sv_of(A, 0, q) + r, false, e_err, e_brk, e_wb);
          S.st[1] += e_brk;
          S.st[3] += e_wb;
          if (qk == PK_V) {
            const int t = (q + 1) / 2;
            if (t >= 2) {
              S.st[0] = e_err;
              if (A.tol_mode && e_err < A.tol) {
                S.ist[0] = t - 1;
                S.st[2] = e_err;
                S.ist[1] = 1;
              }
            }
          } else if (qk == PK_ERR) {
            S.st[0] = e_err;
          }
          if (S.ist[0] < 0 && q == A.num_passes - 1) {
            S.ist[0] = A.T;
            S.st[2] = A.want_err ? S.st[0] : -1.0;
            S.ist[1] = A.tol_mode ? (S.st[0] < A.tol ? 1 : 0) : 0;
          }
        }
        named_bar(1, NT);
        if (S.ist[0] >= 0) break;
      }
      if (p >= A.pass_end) break;
      const int kind = pass_kind(p, A);
      if (kind == PK_NONE) continue;
      const int f = (kind == PK_V || kind == PK_ERR) ? 1 : 0;
      if (kind != PK_INIT) {
        for (int gg = tid; gg < NV * TS; gg += NT) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gg < R4) {
            double2 lo, hi;
            sv_load4(sv_of(A, 0, p - 1) + 4 * gg, false, lo, hi);
            v = make_float4((float)lo.x, (float)lo.y, (float)hi.x, (float)hi.y);
          }
          s_sm[gg] = v;
        }
        named_bar(1, NT);
#pragma unroll
        for (int j = 0; j < NV; ++j) s[j] = s_sm[g[j]];
      }
#pragma unroll
      for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc_s[j * 4 + q][tid] = 0.0;
      float4 acc32[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      float* outp0 = nullptr;

      auto flush = [&]() {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          acc_s[j * 4 + 0][tid] += (double)acc32[j].x;
          acc_s[j * 4 + 1][tid] += (double)acc32[j].y;
          acc_s[j * 4 + 2][tid] += (double)acc32[j].z;
          acc_s[j * 4 + 3][tid] += (double)acc32[j].w;
          acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };

      if constexpr (!STRM) {
        // ================= recompute teams: the implicit_kernel (128,2,2,16) tile loop =======
        const Feed feed = make_feed(p);
        const int nrows = feed.nrows, ntiles = feed.ntiles;
        const bool need_vold = feed.vold != nullptr;
        if (kind == PK_U) outp0 = A.out[0] + rbeg[0];
        if (kind == PK_V) outp0 = vbuf_ptr(A, 0, (p + 1) / 2) + rbeg[1];
        const uint32_t gt0 = gt;
        auto run_tiles = [&](auto kind_tag) {
          constexpr int KIND = decltype(kind_tag)::value;
          constexpr bool kDot = KIND != PK_INIT;
          constexpr bool kAcc = KIND != PK_ERR;
          constexpr bool kOut = KIND == PK_U || KIND == PK_V;
          if (twarp == 0) {
            if (!prefetched)
              for (int t = 0; t < kAhead; ++t) issue_tile(feed, gt0, t);
            cp_async_wait<kAhead - 1>();
          }
          named_bar(team_bar, TS);
          int nfin = 0;
          for (int t = 0; t < ntiles; ++t) {
            float2 fr[TR][NV][2];
            if (twarp == 0) issue_tile(feed, gt0, t + kAhead);
            const uint32_t gi = gt0 + (uint32_t)t;
            const float* sl = tslots + (gi % kRing) * SLOT;
#pragma unroll
            for (int i = 0; i < TR; ++i) {
              float x[XS];
              {
                const float4 x0 = lds128(sl + 96 + i * XS);
                x[0] = x0.x; if (XS > 1) x[1] = x0.y;
                if (XS > 2) x[2] = x0.z;
                if (XS > 3) x[3] = x0.w;
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
            const int rb = (int)(gi % 3u);
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
              if ((lane & (LPR - 1)) == 0) S.red[team][rb][lane / LPR][twarp] = tot;
            }
            if (twarp == 0) cp_async_wait<kAhead - 1>();
            named_bar(team_bar, TS);
            // finish tile t
            const int lr = (team + t * TEAMS) * TR;
            const int rows = min(TR, nrows - lr);
            const int row = lane / G;
            const bool valid = (lane < TR * G) && (row < rows);
            float wt = 0.f;
            if constexpr (kDot) {
              float tot = 0.f;
              if (lane < TR * G) {
                const float* rp = &S.red[team][rb][row][(lane % G) * PER];
#pragma unroll
                for (int q = 0; q < PER; ++q) tot += rp[q];
              }
#pragma unroll
              for (int off = 1; off < G; off <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
              if (valid) {
                const float c = sl[row];
                const float h = FACT ? sl[32 + row] : 1.f;
                const float tj = FACT ? h * tot : tot;
                const float w = c * rcp_approx(tj);
                wt = FACT ? w * h : w;
                if (twarp == NWT - 1 && (lane % G) == 0) {
                  if (bad_weight(c)) S.wbL[team][lane] += 1.0;
                  if (need_vold) S.errL[team][lane] += fabs((double)sl[64 + row] * (double)tj - (double)c);
                  if constexpr (kOut) {
                    if (!(w > 0.f) || !isfinite(w)) S.brkL[team][lane] += 1.0;
                    outp0[lr + row] = w;
                  }
                }
              }
              if constexpr (!kAcc) wt = 0.f;
            } else {
              if (valid) wt = FACT ? sl[32 + row] : 1.f;   // u^0 = 1 (reading C6): w~ = h
            }
            if constexpr (kAcc) {
#pragma unroll
              for (int i = 0; i < TR; ++i) {
                const float vi = __shfl_sync(0xffffffffu, wt, i * G);
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
                flush();
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
        gt += (uint32_t)ntiles;
      } else {
        // ================= stream team: materialised rows from the TMA ring ==================
        // The same column ownership and tile structure as a recompute team (8-row tiles, warp
        // transpose-reduce, one team barrier per tile), the rows read from the stage instead of
        // generated: a second read of the stage feeds the accumulation.  Stream warp 0 issues
        // the stages (NSTG - 1 ahead); after the team barrier of tile t every thread is past
        // tile t - 1, so its stage takes tile t + NSTG - 1.
        const SFeed feed = make_sfeed(p);
        const int nrows = feed.nrows, ntiles = feed.ntiles;
        const bool need_vold = feed.vold != nullptr;
        if (kind == PK_U) outp0 = A.out[0] + sbeg[0];
        if (kind == PK_V) outp0 = vbuf_ptr(A, 0, (p + 1) / 2) + sbeg[1];
        const uint32_t gs0 = gs;
        auto run_stiles = [&](auto kind_tag) {
          constexpr int KIND = decltype(kind_tag)::value;
          constexpr bool kDot = KIND != PK_INIT;
          constexpr bool kAcc = KIND != PK_ERR;
          constexpr bool kOut = KIND == PK_U || KIND == PK_V;
          if (twarp == 0 && !prefetched)
            for (int t = 0; t < NSTG - 1; ++t) issue_stage(feed, gs0, t);
          int nfin = 0;
          for (int t = 0; t < ntiles; ++t) {
            const uint32_t gi = gs0 + (uint32_t)t;
            mbar_wait(&S.sfull[gi % NSTG], (gi / NSTG) & 1u);
            const float* st = ring + (int64_t)(gi % NSTG) * STG;
            const float* feat = st + HDR;
            const int rb = (int)(gi % 3u);
            if constexpr (kDot) {
              float pr[TRS];
#pragma unroll
              for (int i = 0; i < TRS; ++i) {
                float2 pp = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                  if (gv[j]) {
                    const float4 fv = lds128(feat + (int64_t)i * r + 4 * g[j]);
                    pp = fma2(make_float2(fv.x, fv.y), make_float2(s[j].x, s[j].y), pp);
                    pp = fma2(make_float2(fv.z, fv.w), make_float2(s[j].z, s[j].w), pp);
                  }
                }
                pr[i] = pp.x + pp.y;
              }
              const float tot = warp_transpose_reduce<TRS>(pr, lane);
              if ((lane & (LPRS - 1)) == 0) S.red[TEAMS][rb][lane / LPRS][twarp] = tot;
            }
            named_bar(team_bar, TS);
            if (twarp == 0) issue_stage(feed, gs0, t + NSTG - 1);
            const int lr = t * TRS;
            const int rows = min(TRS, nrows - lr);
            const int row = lane / GS;
            const bool valid = (lane < TRS * GS) && (row < rows);
            float wt = 0.f;
            if constexpr (kDot) {
              float tot = 0.f;
              if (lane < TRS * GS) {
                const float* rp = &S.red[TEAMS][rb][row][(lane % GS) * PERS];
#pragma unroll
                for (int q = 0; q < PERS; ++q) tot += rp[q];
              }
#pragma unroll
              for (int off = 1; off < GS; off <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
              if (valid) {
                const float c = st[row];
                const float w = c * rcp_approx(tot);   // t_j = F_j . s of the materialised row
                wt = w;
                if (twarp == NWT - 1 && (lane % GS) == 0) {
                  if (bad_weight(c)) S.wbL[TEAMS][lane] += 1.0;
                  if (need_vold) S.errL[TEAMS][lane] += fabs((double)st[32 + row] * (double)tot - (double)c);
                  if constexpr (kOut) {
                    if (!(w > 0.f) || !isfinite(w)) S.brkL[TEAMS][lane] += 1.0;
                    outp0[lr + row] = w;
                  }
                }
              }
              if constexpr (!kAcc) wt = 0.f;
            } else {
              if (valid) wt = 1.f;   // u^0 = 1 (reading C6)
            }
            if constexpr (kAcc) {
#pragma unroll
              for (int i = 0; i < TRS; ++i) {
                const float vi = __shfl_sync(0xffffffffu, wt, i * GS);
                const float2 v2 = make_float2(vi, vi);
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                  if (gv[j]) {
                    const float4 fv = lds128(feat + (int64_t)i * r + 4 * g[j]);
                    const float2 lo = fma2(make_float2(fv.x, fv.y), v2, make_float2(acc32[j].x, acc32[j].y));
                    const float2 hi = fma2(make_float2(fv.z, fv.w), v2, make_float2(acc32[j].z, acc32[j].w));
                    acc32[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
                  }
                }
              }
              if (++nfin == kFlushTilesS) {
                nfin = 0;
                flush();
              }
            }
          }
        };
        switch (kind) {
          case PK_INIT: run_stiles(std::integral_constant<int, PK_INIT>{}); break;
          case PK_V: run_stiles(std::integral_constant<int, PK_V>{}); break;
          case PK_U: run_stiles(std::integral_constant<int, PK_U>{}); break;
          default: run_stiles(std::integral_constant<int, PK_ERR>{}); break;
        }
        gs += (uint32_t)ntiles;
      }
      flush();

      // ---------------- end of pass: teams combined (fixed order), cross-CTA fp64 reduction ---
      double e0 = 0.0, e1 = 0.0, e2 = 0.0;
      if (twarp == NWT - 1) {   // each team's output warp
        e0 = warp_sum_f64(S.errL[team][lane]);
        e1 = warp_sum_f64(S.brkL[team][lane]);
        e2 = warp_sum_f64(S.wbL[team][lane]);
        S.errL[team][lane] = 0.0;
        S.brkL[team][lane] = 0.0;
        S.wbL[team][lane] = 0.0;
        if (lane == 0) {
          S.xs[0][team] = e0;
          S.xs[1][team] = e1;
          S.xs[2][team] = e2;
        }
      }
      named_bar(1, NT);
      if (team == 0) {   // fixed order: team 0 + team 1 + stream team (deterministic)
#pragma unroll
        for (int tm = 1; tm <= TEAMS; ++tm)
#pragma unroll
          for (int e = 0; e < NV * 4; ++e) acc_s[e][ttid] += acc_s[e][ttid + tm * TS];
        if (ttid == 0) {
          e0 = S.xs[0][0];
          e1 = S.xs[1][0];
          e2 = S.xs[2][0];
          for (int tm = 1; tm <= TEAMS; ++tm) {
            e0 += S.xs[0][tm];
            e1 += S.xs[1][tm];
            e2 += S.xs[2][tm];
          }
        }
      }
      named_bar(1, NT);
      if (team == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (gv[j])
            part_store4(part, A.gpp, g[j], cta, acc_s[j * 4 + 0][ttid], acc_s[j * 4 + 1][ttid],
                        acc_s[j * 4 + 2][ttid], acc_s[j * 4 + 3][ttid]);
        }
      }
      if (tid == 0) part_store4(part, A.gpp, R4, cta, e0, e1, e2, 0.0);
      group_barrier<NT>(A.bar, (++nbar) * (unsigned)A.gpp, tid);
      r2_cta(A, 0, p, part, cta, warp, NW, lane);
      // the next pass's first tiles now: they land while this CTA waits for the totals
      prefetched = false;
      const int q = p + 1;
      if (q < A.pass_end && pass_kind(q, A) != PK_NONE) {
        if (twarp == 0) {
          if constexpr (STRM) {
            const SFeed nf = make_sfeed(q);
            for (int t = 0; t < NSTG - 1; ++t) issue_stage(nf, gs, t);
          } else {
            const Feed nf = make_feed(q);
            for (int t = 0; t < kAhead; ++t) issue_tile(nf, gt, t);
          }
        }
        prefetched = true;
      }
    }

    if constexpr (!STRM) {
      if (twarp == 0) cp_async_wait<0>();
    }
    // ---------------- returned v into the user buffer, then the fp64 read-out ---------------
    const int final_t = S.ist[0];
    int64_t u0, u1, v0, v1;
    cta_rows(A.rows[0], A.gpp, cta, &u0, &u1);
    cta_rows(A.rows[1], A.gpp, cta, &v0, &v1);
    if ((final_t ^ A.T) & 1)
      for (int64_t i = v0 + tid; i < v1; i += NT) A.out[1][i] = __ldcg(A.vbuf1 + i);
    named_bar(1, NT);
    double la = 0.0, lb = 0.0;
    for (int64_t i = u0 + tid; i < u1; i += NT) la += (double)A.w[0][i] * log((double)__ldcg(A.out[0] + i));
    for (int64_t i = v0 + tid; i < v1; i += NT) lb += (double)A.w[1][i] * log((double)__ldcg(A.out[1] + i));
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
      *part_at(part, A.gpp, (int)rstride, cta) = la;
      *part_at(part, A.gpp, (int)rstride + 1, cta) = lb;
    }
    group_barrier<NT>(A.bar, (++nbar) * (unsigned)A.gpp, tid);
    if (cta == 0 && tid == 0) {
      la = 0.0;
      lb = 0.0;
      for (int c = 0; c < A.gpp; ++c) {
        la += __ldcg(part_at(part, A.gpp, (int)rstride, c));
        lb += __ldcg(part_at(part, A.gpp, (int)rstride + 1, c));
      }
      if (A.nranks > 1) {
        la = xrank_total(A, 0, 0, (int)rstride, la);
        lb = xrank_total(A, 0, 0, (int)rstride + 1, lb);
      }
      stg_state[ST_ITERS] = (double)final_t;
      stg_state[ST_FINAL_A] = la;
      stg_state[ST_FINAL_B] = lb;
      stg_state[ST_ROT] = A.eps * (la + lb);
      stg_state[ST_ERR] = S.st[2];
      stg_state[ST_CONV] = (double)S.ist[1];
      stg_state[ST_BRK] = S.st[1];
      stg_state[ST_WBAD] = S.st[3];
      sticky_flags(A, S.st[1], S.st[3]);
      __threadfence();
      stg_state[ST_STOP] = 1.0;
    }
  };

  if (team == TEAMS) {
    reg_lower();
    body(std::true_type{});
  } else {
    reg_raise();
    body(std::false_type{});
  }
}

}  // namespace hyb

bool hybrid_supported(const SinkArgs& a) {
  return a.r <= hyb::NV * hyb::TS * 4 && a.d >= 1 && a.d <= 3 && !a.stab && !a.multi_launch &&
         a.nprob == 1 && !a.cx && !a.emul && a.gpp > 1;
}

size_t hybrid_smem(int r, int d) {
  size_t fixed = 0;
  switch (d) {
    case 1: fixed = hyb::dyn_smem_fixed<1>(); break;
    case 2: fixed = hyb::dyn_smem_fixed<2>(); break;
    default: fixed = hyb::dyn_smem_fixed<3>(); break;
  }
  return fixed + sizeof(float) * hyb::NSTG * hyb::stage_floats(r);
}

template <int D, int MODE>
static cudaError_t launch_h(const SinkArgs& a, int grid, cudaStream_t s) {
  auto kern = hyb::hybrid_kernel<D, MODE>;
  const size_t dyn = hybrid_smem(a.r, D);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&a};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(hyb::NT), args, dyn, s);
  count_launch();
  return e;
}

cudaError_t launch_hybrid_ws(const SinkArgs& a, int grid, cudaStream_t s) {
  const int mode = a.hrow[0] != nullptr ? 1 : 0;
#define H(D_, M_) \
  if (a.d == D_ && mode == M_) return launch_h<D_, M_>(a, grid, s);
  H(1, 0) H(1, 1) H(2, 0) H(2, 1) H(3, 0) H(3, 1)
#undef H
  return cudaErrorInvalidConfiguration;
}

}  // namespace lsk
