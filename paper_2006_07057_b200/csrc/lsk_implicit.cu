// lsk_implicit.cu — Alg. 1 on K_theta = xi zeta^T WITHOUT materialising
// the factors: every pass regenerates F_jk = phi(p_j, u_k)/sqrt(r) in registers from the
// point rows and the anchors (Lemma decomp-RBF, expanded in base 2):
//     F_jk = 2^( alpha2_j + beta2_k + sum_c W_kc p_jc ),
//     alpha2_j = -(2 log2e/eps)|p_j|^2, W_kc = (4 log2e/eps) U_kc,
//     beta2_k = log2e (-(2/eps)|U_k|^2 + |U_k|^2/(eps q) + log_scale).
//
// Factored exponent (FACT, DESIGN.md §6 K5): the row term is pulled out of the entry,
//     F_jk = h_j G_jk,  G_jk = 2^(beta2_k + abar + sum_c W_kc p_jc),  h_j = 2^(alpha2_j - abar),
// with abar = -(log2e/eps) R^2 (mid-range of alpha2, so h_j is within 2^{+-(log2e/eps)R^2}).
// Then t_j = h_j (G_j . s), w_j = c_j / t_j, and the accumulation s'_k = sum_j F_jk w_j =
// sum_j G_jk (h_j w_j): per entry only the d-term dot W_k . p_j and one MUFU ex2 remain
// (d FFMA2 per column pair instead of d+1, and no per-entry |p|^2 work).  The host uses it
// when (log2e/eps) R^2 <= 60 (G, h stay far from the fp32 range limits); otherwise the plain
// expanded form (h = 1, abar folded per row) runs.
//
// Stabilised mode (MODE 2, reading C30): each row's exponent is shifted by its maximum
// m_j = max_k (beta2_k + W_k . p_j) (precomputed, row_shift_kernel), so every regenerated entry
// is <= ~1, and the kernel returns the scalings of the row-normalised problem.
//
// Layout: one CTA per SM made of TEAMS teams of TS threads (all consumers).  A team owns every
// column: thread t of a team owns float4 column groups {t, t+TS, ...} (its W, beta2, slice of
// s and fp32 accumulators live in registers; the fp64 accumulators in shared memory).  Teams
// take alternate tiles of TR rows of the CTA's row range.  Each team's warp 0 stages tiles
// (point rows, c_j, h_j, v_old_j) kAhead = 2 tiles ahead with cp.async into an 8-slot ring
// (measured: 16 slots 8 ahead 20.3 us/pass on config 2, 32 / 16 21.0, 8 / 2 20.1).
//
// Per tile (default, PIPE = 0): features -> row-dot partials -> warp transpose-reduce -> one
// named barrier per team (publishes the partials and the next slot) -> the exchange: row i's
// NWT warp partials are summed by G lanes (NWT/G each) and a fixed xor butterfly — every lane of
// the group ends with the same bits, and the order never changes (deterministic) -> scalings
// -> FFMA2 accumulation.  PIPE = 1 (tuning alternative) holds two feature tiles: tile t's
// partials are published with a split mbarrier arrive before tile t-1 is finished.  Pass
// boundary, stopping test and the fp64 read-out are those of the streaming kernel
// (lsk_sinkhorn.cu); s is staged once per CTA into shared memory at each pass start.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {

namespace impl {

constexpr int kRing = 8;    // tile slots per team
constexpr int kSRing = 6;   // hybrid: row slots per stream warp (bulk copies in flight)
constexpr int kSRow = 1024; // hybrid: floats per row slot (r <= 1024)
constexpr int kAhead = 2;   // the loader stages tile t+kAhead when tile t starts (<= kRing/2)

template <int D>
struct Geo {
  static constexpr int XS = D <= 4 ? 4 : 8;        // floats per staged point row
  static constexpr int SLOT = 96 + 32 * XS;        // c[32] h[32] vold[32] x[32][XS]
};

// lanes per row in the row-dot exchange: the largest divisor of the team's warp count that
// fits the lanes a row has after the transpose-reduce
__host__ __device__ constexpr int exchange_lanes(int nwt, int lpr) {
  int g = nwt < lpr ? nwt : lpr;
  while (nwt % g) --g;
  return g;
}

template <int TS, int TEAMS, int TR, int NWALL, int SW>
struct Smem {
  uint64_t full[TEAMS][kRing];     // slot landed (32 cp.async arrivals of the loader warp)
  uint64_t redbar[TEAMS][3];       // row-dot partials of a tile published (TS arrivals)
  float red[TEAMS][3][TR][TS / 32];
  double xs[3][NWALL];
  double xsS[2][SW > 0 ? SW : 1];  // stream warps' error / breakdown sums of a pass
  uint64_t sfull[SW > 0 ? SW : 1][kSRing];   // stream warps' row slots landed (bulk copy tx)
  double ext[kExtra];
  double cxext[8];                 // cluster mode: this CTA's extras [0..3], read-out [4..5]
  uint64_t cxbar;                  // cluster mode: cluster-scope pass barrier
  double errL[TEAMS][32];          // per-lane marginal-error sums of the output warps
  double brkL[TEAMS][32];          // per-lane breakdown counts of the output warps
  double wbL[TEAMS][32];           // per-lane bad-weight counts of the output warps
  double st[4];                    // running solve state: err, breakdowns, final err, bad weights
  int ist[2];                      // final_t, conv
};

// MODE 0: expanded exponent; 1: factored (row factor h_j); 2: stabilised (per-row shift m_j,
// scalings of the row-normalised problem, reading C30)
// SW > 0 (hybrid): SW more warps stream the materialised factor rows [0, nstream) of each side
// (read once per pass from HBM, which the recompute teams leave idle) while the teams
// regenerate the rest; both add into the same fixed-order reductions.
template <int TS, int TEAMS, int NV, int TR, int D, int MODE, bool PIPE, int SW = 0>
__global__ void __launch_bounds__(TS * TEAMS + 32 * SW, 1) implicit_kernel(const SinkArgs A) {
  constexpr bool FACT = MODE == 1, STAB = MODE == 2;
  constexpr int NTI = TS * TEAMS;      // recompute threads
  constexpr int NT = NTI + 32 * SW;    // CTA threads
  constexpr int NWT = TS / 32;         // warps per team
  constexpr int NW = NT / 32;
  constexpr int GPL = NV * TS / 32;    // stream lanes: float4 column groups lane + 32 i
  constexpr int XS = Geo<D>::XS, SLOT = Geo<D>::SLOT;
  // fp32 partials over <= 64 rows, then fp64 (all terms are positive, so the
  // fp32 partial's relative error is <= 64 u; measured: config 5 -1.6% per pass vs 32 rows)
  constexpr int kFlushTiles = (64 / TR) > 0 ? (64 / TR) : 1;
  constexpr int LPR = 32 / TR;                                   // lanes per row after the transpose-reduce
  constexpr int G = exchange_lanes(NWT, LPR);                     // lanes per row in the exchange
  constexpr int PER = NWT / G;                                   // partials summed per lane
  static_assert(TEAMS >= 1 && TEAMS <= 8, "1 to 8 teams (named barriers 2..9)");
  static_assert(TR * G <= 32 && NWT % G == 0, "exchange layout");
  __shared__ __align__(16) Smem<TS, TEAMS, TR, NW, SW> S;
  // dynamic: fp64 accumulators [NV*4][NT] (element-major: consecutive threads, consecutive
  // words), then the tile slots [TEAMS][kRing][SLOT]
  extern __shared__ double acc_dyn[];
  double (*acc_s)[NT] = reinterpret_cast<double (*)[NT]>(acc_dyn);
  float* slots = reinterpret_cast<float*>(acc_dyn + NV * 4 * NT);
  float4* s_sm = reinterpret_cast<float4*>(slots + TEAMS * kRing * SLOT);   // [NV * TS] s in fp32
  double* sacc0 = reinterpret_cast<double*>(s_sm + NV * TS);   // [SW][GPL * 4][32] stream partials
  float* sring0 = reinterpret_cast<float*>(sacc0 + SW * GPL * 4 * 32);   // [SW][kSRing][kSRow]
  double* cxtot = reinterpret_cast<double*>(sring0 + SW * kSRing * kSRow);  // cx: [(r/4+1)*4]
  float4* stash4 = reinterpret_cast<float4*>(cxtot + (A.cx ? ((A.r >> 2) + 1) * 4 : 0));   // [TR*NV][NT]
  uint32_t cxphase = 0;

  const int tid = threadIdx.x;
  const bool strm = SW > 0 && tid >= NTI;   // a stream warp
  const int team = strm ? TEAMS : tid / TS, ttid = strm ? tid - NTI : tid - team * TS;
  const int warp = tid >> 5, lane = tid & 31;
  const int twarp = ttid >> 5;          // warp index within the team
  const uint32_t team_bar = 2u + (uint32_t)team;   // named barrier ids 2..9 (1 = whole CTA)
  const int prob = blockIdx.x / A.gpp;
  const int cta = blockIdx.x - prob * A.gpp;
  const int r = A.r;
  double* stg_state = A.state + (int64_t)prob * kStateDoubles;
  if (__ldcg(stg_state + ST_STOP) != 0.0) return;   // finished (multi-launch mode)

  if (tid == 0) {
    for (int tm = 0; tm < TEAMS; ++tm) {
      for (int i = 0; i < kRing; ++i) mbar_init(&S.full[tm][i], 32);
      for (int i = 0; i < 3; ++i) mbar_init(&S.redbar[tm][i], TS);
    }
    if constexpr (SW > 0) {
      for (int w = 0; w < SW; ++w)
        for (int i = 0; i < kSRing; ++i) mbar_init(&S.sfull[w][i], 1);
    }
    if (A.cx) mbar_init(&S.cxbar, (uint32_t)A.gpp);
    fence_mbar_init();
  }
  // zero the slots once: tail rows then compute on finite data without per-row predicates
  for (int i = tid; i < TEAMS * kRing * SLOT; i += NT) slots[i] = 0.f;

  // per-thread anchor constants for the owned column groups (as float pairs for FFMA2)
  const int R4 = r >> 2;
  int g[NV];
  bool gv[NV];
  float2 W2[NV][D][2];
  float2 B2[NV][2];
  const float boff = FACT ? A.abar : 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    g[j] = ttid + j * TS;
    gv[j] = g[j] < R4;
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
  __syncthreads();

  float4 s[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc_s[j * 4 + q][tid] = 0.0;
  }

  // running solve state in shared memory (uniform; keeps registers for the tile loop)
  double& stErr = S.st[0];
  double& stBrk = S.st[1];
  double& ferr = S.st[2];
  double& stWb = S.st[3];
  int& final_t = S.ist[0];
  int& conv = S.ist[1];
  if (tid == 0) {
    stErr = __ldcg(stg_state + ST_ERR);
    stBrk = __ldcg(stg_state + ST_BRK);
    stWb = __ldcg(stg_state + ST_WBAD);
    ferr = -1.0;
    final_t = -1;
    conv = 0;
  }
  if (tid < 32) {
    for (int tm = 0; tm < TEAMS; ++tm) S.errL[tm][tid] = S.brkL[tm][tid] = S.wbL[tm][tid] = 0.0;
  }
  __syncthreads();
  if (A.cx) cluster_sync_all();   // every CTA's cluster barrier is initialised before any arrive
  const int64_t rstride = r + kExtra;
  double* part = A.part + prob * part_per_problem(r, A.gpp);   // [blk][gpp][4]
  const bool multi = A.multi_launch != 0;
  unsigned int nbar = 0;
  uint32_t gt = 0;   // tiles of this team so far in this launch: slot gt % kRing, red gt % 3

  float* tslots = slots + team * kRing * SLOT;

  // What the loader streams for pass p: this CTA's rows of the pass's factor side (c_j, h_j,
  // v_old_j, point rows).  Pass p+1's first kAhead tiles are issued at the end of pass p, so
  // their latency hides behind the pass boundary (the inputs are static; v_old was written by
  // this CTA two passes earlier).
  struct Feed {
    const float *w, *X, *h, *vold;
    int nrows, ntiles;
  };
  int64_t rbeg[2];   // this CTA's rows of each side (pass-invariant)
  int rcnt[2];
#pragma unroll
  for (int fs = 0; fs < 2; ++fs) {   // hybrid: the recompute rows follow the streamed prefix
    const int64_t ns = SW > 0 ? A.nstream[fs] : 0;
    int64_t q1;
    cta_rows(A.rows[fs] - ns, A.gpp, cta, &rbeg[fs], &q1);
    rcnt[fs] = (int)(q1 - rbeg[fs]);
    rbeg[fs] += ns;
  }
  auto make_feed = [&](int q) {
    const int kq = pass_kind(q, A);
    const int fq = (kq == PK_V || kq == PK_ERR) ? 1 : 0;
    const int64_t q0 = rbeg[fq];
    Feed fd;
    fd.nrows = rcnt[fq];
    fd.ntiles = ((fd.nrows + TR - 1) / TR - team + TEAMS - 1) / TEAMS;   // tiles team, team+TEAMS, ...
    fd.w = A.w[fq] + (int64_t)prob * A.wstride[fq] + q0;
    fd.X = A.X[fq] + (int64_t)prob * A.fstride[fq] + q0 * D;
    fd.h = (FACT || STAB) ? A.hrow[fq] + (int64_t)prob * A.wstride[fq] + q0 : nullptr;
    const bool nv = (kq == PK_ERR) || (kq == PK_V && q >= 3);
    fd.vold = nv ? vbuf_ptr(A, prob, (kq == PK_ERR) ? A.T : (q + 1) / 2 - 1) + q0 : nullptr;
    return fd;
  };
  // loader (team warp 0): tile t of a pass -> slot (g0 + t) % kRing.  PIPE: completion on the
  // slot's mbarrier; !PIPE: one cp.async group per tile (empty ones too), waited by the loader
  // before the team's per-tile named barrier publishes the slot
  auto issue_tile = [&](const Feed& fd, uint32_t g0, int t) {
    if (t >= fd.ntiles) {
      if constexpr (!PIPE) cp_async_commit();
      return;
    }
    const int lr = (team + t * TEAMS) * TR;
    const uint32_t gi = g0 + (uint32_t)t;
    float* sl = tslots + (gi % kRing) * SLOT;
    if (lane < TR && lane < fd.nrows - lr) {
      cp_async4(sl + lane, fd.w + lr + lane);
      if (FACT || STAB) cp_async4(sl + 32 + lane, fd.h + lr + lane);
      if (fd.vold) cp_async4(sl + 64 + lane, fd.vold + lr + lane);
#pragma unroll
      for (int c = 0; c < D; ++c) cp_async4(sl + 96 + lane * XS + c, fd.X + (lr + lane) * D + c);
    }
    if constexpr (PIPE) cp_async_mbar_arrive_noinc(&S.full[team][gi % kRing]);
    else cp_async_commit();
  };
  bool prefetched = false;   // this pass's first kAhead tiles were issued by the previous pass
  uint32_t skw = 0;           // hybrid: rows this stream warp has consumed (ring slot / parity)

  // Stream warps (hybrid): warp sw takes rows sb0 + sw, + SW, ... of this CTA's share of the
  // streamed prefix.  Its lane 0 keeps kSRing rows in flight with 1-D bulk copies (TMA engine)
  // into the warp's own ring (completion: the slot's mbarrier tx count); the warp reads a row
  // from shared memory (lane: float4 groups lane + 32 i), refills the slot, forms the dot with
  // s as a lane partial plus a fixed xor butterfly (every lane gets the same bits), then
  // w_j = c_j / t_j and the fp32 accumulation F_j w_j, flushed to the warp's fp64 partials
  // every 32 rows.  The features are the materialised ones (h_j included), so the init pass
  // accumulates with u^0 = 1.
  auto stream_pass = [&](int kind, int f, int p) {
    if constexpr (SW > 0) {
      const int sw = ttid >> 5;
      double* sacc = sacc0 + sw * (GPL * 4 * 32);
      float* ring = sring0 + sw * (kSRing * kSRow);
      const bool kDot = kind != PK_INIT, kAcc = kind != PK_ERR;
      const bool kOut = kind == PK_U || kind == PK_V;
      int64_t sb0, sb1;
      cta_rows(A.nstream[f], A.gpp, cta, &sb0, &sb1);
      // this warp's rows: sb0 + sw + SW k, k < K (one bulk copy each into its ring)
      const int K = (sb1 - sb0 > sw) ? (int)((sb1 - sb0 - sw + SW - 1) / SW) : 0;
      const float* Fp = A.F[f];
      const float* wp = A.w[f] + (int64_t)prob * A.wstride[f];
      const bool nvo = (kind == PK_ERR) || (kind == PK_V && p >= 3);
      const float* vold = nvo ? vbuf_ptr(A, prob, (kind == PK_ERR) ? A.T : (p + 1) / 2 - 1) : nullptr;
      float* outp = kind == PK_U ? A.out[0] + (int64_t)prob * A.wstride[0]
                                 : (kind == PK_V ? vbuf_ptr(A, prob, (p + 1) / 2) : nullptr);
      const uint32_t rowbytes = (uint32_t)r * 4u;
      const uint32_t k0 = skw;
      auto issue = [&](int k) {   // lane 0
        const uint32_t slot = (k0 + (uint32_t)k) % kSRing;
        mbar_arrive_expect_tx(&S.sfull[sw][slot], rowbytes);
        bulk_g2s(ring + slot * kSRow, Fp + (sb0 + sw + (int64_t)SW * k) * r, rowbytes,
                 &S.sfull[sw][slot], policy_evict_first());
      };
      if (lane == 0)
        for (int k = 0; k < K && k < kSRing; ++k) issue(k);
      float4 sv[GPL], acc[GPL];
#pragma unroll
      for (int i = 0; i < GPL; ++i) {
        const int g = lane + 32 * i;
        sv[i] = (kDot && g < R4) ? s_sm[g] : make_float4(0.f, 0.f, 0.f, 0.f);
        acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int e = lane; e < GPL * 4 * 32; e += 32) sacc[e] = 0.0;
      auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < GPL; ++i) {
          sacc[(i * 4 + 0) * 32 + lane] += (double)acc[i].x;
          sacc[(i * 4 + 1) * 32 + lane] += (double)acc[i].y;
          sacc[(i * 4 + 2) * 32 + lane] += (double)acc[i].z;
          sacc[(i * 4 + 3) * 32 + lane] += (double)acc[i].w;
          acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      double errw = 0.0, brkw = 0.0;
      float creg = 0.f, vreg = 0.f;   // c_j, v_old_j of rows k0..k0+31 (lane l: row k0 + l)
      for (int k = 0; k < K; ++k) {
        if ((k & 31) == 0) {
          const int kk = k + lane;
          const int64_t j = sb0 + sw + (int64_t)SW * kk;
          creg = kk < K ? __ldg(wp + j) : 0.f;
          vreg = (kk < K && nvo) ? __ldcg(vold + j) : 0.f;
        }
        const float cj = __shfl_sync(0xffffffffu, creg, k & 31);
        const float vo = __shfl_sync(0xffffffffu, vreg, k & 31);
        const int64_t j = sb0 + sw + (int64_t)SW * k;
        const uint32_t gk = k0 + (uint32_t)k;
        mbar_wait(&S.sfull[sw][gk % kSRing], (gk / kSRing) & 1u);
        const float* row = ring + (gk % kSRing) * kSRow;
        float4 fr[GPL];
#pragma unroll
        for (int i = 0; i < GPL; ++i) {
          const int g = lane + 32 * i;
          fr[i] = g < R4 ? lds128(row + 4 * g) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncwarp();
        if (lane == 0 && k + kSRing < K) {   // the slot is free again: refill it
          fence_proxy_async_smem();
          issue(k + kSRing);
        }
        float w = 1.f;
        if (kDot) {
          float2 pp = make_float2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < GPL; ++i) {
            pp = fma2(make_float2(fr[i].x, fr[i].y), make_float2(sv[i].x, sv[i].y), pp);
            pp = fma2(make_float2(fr[i].z, fr[i].w), make_float2(sv[i].z, sv[i].w), pp);
          }
          float t = pp.x + pp.y;
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
          w = cj * rcp_approx(t);   // w_j = c_j / t_j (as the recompute teams)
          if (lane == 0) {
            if (nvo) errw += fabs((double)vo * (double)t - (double)cj);
            if (kOut) {
              if (!(w > 0.f) || !isfinite(w)) brkw += 1.0;
              outp[j] = w;
            }
          }
          if (!kAcc) w = 0.f;
        }
        if (kAcc) {
          const float2 w2 = make_float2(w, w);
#pragma unroll
          for (int i = 0; i < GPL; ++i) {
            const float2 lo = fma2(make_float2(fr[i].x, fr[i].y), w2, make_float2(acc[i].x, acc[i].y));
            const float2 hi = fma2(make_float2(fr[i].z, fr[i].w), w2, make_float2(acc[i].z, acc[i].w));
            acc[i] = make_float4(lo.x, lo.y, hi.x, hi.y);
          }
          if ((k & 31) == 31) flush();
        }
      }
      skw += (uint32_t)K;
      if (kAcc) flush();
      if (lane == 0) {
        S.xsS[0][sw] = errw;
        S.xsS[1][sw] = brkw;
      }
    }
  };

  // one tile's features of this thread's columns: F_jk (or G_jk) = 2^(exponent) for the TR
  // staged point rows of slot sl (independent of s: also generated ahead, across a boundary)
  auto gen_features = [&](const float* sl, float2 (&fr)[TR][NV][2]) {
#pragma unroll
    for (int i = 0; i < TR; ++i) {
      float x[XS];
      {
        const float4 x0 = lds128(sl + 96 + i * XS);
        x[0] = x0.x; if (XS > 1) x[1] = x0.y;
        if (XS > 2) x[2] = x0.z;
        if (XS > 3) x[3] = x0.w;
        if constexpr (XS > 4) {
          const float4 x1 = lds128(sl + 96 + i * XS + 4);
          x[4] = x1.x; x[5] = x1.y; x[6] = x1.z; x[7] = x1.w;
        }
      }
      float2 al2 = make_float2(0.f, 0.f);
      if constexpr (STAB) {
        const float mj = -sl[32 + i];   // the row's shift: every G_jk <= ~1
        al2 = make_float2(mj, mj);
      } else if constexpr (!FACT) {
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
          float2 e = FACT ? B2[j][h] : add2(al2, B2[j][h]);   // STAB: al2 = -m_j
#pragma unroll
          for (int c = 0; c < D; ++c) e = fma2(W2[j][c][h], make_float2(x[c], x[c]), e);
          fr[i][j][h] = make_float2(ex2(e.x), ex2(e.y));
        }
      }
    }
  };
  // boundary overlap (DESIGN.md §6 K5): tile 0 of the next pass is generated while the CTA
  // waits at the pass boundary and parked in shared memory (element-major: conflict-free
  // 128-bit stores and loads); pre_done: the stash holds this pass's tile 0
  constexpr bool kPre = !PIPE && SW == 0;
  bool pre_done = false;
  auto stash_store = [&](const float2 (&fr)[TR][NV][2]) {
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < NV; ++j)
        stash4[(i * NV + j) * NT + tid] = make_float4(fr[i][j][0].x, fr[i][j][0].y, fr[i][j][1].x, fr[i][j][1].y);
  };
  auto stash_load = [&](float2 (&fr)[TR][NV][2]) {
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const float4 v = stash4[(i * NV + j) * NT + tid];
        fr[i][j][0] = make_float2(v.x, v.y);
        fr[i][j][1] = make_float2(v.z, v.w);
      }
  };
  // generate the features of pass q's tile 0 into the stash (its slot was issued when this pass's
  // tiles ended); A.pre = 1: after R2, 2: between the group barrier's arrive and wait
  auto pre_gen = [&](int q) {
    if constexpr (kPre) {
      if (q >= A.pass_end || pass_kind(q, A) == PK_NONE) return;
      const int nr = rcnt[(pass_kind(q, A) == PK_V || pass_kind(q, A) == PK_ERR) ? 1 : 0];
      if (team * TR >= nr) return;   // this team has no tile in pass q
      if (twarp == 0) cp_async_wait<kAhead - 1>();   // tile 0 landed
      named_bar(team_bar, TS);
      float2 fr[TR][NV][2];
      gen_features(tslots + (gt % kRing) * SLOT, fr);
      stash_store(fr);
      pre_done = true;
    }
  };

  for (int p = A.pass_begin;; ++p) {
    // ---------------- results of pass q = p-1: stopping test (see lsk_sinkhorn.cu) -------
    const bool have_prev = multi ? (p == A.pass_begin && p > 0) : (p > A.pass_begin);
    if (have_prev) {
      if (tid == 0) {
        const int q = p - 1;
        const int qk = pass_kind(q, A);
        double e_err, e_brk, e_wb;
        if (A.cx) {
          double x[4];
          cx_total4(cxtot, A.gpp, r >> 2, x);
          e_err = x[0];
          e_brk = x[1];
          e_wb = x[2];
        } else if (A.gpp > 1) {
          sv_load_extras(sv_of(A, prob, q) + r, multi, e_err, e_brk, e_wb);
        } else {
          e_err = S.ext[0];
          e_brk = S.ext[1];
          e_wb = S.ext[2];
        }
        stBrk += e_brk;
        stWb += e_wb;
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
      // s -> fp32 in shared memory once per CTA (the teams share it; see lsk_implicit_warp.cu)
      for (int gg = tid; gg < NV * TS; gg += NT) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gg < R4) {
          if (A.cx) {
            double x[4];
            cx_total4(cxtot, A.gpp, gg, x);
            v = make_float4((float)x[0], (float)x[1], (float)x[2], (float)x[3]);
          } else if (A.gpp > 1) {
            double2 lo, hi;
            sv_load4(sv_of(A, prob, p - 1) + 4 * gg, multi, lo, hi);
            v = make_float4((float)lo.x, (float)lo.y, (float)hi.x, (float)hi.y);
          } else {   // gpp == 1: the combined accumulator sits in team 0's slots
            const int t0 = gg % TS, j = gg / TS;
            v = make_float4((float)acc_s[j * 4][t0], (float)acc_s[j * 4 + 1][t0],
                            (float)acc_s[j * 4 + 2][t0], (float)acc_s[j * 4 + 3][t0]);
          }
        }
        s_sm[gg] = v;
      }
      named_bar(1, NT);   // s staged; every team is done with team 0's slots
#pragma unroll
      for (int j = 0; j < NV; ++j) s[j] = s_sm[g[j]];
    }
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc_s[j * 4 + q][tid] = 0.0;

    const int64_t r0 = rbeg[f];
    const Feed feed = make_feed(p);
    const int nrows = feed.nrows;
    const int ntiles = feed.ntiles;
    const bool need_vold = feed.vold != nullptr;
    float* outp0 = nullptr;
    if (kind == PK_U) outp0 = A.out[0] + (int64_t)prob * A.wstride[0] + r0;
    if (kind == PK_V) outp0 = vbuf_ptr(A, prob, (p + 1) / 2) + r0;
    float4 acc32[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t gt0 = gt;

    // The tile loop is instantiated per pass kind (compile-time KIND: no per-tile kind
    // branches) with 32-bit row offsets relative to this CTA's first row.
    auto run_tiles = [&](auto kind_tag) {
      constexpr int KIND = decltype(kind_tag)::value;
      constexpr bool kDot = KIND != PK_INIT;
      constexpr bool kAcc = KIND != PK_ERR;
      constexpr bool kOut = KIND == PK_U || KIND == PK_V;
      auto issue = [&](int t) { issue_tile(feed, gt0, t); };
      constexpr bool kPP = !PIPE && SW == 0 && TEAMS == 2;
      const bool pp = kPP && A.pingpong != 0;
      if (twarp == 0) {
        if (!prefetched) {
#pragma unroll
          for (int t = 0; t < kAhead; ++t) issue(t);
        }
        if constexpr (!PIPE) {
          if (!pre_done) cp_async_wait<kAhead - 1>();   // tile 0 landed
        }
      }
      if constexpr (!PIPE) {
        if (!pre_done) named_bar(team_bar, TS);
      }

      // generate tile t's features into fr and publish its row-dot partials
      // GEN = false: fr already holds the tile (generated at the previous pass boundary)
      // Ping-pong (two teams): the teams' feature generations alternate — team 0 generates
      // tile t after team 1's tile t-1 (barrier 10), team 1 tile t after team 0's tile t
      // (barrier 11) — so one team's exchange and accumulation (shuffle / shared-memory work in
      // the MIO queue) run under the other team's ex2 instead of both teams generating at once
      // and then both leaving the MUFU idle.
      auto compute = [&](int t, float2 (&fr)[TR][NV][2], auto gen_tag) {
        if (twarp == 0) issue(t + kAhead);
        const uint32_t gi = gt0 + (uint32_t)t;
        const float* sl = tslots + (gi % kRing) * SLOT;
        if constexpr (PIPE) mbar_wait(&S.full[team][gi % kRing], (gi / kRing) & 1u);
        if constexpr (kPP) {
          if (pp && (team == 1 || t > 0)) named_bar(team == 0 ? 10u : 11u, 2 * TS);
        }
        if constexpr (decltype(gen_tag)::value) gen_features(sl, fr);
        else stash_load(fr);
        if constexpr (kPP) {
          if (pp) named_arrive(team == 0 ? 11u : 10u, 2 * TS);
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
        if constexpr (PIPE) {
          mbar_arrive(&S.redbar[team][rb]);   // also the per-tile team sync of the init pass
        } else {
          if (twarp == 0) cp_async_wait<kAhead - 1>();   // tile t+1 landed
          named_bar(team_bar, TS);   // publishes red[rb] and slot t+1 to the team
        }
      };

      // finish tile t: wait for the team's partials, derive the TR scalings (every warp the
      // same bits), write them (last warp), accumulate G^T w~ (w~ = h w)
      int nfin = 0;
      auto finish = [&](int t, float2 (&fr)[TR][NV][2]) {
        const uint32_t gi = gt0 + (uint32_t)t;
        const int lr = (team + t * TEAMS) * TR;
        const int rows = min(TR, nrows - lr);
        const float* sl = tslots + (gi % kRing) * SLOT;
        const int rb = (int)(gi % 3u);
        if constexpr (PIPE) mbar_wait(&S.redbar[team][rb], (gi / 3u) & 1u);
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
            const float tj = FACT ? h * tot : tot;     // t_j = F_j . s (STAB: of the normalised K)
            const float w = c * rcp_approx(tj);        // w_j = c_j / t_j
            wt = FACT ? w * h : w;
            if (twarp == NWT - 1 && (lane % G) == 0) {   // outputs: one lane per row
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
          if (valid) wt = FACT ? sl[32 + row] : 1.f;   // u^0 = 1 (reading C6): w~ = h; STAB: u~^0 = 1
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
      };

      if constexpr (PIPE) {
        float2 frA[TR][NV][2];
        float2 frB[TR][NV][2];
        if (ntiles > 0) {
          int t = 0;
          compute(0, frA, std::true_type{});
          while (true) {   // frA holds tile t
            if (t + 1 >= ntiles) { finish(t, frA); break; }
            compute(t + 1, frB, std::true_type{});
            finish(t, frA);
            ++t;           // frB holds tile t
            if (t + 1 >= ntiles) { finish(t, frB); break; }
            compute(t + 1, frA, std::true_type{});
            finish(t, frB);
            ++t;
          }
        }
      } else {
        float2 frA[TR][NV][2];
        int t0 = 0;
        if constexpr (kPre) {
          if (pre_done && ntiles > 0) {   // tile 0 from the stash (peeled: the loop always generates)
            compute(0, frA, std::false_type{});
            finish(0, frA);
            t0 = 1;
          }
        }
        for (int t = t0; t < ntiles; ++t) {
          compute(t, frA, std::true_type{});
          finish(t, frA);
        }
        if constexpr (kPP) {   // balance the ping-pong barriers when the teams' tile counts differ
          if (pp) {
            const int nt = (nrows + TR - 1) / TR, n0 = (nt + 1) / 2, n1 = nt / 2;
            if (team == 1 && n1 < n0) named_bar(11u, 2 * TS);
            if (team == 0 && n1 == n0 && n0 > 0) named_bar(10u, 2 * TS);
          }
        }
      }
    };
    if (strm) {
      stream_pass(kind, f, p);
    } else {
      switch (kind) {
        case PK_INIT: run_tiles(std::integral_constant<int, PK_INIT>{}); break;
        case PK_V: run_tiles(std::integral_constant<int, PK_V>{}); break;
        case PK_U: run_tiles(std::integral_constant<int, PK_U>{}); break;
        default: run_tiles(std::integral_constant<int, PK_ERR>{}); break;
      }
      gt += (uint32_t)ntiles;
      pre_done = false;
      if constexpr (!PIPE && SW == 0) {
        // boundary overlap: the next pass's first tiles are issued now (their slots are free),
        // so they have landed when the team generates tile 0's features at the boundary
        if (A.pre && twarp == 0) {
          const int q = p + 1;
          if (q < A.pass_end && pass_kind(q, A) != PK_NONE) {
            const Feed nf = make_feed(q);
#pragma unroll
            for (int t = 0; t < kAhead; ++t) issue_tile(nf, gt, t);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      acc_s[j * 4 + 0][tid] += (double)acc32[j].x;
      acc_s[j * 4 + 1][tid] += (double)acc32[j].y;
      acc_s[j * 4 + 2][tid] += (double)acc32[j].z;
      acc_s[j * 4 + 3][tid] += (double)acc32[j].w;
    }

    // ---------------- end of pass: teams combined (fixed order), cross-CTA fp64 reduction ---
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    if (!strm && twarp == NWT - 1) {
      e0 = warp_sum_f64(S.errL[team][lane]);
      e1 = warp_sum_f64(S.brkL[team][lane]);
      e2 = warp_sum_f64(S.wbL[team][lane]);
      S.errL[team][lane] = 0.0;
      S.brkL[team][lane] = 0.0;
      S.wbL[team][lane] = 0.0;
    }
    if (!strm && twarp == NWT - 1 && lane == 0) {   // hand the team's extras to its thread 0
      S.xs[0][NW - 1 - team] = e0;
      S.xs[1][NW - 1 - team] = e1;
      S.xs[2][NW - 1 - team] = e2;
    }
    named_bar(1, NT);   // every team's accumulators and extras are in shared memory
    if (!strm && tid == 0) {   // the extras, fixed order: team 0 + team 1 + ... (deterministic)
      e0 = S.xs[0][NW - 1];
      e1 = S.xs[1][NW - 1];
      e2 = S.xs[2][NW - 1];
#pragma unroll
      for (int tm = 1; tm < TEAMS; ++tm) {
        e0 += S.xs[0][NW - 1 - tm];
        e1 += S.xs[1][NW - 1 - tm];
        e2 += S.xs[2][NW - 1 - tm];
      }
    }
    if constexpr (TEAMS > 1) {
      if (team == 0) {   // fixed order: team 0 + team 1 + ... (deterministic)
#pragma unroll
        for (int tm = 1; tm < TEAMS; ++tm) {
#pragma unroll
          for (int e = 0; e < NV * 4; ++e) acc_s[e][ttid] += acc_s[e][ttid + tm * TS];
        }
      }
      // R1 (gpp > 1, no cluster) stores each team-0 thread's own combined columns and starts
      // with a CTA barrier of its own; the other boundary forms read other threads' columns
      if (A.gpp == 1 || A.cx || SW > 0) named_bar(1, NT);
    }
    if constexpr (SW > 0) {   // then the stream warps' partials, warp 0, 1, ... (fixed order)
      if (team == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const int gg = ttid + j * TS;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double a = acc_s[j * 4 + q][ttid];
            for (int w = 0; w < SW; ++w) a += sacc0[w * (GPL * 4 * 32) + ((gg >> 5) * 4 + q) * 32 + (gg & 31)];
            acc_s[j * 4 + q][ttid] = a;
          }
        }
        if (ttid == 0) {
          for (int w = 0; w < SW; ++w) {
            e0 += S.xsS[0][w];
            e1 += S.xsS[1][w];
          }
        }
      }
      named_bar(1, NT);
    }
    unsigned long long* trc = (A.trace && tid == 0) ? A.trace + ((int64_t)p * A.gpp + cta) * 4 : nullptr;
    if (trc) trc[0] = globaltimer();
    if (A.cx) {
      // partials: team 0's acc_s columns (teams already combined) + the extras, in this CTA's
      // shared memory; owners sum them over DSMEM (lsk_sink_common.cuh cx_*)
      if (tid == 0) {
        S.cxext[0] = e0;
        S.cxext[1] = e1;
        S.cxext[2] = e2;
        S.cxext[3] = 0.0;
      }
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);
      cx_r2<NT>(A, cxtot, cta, tid, [&](int kb, int q) -> uint32_t {
        if (kb >= R4) return smem_u32(&S.cxext[q]);
        return smem_u32(&acc_s[(kb / TS) * 4 + q][kb % TS]);
      });
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);
    } else if (A.gpp > 1) {
      if (team == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (gv[j])
            part_store4(part, A.gpp, g[j], cta, acc_s[j * 4 + 0][ttid], acc_s[j * 4 + 1][ttid],
                        acc_s[j * 4 + 2][ttid], acc_s[j * 4 + 3][ttid]);
        }
      }
      if (tid == 0) part_store4(part, A.gpp, r >> 2, cta, e0, e1, e2, 0.0);
      if (A.pre == 2) {   // the group barrier, with the next tile's features between arrive and wait
        named_bar(1, NT);
        if (tid == 0) red_release_add(A.bar + prob, 1u);
        ++nbar;
        pre_gen(p + 1);
        if (tid == 0) {
          while (ld_acquire(A.bar + prob) < nbar * (unsigned)A.gpp) {
          }
        }
        named_bar(1, NT);
      } else {
        group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
      }
      if (trc) trc[1] = globaltimer();
      // R2: this CTA reduces column blocks kb = cta, cta+gpp, ... (block r/4: the extras)
      r2_cta(A, prob, p, part, cta, warp, NW, lane);
      if (trc) trc[2] = globaltimer();
      if (trc) trc[3] = globaltimer();
    } else {
      if (tid == 0) {
        S.ext[0] = e0;
        S.ext[1] = e1;
        S.ext[2] = e2;
      }
      named_bar(1, NT);
    }
    // issue the next pass's first tiles now, after this CTA's share of the boundary work, so
    // they land while the CTA waits for the other CTAs' totals (slots gt.. are free: the ring
    // holds 2 * kAhead tiles)
    prefetched = false;
    if constexpr (!PIPE) {
      const int q = p + 1;
      if (q < A.pass_end && pass_kind(q, A) != PK_NONE) {
        if (!strm && twarp == 0 && !A.pre) {
          const Feed nf = make_feed(q);
#pragma unroll
          for (int t = 0; t < kAhead; ++t) issue_tile(nf, gt, t);
        }
        prefetched = true;
      }
    }
    // boundary overlap (after this CTA's share of R2, while the other owners finish theirs)
    if (A.pre && !strm && !pre_done) pre_gen(p + 1);
  }

  if constexpr (!PIPE) {
    if (twarp == 0) cp_async_wait<0>();   // a prefetch for a pass that did not run
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
    if (A.cx) {
      if (tid == 0) {
        S.cxext[4] = la;
        S.cxext[5] = lb;
      }
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);
      if (cta == 0 && tid == 0) {
        la = 0.0;
        lb = 0.0;
        for (int c = 0; c < A.gpp; ++c) {
          la += ld_dsmem_f64(mapa_shared(smem_u32(&S.cxext[4]), (uint32_t)c));
          lb += ld_dsmem_f64(mapa_shared(smem_u32(&S.cxext[5]), (uint32_t)c));
        }
      }
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);   // no CTA exits while CTA 0 reads it
    } else if (A.gpp > 1) {
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
      stg_state[ST_WBAD] = stWb;
      sticky_flags(A, stBrk, stWb);
      __threadfence();
      stg_state[ST_STOP] = 1.0;
    }
  } else if (multi && cta == 0 && tid == 0) {
    stg_state[ST_ERR] = stErr;
    stg_state[ST_BRK] = stBrk;
    stg_state[ST_WBAD] = stWb;
  }
}

// h_j = 2^(c2 |p_j|^2 - abar): the row factor of the factored exponent (same fp32 arithmetic
// as the expanded form's alpha2_j)
template <int D>
__global__ void row_scale_kernel(const float* __restrict__ X, int64_t n, float c2, float abar,
                                 float* __restrict__ h) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float al = 0.f;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float x = X[j * D + c];
    al = fmaf(x, x, al);
  }
  h[j] = ex2(al * c2 - abar);
}

// Stabilised mode (reading C30): m_j = max_k (beta2_k + sum_c W_kc p_jc) (log2 units, the same
// fp32 FMA order as the kernel's exponent) and the fp64 natural-log row offset
// A_j = (alpha2_j + m_j) ln 2 with alpha2_j = c2 |p_j|^2, so F_jk = e^{A_j} 2^{beta2_k + W_k.p_j - m_j}.
// Anchor constants staged in shared memory; one thread per row.
template <int D>
__global__ void __launch_bounds__(256) row_shift_kernel(const float* __restrict__ X, int64_t n,
                                                        const float* __restrict__ Wt,
                                                        const float* __restrict__ beta2, int r,
                                                        float c2, float* __restrict__ m2,
                                                        double* __restrict__ A) {
  extern __shared__ float cst[];   // [D + 1][r]: W rows, then beta2
  for (int i = threadIdx.x; i < (D + 1) * r; i += blockDim.x)
    cst[i] = i < D * r ? Wt[i] : beta2[i - D * r];
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float x[D];
  float al = 0.f;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    x[c] = X[j * D + c];
    al = fmaf(x[c], x[c], al);
  }
  float mx = -INFINITY;
  for (int k = 0; k < r; ++k) {
    float e = cst[D * r + k];
#pragma unroll
    for (int c = 0; c < D; ++c) e = fmaf(cst[c * r + k], x[c], e);
    mx = fmaxf(mx, e);
  }
  m2[j] = mx;
  A[j] = ((double)(al * c2) + (double)mx) * 0.69314718055994530942;
}

template <int TS, int TEAMS, int NV, int TR, int D, int SW = 0, bool PIPE = false>
constexpr size_t dyn_smem() {
  return sizeof(double) * NV * 4 * (TS * TEAMS + 32 * SW) +
         sizeof(float) * TEAMS * kRing * Geo<D>::SLOT + sizeof(float4) * NV * TS +
         sizeof(double) * SW * NV * TS * 4 + sizeof(float) * SW * kSRing * kSRow +
         ((!PIPE && SW == 0) ? sizeof(float4) * TR * NV * TS * TEAMS : 0);   // boundary stash
}

}  // namespace impl

// (TS, TEAMS, NV, TR, PIPE) per r and d, one CTA per SM.  Larger tiles amortise the per-tile
// team exchange (measured, DESIGN.md §6 K5); they need the registers of fewer threads.
// PIPE = 1 holds two feature tiles (lag-one software pipeline).
//   r <= 128:          eight one-warp teams, 4 columns per thread, 16-row tiles (small r: the
//                      per-tile exchange stays inside a warp, no padded columns);
//   r <= 1024, d <= 3: two 128-thread teams, 8 columns per thread, 16-row tiles (255 regs);
//   r <= 1024, d > 3:  four 128-thread teams, 8 columns per thread, 4-row tiles;
//   r <= 2048:         one 512-thread team, 4 columns per thread, 8-row tiles;
//   r <= 4096, d <= 3: one 256-thread team, 16 columns per thread, 8-row tiles;
//   r <= 4096, d > 3:  one 512-thread team, 8 columns per thread, 4-row tiles.
// LSK_ICFG="ts,teams,nv,tr,pipe" selects another instantiated configuration (tuning knob).
ImplCfg implicit_config(int r, int d) {
  const int r4 = (r + 3) / 4;
  ImplCfg c{};
#ifdef LSK_TUNING
  {
    // the warp-private kernel is opt-in (LSK_IWARP=1): measured slower than the team kernel on
    // config 2 (26.6 vs 24.0 us per pass, DESIGN.md §6 K5)
    const char* e = getenv("LSK_IWARP");
    int nw, nv, tr;
    if (e && atoi(e) == 1 && implicit_warp_config(r, d, &nw, &nv, &tr)) {
      c.ts = 32 * nw; c.teams = 1; c.nv = nv; c.tr = tr; c.pipe = 0; c.warp = 1;
      return c;
    }
  }
#endif
  if (r4 <= 32) c = ImplCfg{32, 8, 1, 16, 0, 0};   // small r: one warp per team, 8 teams
  else if (r4 <= 256) c = d <= 3 ? ImplCfg{128, 2, 2, 16, 0, 0} : ImplCfg{128, 4, 2, 4, 0, 0};
  else if (r4 <= 512) c = {512, 1, 1, 8, 0, 0};
  else c = d <= 3 ? ImplCfg{256, 1, 4, 8, 0, 0} : ImplCfg{512, 1, 2, 4, 0, 0};
#ifdef LSK_TUNING
  if (const char* e = getenv("LSK_ICFG")) {
    ImplCfg x{};
    if (sscanf(e, "%d,%d,%d,%d,%d", &x.ts, &x.teams, &x.nv, &x.tr, &x.pipe) == 5 &&
        x.ts * x.nv * 4 >= r)
      c = x;
  }
#endif
  return c;
}

#define LSK_IMPL_D(X, TS, TM, NV, TR, P) X(TS, TM, NV, TR, P, 1) X(TS, TM, NV, TR, P, 2) \
  X(TS, TM, NV, TR, P, 3) X(TS, TM, NV, TR, P, 4) X(TS, TM, NV, TR, P, 5)                  \
  X(TS, TM, NV, TR, P, 6) X(TS, TM, NV, TR, P, 7) X(TS, TM, NV, TR, P, 8)
#define LSK_IMPL_D123(X, TS, TM, NV, TR, P) X(TS, TM, NV, TR, P, 1) X(TS, TM, NV, TR, P, 2) \
  X(TS, TM, NV, TR, P, 3)
#define LSK_IMPL_D23(X, TS, TM, NV, TR, P) X(TS, TM, NV, TR, P, 2) X(TS, TM, NV, TR, P, 3)
// the configurations implicit_config selects (every d; the big-tile ones for d <= 3); tuning
// builds (-DLSK_TUNING) add the measured alternatives for d = 2, 3 and any LSK_IMPL_EXTRA_H
#define LSK_IMPL_DEFAULT(X) LSK_IMPL_D(X, 32, 8, 1, 16, 0)                                 \
  LSK_IMPL_D(X, 128, 4, 2, 4, 0) LSK_IMPL_D(X, 512, 1, 1, 8, 0)                           \
  LSK_IMPL_D(X, 512, 1, 2, 4, 0) LSK_IMPL_D123(X, 128, 2, 2, 16, 0)                       \
  LSK_IMPL_D123(X, 256, 1, 4, 8, 0)
#if defined(LSK_AB_ONLY)   // quick A/B builds: the config 1, 2 and 5 kernels only
#define LSK_IMPL_ALL(X) X(32, 8, 1, 16, 0, 2) X(128, 2, 2, 16, 0, 2) X(256, 1, 4, 8, 0, 3)
#elif defined(LSK_TUNING)
#define LSK_IMPL_ALL(X) LSK_IMPL_DEFAULT(X) LSK_IMPL_D23(X, 128, 2, 2, 8, 1) \
  LSK_IMPL_D23(X, 256, 1, 4, 2, 1) X(128, 3, 2, 8, 0, 2) LSK_IMPL_EXTRA(X)
#ifdef LSK_IMPL_EXTRA_H
#include LSK_IMPL_EXTRA_H
#else
#define LSK_IMPL_EXTRA(X)
#endif
#else
#define LSK_IMPL_ALL(X) LSK_IMPL_DEFAULT(X)
#endif

// cluster mode: the owners' fp64 totals follow the dynamic layout
static size_t cx_smem(const SinkArgs& a) {
  return a.cx ? sizeof(double) * (size_t)((a.r >> 2) + 1) * 4 : 0;
}

template <int TS, int TM, int NV, int TR, int D, int MODE, bool PIPE, int SW = 0>
static cudaError_t launch_cfg(const SinkArgs& a, bool coop, int grid, cudaStream_t s) {
  auto kern = impl::implicit_kernel<TS, TM, NV, TR, D, MODE, PIPE, SW>;
  const size_t dyn = impl::dyn_smem<TS, TM, NV, TR, D, SW, PIPE>() + cx_smem(a);
  constexpr int nthr = TS * TM + 32 * SW;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  if (a.cx) {   // one thread-block cluster per problem (gpp CTAs); clusters never wait on each other
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nthr);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)a.gpp;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, a);
  } else if (coop) {
    void* args[] = {(void*)&a};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(nthr), args, dyn, s);
  } else {
    kern<<<grid, nthr, dyn, s>>>(a);
    e = cudaGetLastError();
  }
  count_launch();
  return e;
}

template <int TS, int TM, int NV, int TR, int D, int MODE, bool PIPE, int SW = 0>
static int occupancy_cfg() {
  auto kern = impl::implicit_kernel<TS, TM, NV, TR, D, MODE, PIPE, SW>;
  constexpr size_t dyn = impl::dyn_smem<TS, TM, NV, TR, D, SW, PIPE>();
  int nb = 0;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, TS * TM + 32 * SW, dyn);
  return nb;
}

#ifdef LSK_TUNING
// Hybrid (a.nstream > 0): one 128-thread recompute team (measured 21.7 vs 20.5 us per pass for
// the two-team default on config 2 — the team's registers are what the stream warps use) plus
// four stream warps; r <= 1024, d <= 3, plain or factored exponent.
static cudaError_t launch_hybrid(const SinkArgs& a, bool coop, int grid, cudaStream_t s, int* occ) {
  if (a.r > 1024 || a.d > 3 || a.stab) return cudaErrorInvalidConfiguration;
  const int mode = a.hrow[0] != nullptr ? 1 : 0;
#define H(D_, M_)                                                                                if (a.d == D_ && mode == M_) {                                                                   if (occ) {                                                                                       *occ = occupancy_cfg<128, 1, 2, 16, D_, M_, false, 4>();                                       return cudaSuccess;                                                                          }                                                                                              return launch_cfg<128, 1, 2, 16, D_, M_, false, 4>(a, coop, grid, s);                        }
  H(1, 0) H(1, 1) H(2, 0) H(2, 1) H(3, 0) H(3, 1)
#undef H
  return cudaErrorInvalidConfiguration;
}
#endif

// the stabilised mode is instantiated for the default (non-pipelined) configurations only
template <int TS, int TM, int NV, int TR, int D, int P>
static cudaError_t stab_cfg(const SinkArgs& a, bool coop, int grid, cudaStream_t s, int* occ) {
  if constexpr (P == 0 && !(TS == 128 && TM == 3)) {
    if (occ) {
      *occ = occupancy_cfg<TS, TM, NV, TR, D, 2, false>();
      return cudaSuccess;
    }
    return launch_cfg<TS, TM, NV, TR, D, 2, false>(a, coop, grid, s);
  } else {
    return cudaErrorInvalidConfiguration;
  }
}

cudaError_t launch_implicit(const SinkArgs& a, bool coop, int grid, cudaStream_t s) {
  const ImplCfg c = implicit_config(a.r, a.d);
#ifdef LSK_TUNING
  if (itc_supported(a)) return launch_itc(a, grid, s);
#endif
  if (a.nstream[0] + a.nstream[1] > 0 && hybrid_supported(a)) return launch_hybrid_ws(a, grid, s);
#ifdef LSK_TUNING
  if (a.nstream[0] + a.nstream[1] > 0) return launch_hybrid(a, coop, grid, s, nullptr);
  if (c.warp && a.stab) return cudaErrorInvalidConfiguration;   // team kernel only
  if (c.warp) return launch_implicit_warp(a, coop, grid, s, nullptr);
#else
  if (a.nstream[0] + a.nstream[1] > 0 || c.warp) return cudaErrorInvalidConfiguration;
#endif
  const int mode = a.stab ? 2 : (a.hrow[0] != nullptr ? 1 : 0);
#define X(TS_, TM_, NV_, TR_, P_, D_)                                                          \
  if (c.ts == TS_ && c.teams == TM_ && c.nv == NV_ && c.tr == TR_ && c.pipe == P_ && a.d == D_) { \
    if (mode == 2) return stab_cfg<TS_, TM_, NV_, TR_, D_, P_>(a, coop, grid, s, nullptr);       \
    return mode == 1 ? launch_cfg<TS_, TM_, NV_, TR_, D_, 1, P_>(a, coop, grid, s)             \
                     : launch_cfg<TS_, TM_, NV_, TR_, D_, 0, P_>(a, coop, grid, s);            \
  }
  LSK_IMPL_ALL(X)
#undef X
  return cudaErrorInvalidConfiguration;
}

int implicit_max_ctas_per_sm(const SinkArgs& a) {
  const ImplCfg c = implicit_config(a.r, a.d);
  if (a.bimg[0] != nullptr) return 1;   // tensor-core exponent kernel (all of TMEM per CTA)
  if (a.nstream[0] + a.nstream[1] > 0 && a.r <= 1024 && a.d <= 3 && !a.stab) return 1;   // hybrid
#ifdef LSK_TUNING
  if (a.nstream[0] + a.nstream[1] > 0) {
    int occ = 0;
    return launch_hybrid(a, false, 0, nullptr, &occ) == cudaSuccess ? occ : 0;
  }
  if (c.warp) {
    int occ = 0;
    return launch_implicit_warp(a, false, 0, nullptr, &occ) == cudaSuccess ? occ : 0;
  }
#else
  if (a.nstream[0] + a.nstream[1] > 0 || c.warp) return 0;
#endif
  const int mode = a.stab ? 2 : (a.hrow[0] != nullptr ? 1 : 0);
#define X(TS_, TM_, NV_, TR_, P_, D_)                                                          \
  if (c.ts == TS_ && c.teams == TM_ && c.nv == NV_ && c.tr == TR_ && c.pipe == P_ && a.d == D_) { \
    if (mode == 2) {                                                                           \
      int occ = 0;                                                                             \
      return stab_cfg<TS_, TM_, NV_, TR_, D_, P_>(a, false, 0, nullptr, &occ) == cudaSuccess ? occ : 0; \
    }                                                                                          \
    return mode == 1 ? occupancy_cfg<TS_, TM_, NV_, TR_, D_, 1, P_>()                          \
                     : occupancy_cfg<TS_, TM_, NV_, TR_, D_, 0, P_>();                         \
  }
  LSK_IMPL_ALL(X)
#undef X
  return 0;
}

cudaError_t launch_row_shift(const float* X, int64_t n, int d, const float* Wt,
                             const float* beta2, int r, float c2, float* m2, double* A,
                             cudaStream_t s) {
  const unsigned blocks = (unsigned)((n + 255) / 256);
  const size_t dyn = sizeof(float) * (d + 1) * r;
  switch (d) {
#define C(D_)                                                                                  \
  case D_:                                                                                     \
    cudaFuncSetAttribute(impl::row_shift_kernel<D_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn); \
    impl::row_shift_kernel<D_><<<blocks, 256, dyn, s>>>(X, n, Wt, beta2, r, c2, m2, A);         \
    break;
    C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_row_scale(const float* X, int64_t n, int d, float c2, float abar, float* h,
                             cudaStream_t s) {
  const unsigned blocks = (unsigned)((n + 255) / 256);
  switch (d) {
#define C(D_) case D_: impl::row_scale_kernel<D_><<<blocks, 256, 0, s>>>(X, n, c2, abar, h); break;
    C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace lsk
