// lsk_sinkhorn.cu — Alg. 1 on K_theta = xi zeta^T as ONE
// persistent launch per solve (or one launch per pass when an NCCL all-reduce sits between
// passes).
//
// Schedule ("row-fused passes"): an iteration is a v-pass over zeta then a u-pass over xi.
// For each factor row j the pass computes t_j = F_j . s (fp32, r-long dot), w_j = c_j / t_j
// (c = b for the v-pass, a for the u-pass), and accumulates s'_k += F_jk w_j — so each factor
// is read from HBM exactly once per iteration: 4 r (n+m) bytes.  The
// naive 4-GEMV schedule would read 8 r (n+m).
//
// CTA layout: 8 consumer warps + 1 producer warp.  The producer streams a contiguous row
// range of the factor through a shared-memory ring with 1-D bulk async copies (TMA engine,
// cp.async.bulk + mbarrier complete_tx) and fetches per-row scalars (c_j, v_old_j) with
// cp.async; the factor stream does not depend on s, so the ring keeps HBM busy across the
// grid barriers between passes.  Consumer thread t owns float4 column groups
// {t, t+256, ...}: its slice of s and of the fp64 accumulator live in registers, so the
// accumulation needs no intra-CTA reduction.  Row dots are reduced with a warp
// transpose-reduce (TR rows in TR-1+5-log2(TR) shuffles) and one smem exchange.
//
// Precision (C13): r-long dots in fp32; the n-long accumulation of s in fp32 over
// <= 32 rows, then fp64; cross-CTA reduction in fp64 in a fixed order (deterministic, no
// float atomics).  Marginal error and a^T log u / b^T log v in fp64.
//
// The recompute (implicit) variant has its own kernels: lsk_implicit.cu.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {

constexpr int NT = kConsumerThreads;
constexpr int NW = NT / 32;
constexpr int kHdr = 64 + 32 * 16;   // stage header floats: c[32], vold[32], (pad) — keeps the
                                     // factor rows 16-byte aligned after the header
constexpr int kMaxStages = 16;

struct Smem {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t redbar[3];
  float red[3][NW][32];
  double xs[2][NW];
  double ext[kExtra];
  double cxext[2];  // cluster mode: this CTA's read-out partials
  uint64_t cxbar;   // cluster mode: cluster-scope pass barrier
  int done_seq;   // last pass finished by the consumers: base(k) + pass, k-th problem of the CTA
  int stop_seq;   // base(k) once the k-th problem of the CTA has stopped (tolerance mode)
  int mstop;      // multi-launch mode: the consumers stop at the top of this launch
};

// CW: columns per consumer group — 4 (float4 groups) or, for r <= 512 (fewer float4 groups than
// consumer threads), 2 (float2 groups: every consumer thread owns columns, round 2; with float4
// groups half the threads would load and multiply duplicate data, the per-tile cost of r = 1024
// for half the bytes)
template <int NV, int TR, int CW = 4>
__global__ void __launch_bounds__(kThreads, 1) sinkhorn_kernel(const SinkArgs A) {
  static_assert(CW == 4 || (CW == 2 && NV == 1), "float2 groups: one group per thread");
  extern __shared__ __align__(128) float ring[];
  __shared__ Smem S;
  constexpr int kFlushTiles = (32 / TR) > 0 ? (32 / TR) : 1;   // fp32 partial over <= 32 rows

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // groups of gpp CTAs; a group runs problems group, group + ngroups, ... (persistent)
  const int group = blockIdx.x / A.gpp;
  const int cta = blockIdx.x - group * A.gpp;
  const int ngroups = (int)gridDim.x / A.gpp;
  const int r = A.r;
  const int seq_stride = A.num_passes + 2;

  if (A.multi_launch && __ldcg(A.state + ST_STOP) != 0.0) return;   // solve already finished

  if (tid == 0) {
    for (int i = 0; i < A.nstage; ++i) {
      mbar_init(&S.full[i], 33);   // producer lane-0 arrive (+tx) + 32 cp.async arrivals
      mbar_init(&S.empty[i], NW);  // one arrival per consumer warp
    }
    for (int i = 0; i < 3; ++i) mbar_init(&S.redbar[i], NT);
    S.done_seq = A.pass_begin - 1;
    S.stop_seq = -1;
    // Multi-launch mode (one pass per launch, batch 1, gpp >= 2): the consumers' stopping test
    // on pass pass_begin - 1 runs at the top of the launch, before any tile; decide it here for
    // the producer too (same inputs, same comparisons), so it never streams a pass the
    // consumers will not consume (it would block on a full ring).
    S.mstop = 0;
    if (A.multi_launch && A.pass_begin > 0) {
      const int q = A.pass_begin - 1;
      bool stop = q == A.num_passes - 1;
      if (A.tol_mode && pass_kind(q, A) == PK_V && (q + 1) / 2 >= 2)
        stop = stop || __ldcg(sv_of(A, 0, q) + r) < A.tol;
      S.mstop = stop ? 1 : 0;
    }
    if (A.cx) mbar_init(&S.cxbar, (uint32_t)A.gpp);
    fence_mbar_init();
  }
  // zero the ring once: tail tiles then compute on finite data without per-row predicates
  for (int64_t i = tid; i < (int64_t)A.nstage * A.stage_floats / 4; i += kThreads)
    reinterpret_cast<float4*>(ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_proxy_async_smem();
  __syncthreads();
  if (A.cx) cluster_sync_all();   // all threads (producer too): barriers initialised cluster-wide
  // cluster mode: this CTA's fp64 partials and the owners' totals, after the ring
  double* cxpart = reinterpret_cast<double*>(ring + (int64_t)A.nstage * A.stage_floats);
  double* cxtot = cxpart + ((r >> 2) + 1) * 4;
  uint32_t cxphase = 0;

  // ======================================= producer =======================================
  if (warp == NW) {
    if (S.mstop) return;
    uint32_t stage = 0, phase = 0;
    const uint64_t pol = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    int pk = 0;
    for (int prob = group; prob < A.nprob; prob += ngroups, ++pk) {
    const int base = pk * seq_stride;
    bool stopped_here = false;
    for (int p = A.pass_begin; p < A.pass_end; ++p) {
      const int kind = pass_kind(p, A);
      if (kind == PK_NONE) continue;
      const int f = (kind == PK_V || kind == PK_ERR) ? 1 : 0;
      const bool need_vold = (kind == PK_ERR) || (kind == PK_V && p >= 3);
      int wait_for = -1;
      if (need_vold) wait_for = p - 2;                      // v_old written by pass p-2
      if (A.tol_mode && kind == PK_U && p >= 4) wait_for = p - 1;   // stop decision
      if (wait_for >= A.pass_begin) {
        while (*(volatile int*)&S.done_seq < base + wait_for) __nanosleep(32);
        __syncwarp();
        __threadfence_block();
        if (*(volatile int*)&S.stop_seq == base) {
          stopped_here = true;
          break;
        }
      }
      int64_t r0, r1;
      cta_rows(A.rows[f], A.gpp, cta, &r0, &r1);
      const float* wp = A.w[f] + (int64_t)prob * A.wstride[f];
      const float* vold = nullptr;
      if (need_vold) vold = vbuf_ptr(A, prob, (kind == PK_ERR) ? A.T : (p + 1) / 2 - 1);
      const float* Fp = A.F[f] + (int64_t)prob * A.fstride[f];
      // the first l2_resident of this CTA's rows stay in L2 across iterations (evict_last)
      const int64_t keep_end = r0 + (int64_t)((double)(r1 - r0) * (double)A.l2_resident);
      for (int64_t row0 = r0; row0 < r1; row0 += TR) {
        const int rows = (int)min((int64_t)TR, r1 - row0);
        mbar_wait(&S.empty[stage], phase ^ 1u);
        float* st = ring + (int64_t)stage * A.stage_floats;
        if (lane == 0) {
          const uint32_t bytes = (uint32_t)rows * (uint32_t)r * 4u;
          mbar_arrive_expect_tx(&S.full[stage], bytes);
          bulk_g2s(st + kHdr, Fp + row0 * r, bytes, &S.full[stage], row0 < keep_end ? pol_keep : pol);
        }
        if (lane < rows) {
          cp_async4(st + lane, wp + row0 + lane);
          if (need_vold) cp_async4(st + 32 + lane, vold + row0 + lane);
        }
        cp_async_mbar_arrive_noinc(&S.full[stage]);
        if (++stage == (uint32_t)A.nstage) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    (void)stopped_here;
    }   // problems
    return;
  }

  // ======================================= consumers ======================================
  const int RG = r / CW;   // column groups
  int g[NV];
  bool gv[NV];
  int ge[NV];   // clamped group index: invalid groups read column group 0 and use s = 0
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    g[j] = tid + j * NT;
    gv[j] = g[j] < RG;
    ge[j] = gv[j] ? g[j] : 0;
  }
  // one column group of a feature row in shared memory (float2 groups: z, w = 0)
  auto load_group = [](const float* rowp, int grp) -> float4 {
    if constexpr (CW == 4) {
      return *reinterpret_cast<const float4*>(rowp + 4 * grp);
    } else {
      const float2 v = *reinterpret_cast<const float2*>(rowp + 2 * grp);
      return make_float4(v.x, v.y, 0.f, 0.f);
    }
  };
  float4 s[NV];
  double acc64[NV][4];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc64[j][q] = 0.0;
  }

  uint32_t stage = 0, phase = 0;
  uint32_t tk = 0;         // tiles that used a red buffer (buffer tk % 3, phase (tk / 3) & 1)
  const bool multi = A.multi_launch != 0;
  const int64_t rstride = r + kExtra;
  int pk = 0;
  for (int prob = group; prob < A.nprob; prob += ngroups, ++pk) {
  const int base = pk * seq_stride;
  double* stg_state = A.state + (int64_t)prob * kStateDoubles;
  // running solve state (identical in every CTA of the problem)
  double stErr = __ldcg(stg_state + ST_ERR);
  double stBrk = __ldcg(stg_state + ST_BRK);
  double stWb = __ldcg(stg_state + ST_WBAD);
  double* part = A.part + prob * part_per_problem(r, A.gpp);   // [blk][gpp][4]
  unsigned int nbar = 0;   // group barriers passed for this problem in this launch
  int final_t = -1, conv = 0;
  double ferr = -1.0;

  for (int p = A.pass_begin;; ++p) {
    // ---------------- results of pass q = p-1: stopping test ----------------------------------
    const bool have_prev = multi ? (p == A.pass_begin && p > 0) : (p > A.pass_begin);
    if (have_prev) {
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
          stErr = e_err;   // err_{t-1} = |v^{t-1} o K^T u^{t-1} - b|_1
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
      if (tid == 0) {
        if (final_t >= 0) *(volatile int*)&S.stop_seq = base;
        __threadfence_block();
        *(volatile int*)&S.done_seq = base + q;
      }
      if (final_t >= 0) break;
    }
    if (p >= A.pass_end) break;

    // ---------------- pass p ---------------------------------------------------------------
    const int kind = pass_kind(p, A);
    if (kind == PK_NONE) continue;
    const int f = (kind == PK_V || kind == PK_ERR) ? 1 : 0;
    if (kind != PK_INIT) {
      if (A.cx) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (gv[j]) {
            double x[4];
            if constexpr (CW == 4) {
              cx_total4(cxtot, A.gpp, g[j], x);
              s[j] = make_float4((float)x[0], (float)x[1], (float)x[2], (float)x[3]);
            } else {
              cx_total4(cxtot, A.gpp, g[j] >> 1, x);
              const int o = 2 * (g[j] & 1);
              s[j] = make_float4((float)x[o], (float)x[o + 1], 0.f, 0.f);
            }
          } else {
            s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      } else if (A.gpp > 1) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (gv[j]) {
            if constexpr (CW == 4) {
              double2 lo, hi;
              sv_load4(sv_of(A, prob, p - 1) + 4 * g[j], multi, lo, hi);
              s[j] = make_float4((float)lo.x, (float)lo.y, (float)hi.x, (float)hi.y);
            } else {
              const double2 lo = sv_load2(sv_of(A, prob, p - 1) + 2 * g[j], multi);
              s[j] = make_float4((float)lo.x, (float)lo.y, 0.f, 0.f);
            }
          } else {
            s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j)
          s[j] = gv[j] ? make_float4((float)acc64[j][0], (float)acc64[j][1], (float)acc64[j][2],
                                     (float)acc64[j][3])
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc64[j][q] = 0.0;

    int64_t r0, r1;
    cta_rows(A.rows[f], A.gpp, cta, &r0, &r1);
    float* outp = nullptr;
    if (kind == PK_U) outp = A.out[0] + (int64_t)prob * A.wstride[0];
    if (kind == PK_V) outp = vbuf_ptr(A, prob, (p + 1) / 2);
    const bool err_here = (kind == PK_ERR) || (kind == PK_V && p >= 3);
    double errsum = 0.0, brksum = 0.0, wbsum = 0.0;   // warp 0, lanes < TR
    float4 acc32[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    int tiles_since_flush = 0;

    // Software-pipelined tile loop: tile k's row dots are reduced across warps through
    // red[k % 3] + an mbarrier (split arrive / wait), and finished (scaling, accumulation,
    // stage release) only after tile k+1's dots are issued — no CTA-wide barrier per tile.
    int64_t row0 = r0;
    bool pend = false;              // a tile whose dots are issued but not finished
    int64_t p_row0 = 0;
    int p_rows = 0;
    uint32_t p_stage = 0, p_tk = 0;

    // finish a tile: wait for all warps' partial dots, derive the TR scalings (every warp
    // computes them identically), write them (warp 0), accumulate F_j^T w_j, release the stage
    auto finish = [&](uint32_t fstage, int64_t frow0, int frows, uint32_t ftk) {
      const float* st = ring + (int64_t)fstage * A.stage_floats;
      const float* feat = st + kHdr;
      float vr_l = 0.f;
      if (kind == PK_INIT) {
        vr_l = (lane < frows) ? 1.f : 0.f;   // u^0 = 1 (reading C6): s_v^0 = xi^T 1
      } else {
        const int rb = (int)(ftk % 3u);
        mbar_wait(&S.redbar[rb], (ftk / 3u) & 1u);
        if (lane < frows) {
          float t = 0.f;
#pragma unroll
          for (int w = 0; w < NW; ++w) t += S.red[rb][w][lane];   // fixed order: all warps agree
          const float c = st[lane];
          if (kind != PK_ERR) vr_l = __fdiv_rn(c, t);
          if (warp == 0) {
            if (bad_weight(c)) wbsum += 1.0;
            if (err_here) errsum += fabs((double)st[32 + lane] * (double)t - (double)c);
            if (kind != PK_ERR) {
              if (!(vr_l > 0.f) || !isfinite(vr_l)) brksum += 1.0;
              outp[frow0 + lane] = vr_l;
            }
          }
        }
      }
      if (kind != PK_ERR) {
        // vr_l = 0 in lanes >= frows, so tail rows add 0 x (finite stale/zero data)
        float vis[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) vis[i] = __shfl_sync(0xffffffffu, vr_l, i);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          float4 fvv[TR];
#pragma unroll
          for (int i = 0; i < TR; ++i) fvv[i] = load_group(feat + i * r, ge[j]);
#pragma unroll
          for (int i = 0; i < TR; ++i) {
            const float vi = vis[i];
            const float4 fv = fvv[i];
            acc32[j].x = fmaf(fv.x, vi, acc32[j].x);
            acc32[j].y = fmaf(fv.y, vi, acc32[j].y);
            if constexpr (CW == 4) {
              acc32[j].z = fmaf(fv.z, vi, acc32[j].z);
              acc32[j].w = fmaf(fv.w, vi, acc32[j].w);
            }
          }
        }
        if (++tiles_since_flush == kFlushTiles) {
          tiles_since_flush = 0;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            acc64[j][0] += (double)acc32[j].x;
            acc64[j][1] += (double)acc32[j].y;
            acc64[j][2] += (double)acc32[j].z;
            acc64[j][3] += (double)acc32[j].w;
            acc32[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[fstage]);
    };

    // issue the dots of the tile at row0; then finish the pending tile
    auto step = [&]() -> bool {
      if (row0 >= r1) return false;
      const int rows = (int)min((int64_t)TR, r1 - row0);
      mbar_wait(&S.full[stage], phase);
      if (A.dbg == 1) {   // tuning probe: pure streaming rate of the producer / TMA ring
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[stage]);
        if (++stage == (uint32_t)A.nstage) { stage = 0; phase ^= 1u; }
        row0 += TR;
        return true;
      }
      const float* st = ring + (int64_t)stage * A.stage_floats;
      const float* feat = st + kHdr;
      uint32_t my_tk = tk;
      if (kind != PK_INIT) {
        // rows >= `rows` of a tail tile hold finite stale/zero data; their dots are unused
        float pr[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) pr[i] = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          float4 fvv[TR];
#pragma unroll
          for (int i = 0; i < TR; ++i)   // all loads of this column group first
            fvv[i] = load_group(feat + i * r, ge[j]);
#pragma unroll
          for (int i = 0; i < TR; ++i) {
            const float4 fv = fvv[i];
            pr[i] = fmaf(fv.x, s[j].x, pr[i]);
            pr[i] = fmaf(fv.y, s[j].y, pr[i]);
            if constexpr (CW == 4) {
              pr[i] = fmaf(fv.z, s[j].z, pr[i]);
              pr[i] = fmaf(fv.w, s[j].w, pr[i]);
            }
          }
        }
        const float tot = warp_transpose_reduce<TR>(pr, lane);
        constexpr int kLanesPerRow = 32 / TR;
        const int rb = (int)(tk % 3u);
        if ((lane & (kLanesPerRow - 1)) == 0) S.red[rb][warp][lane / kLanesPerRow] = tot;
        mbar_arrive(&S.redbar[rb]);   // every consumer lane arrives (count NT)
        ++tk;
      }
      if (pend) finish(p_stage, p_row0, p_rows, p_tk);
      pend = true;
      p_stage = stage;
      p_row0 = row0;
      p_rows = rows;
      p_tk = my_tk;
      if (++stage == (uint32_t)A.nstage) {
        stage = 0;
        phase ^= 1u;
      }
      row0 += TR;
      return true;
    };
    while (step()) {
    }
    if (pend) finish(p_stage, p_row0, p_rows, p_tk);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      acc64[j][0] += (double)acc32[j].x;
      acc64[j][1] += (double)acc32[j].y;
      acc64[j][2] += (double)acc32[j].z;
      acc64[j][3] += (double)acc32[j].w;
    }

    // ---------------- end of pass: CTA extras, then cross-CTA fp64 reduction ----------------
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    if (warp == 0) {
      e0 = warp_sum_f64(errsum);
      e1 = warp_sum_f64(brksum);
      e2 = warp_sum_f64(wbsum);
    }
    unsigned long long* trc = (A.trace && tid == 0) ? A.trace + ((int64_t)p * A.gpp + cta) * 4 : nullptr;
    if (trc) trc[0] = globaltimer();   // tiles done
    if (A.cx) {
      // this CTA's partials to its shared memory; owners sum them over DSMEM
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if (gv[j]) {
          double2* d2 = reinterpret_cast<double2*>(cxpart + CW * g[j]);
          d2[0] = make_double2(acc64[j][0], acc64[j][1]);
          if constexpr (CW == 4) d2[1] = make_double2(acc64[j][2], acc64[j][3]);
        }
      }
      if (tid == 0) {
        cxpart[4 * (r >> 2) + 0] = e0;
        cxpart[4 * (r >> 2) + 1] = e1;
        cxpart[4 * (r >> 2) + 2] = e2;
        cxpart[4 * (r >> 2) + 3] = 0.0;
      }
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);
      cx_r2<NT>(A, cxtot, cta, tid,
                [&](int kb, int q) -> uint32_t { return smem_u32(cxpart + 4 * kb + q); });
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);
    } else if (A.gpp > 1) {
      // R1: block partials part[blk][cta][4] (lsk_sink_common.cuh)
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if (gv[j]) {
          if constexpr (CW == 4) {
            part_store4(part, A.gpp, g[j], cta, acc64[j][0], acc64[j][1], acc64[j][2], acc64[j][3]);
          } else {   // half of block g/2: columns 2g, 2g+1
            double2* d = reinterpret_cast<double2*>(part + ((((int64_t)(g[j] >> 1)) * A.gpp + cta) << 2) +
                                                    2 * (g[j] & 1));
            *d = make_double2(acc64[j][0], acc64[j][1]);
          }
        }
      }
      if (tid == 0) part_store4(part, A.gpp, r >> 2, cta, e0, e1, e2, 0.0);
      group_barrier<NT>(A.bar + prob, (++nbar) * (unsigned)A.gpp, tid);
      if (trc) trc[1] = globaltimer();   // barrier 1 passed
      // R2: this CTA reduces columns k = cta, cta+gpp, ... in a fixed order
      // R2: this CTA reduces column blocks kb = cta, cta+gpp, ... (block r/4: the extras)
      r2_cta(A, prob, p, part, cta, warp, NW, lane);
      if (trc) trc[2] = globaltimer();   // R2 done
      if (trc) trc[3] = globaltimer();   // barrier 2 passed
    } else {
      if (tid == 0) {
        S.ext[0] = e0;
        S.ext[1] = e1;
        S.ext[2] = e2;
      }
      named_bar(1, NT);
    }
  }

  if (final_t >= 0) {
    // ---------------- final phase: returned v to the user buffer, then the fp64 read-out
    // W_hat = eps (a^T log u + b^T log v) of the returned state
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
        S.cxext[0] = la;
        S.cxext[1] = lb;
      }
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);
      if (cta == 0 && tid == 0) {
        la = 0.0;
        lb = 0.0;
        for (int c = 0; c < A.gpp; ++c) {
          la += ld_dsmem_f64(mapa_shared(smem_u32(&S.cxext[0]), (uint32_t)c));
          lb += ld_dsmem_f64(mapa_shared(smem_u32(&S.cxext[1]), (uint32_t)c));
        }
      }
      cx_barrier<NT>(&S.cxbar, cxphase, A.gpp, tid);   // no CTA moves on while CTA 0 reads it
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
    // multi-launch mode: persist the running state for the next launch
    stg_state[ST_ERR] = stErr;
    stg_state[ST_BRK] = stBrk;
    stg_state[ST_WBAD] = stWb;
  }
  }   // problems
}

// ------------------------------------------------------------------------------------------
void sinkhorn_tile_config(int r, int max_stage_bytes, int* tr, int* nv) {
  const int r4 = (r + 3) / 4;
  int v = (r4 + NT - 1) / NT;
  int p2 = 1;
  while (p2 < v) p2 <<= 1;
  *nv = (2 * r4 <= NT) ? 0 : p2;   // 0: one float2 group per consumer thread (r <= 512)
  // largest instantiated TR whose stage fits the budget (target 64 KB: long tiles amortise
  // the per-tile cross-warp exchange; measured on config 2: 32 KB stages 4.6 TB/s, 64 KB
  // stages 5.3 TB/s)
  const int lo = std::max(1, 8 / p2), hi = std::max(1, 32 / p2);
  int tt = hi;
  const int budget = std::min(max_stage_bytes, 65536 + kHdr * 4);
  while (tt > lo && (kHdr + tt * r) * 4 > budget) tt >>= 1;
#ifdef LSK_TUNING
  if (const char* e = getenv("LSK_TR")) {   // tuning knob
    const int x = atoi(e);
    if (x >= lo && x <= hi) tt = x;
  }
#endif
  *tr = tt;
}

size_t sinkhorn_static_smem() { return sizeof(Smem); }

template <int NV, int TR, int CW = 4>
static cudaError_t launch_t(const SinkArgs& a, bool coop, int grid, size_t smem,
                            cudaStream_t s) {
  auto kern = sinkhorn_kernel<NV, TR, CW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (a.cx) {   // one thread-block cluster per group of gpp CTAs (groups never wait on each other)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
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
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kThreads), args, smem, s);
  } else {
    kern<<<grid, kThreads, smem, s>>>(a);
    e = cudaGetLastError();
  }
  count_launch();
  return e;
}

template <int NV, int TR, int CW = 4>
static int occupancy_t(size_t smem) {
  int nb = 0;
  auto kern = sinkhorn_kernel<NV, TR, CW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, smem);
  return nb;
}

// nv = 0: NV = 1 with float2 column groups (r <= 512)
#define LSK_STREAM_CASES(X) X(1, 32) X(1, 16) X(1, 8) X(2, 16) X(2, 8) X(2, 4) X(4, 8) X(4, 4) \
  X(4, 2) X(8, 4) X(8, 2) X(8, 1)
#define LSK_STREAM_HALF_CASES(Y) Y(32) Y(16) Y(8)

cudaError_t launch_sinkhorn(const SinkArgs& a, bool coop, int grid, size_t smem, cudaStream_t s) {
  const int tr = a.tr, nv = a.nv;
#define X(NV_, TR_) if (nv == NV_ && tr == TR_) return launch_t<NV_, TR_>(a, coop, grid, smem, s);
  LSK_STREAM_CASES(X)
#undef X
#define Y(TR_) if (nv == 0 && tr == TR_) return launch_t<1, TR_, 2>(a, coop, grid, smem, s);
  LSK_STREAM_HALF_CASES(Y)
#undef Y
  return cudaErrorInvalidConfiguration;
}

template <int NV, int TR, int CW = 4>
static int active_clusters_t(size_t smem, int csize) {
  auto kern = sinkhorn_kernel<NV, TR, CW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

int sinkhorn_max_active_clusters(int nv, int tr, size_t smem, int csize) {
#define X(NV_, TR_) if (nv == NV_ && tr == TR_) return active_clusters_t<NV_, TR_>(smem, csize);
  LSK_STREAM_CASES(X)
#undef X
#define Y(TR_) if (nv == 0 && tr == TR_) return active_clusters_t<1, TR_, 2>(smem, csize);
  LSK_STREAM_HALF_CASES(Y)
#undef Y
  return 0;
}

int sinkhorn_max_ctas_per_sm(int nv, int tr, size_t smem) {
#define X(NV_, TR_) if (nv == NV_ && tr == TR_) return occupancy_t<NV_, TR_>(smem);
  LSK_STREAM_CASES(X)
#undef X
#define Y(TR_) if (nv == 0 && tr == TR_) return occupancy_t<1, TR_, 2>(smem);
  LSK_STREAM_HALF_CASES(Y)
#undef Y
  return 0;
}

}  // namespace lsk
