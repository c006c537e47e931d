// lsk_implicit_tc.cu — Alg. 1 on K_theta = xi zeta^T without materialising
// the factors, with the exponent of every regenerated entry computed on the 5th-generation
// tensor cores (DESIGN.md §6 K9, round 2).
//
// The recompute kernel (lsk_implicit.cu) spends, per entry, one FFMA2 on the exponent
// E_kj = beta2_k + abar + W_k . p_j (d = 2; the factored form of Lemma decomp-RBF, PAPER.md:934,
// see lsk_implicit.cu's header), plus the register moves that broadcast p_j, next to the one
// MUFU ex2 — and its tile loop is issue/latency bound, not MUFU bound (DESIGN.md §6 K5).  Here
// the exponents of a whole tile come from ONE kind::tf32 tcgen05.mma per 128 anchors, with the
// 3xTF32 split packed into K = 8:
//     A row k = [Wh_k1 .. Wh_kd | Wl_k1 .. Wl_kd | Wh_k1 .. Wh_kd | bh_k  bl_k | 0 ..]
//     B row j = [ph_j1 .. ph_jd | ph_j1 .. ph_jd | pl_j1 .. pl_jd |  1     1   | 0 ..]
// (hi = cvt.rna.tf32(x), lo = cvt.rna.tf32(x - hi); the dropped Wl.pl term is ~2^-22 of |W||p|),
// so D[k][j] = E_kj lands in TMEM with the anchors k on the lanes and the tile's rows j on the
// columns — the recompute kernel's ownership (a thread owns columns, rows run in registers).
// Each thread then reads its 8 anchors x 16 rows with tcgen05.ld and does only the ex2, the
// row-dot FFMA2 and the accumulation FFMA2.  Measured on B200 (scripts/micro/tmem_ex2.cu):
// tcgen05.ld sustains > 150 B/clk/SM, ex2 fed from TMEM runs at 15.2 of 16 /clk/SM, and the
// packed MMA's exponent error is 7.2e-6 at |E| <= 89 (the fp32 FMA chain's: 4.0e-6).
//
// Layout: one CTA per SM (the TMEM allocation takes all 512 columns), two teams of 128 threads
// (one warp per TMEM lane quarter).  Thread (q, l) of a team owns anchors k = 128 b + 32 q + l,
// b = 0..7 (r <= 1024).  Teams take alternate 16-row tiles; each team double-buffers its TMEM
// tile (8 blocks x 16 columns): the MMA of tile t+1 runs while the team finishes tile t.  The
// team's warp 0 stages tiles (the precomputed B image rows, c_j, h_j, v_old_j) 2 ahead with
// cp.async into an 8-slot ring; its lane 0 issues the MMAs (tcgen05.commit -> the buffer's
// mbarrier).  Per tile: wait MMA -> tcgen05.ld -> ex2 -> row-dot partials (FFMA2 over row pairs)
// -> warp transpose-reduce -> one named barrier per team -> the exchange (a fixed xor
// butterfly: every lane of a group gets the same bits) -> t_j, w_j = c_j rcp(t_j) -> FFMA2
// accumulation -> fp64 every 64 rows.  Pass boundary, stopping test and read-out are those of
// the other persistent kernels (lsk_sink_common.cuh; deterministic fixed-order reductions).
#include <cmath>
#include <type_traits>

#include "lsk_internal.h"
#include "lsk_ptx.cuh"
#include "lsk_sink_common.cuh"

namespace lsk {
namespace itc {

constexpr int TS = 128;            // threads per team (one warp per TMEM lane quarter)
constexpr int TEAMS = 2;
constexpr int NT = TS * TEAMS;
constexpr int NW = NT / 32;
constexpr int NWT = TS / 32;
constexpr int NB = 8;              // 128-anchor blocks: r <= 1024, anchors per thread
constexpr int TR = 8;              // rows per tile = the MMA's N
constexpr int NBUF = 4;            // TMEM tile buffers per team (NB x TR columns each)
constexpr int kRing = 8;           // tile slots per team
constexpr int kAhead = 4;          // slots staged ahead
constexpr int kMmaAhead = 2;       // MMAs issued ahead of the tile being computed
constexpr int kSlot = 384;         // bytes: B image [8 rows x 32 B] | c[8] | h[8] | vold[8] (| pad)
constexpr int kImgBlk = 128 * 32;  // bytes of one 128-row K = 8 tf32 image block
constexpr int kTmemCols = 512;
constexpr int kDynSmem = 120 * 1024;   // > half an SM: one CTA per SM (TMEM: all 512 columns)
// instruction descriptor: D f32, A = B = tf32, both K-major, N = TR, M = 128
static_assert(TEAMS * NBUF * NB * TR == 512, "TMEM columns");
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TR >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);

// byte offset of (row, k) in a K-major SWIZZLE_NONE tf32 image with K = 8: core matrices of
// 8 rows x 16 B; the two K halves of an 8-row group 128 B apart (LBO), groups 256 B apart (SBO)
__host__ __device__ __forceinline__ uint32_t img_off(int row, int k) {
  return (uint32_t)((row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

struct Smem {
  uint64_t mma[TEAMS][NBUF];       // MMA of the team's TMEM buffer done (tcgen05.commit)
  uint32_t tmem;
  float red[TEAMS][3][TR][NWT];
  double xs[3][NW];
  double errL[TEAMS][32];
  double brkL[TEAMS][32];
  double wbL[TEAMS][32];
  double st[4];                    // err, breakdowns, final err, bad weights
  int ist[2];                      // final_t, conv
};

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void ldtm16(uint32_t (&r)[16], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void ldtm8(uint32_t (&r)[8], uint32_t taddr) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void sttm8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void sttm_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void ldtm_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int D>
__global__ void __launch_bounds__(NT, 1) itc_kernel(const SinkArgs A) {
  constexpr int kFlushTiles = 64 / TR;
  constexpr int LPR = 32 / TR;   // lanes per row after the transpose-reduce
  constexpr int G = NWT < LPR ? NWT : LPR, PER = NWT / G;
  static_assert(3 * D + 2 <= 8, "K = 8 packing holds d <= 2");
  __shared__ __align__(16) Smem S;
  extern __shared__ __align__(1024) unsigned char dyn[];
  unsigned char* wimg = dyn;                                   // [NB][128 x 32 B]
  unsigned char* slots = wimg + NB * kImgBlk;                  // [TEAMS][kRing][kSlot]
  float* s_sm = reinterpret_cast<float*>(slots + TEAMS * kRing * kSlot);   // [NB * 128]
  double* acc_col = reinterpret_cast<double*>(s_sm + NB * 128);          // [TEAMS][NB * 128]

  const int tid = threadIdx.x;
  const int team = tid / TS, ttid = tid - team * TS;
  const int warp = tid >> 5, lane = tid & 31, twarp = ttid >> 5;
  const int cta = blockIdx.x;
  const int r = A.r;
  const int R4 = r >> 2;
  double* stg_state = A.state;
  const uint32_t team_bar = 2u + (uint32_t)team;

  // ---- setup: TMEM, barriers, the anchor image (A operand), zeroed slots ----------------
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem)), "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int tm = 0; tm < TEAMS; ++tm)
      for (int i = 0; i < NBUF; ++i) mbar_init(&S.mma[tm][i], 1);
    fence_mbar_init();
    S.st[0] = __ldcg(stg_state + ST_ERR);
    S.st[1] = __ldcg(stg_state + ST_BRK);
    S.st[2] = -1.0;
    S.st[3] = __ldcg(stg_state + ST_WBAD);
    S.ist[0] = -1;
    S.ist[1] = 0;
  }
  for (int k = tid; k < NB * 128; k += NT) {   // anchor row k of the packed 3xTF32 image
    float row[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (k < r) {
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const float w = A.Wt[(int64_t)c * r + k];
        const float wh = tf32_rna(w);
        row[c] = wh;
        row[D + c] = tf32_rna(w - wh);
        row[2 * D + c] = wh;
      }
      const float b = A.beta2[k] + A.abar;
      const float bh = tf32_rna(b);
      row[3 * D] = bh;
      row[3 * D + 1] = tf32_rna(b - bh);
    } else {
      row[3 * D] = -1e30f;   // padding anchors: E = -1e30, ex2 -> exact 0
    }
    unsigned char* blk = wimg + (k >> 7) * kImgBlk;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      *reinterpret_cast<float4*>(blk + img_off(k & 127, 4 * h)) =
          make_float4(row[4 * h], row[4 * h + 1], row[4 * h + 2], row[4 * h + 3]);
  }
  for (int i = tid; i < TEAMS * kRing * kSlot / 16; i += NT)
    reinterpret_cast<float4*>(slots)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid < 32)
    for (int tm = 0; tm < TEAMS; ++tm) S.errL[tm][tid] = S.brkL[tm][tid] = S.wbL[tm][tid] = 0.0;
  fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem;
  const uint32_t wimg_a = smem_u32(wimg);
  unsigned char* tslots = slots + team * kRing * kSlot;

  int64_t rbeg[2];
  int rcnt[2];
#pragma unroll
  for (int fs = 0; fs < 2; ++fs) {
    int64_t q1;
    cta_rows(A.rows[fs], A.gpp, cta, &rbeg[fs], &q1);
    rcnt[fs] = (int)(q1 - rbeg[fs]);
  }
  double* part = A.part;
  const int64_t rstride = r + kExtra;

  // owned anchors k_b = 128 b + 32 twarp + lane
  const int kown = 32 * twarp + lane;
  float2 s2[NB];   // (s_k, s_k) pairs for the row-pair FFMA2
#pragma unroll
  for (int b = 0; b < NB; ++b) s2[b] = make_float2(0.f, 0.f);
  for (int k = ttid; k < NB * 128; k += TS) acc_col[team * NB * 128 + k] = 0.0;
  unsigned int nbar = 0;
  uint32_t gt = 0;   // tiles of this team so far: slot gt % kRing, TMEM buffer gt % NBUF
  bool prefetched = false;
  int mma_pref = 0;   // MMAs of the next pass already issued (its first tiles)

  struct Feed {
    const float *w, *img, *h, *vold;
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
    fd.img = A.bimg[fq] + q0 * 8;   // the B image rows (8 floats per point row)
    fd.h = A.hrow[fq] + q0;
    const bool nv = (kq == PK_ERR) || (kq == PK_V && q >= 3);
    fd.vold = nv ? vbuf_ptr(A, 0, (kq == PK_ERR) ? A.T : (q + 1) / 2 - 1) + q0 : nullptr;
    return fd;
  };
  // team warp 0: tile t of a pass -> slot (g0 + t) % kRing; one cp.async group per tile
  auto issue_tile = [&](const Feed& fd, uint32_t g0, int t) {
    if (t < fd.ntiles) {
      const int lr = (team + t * TEAMS) * TR;
      unsigned char* sl = tslots + ((g0 + (uint32_t)t) % kRing) * kSlot;
      const int rows = min(TR, fd.nrows - lr);
      {   // B image: lane -> row lane / 2, K half lane % 2 (16 B each)
        const int row = lane >> 1, hk = lane & 1;
        if (lane < 2 * TR && row < rows)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sl + img_off(row, 4 * hk))),
                       "l"(fd.img + (int64_t)(lr + row) * 8 + 4 * hk)
                       : "memory");
      }
      float* sc = reinterpret_cast<float*>(sl + 32 * TR);
      if (lane < rows) {
        cp_async4(sc + lane, fd.w + lr + lane);
        cp_async4(sc + TR + lane, fd.h + lr + lane);
        if (fd.vold) cp_async4(sc + 2 * TR + lane, fd.vold + lr + lane);
      }
    }
    cp_async_commit();
  };
  // team lane 0 of warp 0: the 8 MMAs of tile gi into TMEM buffer gi % NBUF
  auto tbuf = [&](uint32_t gi) { return (uint32_t)((team * NBUF + (int)(gi % NBUF)) * NB * TR); };
  auto issue_mma = [&](uint32_t gi) {
    tc_fence_after();
    const uint32_t bsl = smem_u32(tslots + (gi % kRing) * kSlot);
    const uint64_t bdesc = desc_none(bsl);
    const uint32_t dcol = tmem + tbuf(gi);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint64_t adesc = desc_none(wimg_a + b * kImgBlk);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol + b * TR),
          "l"(adesc), "l"(bdesc), "r"(kIdesc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&S.mma[team][gi % NBUF]))
                 : "memory");
  };

  for (int p = A.pass_begin;; ++p) {
    // ---------------- results of pass p-1: stopping test (as implicit_kernel) ------------
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
    if (kind != PK_INIT) {   // s -> fp32 in shared memory once per CTA
      for (int k = tid; k < NB * 128; k += NT) {
        float v = 0.f;
        if (k < r) v = (float)sv_load(sv_of(A, 0, p - 1) + k, false);
        s_sm[k] = v;
      }
      named_bar(1, NT);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const float v = s_sm[128 * b + kown];
        s2[b] = make_float2(v, v);
      }
    }
    float2 acc2[NB];   // (even rows, odd rows) fp32 partials per owned anchor
#pragma unroll
    for (int b = 0; b < NB; ++b) acc2[b] = make_float2(0.f, 0.f);
    double* accd = acc_col + team * NB * 128;
    auto flush = [&]() {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        accd[128 * b + kown] += (double)acc2[b].x + (double)acc2[b].y;
        acc2[b] = make_float2(0.f, 0.f);
      }
    };

    const Feed feed = make_feed(p);
    const int nrows = feed.nrows, ntiles = feed.ntiles;
    const bool need_vold = feed.vold != nullptr;
    float* outp0 = nullptr;
    if (kind == PK_U) outp0 = A.out[0] + rbeg[0];
    if (kind == PK_V) outp0 = vbuf_ptr(A, 0, (p + 1) / 2) + rbeg[1];
    const uint32_t gt0 = gt;
    // Phase-split tile pipeline (per team): phase A of tile t (TMEM exponents -> ex2 -> row-dot
    // partials -> the features written back over the exponents), one team barrier, then phase
    // B of tile t-1 (its exchange, whose partials were published a whole phase A earlier, and
    // the accumulation from the features read back from TMEM).  The registers hold one block of
    // 8 x 8 features at a time, and the exchange latency hides behind the next tile's MUFU work.
    auto run_tiles = [&](auto kind_tag) {
      constexpr int KIND = decltype(kind_tag)::value;
      constexpr bool kDot = KIND != PK_INIT;
      constexpr bool kAcc = KIND != PK_ERR;
      constexpr bool kOut = KIND == PK_U || KIND == PK_V;
      if (twarp == 0) {
        if (!prefetched)
          for (int t = 0; t < kAhead; ++t) issue_tile(feed, gt0, t);
        const int want = min(ntiles, kMmaAhead);
        if (mma_pref < want) {
          cp_async_wait<kAhead - kMmaAhead>();   // tiles 0 .. kMmaAhead-1 landed
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0)
            for (int t = mma_pref; t < want; ++t) issue_mma(gt0 + (uint32_t)t);
        }
      }
      int nfin = 0;
      // phase B of tile u: scalings from the team's partials, outputs, accumulation
      auto phase_b = [&](int u) {
        const uint32_t gi = gt0 + (uint32_t)u;
        const float* sc = reinterpret_cast<const float*>(tslots + (gi % kRing) * kSlot + 32 * TR);
        const int rb = (int)(gi % 3u);
        const int lr = (team + u * TEAMS) * TR;
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
            const float c = sc[row];
            const float h = sc[TR + row];
            const float tj = h * tot;               // t_j = F_j . s = h_j (G_j . s)
            const float w = c * rcp_approx(tj);     // w_j = c_j / t_j
            wt = w * h;                             // w~_j = h_j w_j
            if (twarp == NWT - 1 && (lane % G) == 0) {
              if (bad_weight(c)) S.wbL[team][row] += 1.0;
              if (need_vold) S.errL[team][row] += fabs((double)sc[2 * TR + row] * (double)tj - (double)c);
              if constexpr (kOut) {
                if (!(w > 0.f) || !isfinite(w)) S.brkL[team][row] += 1.0;
                outp0[lr + row] = w;
              }
            }
          }
          if constexpr (!kAcc) wt = 0.f;
        } else {
          if (valid) wt = sc[TR + row];   // u^0 = 1 (reading C6): w~ = h
        }
        if constexpr (kAcc) {
          float2 v2[TR / 2];
#pragma unroll
          for (int i = 0; i < TR / 2; ++i)
            v2[i] = make_float2(__shfl_sync(0xffffffffu, wt, (2 * i) * G),
                                __shfl_sync(0xffffffffu, wt, (2 * i + 1) * G));
          const uint32_t tb = tmem + ((uint32_t)(32 * twarp) << 16) + tbuf(gi);
          uint32_t f[NB][TR];
#pragma unroll
          for (int b = 0; b < NB; ++b) ldtm8(f[b], tb + b * TR);
          ldtm_wait();
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int i = 0; i < TR / 2; ++i)
              acc2[b] = fma2(make_float2(__uint_as_float(f[b][2 * i]), __uint_as_float(f[b][2 * i + 1])),
                             v2[i], acc2[b]);
          if (++nfin == kFlushTiles) {
            nfin = 0;
            flush();
          }
        }
      };
      for (int t = 0; t < ntiles; ++t) {
        const uint32_t gi = gt0 + (uint32_t)t;
        // the loader first makes tile t + kMmaAhead visible to the tensor core (it was staged
        // kAhead - kMmaAhead tiles ago), THEN stages tile t + kAhead: the proxy fence must not
        // wait for loads still in flight
        if (twarp == 0) {
          cp_async_wait<kAhead - kMmaAhead - 1>();   // tiles <= t + kMmaAhead landed
          fence_proxy_async_smem();
          issue_tile(feed, gt0, t + kAhead);
        }
        // ---- phase A of tile t ----
        mbar_wait(&S.mma[team][gi % NBUF], (gi / NBUF) & 1u);
        tc_fence_after();
        const uint32_t tb = tmem + ((uint32_t)(32 * twarp) << 16) + tbuf(gi);
        float2 pp[TR / 2];
#pragma unroll
        for (int i = 0; i < TR / 2; ++i) pp[i] = make_float2(0.f, 0.f);
        {
          uint32_t e[NB][TR];
#pragma unroll
          for (int b = 0; b < NB; ++b) ldtm8(e[b], tb + b * TR);
          ldtm_wait();
#pragma unroll
          for (int b = 0; b < NB; ++b) {
#pragma unroll
            for (int i = 0; i < TR; ++i) e[b][i] = __float_as_uint(ex2(__uint_as_float(e[b][i])));
            if constexpr (kDot) {
#pragma unroll
              for (int i = 0; i < TR / 2; ++i)
                pp[i] = fma2(make_float2(__uint_as_float(e[b][2 * i]), __uint_as_float(e[b][2 * i + 1])),
                             s2[b], pp[i]);
            }
            if constexpr (kAcc) sttm8(tb + b * TR, e[b]);   // the features over the exponents
          }
        }
        const int rb = (int)(gi % 3u);
        if constexpr (kDot) {
          float pr[TR];
#pragma unroll
          for (int i = 0; i < TR / 2; ++i) {
            pr[2 * i] = pp[i].x;
            pr[2 * i + 1] = pp[i].y;
          }
          const float tot = warp_transpose_reduce<TR>(pr, lane);
          if ((lane & (LPR - 1)) == 0) S.red[team][rb][lane / LPR][twarp] = tot;
        }
        if constexpr (kAcc) sttm_wait();
        tc_fence_before();
        named_bar(team_bar, TS);   // red[t] and the slots published; phase B(t-1) reads done
        // tile t + kMmaAhead -> TMEM buffer of tile t + kMmaAhead - NBUF (its phase B was before
        // this barrier)
        if (ttid == 0 && t + kMmaAhead < ntiles) issue_mma(gi + (uint32_t)kMmaAhead);
        tc_fence_after();
        // ---- phase B of tile t-1 ----
        if (t > 0) phase_b(t - 1);
      }
      if (ntiles > 0) {   // drain: phase B of the last tile after its partials are published
        tc_fence_before();
        named_bar(team_bar, TS);
        tc_fence_after();
        phase_b(ntiles - 1);
      }
    };
    switch (kind) {
      case PK_INIT: run_tiles(std::integral_constant<int, PK_INIT>{}); break;
      case PK_V: run_tiles(std::integral_constant<int, PK_V>{}); break;
      case PK_U: run_tiles(std::integral_constant<int, PK_U>{}); break;
      default: run_tiles(std::integral_constant<int, PK_ERR>{}); break;
    }
    gt += (uint32_t)ntiles;
    flush();

    // ---------------- end of pass: teams combined (fixed order), cross-CTA fp64 reduction ---
    if (twarp == NWT - 1) {   // each team's output warp
      const double e0 = warp_sum_f64(S.errL[team][lane]);
      const double e1 = warp_sum_f64(S.brkL[team][lane]);
      const double e2 = warp_sum_f64(S.wbL[team][lane]);
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
    // column groups g = tid: team 0 + team 1 (fixed order: deterministic), then R1
    for (int g4 = tid; g4 < R4; g4 += NT) {
      double v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[e] = acc_col[4 * g4 + e];
#pragma unroll
        for (int tm = 1; tm < TEAMS; ++tm) v[e] += acc_col[tm * NB * 128 + 4 * g4 + e];
      }
      part_store4(part, A.gpp, g4, cta, v[0], v[1], v[2], v[3]);
    }
    if (tid == 0) {
      double e0 = S.xs[0][0], e1 = S.xs[1][0], e2 = S.xs[2][0];
      for (int tm = 1; tm < TEAMS; ++tm) {
        e0 += S.xs[0][tm];
        e1 += S.xs[1][tm];
        e2 += S.xs[2][tm];
      }
      part_store4(part, A.gpp, R4, cta, e0, e1, e2, 0.0);
    }
    named_bar(1, NT);   // every team's columns read before they are zeroed
    for (int k = ttid; k < NB * 128; k += TS) acc_col[team * NB * 128 + k] = 0.0;
    group_barrier<NT>(A.bar, (++nbar) * (unsigned)A.gpp, tid);
    r2_cta(A, 0, p, part, cta, warp, NW, lane);
    // the next pass's first tiles and its first MMA now: they land while this CTA waits for
    // the totals (the exponents do not depend on s)
    prefetched = false;
    mma_pref = 0;
    const int q = p + 1;
    if (q < A.pass_end && pass_kind(q, A) != PK_NONE) {
      if (twarp == 0) {
        const Feed nf = make_feed(q);
        for (int t = 0; t < kAhead; ++t) issue_tile(nf, gt, t);
        const int want = min(nf.ntiles, kMmaAhead);
        if (want > 0) {
          cp_async_wait<kAhead - kMmaAhead>();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0)
            for (int t = 0; t < want; ++t) issue_mma(gt + (uint32_t)t);
        }
        mma_pref = want;
      }
      prefetched = true;
    }
  }

  if (twarp == 0) cp_async_wait<0>();
  // an early stop leaves the next pass's prefetched MMA in flight: wait for it before the
  // TMEM is released
  if (ttid == 0)
    for (int t = 0; t < mma_pref; ++t) {
      const uint32_t gi = gt + (uint32_t)t;
      mbar_wait(&S.mma[team][gi % NBUF], (gi / NBUF) & 1u);
    }
  // ---------------- returned v into the user buffer, then the fp64 read-out -----------------
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
  // every MMA was waited on (each issued tile was consumed); release TMEM
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
}

// B image of a side: row j = [ph | ph | pl | 1 1 | 0 ..] (K = 8 tf32), one thread per row
__global__ void bimg_kernel(const float* __restrict__ X, int64_t n, int d, float* __restrict__ img) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float row[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int c = 0; c < d; ++c) {
    const float x = X[j * d + c];
    const float xh = tf32_rna(x);
    row[c] = xh;
    row[d + c] = xh;
    row[2 * d + c] = tf32_rna(x - xh);
  }
  row[3 * d] = 1.f;
  row[3 * d + 1] = 1.f;
  float4* o = reinterpret_cast<float4*>(img + j * 8);
  o[0] = make_float4(row[0], row[1], row[2], row[3]);
  o[1] = make_float4(row[4], row[5], row[6], row[7]);
}

}  // namespace itc

bool itc_supported(const SinkArgs& a) {
  return a.bimg[0] != nullptr && a.bimg[1] != nullptr && a.r <= itc::NB * 128 && a.d >= 1 &&
         a.d <= 2 && a.hrow[0] != nullptr && !a.stab &&
         !a.multi_launch && a.nprob == 1 && !a.cx && !a.emul && a.gpp > 1 &&
         a.nstream[0] + a.nstream[1] == 0;
}

size_t itc_image_floats(int64_t rows) { return (size_t)rows * 8; }

cudaError_t launch_itc_image(const float* X, int64_t n, int d, float* img, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  itc::bimg_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(X, n, d, img);
  count_launch();
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_d(const SinkArgs& a, int grid, cudaStream_t s) {
  auto kern = itc::itc_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, itc::kDynSmem);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&a};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(itc::NT), args, itc::kDynSmem, s);
  count_launch();
  return e;
}

cudaError_t launch_itc(const SinkArgs& a, int grid, cudaStream_t s) {
  if (a.d == 1) return launch_d<1>(a, grid, s);
  if (a.d == 2) return launch_d<2>(a, grid, s);
  return cudaErrorInvalidConfiguration;
}

}  // namespace lsk
