// lsk_sink_common.cuh — device helpers shared by the streaming and the implicit Sinkhorn
// kernels: pass schedule, row partition, deterministic warp reductions, group barrier.
#pragma once
#include "lsk_internal.h"
#include "lsk_ptx.cuh"

namespace lsk {

__device__ __forceinline__ int pass_kind(int p, const SinkArgs& A) {
  if (p == 0) return PK_INIT;
  if (p <= 2 * A.T) return (p & 1) ? PK_V : PK_U;
  if (p == 2 * A.T + 1 && A.want_err) return PK_ERR;
  return PK_NONE;
}

__device__ __forceinline__ void cta_rows(int64_t total, int gpp, int cta, int64_t* r0,
                                         int64_t* r1) {
  *r0 = (total * cta) / gpp;
  *r1 = (total * (cta + 1)) / gpp;
}

// Warp transpose-reduce: each lane holds v[0..TR) (one partial per row).  Returns, in every
// lane, the warp total of row (lane >> (5 - log2 TR)).  Fixed shuffle pattern: deterministic.
template <int TR>
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[TR], int lane) {
#pragma unroll
  for (int w = TR / 2, off = 16; w >= 1; w >>= 1, off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = upper ? v[i] : v[i + w];
      const float keep = upper ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  constexpr int kLog = (TR >= 32) ? 5 : (TR >= 16) ? 4 : (TR >= 8) ? 3 : (TR >= 4) ? 2 : (TR >= 2) ? 1 : 0;
#pragma unroll
  for (int off = 16 >> kLog; off >= 1; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
  return v[0];
}

__device__ __forceinline__ double warp_sum_f64(double x) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// Barrier among the gpp CTAs of one problem: monotone counter, k-th barrier waits for
// k * gpp arrivals (counter zeroed once per solve by the host).
// bar.sync orders the CTA's writes before thread 0's gpu-scope release; thread 0's acquire
// is ordered before the other threads' reads by the second bar.sync (cumulativity) — the
// same pattern as CUTLASS's GenericBarrier.  Readers use ld.global.cg (L2), so no L1 flush.
template <int NTHR>
__device__ __forceinline__ void group_barrier(unsigned int* ctr, unsigned int target, int tid) {
  named_bar(1, NTHR);
  if (tid == 0) {
    red_release_add(ctr, 1u);
    while (ld_acquire(ctr) < target) {
    }
  }
  named_bar(1, NTHR);
}

// ---- cross-CTA r-vector exchange without a second barrier ----------------------------------
// The fp64 result of pass p (R2) goes to svec buffer p & 1 of the problem ([2][r + kExtra]).
// Its readers (the next pass) poll each value until it differs from the sentinel (all-ones
// bits: a NaN that no arithmetic produces), so no group barrier is needed between R2 and the
// next pass.  The R2 owner of a column re-arms the other buffer (pass p-1's result, whose
// readers all passed this pass's barrier 1) — visible to the readers of pass p+1's result
// through barrier 1 of pass p+1.  Multi-launch mode (NCCL all-reduce between launches) keeps
// one buffer and plain loads: the launch boundary orders everything.
constexpr unsigned long long kSvSentinel = ~0ull;

__device__ __forceinline__ double* sv_of(const SinkArgs& A, int prob, int pass) {
  double* base = A.svec + (int64_t)prob * 2 * (A.r + kExtra);
  return (A.multi_launch || !(pass & 1)) ? base : base + (A.r + kExtra);
}

__device__ __forceinline__ double sv_load(const double* p, bool multi) {
  if (multi) return __ldcg(p);
  unsigned long long b;
  for (;;) {   // back off between polls: early CTAs must not flood the L2 lines being written
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
    if (b != kSvSentinel) break;
    __nanosleep(100);
  }
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ double2 sv_load2(const double* p, bool multi) {
  if (multi) return __ldcg(reinterpret_cast<const double2*>(p));
  unsigned long long b0, b1;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(b0), "=l"(b1) : "l"(p) : "memory");
    if (b0 != kSvSentinel && b1 != kSvSentinel) break;
    __nanosleep(100);
  }
  return make_double2(__longlong_as_double((long long)b0), __longlong_as_double((long long)b1));
}

// four consecutive values (a float4 column group) in one poll: one L2 round trip instead of
// the two of back-to-back sv_load2 calls
__device__ __forceinline__ void sv_load4(const double* p, bool multi, double2& lo, double2& hi) {
  if (multi) {
    lo = __ldcg(reinterpret_cast<const double2*>(p));
    hi = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    return;
  }
  unsigned long long b0, b1, b2, b3;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%4];\n\t"
                 "ld.relaxed.gpu.global.v2.b64 {%2, %3}, [%5];"
                 : "=l"(b0), "=l"(b1), "=l"(b2), "=l"(b3) : "l"(p), "l"(p + 2) : "memory");
    if (b0 != kSvSentinel && b1 != kSvSentinel && b2 != kSvSentinel && b3 != kSvSentinel) break;
    __nanosleep(100);
  }
  lo = make_double2(__longlong_as_double((long long)b0), __longlong_as_double((long long)b1));
  hi = make_double2(__longlong_as_double((long long)b2), __longlong_as_double((long long)b3));
}

// the pass's extras (block r/4: err, breakdowns, bad weights, 0) in one poll: both 16-byte
// loads are issued before either is tested, so the three values cost one L2 round trip
// (three sequential sv_load calls cost three, on the path every CTA waits on)
__device__ __forceinline__ void sv_load_extras(const double* p, bool multi, double& e_err,
                                               double& e_brk, double& e_wb) {
  if (multi) {
    const double2 lo = __ldcg(reinterpret_cast<const double2*>(p));
    e_err = lo.x;
    e_brk = lo.y;
    e_wb = __ldcg(p + 2);
    return;
  }
  unsigned long long b0, b1, b2, b3;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%4];\n\t"
                 "ld.relaxed.gpu.global.v2.b64 {%2, %3}, [%5];"
                 : "=l"(b0), "=l"(b1), "=l"(b2), "=l"(b3) : "l"(p), "l"(p + 2) : "memory");
    if (b0 != kSvSentinel && b1 != kSvSentinel && b2 != kSvSentinel && b3 != kSvSentinel) break;
    __nanosleep(100);
  }
  e_err = __longlong_as_double((long long)b0);
  e_brk = __longlong_as_double((long long)b1);
  e_wb = __longlong_as_double((long long)b2);
}

// ---- cross-GPU exchange over NVLink peer memory (one persistent launch per GPU) -----------
// The owner of column k on every rank (same CTA partition on every rank) adds the ranks' local
// totals in rank order: it stores its own total into slot [par][my rank][k] of EVERY rank's
// inbox (through NVLink), polls its own inbox slots [par][src][k] until they differ from the
// all-ones sentinel, sums them src = 0, 1, ... (the same bits on every rank: deterministic),
// and re-arms the slots it consumed.  par alternates with the pass: ranks can be at most one
// pass apart (pass p+1 needs every rank's pass-p totals), and a slot consumed in pass p is
// rewritten (by its source, in pass p+2) only after that source saw this rank's pass p+1
// total.  Ordering: each value is one aligned 64-bit store (single-copy atomic, so a poll sees
// the sentinel or the whole value), and ONE fence.acq_rel.sys at the top of each call orders
// everything this thread did in the previous call — its polls (acquire side: the values it
// read) and its re-arms (release side) — before the stores of this call; a source's store of
// pass p+2 therefore follows its poll of this rank's pass-p+1 total, which follows this rank's
// re-arm of pass p.  (Round 1 used a st.release.sys per store, N fences per call.)  A poll that
// outlives A.xtimeout_ns sets ST_XERR (and the sticky status) and yields NaN, so a broken
// peer cannot hang the GPU.  In emulation mode (A.emul) the ranks are the problems of one
// cooperative launch on one GPU (rank = problem index) — the same code and protocol.
__device__ __forceinline__ double xpoll(const double* p, long long deadline, int* timed_out) {
  unsigned long long b;
  for (;;) {
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
    if (b != kSvSentinel) return __longlong_as_double((long long)b);
    if (*timed_out || (long long)globaltimer() > deadline) {
      *timed_out = 1;
      return __longlong_as_double(0x7ff8000000000000ll);   // NaN
    }
    __nanosleep(64);
  }
}

__device__ __forceinline__ double xrank_total(const SinkArgs& A, int prob, int par, int k,
                                              double local) {
  const int N = A.nranks;
  const int me = A.emul ? prob : A.rank;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int d = 0; d < N; ++d)
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(A.xbox[d] + ((int64_t)(par * N + me) * A.xrs + k)),
                 "d"(local)
                 : "memory");
  double* mine = A.xbox[me] + (int64_t)par * N * A.xrs + k;
  const long long deadline = (long long)globaltimer() + A.xtimeout_ns;
  int timed_out = 0;
  double tot = 0.0;
  for (int src = 0; src < N; ++src) tot += xpoll(mine + (int64_t)src * A.xrs, deadline, &timed_out);
  for (int src = 0; src < N; ++src)
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(mine + (int64_t)src * A.xrs), "l"(kSvSentinel)
                 : "memory");
  if (timed_out) {
    A.state[(int64_t)prob * kStateDoubles + ST_XERR] = 1.0;
    if (A.sticky) atomicOr(A.sticky, STICKY_XERR);
  }
  return tot;
}

// R2 owner: publish column k of pass p (the all-rank total when the launch spans GPUs) and
// re-arm the same column of pass p-1's buffer
__device__ __forceinline__ void sv_publish(const SinkArgs& A, int prob, int pass, int k, double v) {
  if (A.nranks > 1) v = xrank_total(A, prob, pass & 1, k, v);
  double* cur = sv_of(A, prob, pass);
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(cur + k), "d"(v) : "memory");
  if (!A.multi_launch) {
    double* prv = sv_of(A, prob, pass + 1);   // the other buffer
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(prv + k), "l"(kSvSentinel) : "memory");
  }
}

// ---- R1/R2 partial layout: column blocks of 4, part[blk][cta][4] ---------------------------
// Per problem (r + kExtra + 4) * gpp doubles: blocks 0..r/4-1 the r-vector, block r/4 the
// extras (err, breakdowns, 0, 0), block r/4+1 the read-out partials.  A CTA's four partials
// of a block are one 32-byte sector (R1: one coalesced store pair per float4 group instead of
// four scattered 8-byte stores, so the barrier's release drains fewer stores), and a block's
// partials of all CTAs are contiguous (R2 reads 32 * gpp consecutive bytes).
__device__ __forceinline__ int64_t part_per_problem(int r, int gpp) {
  return (int64_t)(r + kExtra + 4) * gpp;
}
__device__ __forceinline__ double* part_at(double* part, int gpp, int k, int cta) {
  return part + (((int64_t)(k >> 2) * gpp + cta) << 2) + (k & 3);
}
__device__ __forceinline__ void part_store4(double* part, int gpp, int blk, int cta, double a0,
                                            double a1, double a2, double a3) {
  double2* d = reinterpret_cast<double2*>(part + (((int64_t)blk * gpp + cta) << 2));
  d[0] = make_double2(a0, a1);
  d[1] = make_double2(a2, a3);
}

// R2 of column block kb (columns 4kb..4kb+3) by G2 lanes of a warp: every lane adds the
// partials of the CTAs it reads in increasing CTA order (double2 e = sub + G2 i holds CTA e/2's
// columns 2(e&1), 2(e&1)+1), then an xor butterfly over the group's lanes of equal parity — a
// fixed order, the same bits on every run — and the group's lanes 0, 1 publish the four totals.
// G2 = 2 gpp rounded up to a power of two (<= 32): small groups reduce 32 / G2 blocks per warp
// in one round trip.
__device__ __forceinline__ void sv_publish(const SinkArgs& A, int prob, int pass, int k, double v);
__device__ __forceinline__ int r2_lanes(int gpp) {
  int g = 2;
  while (g < 2 * gpp && g < 32) g <<= 1;
  return g;
}
__device__ __forceinline__ void r2_block(const SinkArgs& A, int prob, int pass, const double* part,
                                         int kb, int sub, int G2, bool active) {
  const double2* src = reinterpret_cast<const double2*>(part + (((int64_t)kb * A.gpp) << 2));
  const int n2 = 2 * A.gpp;
  double ax = 0.0, ay = 0.0;
  constexpr int kBatch = 10;   // loads in flight per lane (one L2 round trip for gpp <= 160)
  if (active) {
    for (int e0 = sub; e0 < n2; e0 += G2 * kBatch) {
      double2 v[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; ++i)
        v[i] = (e0 + G2 * i < n2) ? __ldcg(src + e0 + G2 * i) : make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        ax += v[i].x;
        ay += v[i].y;
      }
    }
  }
  for (int off = 2; off < G2; off <<= 1) {
    ax += __shfl_xor_sync(0xffffffffu, ax, off);
    ay += __shfl_xor_sync(0xffffffffu, ay, off);
  }
  if (active && sub < 2) {
    sv_publish(A, prob, pass, 4 * kb + 2 * sub, ax);
    sv_publish(A, prob, pass, 4 * kb + 2 * sub + 1, ay);
  }
}

// R2 of every column block this CTA owns (kb = cta, cta + gpp, ...; block r/4: the extras),
// spread over the CTA's nw warps, 32 / G2 blocks per warp at a time
__device__ __forceinline__ void r2_cta(const SinkArgs& A, int prob, int pass, const double* part,
                                       int cta, int warp, int nw, int lane) {
  const int G2 = r2_lanes(A.gpp);
  const int bpw = 32 / G2;
  const int nblk = (A.r >> 2) + 1;
  const int mine = (nblk - cta + A.gpp - 1) / A.gpp;   // blocks owned by this CTA
  for (int m0 = warp * bpw; m0 < mine; m0 += nw * bpw) {
    const int m = m0 + lane / G2;
    r2_block(A, prob, pass, part, cta + A.gpp * m, lane % G2, G2, m < mine);
  }
}

// end of solve: fold the problem's breakdown / bad-weight counts into the sticky status word
__device__ __forceinline__ void sticky_flags(const SinkArgs& A, double brk, double wbad) {
  if (!A.sticky) return;
  int bits = 0;
  if (brk > 0.0) bits |= STICKY_BREAKDOWN;
  if (wbad > 0.0) bits |= STICKY_WEIGHTS;
  if (bits) atomicOr(A.sticky, bits);
}

// a Sinkhorn weight (a_i or b_j; mu, nu are probability measures with positive masses,
// PAPER.md:220) that is not finite and > 0
__device__ __forceinline__ bool bad_weight(float c) { return !(c > 0.f) || !isfinite(c); }

// ---- pass boundary inside a thread-block cluster (A.cx: a problem's gpp <= 8 CTAs are one
// cluster; small problems) ---------------------------------------------------
// Each CTA keeps its fp64 partial r-vector (+ extras) in its own shared memory; the owner CTA
// of column block kb (kb % gpp) sums the gpp partials over DSMEM in CTA order (fixed order:
// deterministic) into its tot array; every CTA then reads the totals it needs from the owners.
// Two cluster barriers per pass (partials ready; totals ready) replace the global-memory
// partials, the atomic group barrier and the svec round trips.
//
// cx barrier: consumer thread 0 of every CTA arrives (release, cluster scope) on the mbarrier
// of every CTA of the cluster (expected count gpp), then waits (acquire) on its own; the named
// barriers around it order the CTA's other consumer threads (the stream kernel's producer warp
// never joins: it only talks to its own CTA through the ring).  One mbarrier per CTA is enough:
// a CTA cannot arrive for instance k+1 on a barrier whose owner has not passed instance k
// (instance k+1 needs the owner's own arrival, made after its wait on k).
template <int NTHR>
__device__ __forceinline__ void cx_barrier(uint64_t* cxbar, uint32_t& cxphase, int G, int tid) {
  named_bar(1, NTHR);
  if (tid == 0) {
    const uint32_t a = smem_u32(cxbar);
    for (int c = 0; c < G; ++c) mbar_arrive_remote_cluster(mapa_shared(a, (uint32_t)c));
    while (!mbar_try_wait_cluster(cxbar, cxphase)) {
    }
  }
  cxphase ^= 1u;
  named_bar(1, NTHR);
}

// R2 inside the cluster: this CTA (rank cta) sums column blocks kb = cta, cta + G, ...
// (block r/4: the extras) over the G CTAs' partials; part_addr(kb, q) is the local shared
// address of element q of block kb of a CTA's partials (the same offset in every CTA).
// Thread i of the NTHR handles element (i & 3) of the (i >> 2)-th owned block, and so on.
template <int NTHR, typename PartAddr>
__device__ __forceinline__ void cx_r2(const SinkArgs& A, double* tot, int cta, int tid,
                                      PartAddr part_addr) {
  const int G = A.gpp;
  const int nblk = (A.r >> 2) + 1;
  const int mine = (nblk - cta + G - 1) / G;
  for (int e = tid; e < mine * 4; e += NTHR) {
    const int kb = cta + G * (e >> 2), q = e & 3;
    const uint32_t a = part_addr(kb, q);
    double x = 0.0;
    for (int c = 0; c < G; ++c) x += ld_dsmem_f64(mapa_shared(a, (uint32_t)c));
    tot[kb * 4 + q] = x;
  }
}

// the four totals of column block kb (its owner's tot array)
__device__ __forceinline__ void cx_total4(const double* tot, int G, int kb, double (&o)[4]) {
  const uint32_t a = mapa_shared(smem_u32(tot + kb * 4), (uint32_t)(kb % G));
  const double2 lo = ld_dsmem_v2f64(a), hi = ld_dsmem_v2f64(a + 16);
  o[0] = lo.x; o[1] = lo.y; o[2] = hi.x; o[3] = hi.y;
}

__device__ __forceinline__ float* vbuf_ptr(const SinkArgs& A, int prob, int t) {
  return (((t ^ A.T) & 1) ? A.vbuf1 : A.out[1]) + (int64_t)prob * A.wstride[1];
}

}  // namespace lsk
