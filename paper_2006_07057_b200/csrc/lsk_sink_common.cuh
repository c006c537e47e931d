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

__device__ __forceinline__ float* vbuf_ptr(const SinkArgs& A, int prob, int t) {
  return (((t ^ A.T) & 1) ? A.vbuf1 : A.out[1]) + (int64_t)prob * A.wstride[1];
}

}  // namespace lsk
