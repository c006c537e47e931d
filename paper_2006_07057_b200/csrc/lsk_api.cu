// lsk_api.cu — host side of the C ABI declared in include/lsk.h: validation, fp64 feature
// parameters (Lambert W_0), workspace cache, launch configuration, NCCL (dlopen'ed) and the
// host-buffer end-to-end entry point.  No torch types anywhere.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nccl.h>

#include "lsk_internal.h"

namespace lsk {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;
void count_launch(int k) { g_launches += k; }

static lsk_status fail(lsk_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
#define LSK_CU(call)                                                                      \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(LSK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)
#define LSK_TRY(call)                 \
  do {                                \
    lsk_status st_ = (call);          \
    if (st_ < 0) return st_;          \
  } while (0)

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Tuning knobs (LSK_GPP, LSK_ICFG, ...) exist only in tuning builds (-DLSK_TUNING,
// scripts/build_variant.sh): the product library never reads them, so nothing in the
// environment can change the kernel that runs.
static const char* tuning_env(const char* name) {
#ifdef LSK_TUNING
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// ------------------------------------------------------------------ device properties ---
static int num_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = v > 0 ? v : 1;
  return cache[dev];
}
static int max_smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

// ------------------------------------------------------------------ workspace cache -----
// Two growable buffers per (device, stream): slot 0 for the caller-level carve (anchor
// constants, row factors, scratch), slot 1 for the solve state that run_solve sizes AFTER
// planning (fp64 CTA partials for the planned number of CTAs, r-vectors, barrier counters,
// state blocks, second v buffer) — growing slot 1 never invalidates slot-0 pointers.  Plus
// one never-moving device int: the sticky status word (StickyBits).
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
};
static std::mutex g_ws_mu;
static std::map<std::tuple<int, cudaStream_t, int>, Workspace> g_ws;
static std::map<std::pair<int, cudaStream_t>, int*> g_sticky;

static lsk_status get_sticky(cudaStream_t s, int** out) {
  int dev = 0;
  LSK_CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int*& p = g_sticky[{dev, s}];
  if (!p) {
    if (cudaMalloc(&p, 256) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(LSK_ENOMEM, "status word cudaMalloc failed");
    }
    if (cudaMemset(p, 0, 256) != cudaSuccess) return fail(LSK_ECUDA, "status word memset failed");
  }
  *out = p;
  return LSK_OK;
}

// read and clear the sticky status of stream s (synchronises s); returns the status it encodes
static lsk_status take_sticky(cudaStream_t s) {
  int* dp;
  LSK_TRY(get_sticky(s, &dp));
  int bits = 0;
  LSK_CU(cudaMemcpyAsync(&bits, dp, sizeof(int), cudaMemcpyDeviceToHost, s));
  LSK_CU(cudaStreamSynchronize(s));
  if (bits == 0) return LSK_OK;
  LSK_CU(cudaMemsetAsync(dp, 0, sizeof(int), s));
  if (bits & STICKY_XERR)
    return fail(LSK_ENCCL, "an earlier solve on this stream: cross-GPU peer exchange timed out");
  if (bits & STICKY_WEIGHTS)
    return fail(LSK_EWEIGHTS, "an earlier solve on this stream: a weight a_i or b_j is not finite and > 0");
  return fail(LSK_EBREAKDOWN, "an earlier solve on this stream: zero or non-finite row dot");
}

static lsk_status get_ws(cudaStream_t s, size_t bytes, char** out, int slot = 0) {
  int dev = 0;
  LSK_CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Workspace& w = g_ws[{dev, s, slot}];
  if (w.bytes < bytes) {
    if (w.ptr) {
      cudaStreamSynchronize(s);
      cudaFree(w.ptr);
      w.ptr = nullptr;
      w.bytes = 0;
    }
    const size_t nb = bytes + bytes / 4 + (1u << 20);
    if (cudaMalloc(&w.ptr, nb) != cudaSuccess) {
      cudaGetLastError();
      return fail(LSK_ENOMEM, "workspace cudaMalloc failed");
    }
    w.bytes = nb;
  }
  *out = static_cast<char*>(w.ptr);
  return LSK_OK;
}

struct Carve {
  size_t off = 0;
  size_t take(size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  }
};

// ------------------------------------------------------------------ NCCL (dlopen) -------
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};
static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOLOAD | RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* env = getenv("LSK_NCCL_PATH");
      if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce;
  });
  return api;
}

}  // namespace lsk

struct lsk_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
  // in-kernel NVLink exchange (lsk_comm_enable_p2p): every rank's inbox, own one allocated
  bool p2p = false;
  int xrs = 0;
  double* xbox[lsk::kMaxRanks] = {};
};

namespace lsk {

static lsk_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return LSK_OK;
  const char* s = nccl().errStr ? nccl().errStr(r) : "?";
  return fail(LSK_ENCCL, std::string(what) + ": " + s);
}

// ------------------------------------------------------------------ Lambert W_0 ---------
static lsk_status lambert_w0(double z, double* w) {
  if (!(z >= -1.0 / M_E)) return fail(LSK_EDOMAIN, "lambert_w0: argument < -1/e");
  if (z == 0.0) {
    *w = 0.0;
    return LSK_OK;
  }
  double x = z > 0 ? std::log1p(z) : -0.5;
  for (int it = 0; it < 100; ++it) {
    const double ex = std::exp(x);
    const double f = x * ex - z;
    const double xp1 = x + 1.0;
    const double step = f / (ex * xp1 - (x + 2.0) * f / (2.0 * xp1));
    x -= step;
    if (std::fabs(step) <= 1e-15 * (1.0 + std::fabs(x))) break;
  }
  *w = x;
  return LSK_OK;
}

// ------------------------------------------------------------------ Sinkhorn driver -----
struct SolveCfg {
  bool impl = false;
  int batch = 1;
  int gpp = 1;
  int grid = 1;
  size_t smem = 0;
  int nstage = 2;
  int stage_floats = 0;
  bool coop = false;
};

// Cluster mode (A.cx, DESIGN.md §6 "pass boundary in a cluster"): a problem's gpp CTAs form one
// thread-block cluster and the per-pass r-vector reduction runs over DSMEM — for groups of 2..8
// CTAs (portable cluster sizes) and r <= 1024 (the fp64 partials + totals take 2 x 8 (r+4) B of
// shared memory).  Not with a communicator or emulated ranks (those reduce through svec).
constexpr int kCxMaxGpp = 8;
constexpr int kCxMaxR = 1024;
static bool cx_size_ok(int gpp, int r) { return gpp >= 2 && gpp <= kCxMaxGpp && r <= kCxMaxR; }
// a single small problem that would want up to 2 x kCxMaxGpp CTAs runs as one cluster of
// kCxMaxGpp: each CTA takes up to twice its rows (one more tile per team), the pass boundary
// drops from ~3 us through global memory to ~1 us over DSMEM
static int cx_cap(int64_t want, int r, bool allow_cx) {
  if (!allow_cx || r > kCxMaxR || want < 2 || want > 2 * kCxMaxGpp) return 0;
  return (int)std::min<int64_t>(want, kCxMaxGpp);
}

static lsk_status plan_implicit(SinkArgs& A, int batch, const lsk_solve_opts* o, SolveCfg* c,
                                bool allow_cx) {
  if (A.r > 4096) return fail(LSK_EDIM, "implicit variant supports r <= 4096");
  const ImplCfg ic = implicit_config(A.r, A.d);
  A.tr = ic.tr;
  A.nv = ic.nv;
  const int tr = ic.tr;
  c->impl = true;
  c->batch = batch;
  c->smem = 0;
  c->nstage = 0;
  c->stage_floats = 0;
  int occ = implicit_max_ctas_per_sm(A);
  if (occ < 1) return fail(LSK_EUNSUPPORTED, "implicit kernel does not fit on an SM");
  int cps = (o && o->ctas_per_sm > 0) ? std::min(o->ctas_per_sm, occ) : occ;
  // one tile per team per pass at least: rows / (teams x tr) CTAs
  const int64_t rows = std::max(A.rows[0], A.rows[1]);
  const int64_t rpc = (int64_t)ic.teams * tr;
  const int64_t want = std::max<int64_t>(1, (rows + rpc - 1) / rpc);
  const int slots = num_sms() * cps;
  A.cx = 0;
  if (batch > 1) {
    // one CTA per problem when the batch fills the device; else a cluster of CTAs per problem
    c->gpp = 1;
    const int g = (int)std::min<int64_t>(std::min(kCxMaxGpp, slots / batch), want);
    if (allow_cx && cx_size_ok(g, A.r)) {
      c->gpp = g;
      A.cx = 1;
    }
    c->grid = batch * c->gpp;
    c->coop = false;
  } else {
    c->gpp = (int)std::min<int64_t>((int64_t)slots, want);
    if (const int g = cx_cap(want, A.r, allow_cx)) c->gpp = g;
    if (const char* e = tuning_env("LSK_GPP")) c->gpp = std::max(1, std::min(c->gpp, atoi(e)));   // tuning knob
    c->grid = c->gpp;
    A.cx = (allow_cx && cx_size_ok(c->gpp, A.r)) ? 1 : 0;
    c->coop = c->gpp > 1 && !A.cx;
  }
  return LSK_OK;
}

// Factored exponent of the implicit kernel (lsk_implicit.cu header): used when the row factor
// h_j = 2^(alpha2_j - abar) stays within 2^{+-60}, i.e. (log2e/eps) R^2 <= 60.  LSK_FACT=0
// forces the plain expanded form (tests cover both).
static lsk_status setup_fact(SinkArgs& A, double R, int batch, cudaStream_t s, char* ws,
                             Carve& cv) {
  A.hrow[0] = A.hrow[1] = nullptr;
  A.abar = 0.f;
  const char* e = tuning_env("LSK_FACT");
  if (e && atoi(e) == 0) return LSK_OK;
  const double span = 1.4426950408889634074 / A.eps * R * R;
  if (!(R > 0.0) || !(span <= 60.0)) return LSK_OK;
  A.abar = (float)(-span);   // = c2 R^2 / 2, the middle of alpha2's range [c2 R^2, 0]
  for (int f = 0; f < 2; ++f) {
    float* h = reinterpret_cast<float*>(ws + cv.take(sizeof(float) * A.rows[f] * batch));
    LSK_CU(launch_row_scale(A.X[f], A.rows[f] * batch, A.d, A.c2, A.abar, h, s));
    A.hrow[f] = h;
  }
  return LSK_OK;
}

static lsk_status plan_solve(SinkArgs& A, bool impl, int batch, const lsk_solve_opts* o,
                             SolveCfg* c, bool allow_cx = true) {
  if (impl) return plan_implicit(A, batch, o, c, allow_cx);
  c->impl = impl;
  c->batch = batch;
  const int hdr = 64 + 32 * 16;
  int cps = (o && o->ctas_per_sm > 0) ? o->ctas_per_sm : 1;
  const size_t static_smem = sinkhorn_static_smem();
  const size_t smem_sm = 227 * 1024;   // B200: 228 KB per SM, 227 KB usable per CTA
  int tr = 0, nv = 0, nst = 0, sf = 0;
  const size_t cxb = A.r <= kCxMaxR ? cx_part_bytes(A.r) : 0;   // reserved for cluster mode
  for (;; cps = 1) {
    const size_t per_cta =
        std::min<size_t>(max_smem_optin(), smem_sm / cps - (cps > 1 ? 1024 : 0)) - static_smem - 512 - cxb;
    sinkhorn_tile_config(A.r, (int)(per_cta / 3), &tr, &nv);
    sf = (hdr + tr * A.r + 31) & ~31;
    nst = std::min<int>((int)(per_cta / ((size_t)sf * 4)), 16);
    if (nst >= 3 || cps == 1) break;
  }
  if (nv > 8) return fail(LSK_EDIM, "r too large for this variant");
  // the pipelined tile loop holds two stages while the producer fills a third
  if (nst < 3) return fail(LSK_EDIM, "r too large: three ring stages do not fit in shared memory");
  if (const char* e = tuning_env("LSK_NSTAGE")) nst = std::max(3, std::min(nst, atoi(e)));   // tuning knob
  A.tr = tr;
  A.nv = nv;
  c->stage_floats = sf;
  c->nstage = nst;
  c->smem = (size_t)nst * sf * 4 + cxb;
  int occ = sinkhorn_max_ctas_per_sm(nv, tr, c->smem);
  if (occ < 1) return fail(LSK_EUNSUPPORTED, "sinkhorn kernel does not fit on an SM");
  cps = std::min(cps, occ);
  const int sms = num_sms();
  if (batch > 1) {
    // persistent groups of gpp CTAs, each looping over problems; pick the group size that
    // keeps the most SMs busy over all rounds, charging gpp > 1 its per-pass group exchange
    // against the pass's streaming time at the slot's share of HBM: t_x ~ 6.4 us through
    // global memory (measured round 1, config 4: gpp 1 / 2 / 4 / 8 -> 1282 / 1212 / 1312 /
    // 1106 it/s), ~1 us as a cluster over DSMEM (2 cluster barriers + DSMEM reads), whose
    // groups are limited to the clusters that can be resident at once
    const int slots = sms * cps;
    const int64_t rows = std::max(A.rows[0], A.rows[1]);
    const double slot_bw = 6.4e12 / slots;   // bytes/s per CTA slot when all stream
    int best_g = 1, best_ng = std::min(slots, batch);
    bool best_cx = false;
    double best_eff = -1.0;
    for (int gsz = 1; gsz <= 64 && gsz <= slots; gsz *= 2) {
      if (gsz > 1 && rows / gsz < 2 * tr) break;
      const bool cx = allow_cx && cx_size_ok(gsz, A.r);
      int ngroups = slots / gsz;
      if (cx) ngroups = std::min(ngroups, sinkhorn_max_active_clusters(nv, tr, c->smem, gsz));
      if (ngroups < 1) continue;
      const int rounds = (batch + ngroups - 1) / ngroups;
      const double t_pass = 4.0 * A.r * (double)rows / gsz / slot_bw;
      const double t_x = cx ? 1.0e-6 : 6.4e-6;
      const double eff = (double)batch * gsz / ((double)rounds * ngroups * gsz) *
                         ((double)ngroups * gsz / slots) *
                         (gsz == 1 ? 1.0 : t_pass / (t_pass + t_x));
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        best_g = gsz;
        best_ng = std::min(ngroups, batch);
        best_cx = cx;
      }
    }
    if (const char* e = tuning_env("LSK_BGPP")) {   // tuning knob, clamped to what the grid holds
      best_g = std::max(1, std::min(atoi(e), std::min(64, slots)));
      best_ng = std::min(slots / best_g, batch);
      best_cx = false;
    }
    c->gpp = best_g;
    c->grid = best_ng * best_g;
    A.cx = best_cx ? 1 : 0;
    c->coop = best_g > 1 && !best_cx;
  } else {
    const int64_t rows = std::max(A.rows[0], A.rows[1]);
    const int64_t want = std::max<int64_t>(1, (rows + 2 * tr - 1) / (2 * tr));
    c->gpp = (int)std::min<int64_t>((int64_t)sms * cps, want);
    if (const int g = cx_cap(want, A.r, allow_cx)) c->gpp = g;
    if (const char* e = tuning_env("LSK_GPP")) c->gpp = std::max(1, std::min(c->gpp, atoi(e)));   // tuning knob
    c->grid = c->gpp;
    A.cx = (allow_cx && cx_size_ok(c->gpp, A.r)) ? 1 : 0;
    c->coop = c->gpp > 1 && !A.cx;
  }
  return LSK_OK;
}

constexpr int kPreDefault = 2;
constexpr int kPingPongDefault = 1;

static lsk_status collect_reports(const SinkArgs& A, int batch, lsk_report* reps, bool nccl_rot,
                                  cudaStream_t s);

// Small single-GPU problems whose factors fit in the shared memory of one cluster (<= 8 CTAs):
// the resident kernel (lsk_resident.cu, DESIGN.md §6 K10) instead of the persistent grid kernels
static bool resident_allowed(const lsk_solve_opts* o) {
  if (o && (o->flags & LSK_SOLVE_NO_RESIDENT)) return false;
  const char* e = tuning_env("LSK_RESG");   // tuning knob: 0 = off
  return !(e && atoi(e) == 0);
}

static int resident_pick(const SinkArgs& A, int batch, const lsk_comm* comm,
                         const lsk_solve_opts* o) {
  if (!resident_allowed(o) || batch < 1 || comm || A.emul || !A.F[0] || !A.F[1] || A.stab ||
      A.nstream[0] + A.nstream[1] > 0)
    return 0;
  int G = resident_cluster(A.r, A.rows[0], A.rows[1]);
  if (const char* e = tuning_env("LSK_RESG")) {   // tuning knob: 0 = off, else the cluster size
    const int g = atoi(e);
    if (g == 0) return 0;
    if (G > 0 && (g == 1 || g == 2 || g == 4 || g == 8) &&
        resident_smem_bytes(A.r, A.rows[0], A.rows[1], g) <= 227 * 1024)
      G = g;
  }
  return G;
}

static lsk_status run_solve(SinkArgs A, bool impl, int batch, const lsk_solve_opts* o,
                            lsk_report* reps, lsk_comm* comm, cudaStream_t s) {
  if (!o) return fail(LSK_EINVAL, "opts is NULL");
  if (o->max_iters < 1) return fail(LSK_EINVAL, "max_iters < 1");
  A.T = o->max_iters;
  A.tol_mode = o->tol > 0.0 ? 1 : 0;
  A.tol = o->tol;
  A.want_err = (A.tol_mode || o->want_marginal_err) ? 1 : 0;
  A.num_passes = 2 * A.T + 1 + A.want_err;
  if (const int G = resident_pick(A, batch, comm, o)) {   // one cluster per problem
    Carve sz;
    const size_t oState = sz.take(sizeof(double) * kStateDoubles * batch);
    char* ws;
    LSK_TRY(get_ws(s, sz.off, &ws, 1));
    LSK_TRY(get_sticky(s, &A.sticky));
    A.state = reinterpret_cast<double*>(ws + oState);
    LSK_CU(cudaMemsetAsync(A.state, 0, sizeof(double) * kStateDoubles * batch, s));
    A.nranks = 1;
    A.rank = 0;
    A.nprob = batch;
    A.gpp = G;
    A.pass_begin = 0;
    A.pass_end = A.num_passes;
    LSK_CU(launch_resident(A, G, batch, s));
    return collect_reports(A, batch, reps, false, s);
  }
  SolveCfg c;
  LSK_TRY(plan_solve(A, impl, batch, o, &c, !comm && !A.emul));
  // implicit team kernel: the next pass's first feature tile is generated between the group
  // barrier's arrive and wait (DESIGN.md §6 K5, boundary overlap; measured on the grid path
  // only: the cluster boundary has no wait to hide it in)
  A.pre = A.cx ? 0 : kPreDefault;
  if (const char* e = tuning_env("LSK_PRE")) A.pre = std::max(0, std::min(2, atoi(e)));
  A.pingpong = kPingPongDefault;   // implicit two-team kernel: alternating generations (§6 K5)
  if (const char* e = tuning_env("LSK_PP")) A.pingpong = atoi(e) != 0;
  if (impl && A.d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  const bool p2p = !A.emul && comm && comm->p2p && batch == 1 && A.r + kExtra + 2 <= comm->xrs &&
                   !(getenv("LSK_P2P") && atoi(getenv("LSK_P2P")) == 0);
  if (comm && c.gpp < 2) {
    // the cross-GPU paths reduce through svec: force >= 2 CTAs
    c.gpp = std::min(2, num_sms());
    c.grid = c.gpp;
    c.coop = true;
  }
  if (A.emul) {
    // emulated ranks (lsk_*_emulated): the batch is the nranks row shards of ONE problem, each
    // a group of gpp >= 2 CTAs, all co-resident in one cooperative launch (ranks wait on each
    // other); xbox / nranks / xrs were set by the caller
    if (A.r + kExtra + 2 > A.xrs) return fail(LSK_EINVAL, "emulated inboxes too small for r");
    const int slots = num_sms() * std::max(1, impl ? implicit_max_ctas_per_sm(A)
                                                   : sinkhorn_max_ctas_per_sm(A.nv, A.tr, c.smem));
    const int64_t rows = std::max(A.rows[0], A.rows[1]);
    const int want = (int)std::max<int64_t>(2, (rows + 2 * A.tr - 1) / (2 * A.tr));
    c.gpp = std::max(2, std::min(want, slots / batch));
    if (c.gpp * batch > slots) return fail(LSK_EUNSUPPORTED, "emulated ranks do not fit on the device");
    c.grid = c.gpp * batch;
    c.coop = true;
  } else {
    A.nranks = 1;
    A.rank = 0;
  }
  if (p2p && !A.emul) {   // one persistent launch per GPU; the exchange runs over NVLink inside it
    A.nranks = comm->nranks;
    A.rank = comm->rank;
    A.xrs = comm->xrs;
    for (int i = 0; i < comm->nranks; ++i) A.xbox[i] = comm->xbox[i];
    A.xtimeout_ns = 20LL * 1000 * 1000 * 1000;
  }
  A.gpp = c.gpp;
  A.dbg = tuning_env("LSK_DEBUG") ? atoi(tuning_env("LSK_DEBUG")) : 0;
  A.l2_resident = tuning_env("LSK_L2RES") ? (float)atof(tuning_env("LSK_L2RES")) : 0.f;   // tuning knob
  A.nprob = batch;
  A.nstage = c.nstage;
  A.stage_floats = c.stage_floats;
  const int64_t rs = A.r + kExtra;
  // the solve state, sized for the planned CTA count (workspace slot 1):
  // part: [batch][(r + kExtra + 4) / 4 blocks][gpp][4] (block r/4 + 1 carries the read-out
  // partials; lsk_sink_common.cuh);
  // svec: [batch][2][r + kExtra], armed with the all-ones sentinel (lsk_sink_common.cuh)
  Carve sz;
  const size_t oPart = sz.take(sizeof(double) * (rs + 4) * c.gpp * batch);
  const size_t oSvec = sz.take(sizeof(double) * 2 * rs * batch);
  const size_t oState = sz.take(sizeof(double) * kStateDoubles * batch);
  const size_t oBar = sz.take(sizeof(unsigned int) * batch);
  const size_t oVbuf = sz.take(sizeof(float) * A.rows[1] * batch);
  char* ws;
  LSK_TRY(get_ws(s, sz.off, &ws, 1));
  LSK_TRY(get_sticky(s, &A.sticky));
  A.part = reinterpret_cast<double*>(ws + oPart);
  A.svec = reinterpret_cast<double*>(ws + oSvec);
  LSK_CU(cudaMemsetAsync(A.svec, 0xFF, sizeof(double) * 2 * rs * batch, s));
  A.state = reinterpret_cast<double*>(ws + oState);
  A.bar = reinterpret_cast<unsigned int*>(ws + oBar);
  A.vbuf1 = reinterpret_cast<float*>(ws + oVbuf);
  LSK_CU(cudaMemsetAsync(A.state, 0, sizeof(double) * kStateDoubles * batch, s));
  unsigned long long* trace = nullptr;
  const char* trace_path = tuning_env("LSK_TRACE");   // tuning only: per-pass barrier timestamps
  if (trace_path && batch == 1) {
    cudaMalloc(&trace, sizeof(unsigned long long) * 4 * (size_t)A.num_passes * c.gpp);
    cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 4 * (size_t)A.num_passes * c.gpp, s);
  }
  A.trace = trace;
  if (!comm || p2p) {
    A.pass_begin = 0;
    A.pass_end = A.num_passes;
    A.multi_launch = 0;
    LSK_CU(cudaMemsetAsync(A.bar, 0, sizeof(unsigned int) * batch, s));
    LSK_CU(impl ? launch_implicit(A, c.coop, c.grid, s) : launch_sinkhorn(A, c.coop, c.grid, c.smem, s));
  } else {
    if (!nccl().ok) return fail(LSK_ENCCL, "NCCL not loadable");
    A.multi_launch = 1;
    for (int p = 0; p <= A.num_passes; ++p) {
      A.pass_begin = p;
      A.pass_end = std::min(p + 1, A.num_passes);
      if (p == A.num_passes) A.pass_end = p;   // finalise-only launch
      LSK_CU(cudaMemsetAsync(A.bar, 0, sizeof(unsigned int) * batch, s));
      LSK_CU(impl ? launch_implicit(A, c.coop, c.grid, s) : launch_sinkhorn(A, c.coop, c.grid, c.smem, s));
      if (p < A.num_passes)
        LSK_TRY(nccl_check(nccl().allReduce(A.svec, A.svec, (size_t)rs * batch, ncclFloat64,
                                            ncclSum, comm->comm, s),
                           "ncclAllReduce"));
    }
    // read-out partials a^T log u, b^T log v of the local rows -> global sums
    LSK_TRY(nccl_check(nccl().allReduce(A.state + ST_FINAL_A, A.state + ST_FINAL_A, 2,
                                        ncclFloat64, ncclSum, comm->comm, s),
                       "ncclAllReduce(read-out)"));
  }
  if (trace) {
    std::vector<unsigned long long> h(4 * (size_t)A.num_passes * c.gpp);
    cudaMemcpyAsync(h.data(), trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (FILE* fp = fopen(trace_path, "wb")) {
      int hdr[2] = {A.num_passes, c.gpp};
      fwrite(hdr, sizeof(int), 2, fp);
      fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      fclose(fp);
    }
    cudaFree(trace);
  }
  return collect_reports(A, batch, reps, comm && !p2p, s);
}

// reports of a finished solve (state blocks -> lsk_report), sticky status and weight /
// breakdown / convergence statuses; nccl_rot: the read-out partials were all-reduced by NCCL
static lsk_status collect_reports(const SinkArgs& A, int batch, lsk_report* reps, bool nccl_rot,
                                  cudaStream_t s) {
  if (reps) {
    std::vector<double> st((size_t)kStateDoubles * batch);
    LSK_CU(cudaMemcpyAsync(st.data(), A.state, sizeof(double) * st.size(), cudaMemcpyDeviceToHost, s));
    LSK_CU(cudaStreamSynchronize(s));
    bool brk = false, notconv = false, wbad = false;
    for (int b = 0; b < batch; ++b) {
      const double* x = st.data() + (size_t)b * kStateDoubles;
      lsk_report& rp = reps[b];
      rp.iters = (int32_t)x[ST_ITERS];
      rp.converged = (int32_t)x[ST_CONV];
      rp.marginal_err = x[ST_ERR];
      rp.rot = nccl_rot ? A.eps * (x[ST_FINAL_A] + x[ST_FINAL_B]) : x[ST_ROT];
      rp.sum_a_log_u = x[ST_FINAL_A];
      rp.sum_b_log_v = x[ST_FINAL_B];
      rp.breakdown = x[ST_BRK] > 0 ? 1 : 0;
      rp.reserved = 0;
      brk |= rp.breakdown != 0;
      wbad |= x[ST_WBAD] > 0;
      notconv |= A.tol_mode && !rp.converged;
    }
    // reported here: clear the sticky word (it also carries any earlier report-less solve)
    const lsk_status sticky = take_sticky(s);
    if (sticky == LSK_ECUDA || sticky == LSK_ENOMEM) return sticky;
    for (int b = 0; b < batch; ++b)
      if (st[(size_t)b * kStateDoubles + ST_XERR] != 0.0)
        return fail(LSK_ENCCL, "cross-GPU peer exchange timed out (a rank did not arrive)");
    if (wbad) return fail(LSK_EWEIGHTS, "a weight a_i or b_j is not finite and > 0 (PAPER.md:220)");
    if (brk) return fail(LSK_EBREAKDOWN, "zero or non-finite row dot during Sinkhorn");
    if (sticky < 0) return sticky;
    if (notconv) {
      g_err = "tolerance not reached within max_iters";
      return LSK_NOT_CONVERGED;
    }
  }
  return LSK_OK;
}

// Warp-specialised hybrid (lsk_hybrid.cu): off by default.  Its sweep (us per pass on config 2,
// phi = off / 0.1 / 0.15 / 0.2 / 0.25 / 0.3: 20.44 / 20.84 / 20.49 / 19.35 / 19.13 / 21.84,
// profiles/r02e_hybrid_sweep.log) did not hold under the bench protocol (an L2 flush before every
// timed solve, interleaved arms, T = 200 and 500): phi = 0.25 runs at 20.33-20.35 us per pass
// against 20.45 for the pure recompute kernel (scripts/ab_tc.py, profiles/r02_tmem_ex2_microbench.txt)
// — within 1%, so the simpler kernel stays the default and phi > 0 is the caller's choice.
constexpr double kHybridDefault = 0.0;

// slot-0 bytes a solve carves besides the caller's own (the implicit row factors h_j of the
// factored exponent); the solve state lives in slot 1, sized by run_solve after planning
static size_t solve_ws_bytes(int64_t n, int64_t m, int batch) {
  return 256 * 8 + (sizeof(float) * (n + m) + 2 * 256) * batch;
}

static lsk_status check_common(int64_t n, int64_t m, int r, double eps) {
  if (n < 1 || m < 1) return fail(LSK_EINVAL, "n and m must be >= 1");
  if (r < 1 || (r % 4) != 0) return fail(LSK_EINVAL, "r must be >= 1 and a multiple of 4");
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(LSK_EINVAL, "eps must be > 0");
  if (n > (int64_t)1 << 40 || m > (int64_t)1 << 40) return fail(LSK_EINVAL, "n or m too large");
  return LSK_OK;
}

}  // namespace lsk

using namespace lsk;

// ========================================================================================
extern "C" {

const char* lsk_version(void) { return "lsk 0.1.0 (sm_100a)"; }
const char* lsk_last_error(void) { return g_err.c_str(); }
int64_t lsk_launch_count(int32_t reset) {
  const int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

lsk_status lsk_solve_plan(int64_t n, int64_t m, int32_t r, int32_t d, int32_t batch,
                          int32_t variant, int32_t* gpp, int32_t* grid, int32_t* cluster) {
  LSK_TRY(check_common(n, m, r, 1.0));
  if (!gpp || !grid || batch < 1 || d < 1 || (variant != 1 && variant != 2))
    return fail(LSK_EINVAL, "bad plan arguments");
  if (variant == 2 && d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  SinkArgs A{};
  A.rows[0] = n; A.rows[1] = m;
  A.r = r; A.d = variant == 2 ? d : 1;
  static const float dummy = 0.f;   // the factored-exponent instantiation (occupancy only)
  if (variant == 2) A.hrow[0] = A.hrow[1] = &dummy;
  SolveCfg c;
  LSK_TRY(plan_solve(A, variant == 2, batch, nullptr, &c));
  *gpp = c.gpp;
  *grid = c.grid;
  if (cluster) *cluster = A.cx;
  return LSK_OK;
}

lsk_status lsk_resident_plan(int64_t n, int64_t m, int32_t r, int32_t* ctas) {
  if (!ctas) return fail(LSK_EINVAL, "NULL argument");
  LSK_TRY(check_common(n, m, r, 1.0));
  *ctas = resident_cluster(r, n, m);
  return LSK_OK;
}

static void hybrid_rows(const lsk_solve_opts* o, int r, int d, int64_t n, int64_t m,
                        int64_t* ns0, int64_t* ns1);

lsk_status lsk_stream_rows(int64_t n, int64_t m, int32_t r, int32_t d, const lsk_solve_opts* o,
                           int64_t* ns0, int64_t* ns1) {
  if (!ns0 || !ns1) return fail(LSK_EINVAL, "NULL argument");
  LSK_TRY(check_common(n, m, r, 1.0));
  const bool stab = o && (o->flags & LSK_SOLVE_STABILIZE);
  *ns0 = *ns1 = 0;
  if (!stab) hybrid_rows(o, r, d, n, m, ns0, ns1);
  return LSK_OK;
}

lsk_status lsk_stream_status(void* stream) {
  return take_sticky(static_cast<cudaStream_t>(stream));
}

lsk_status lsk_lambert_w0(double z, double* w) {
  if (!w) return fail(LSK_EINVAL, "w is NULL");
  return lambert_w0(z, w);
}

lsk_status lsk_shard_range(int64_t total, int32_t nranks, int32_t rank, int64_t* begin,
                           int64_t* end) {
  if (!begin || !end || nranks < 1 || rank < 0 || rank >= nranks || total < 0)
    return fail(LSK_EINVAL, "bad shard arguments");
  *begin = total * rank / nranks;
  *end = total * (rank + 1) / nranks;
  return LSK_OK;
}

lsk_status lsk_feature_params_init(double eps, int32_t d, int32_t r, double R, uint64_t seed,
                                   const float* X, int64_t n, const float* Y, int64_t m,
                                   lsk_feature_params* out, lsk_comm* comm, void* stream) {
  if (!out) return fail(LSK_EINVAL, "out is NULL");
  if (d < 1 || r < 1) return fail(LSK_EINVAL, "d and r must be >= 1");
  if (!(eps > 0.0)) return fail(LSK_EINVAL, "eps must be > 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool have_pts = (X && n > 0) || (Y && m > 0);
  double maxnorm = -1.0;
  if (have_pts) {
    char* ws;
    LSK_TRY(get_ws(s, 4096, &ws));
    unsigned long long* dmax = reinterpret_cast<unsigned long long*>(ws);
    LSK_CU(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), s));
    if (X && n > 0) LSK_CU(launch_max_sqnorm(X, n, d, dmax, s));
    if (Y && m > 0) LSK_CU(launch_max_sqnorm(Y, m, d, dmax, s));
    if (comm) {
      if (!nccl().ok) return fail(LSK_ENCCL, "NCCL not loadable");
      LSK_TRY(nccl_check(nccl().allReduce(dmax, dmax, 1, ncclUint64, ncclMax, comm->comm, s),
                         "ncclAllReduce(max)"));
    }
    unsigned long long hbits = 0;
    LSK_CU(cudaMemcpyAsync(&hbits, dmax, sizeof(hbits), cudaMemcpyDeviceToHost, s));
    LSK_CU(cudaStreamSynchronize(s));
    double sq;
    std::memcpy(&sq, &hbits, sizeof(sq));
    maxnorm = std::sqrt(sq);
  }
  if (R <= 0.0) {
    if (!have_pts) return fail(LSK_EINVAL, "R <= 0 requires X or Y to compute R");
    R = maxnorm;
    if (!(R > 0.0)) R = 1e-30;   // all points at the origin: any R works (C11)
  } else if (have_pts && maxnorm > R * (1.0 + 1e-12)) {
    return fail(LSK_EDOMAIN, "a point lies outside B(0,R)");
  }
  const double z = R * R / (eps * d);
  double W;
  LSK_TRY(lambert_w0(z, &W));
  const double q = (W > 0.0) ? z / (2.0 * W) : 0.5;   // z -> 0: q -> 1/2
  out->eps = eps;
  out->R = R;
  out->q = q;
  out->sigma = std::sqrt(q * eps / 4.0);
  out->log_scale = 0.25 * d * std::log(2.0 * q) - 0.5 * std::log((double)r);
  out->d = d;
  out->r = r;
  out->seed = seed;
  return LSK_OK;
}

lsk_status lsk_draw_anchors(const lsk_feature_params* p, float* U, void* stream) {
  if (!p || !U) return fail(LSK_EINVAL, "NULL argument");
  if (p->r < 1 || p->d < 1) return fail(LSK_EINVAL, "bad params");
  LSK_CU(launch_anchors(p->seed, p->r, p->d, p->sigma, U, nullptr, static_cast<cudaStream_t>(stream)));
  return LSK_OK;
}

lsk_status lsk_philox_words(uint64_t seed, int32_t r, int32_t d, uint32_t* out, void* stream) {
  if (!out || r < 1 || d < 1) return fail(LSK_EINVAL, "bad arguments");
  LSK_CU(launch_anchors(seed, r, d, 0.0, nullptr, out, static_cast<cudaStream_t>(stream)));
  return LSK_OK;
}

static lsk_status feature_map_impl(const lsk_feature_params* p, const float* U, const float* X,
                                   int64_t rows, float* Xi, cudaStream_t s) {
  if (!p || !U || !X || !Xi) return fail(LSK_EINVAL, "NULL argument");
  if (p->r < 4 || p->r % 4) return fail(LSK_EINVAL, "r must be a multiple of 4");
  if (rows < 1) return fail(LSK_EINVAL, "n must be >= 1");
  if (!aligned16(Xi)) return fail(LSK_EINVAL, "Xi must be 16-byte aligned");
  char* ws;
  Carve cv;
  const bool tensor = p->d > 16 && !tuning_env("LSK_FEATURE_FFMA");   // knob: FFMA A/B only
  const size_t oW = cv.take(sizeof(float) * p->d * p->r);
  const size_t oB = cv.take(sizeof(float) * p->r);
  const size_t oD = cv.take(sizeof(float) * p->r);
  const size_t oI = tensor ? cv.take(feature_map_tc_image_bytes(p->r, p->d)) : 0;
  LSK_TRY(get_ws(s, cv.off, &ws));
  float* Wt = reinterpret_cast<float*>(ws + oW);
  float* b2 = reinterpret_cast<float*>(ws + oB);
  float* bD = reinterpret_cast<float*>(ws + oD);
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, tensor ? nullptr : Wt, b2,
                            bD, s));
  if (tensor) {
    LSK_CU(launch_feature_map_tc(X, rows, p->d, U, b2, p->r, p->eps,
                                 reinterpret_cast<float*>(ws + oI), Xi, s, 0, 0, 0, p->R));
  } else {
    LSK_CU(launch_feature_map(X, rows, p->d, U, Wt, b2, bD, p->r, p->eps, Xi, s));
  }
  return LSK_OK;
}

lsk_status lsk_feature_map(const lsk_feature_params* p, const float* U, const float* X,
                           int64_t n, float* Xi, void* stream) {
  return feature_map_impl(p, U, X, n, Xi, static_cast<cudaStream_t>(stream));
}

lsk_status lsk_feature_map_stabilized(const lsk_feature_params* p, const float* U,
                                      const float* X, int64_t n, float* Xi, double* logoff,
                                      void* stream) {
  if (!p || !U || !X || !Xi || !logoff) return fail(LSK_EINVAL, "NULL argument");
  if (p->r < 4 || p->r % 4) return fail(LSK_EINVAL, "r must be a multiple of 4");
  if (n < 1) return fail(LSK_EINVAL, "n must be >= 1");
  if (p->d > 16) return fail(LSK_EDIM, "the stabilised feature map supports d <= 16");
  if (!aligned16(Xi)) return fail(LSK_EINVAL, "Xi must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  Carve cv;
  const size_t oD = cv.take(sizeof(float) * p->r);
  LSK_TRY(get_ws(s, cv.off, &ws));
  float* bD = reinterpret_cast<float*>(ws + oD);
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, nullptr, nullptr, bD, s));
  LSK_CU(launch_feature_map_stab(X, n, p->d, U, bD, p->r, p->eps, Xi, logoff, s));
  return LSK_OK;
}

lsk_status lsk_rot_value_offset(const float* u, const float* v, const float* a, const float* b,
                                const double* A, const double* B, int64_t n, int64_t m,
                                double eps, double* rot_host, void* stream) {
  if (!u || !v || !a || !b || !A || !B || !rot_host) return fail(LSK_EINVAL, "NULL argument");
  if (n < 1 || m < 1 || !(eps > 0)) return fail(LSK_EINVAL, "bad sizes or eps");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  LSK_TRY(get_ws(s, 8192 + 2 * 64 * sizeof(double), &ws));
  double* part = reinterpret_cast<double*>(ws + 256);
  double* out2 = reinterpret_cast<double*>(ws);
  LSK_CU(launch_rot_value(u, v, a, b, n, m, 1, part, out2, s, A, B));
  double h[2];
  LSK_CU(cudaMemcpyAsync(h, out2, sizeof(h), cudaMemcpyDeviceToHost, s));
  LSK_CU(cudaStreamSynchronize(s));
  *rot_host = eps * (h[0] + h[1]);
  return LSK_OK;
}

lsk_status lsk_feature_map_arccos(const lsk_feature_params* p, int32_t s_degree, double kappa,
                                  const float* U, const float* X, int64_t n, float* Xi,
                                  void* stream) {
  if (!p || !U || !X || !Xi) return fail(LSK_EINVAL, "NULL argument");
  if (p->r < 4 || p->r % 4) return fail(LSK_EINVAL, "r must be a multiple of 4");
  if (n < 1 || p->d < 1) return fail(LSK_EINVAL, "n and d must be >= 1");
  if (s_degree < 0 || s_degree > 2) return fail(LSK_EINVAL, "s must be 0, 1 or 2");
  if (!(kappa > 0.0)) return fail(LSK_EINVAL, "kappa must be > 0");
  if (!(p->sigma > 1.0)) return fail(LSK_EDOMAIN, "the arc-cosine map needs sigma > 1");
  if (!aligned16(Xi)) return fail(LSK_EINVAL, "Xi must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool tensor = p->d > 16;
  char* ws;
  Carve cv;
  const size_t oC = cv.take(sizeof(float) * p->r);
  const size_t oI = tensor ? cv.take(feature_map_tc_image_bytes(p->r, p->d)) : 0;
  LSK_TRY(get_ws(s, cv.off, &ws));
  float* coef = reinterpret_cast<float*>(ws + oC);
  LSK_CU(launch_arccos_coef(U, p->r, p->d, p->sigma, coef, s));
  if (tensor) {
    LSK_CU(launch_feature_map_tc(X, n, p->d, U, coef, p->r, 1.0, reinterpret_cast<float*>(ws + oI),
                                 Xi, s, 1, s_degree, p->r + 4));
    LSK_CU(launch_const_cols(Xi, n, p->r + 4, p->r, (float)std::sqrt(kappa), s));
  } else {
    LSK_CU(launch_feature_map_arccos(X, n, p->d, U, coef, p->r, s_degree, kappa, Xi, s));
  }
  return LSK_OK;
}

lsk_status lsk_feature_map_batched(const lsk_feature_params* p, const float* U, const float* X,
                                   int64_t n, int32_t batch, float* Xi, void* stream) {
  if (batch < 1) return fail(LSK_EINVAL, "batch must be >= 1");
  // one shared anchor draw: the batch is a (batch*n) x d point matrix
  return feature_map_impl(p, U, X, n * batch, Xi, static_cast<cudaStream_t>(stream));
}

lsk_status lsk_factored_sinkhorn(const float* Xi, int64_t n, const float* Zeta, int64_t m,
                                 int32_t r, const float* a, const float* b, double eps,
                                 const lsk_solve_opts* o, float* u, float* v, lsk_report* rep,
                                 lsk_comm* comm, void* stream) {
  LSK_TRY(check_common(n, m, r, eps));
  if (!Xi || !Zeta || !a || !b || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  if (!aligned16(Xi) || !aligned16(Zeta)) return fail(LSK_EINVAL, "factors must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SinkArgs A{};
  A.F[0] = Xi; A.F[1] = Zeta;
  A.rows[0] = n; A.rows[1] = m;
  A.w[0] = a; A.w[1] = b;
  A.out[0] = u; A.out[1] = v;
  A.r = r; A.d = 1; A.eps = eps;
  return run_solve(A, false, 1, o, rep, comm, s);
}

// Fraction of each side's rows the hybrid kernel streams (materialised) instead of regenerating
// (lsk_solve_opts.stream_fraction: 0 = default, < 0 = off), for the shapes the hybrid kernel
// covers (r <= 1024, d <= 3; a single problem spread over every SM), bounded by a memory budget.
static void hybrid_rows(const lsk_solve_opts* o, int r, int d, int64_t n, int64_t m,
                        int64_t* ns0, int64_t* ns1) {
  *ns0 = *ns1 = 0;
  if (r > 1024 || d > 3) return;
  double phi = (o && o->stream_fraction != 0.0) ? o->stream_fraction : kHybridDefault;
  if (const char* e = tuning_env("LSK_HYB")) phi = atof(e);
  if (!(phi > 0.0)) return;   // off
  phi = std::min(phi, 0.9);
  *ns0 = (int64_t)(phi * (double)n);
  *ns1 = (int64_t)(phi * (double)m);
  // rows per CTA must leave the recompute teams whole tiles to work on
  if (std::min(n - *ns0, m - *ns1) < 16 * (int64_t)num_sms()) {
    *ns0 = *ns1 = 0;
    return;
  }
  // at most a quarter of the device memory (queried once: cudaMemGetInfo costs host ms)
  static size_t total = 0;
  if (total == 0) {
    size_t fr = 0;
    if (cudaMemGetInfo(&fr, &total) != cudaSuccess) total = 1;
  }
  const double bytes = (double)(*ns0 + *ns1) * r * 4.0;
  if (bytes > 0.25 * (double)total) *ns0 = *ns1 = 0;
}

lsk_status lsk_factored_sinkhorn_implicit(const lsk_feature_params* p, const float* U,
                                          const float* X, int64_t n, const float* Y, int64_t m,
                                          const float* a, const float* b,
                                          const lsk_solve_opts* o, float* u, float* v,
                                          lsk_report* rep, lsk_comm* comm, void* stream) {
  if (!p) return fail(LSK_EINVAL, "params NULL");
  LSK_TRY(check_common(n, m, p->r, p->eps));
  if (!U || !X || !Y || !a || !b || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  if (p->d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool stab = (o && (o->flags & LSK_SOLVE_STABILIZE));
  if (stab && comm) return fail(LSK_EUNSUPPORTED, "the stabilised implicit solve is single-GPU");
  char* ws;
  Carve cv;
  const size_t oW = cv.take(sizeof(float) * p->d * p->r);
  const size_t oB = cv.take(sizeof(float) * p->r);
  const size_t oM = stab ? cv.take(sizeof(float) * (n + m)) : 0;    // row shifts m_j
  const size_t oA = stab ? cv.take(sizeof(double) * (n + m)) : 0;   // row offsets A_j
  const size_t oR = stab ? cv.take(16384) : 0;                      // read-out scratch
  // tensor-core exponent kernel (lsk_implicit_tc.cu, DESIGN.md §6 K9): measured slower than
  // the FFMA-exponent kernel, so only tuning builds select it (LSK_ITC=1; r <= 1024, d <= 2,
  // factored exponent, not on the NCCL multi-launch path, no streamed fraction)
#ifdef LSK_TUNING
  const char* itc_env = tuning_env("LSK_ITC");
  const bool tc_ok = itc_env && atoi(itc_env) == 1 && !stab && p->d <= 2 && p->r <= 1024 &&
                     (!comm || comm->p2p) && !(o && o->stream_fraction > 0.0);
#else
  const bool tc_ok = false;
#endif
  // hybrid: the first phi n (phi m) rows are materialised and streamed by extra warps of the
  // same persistent launch, the rest regenerated (HBM and MUFU busy at once)
  const bool hyb_ok = !stab && !tc_ok && (!comm || comm->p2p);   // not on the NCCL multi-launch path
  int64_t ns0 = 0, ns1 = 0;
  if (hyb_ok) hybrid_rows(o, p->r, p->d, n, m, &ns0, &ns1);
  const bool hyb = ns0 + ns1 > 0;
  // small problems: the factors are materialised once (FFMA feature map) and the solve runs in
  // the resident cluster kernel (run_solve -> resident_pick), which regenerates nothing
  const bool res = !stab && !hyb && !tc_ok && !comm && resident_allowed(o) &&
                   resident_cluster(p->r, n, m) > 0;
  const size_t oD = (hyb || res) ? cv.take(sizeof(float) * p->r) : 0;
  const size_t oF = hyb ? cv.take(sizeof(float) * (ns0 + ns1) * p->r)
                        : (res ? cv.take(sizeof(float) * (n + m) * p->r) : 0);
#ifdef LSK_TUNING
  const size_t oI = tc_ok ? cv.take(sizeof(float) * itc_image_floats(n + m)) : 0;
#endif
  LSK_TRY(get_ws(s, cv.off + solve_ws_bytes(n, m, 1), &ws));
  float* Wt = reinterpret_cast<float*>(ws + oW);
  float* b2 = reinterpret_cast<float*>(ws + oB);
  float* bD = (hyb || res) ? reinterpret_cast<float*>(ws + oD) : nullptr;
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, Wt, b2, bD, s));
  SinkArgs A{};
  A.X[0] = X; A.X[1] = Y;
  A.rows[0] = n; A.rows[1] = m;
  A.w[0] = a; A.w[1] = b;
  A.out[0] = u; A.out[1] = v;
  A.r = p->r; A.d = p->d; A.eps = p->eps;
  A.Wt = Wt; A.beta2 = b2;
  A.c2 = (float)(-2.0 * 1.4426950408889634074 / p->eps);
  double* offs = nullptr;
  if (stab) {   // reading C30: per-row shifts inside the kernel, offsets folded into the read-out
    float* m2 = reinterpret_cast<float*>(ws + oM);
    offs = reinterpret_cast<double*>(ws + oA);
    LSK_CU(launch_row_shift(X, n, p->d, Wt, b2, p->r, A.c2, m2, offs, s));
    LSK_CU(launch_row_shift(Y, m, p->d, Wt, b2, p->r, A.c2, m2 + n, offs + n, s));
    A.hrow[0] = m2;
    A.hrow[1] = m2 + n;
    A.stab = 1;
  } else {
    LSK_TRY(setup_fact(A, p->R, 1, s, ws, cv));
  }
#ifdef LSK_TUNING
  if (tc_ok && A.hrow[0] != nullptr) {   // the B images of both sides (packed 3xTF32 rows)
    float* img = reinterpret_cast<float*>(ws + oI);
    LSK_CU(launch_itc_image(X, n, p->d, img, s));
    LSK_CU(launch_itc_image(Y, m, p->d, img + itc_image_floats(n), s));
    A.bimg[0] = img;
    A.bimg[1] = img + itc_image_floats(n);
  }
#endif
  if (hyb) {
    float* F0 = reinterpret_cast<float*>(ws + oF);
    float* F1 = F0 + ns0 * p->r;
    if (ns0 > 0) LSK_CU(launch_feature_map(X, ns0, p->d, U, Wt, b2, bD, p->r, p->eps, F0, s));
    if (ns1 > 0) LSK_CU(launch_feature_map(Y, ns1, p->d, U, Wt, b2, bD, p->r, p->eps, F1, s));
    A.F[0] = F0;
    A.F[1] = F1;
    A.nstream[0] = ns0;
    A.nstream[1] = ns1;
  }
  if (res) {
    float* F0 = reinterpret_cast<float*>(ws + oF);
    float* F1 = F0 + n * p->r;
    LSK_CU(launch_feature_map(X, n, p->d, U, Wt, b2, bD, p->r, p->eps, F0, s));
    LSK_CU(launch_feature_map(Y, m, p->d, U, Wt, b2, bD, p->r, p->eps, F1, s));
    A.F[0] = F0;
    A.F[1] = F1;
  }
  lsk_status st = run_solve(A, true, 1, o, rep, comm, s);
  if (stab && rep && st >= 0) {
    double* scratch = reinterpret_cast<double*>(ws + oR);
    LSK_CU(launch_rot_value(u, v, a, b, n, m, 1, scratch + 32, scratch, s, offs, offs + n));
    double h[2];
    LSK_CU(cudaMemcpyAsync(h, scratch, sizeof(h), cudaMemcpyDeviceToHost, s));
    LSK_CU(cudaStreamSynchronize(s));
    rep->sum_a_log_u = h[0];
    rep->sum_b_log_v = h[1];
    rep->rot = p->eps * (h[0] + h[1]);
  }
  return st;
}

lsk_status lsk_factored_sinkhorn_implicit_batched(const lsk_feature_params* p, const float* U,
                                                  const float* X, int64_t n, const float* Y,
                                                  int64_t m, int32_t batch, const float* a,
                                                  const float* b, const lsk_solve_opts* o,
                                                  float* u, float* v, lsk_report* reps,
                                                  void* stream) {
  if (!p) return fail(LSK_EINVAL, "params NULL");
  LSK_TRY(check_common(n, m, p->r, p->eps));
  if (batch < 1) return fail(LSK_EINVAL, "batch must be >= 1");
  if (!U || !X || !Y || !a || !b || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  if (p->d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  if (o && (o->flags & LSK_SOLVE_STABILIZE))
    return fail(LSK_EUNSUPPORTED, "the stabilised implicit solve is single-problem");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  Carve cv;
  const size_t oW = cv.take(sizeof(float) * p->d * p->r);
  const size_t oB = cv.take(sizeof(float) * p->r);
  // small problems: every problem's factors materialised once (one FFMA feature-map launch per
  // side over all batch x n rows: the anchors are shared) for the resident cluster kernel
  const bool res = resident_allowed(o) && resident_cluster(p->r, n, m) > 0;
  const size_t oD = res ? cv.take(sizeof(float) * p->r) : 0;
  const size_t oF = res ? cv.take(sizeof(float) * (size_t)batch * (n + m) * p->r) : 0;
  LSK_TRY(get_ws(s, cv.off + solve_ws_bytes(n, m, batch), &ws));
  float* Wt = reinterpret_cast<float*>(ws + oW);
  float* b2 = reinterpret_cast<float*>(ws + oB);
  float* bD = res ? reinterpret_cast<float*>(ws + oD) : nullptr;
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, Wt, b2, bD, s));
  SinkArgs A{};
  A.X[0] = X; A.X[1] = Y;
  A.rows[0] = n; A.rows[1] = m;
  A.fstride[0] = n * p->d; A.fstride[1] = m * p->d;   // point rows per problem
  A.w[0] = a; A.w[1] = b;
  A.out[0] = u; A.out[1] = v;
  A.wstride[0] = n; A.wstride[1] = m;
  A.r = p->r; A.d = p->d; A.eps = p->eps;
  A.Wt = Wt; A.beta2 = b2;
  A.c2 = (float)(-2.0 * 1.4426950408889634074 / p->eps);
  if (res) {
    float* F0 = reinterpret_cast<float*>(ws + oF);
    float* F1 = F0 + (size_t)batch * n * p->r;
    LSK_CU(launch_feature_map(X, (int64_t)batch * n, p->d, U, Wt, b2, bD, p->r, p->eps, F0, s));
    LSK_CU(launch_feature_map(Y, (int64_t)batch * m, p->d, U, Wt, b2, bD, p->r, p->eps, F1, s));
    A.F[0] = F0;
    A.F[1] = F1;
    A.fstride[0] = n * p->r;   // factor rows per problem
    A.fstride[1] = m * p->r;
    return run_solve(A, false, batch, o, reps, nullptr, s);
  }
  LSK_TRY(setup_fact(A, p->R, batch, s, ws, cv));
  return run_solve(A, true, batch, o, reps, nullptr, s);
}

lsk_status lsk_implicit_row_offsets(const lsk_feature_params* p, const float* U, const float* X,
                                    int64_t n, double* logoff, void* stream) {
  if (!p || !U || !X || !logoff) return fail(LSK_EINVAL, "NULL argument");
  if (n < 1 || p->r < 4 || p->r % 4) return fail(LSK_EINVAL, "bad sizes");
  if (p->d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  Carve cv;
  const size_t oW = cv.take(sizeof(float) * p->d * p->r);
  const size_t oB = cv.take(sizeof(float) * p->r);
  const size_t oM = cv.take(sizeof(float) * n);
  LSK_TRY(get_ws(s, cv.off, &ws));
  float* Wt = reinterpret_cast<float*>(ws + oW);
  float* b2 = reinterpret_cast<float*>(ws + oB);
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, Wt, b2, nullptr, s));
  LSK_CU(launch_row_shift(X, n, p->d, Wt, b2, p->r, (float)(-2.0 * 1.4426950408889634074 / p->eps),
                          reinterpret_cast<float*>(ws + oM), logoff, s));
  return LSK_OK;
}

lsk_status lsk_factored_sinkhorn_batched(const float* Xi, int64_t n, const float* Zeta,
                                         int64_t m, int32_t r, int32_t batch, const float* a,
                                         const float* b, double eps, const lsk_solve_opts* o,
                                         float* u, float* v, lsk_report* reps, void* stream) {
  LSK_TRY(check_common(n, m, r, eps));
  if (batch < 1) return fail(LSK_EINVAL, "batch must be >= 1");
  if (!Xi || !Zeta || !a || !b || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  if (!aligned16(Xi) || !aligned16(Zeta)) return fail(LSK_EINVAL, "factors must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SinkArgs A{};
  A.F[0] = Xi; A.F[1] = Zeta;
  A.rows[0] = n; A.rows[1] = m;
  A.fstride[0] = n * r; A.fstride[1] = m * r;
  A.w[0] = a; A.w[1] = b;
  A.out[0] = u; A.out[1] = v;
  A.wstride[0] = n; A.wstride[1] = m;
  A.r = r; A.d = 1; A.eps = eps;
  return run_solve(A, false, batch, o, reps, nullptr, s);
}

// ---------------------------------------------------------------- emulated ranks ----------
// N ranks of one row-sharded solve as the N problems of one cooperative launch on one GPU:
// rank q owns rows [q n/N, (q+1) n/N) (n, m divisible by N), its own fp64 inbox
// [2][N][xrs] in this GPU's memory, and runs exactly the in-kernel exchange of
// lsk_comm_enable_p2p (lsk_sink_common.cuh xrank_total) — the multi-GPU protocol tested and
// timed where only one GPU exists (B200_PROFILING.md: ranks that wait on one another must not
// be separate launches on one GPU).
static lsk_status setup_emulation(SinkArgs& A, int32_t nranks, int64_t n, int64_t m, int r,
                                  cudaStream_t s) {
  if (nranks < 2 || nranks > kMaxRanks) return fail(LSK_EINVAL, "nranks must be 2..8");
  if (n % nranks || m % nranks) return fail(LSK_EINVAL, "n and m must be divisible by nranks");
  // every r-vector column (r + kExtra) and the two read-out columns, padded to 32
  const int xrs = ((r + kExtra + 2) + 31) & ~31;
  char* ws;
  const size_t per = sizeof(double) * 2 * nranks * xrs;
  LSK_TRY(get_ws(s, per * nranks, &ws, 2));
  LSK_CU(cudaMemsetAsync(ws, 0xFF, per * nranks, s));   // all-ones sentinel
  A.emul = 1;
  A.nranks = nranks;
  A.rank = 0;
  A.xrs = xrs;
  for (int q = 0; q < nranks; ++q) A.xbox[q] = reinterpret_cast<double*>(ws + per * q);
  A.xtimeout_ns = 20LL * 1000 * 1000 * 1000;
  return LSK_OK;
}

lsk_status lsk_factored_sinkhorn_emulated(int32_t nranks, const float* Xi, int64_t n,
                                          const float* Zeta, int64_t m, int32_t r,
                                          const float* a, const float* b, double eps,
                                          const lsk_solve_opts* o, float* u, float* v,
                                          lsk_report* reps, void* stream) {
  LSK_TRY(check_common(n, m, r, eps));
  if (!Xi || !Zeta || !a || !b || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  if (!aligned16(Xi) || !aligned16(Zeta)) return fail(LSK_EINVAL, "factors must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SinkArgs A{};
  LSK_TRY(setup_emulation(A, nranks, n, m, r, s));
  const int64_t nl = n / nranks, ml = m / nranks;
  A.F[0] = Xi; A.F[1] = Zeta;
  A.rows[0] = nl; A.rows[1] = ml;
  A.fstride[0] = nl * r; A.fstride[1] = ml * r;
  A.w[0] = a; A.w[1] = b;
  A.out[0] = u; A.out[1] = v;
  A.wstride[0] = nl; A.wstride[1] = ml;
  A.r = r; A.d = 1; A.eps = eps;
  return run_solve(A, false, nranks, o, reps, nullptr, s);
}

lsk_status lsk_factored_sinkhorn_implicit_emulated(int32_t nranks, const lsk_feature_params* p,
                                                   const float* U, const float* X, int64_t n,
                                                   const float* Y, int64_t m, const float* a,
                                                   const float* b, const lsk_solve_opts* o,
                                                   float* u, float* v, lsk_report* reps,
                                                   void* stream) {
  if (!p) return fail(LSK_EINVAL, "params NULL");
  LSK_TRY(check_common(n, m, p->r, p->eps));
  if (!U || !X || !Y || !a || !b || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  if (p->d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SinkArgs A{};
  LSK_TRY(setup_emulation(A, nranks, n, m, p->r, s));
  const int64_t nl = n / nranks, ml = m / nranks;
  char* ws;
  Carve cv;
  const size_t oW = cv.take(sizeof(float) * p->d * p->r);
  const size_t oB = cv.take(sizeof(float) * p->r);
  LSK_TRY(get_ws(s, cv.off + solve_ws_bytes(n, m, 1), &ws));
  float* Wt = reinterpret_cast<float*>(ws + oW);
  float* b2 = reinterpret_cast<float*>(ws + oB);
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, Wt, b2, nullptr, s));
  A.X[0] = X; A.X[1] = Y;
  A.rows[0] = nl; A.rows[1] = ml;
  A.fstride[0] = nl * p->d; A.fstride[1] = ml * p->d;
  A.w[0] = a; A.w[1] = b;
  A.out[0] = u; A.out[1] = v;
  A.wstride[0] = nl; A.wstride[1] = ml;
  A.r = p->r; A.d = p->d; A.eps = p->eps;
  A.Wt = Wt; A.beta2 = b2;
  A.c2 = (float)(-2.0 * 1.4426950408889634074 / p->eps);
  LSK_TRY(setup_fact(A, p->R, nranks, s, ws, cv));
  return run_solve(A, true, nranks, o, reps, nullptr, s);
}

lsk_status lsk_rot_value(const float* u, const float* v, const float* a, const float* b,
                         int64_t n, int64_t m, double eps, double* rot_host, lsk_comm* comm,
                         void* stream) {
  if (!u || !v || !a || !b || !rot_host) return fail(LSK_EINVAL, "NULL argument");
  if (n < 1 || m < 1 || !(eps > 0)) return fail(LSK_EINVAL, "bad sizes or eps");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  LSK_TRY(get_ws(s, 8192 + 2 * 64 * sizeof(double), &ws));
  double* part = reinterpret_cast<double*>(ws + 256);
  double* out2 = reinterpret_cast<double*>(ws);
  LSK_CU(launch_rot_value(u, v, a, b, n, m, 1, part, out2, s));
  LSK_TRY(take_sticky(s));   // a report-less solve before this read-out broke down
  if (comm) {
    if (!nccl().ok) return fail(LSK_ENCCL, "NCCL not loadable");
    LSK_TRY(nccl_check(nccl().allReduce(out2, out2, 2, ncclFloat64, ncclSum, comm->comm, s),
                       "ncclAllReduce(rot)"));
  }
  double h[2];
  LSK_CU(cudaMemcpyAsync(h, out2, sizeof(h), cudaMemcpyDeviceToHost, s));
  LSK_CU(cudaStreamSynchronize(s));
  *rot_host = eps * (h[0] + h[1]);
  return LSK_OK;
}

lsk_status lsk_rot_value_batched(const float* u, const float* v, const float* a,
                                 const float* b, int64_t n, int64_t m, int32_t batch,
                                 double eps, double* rots_host, void* stream) {
  if (!u || !v || !a || !b || !rots_host) return fail(LSK_EINVAL, "NULL argument");
  if (n < 1 || m < 1 || batch < 1 || !(eps > 0)) return fail(LSK_EINVAL, "bad sizes or eps");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  Carve cv;
  const size_t oOut = cv.take(sizeof(double) * 2 * batch);
  const size_t oPart = cv.take(sizeof(double) * 2 * 64 * batch);
  LSK_TRY(get_ws(s, cv.off, &ws));
  double* out2 = reinterpret_cast<double*>(ws + oOut);
  LSK_CU(launch_rot_value(u, v, a, b, n, m, batch, reinterpret_cast<double*>(ws + oPart), out2, s));
  std::vector<double> h((size_t)2 * batch);
  LSK_CU(cudaMemcpyAsync(h.data(), out2, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
  LSK_CU(cudaStreamSynchronize(s));
  for (int i = 0; i < batch; ++i) rots_host[i] = eps * (h[2 * i] + h[2 * i + 1]);
  return LSK_OK;
}

// ---------------------------------------------------------------- Sinkhorn divergence --
static lsk_status divergence_impl(bool impl, const float* F, int64_t n, const float* G,
                                  int64_t m, int r, int d, const float* a, const float* b,
                                  double eps, const float* Wt, const float* b2, float c2,
                                  double R, const lsk_solve_opts* o, double* out4, lsk_report* reps3,
                                  cudaStream_t s, char* ws, Carve& cv) {
  const int64_t mx = std::max(n, m);
  float* us = reinterpret_cast<float*>(ws + cv.take(sizeof(float) * mx));
  float* vs = reinterpret_cast<float*>(ws + cv.take(sizeof(float) * mx));
  struct Prob { const float *f0, *f1, *w0, *w1; int64_t r0, r1; } probs[3] = {
      {F, G, a, b, n, m}, {F, F, a, a, n, n}, {G, G, b, b, m, m}};
  double W[3];
  lsk_status worst = LSK_OK;
  for (int k = 0; k < 3; ++k) {
    SinkArgs A{};
    if (impl) { A.X[0] = probs[k].f0; A.X[1] = probs[k].f1; }
    else { A.F[0] = probs[k].f0; A.F[1] = probs[k].f1; }
    A.rows[0] = probs[k].r0; A.rows[1] = probs[k].r1;
    A.w[0] = probs[k].w0; A.w[1] = probs[k].w1;
    A.out[0] = us; A.out[1] = vs;
    A.r = r; A.d = d; A.eps = eps;
    A.Wt = Wt; A.beta2 = b2; A.c2 = c2;
    Carve cv2 = cv;   // each solve reuses the same workspace tail
    if (impl) LSK_TRY(setup_fact(A, R, 1, s, ws, cv2));
    lsk_report rep{};
    lsk_status st = run_solve(A, impl, 1, o, &rep, nullptr, s);
    if (st < 0) return st;
    if (st > worst) worst = st;
    W[k] = rep.rot;
    if (reps3) reps3[k] = rep;
  }
  out4[0] = W[0] - 0.5 * (W[1] + W[2]);
  out4[1] = W[0];
  out4[2] = W[1];
  out4[3] = W[2];
  return worst;
}

// ---------------------------------------------------------------- NEXT f4: Alg. 2 --------
// Host side of the accelerated Sinkhorn line search (kernels and data flow: lsk_accel.cu).
// Per trial: 1 lambda launch, 3 factor passes (+2 fixed-order r-vector reductions), 3
// statistics launches, one synchronisation to read the per-CTA partials (summed here in a
// fixed order — the device's block choice repeats the same sums), then the accept launch.
lsk_status lsk_accelerated_sinkhorn(const float* Xi, int64_t n, const float* Zeta, int64_t m,
                                    int32_t r, const float* a, const float* b, double eps,
                                    const lsk_accel_opts* o, double* eta1, double* eta2,
                                    double* F_trace, double* L_trace, int32_t* blk_trace,
                                    lsk_accel_report* rep, void* stream) {
  LSK_TRY(check_common(n, m, r, eps));
  if (!Xi || !Zeta || !a || !b || !o || !eta1 || !eta2) return fail(LSK_EINVAL, "NULL argument");
  if (!aligned16(Xi) || !aligned16(Zeta)) return fail(LSK_EINVAL, "factors must be 16-byte aligned");
  if (o->max_iters < 1 || !(o->L0 > 0.0)) return fail(LSK_EINVAL, "max_iters < 1 or L0 <= 0");
  if (r > 2048) return fail(LSK_EDIM, "accelerated solver supports r <= 2048");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int G = accel_grid(), Gp = accel_pass_grid();
  const int64_t mx = std::max(n, m);
  Carve cv;
  const size_t o_an = cv.take(8 * n), o_bn = cv.take(8 * m);
  const size_t o_z1 = cv.take(8 * n), o_l1 = cv.take(8 * n), o_p1 = cv.take(8 * n), o_t1 = cv.take(8 * n);
  const size_t o_z2 = cv.take(8 * m), o_l2 = cv.take(8 * m), o_p2 = cv.take(8 * m), o_t2 = cv.take(8 * m);
  const size_t o_en = cv.take(8 * mx), o_pt = cv.take(8 * 6 * G), o_sc = cv.take(8 * 32),
               o_tk = cv.take(256);
  const size_t o_pa = cv.take(8 * (size_t)(Gp + 1) * r), o_pb = cv.take(8 * (size_t)(Gp + 1) * r);
  const size_t o_ct = cv.take(8 * CT_COUNT);
  const size_t o_tf = cv.take(8 * (size_t)o->max_iters), o_tl = cv.take(8 * (size_t)o->max_iters),
               o_tb = cv.take(4 * (size_t)o->max_iters);
  char* ws;
  LSK_TRY(get_ws(s, cv.off, &ws));
  auto D = [&](size_t off) { return reinterpret_cast<double*>(ws + off); };
  AccelVecs v{};
  v.n = n; v.m = m;
  v.an = D(o_an); v.bn = D(o_bn);
  v.eta1 = eta1; v.zet1 = D(o_z1); v.lam1 = D(o_l1); v.p1 = D(o_p1); v.t1 = D(o_t1);
  v.eta2 = eta2; v.zet2 = D(o_z2); v.lam2 = D(o_l2); v.p2 = D(o_p2); v.t2 = D(o_t2);
  v.etan = D(o_en); v.part = D(o_pt); v.scal = D(o_sc);
  v.ticket = reinterpret_cast<unsigned int*>(ws + o_tk);
  double* partA = D(o_pa);
  double* partB = D(o_pb);
  // Init: eta^0 = zeta^0 = 0, x_hat^0 = 0; simplex weights (C28)
  LSK_CU(cudaMemsetAsync(eta1, 0, 8 * n, s));
  LSK_CU(cudaMemsetAsync(eta2, 0, 8 * m, s));
  LSK_CU(cudaMemsetAsync(v.zet1, 0, 8 * n, s));
  LSK_CU(cudaMemsetAsync(v.zet2, 0, 8 * m, s));
  LSK_CU(cudaMemsetAsync(v.p1, 0, 8 * n, s));
  LSK_CU(cudaMemsetAsync(v.p2, 0, 8 * m, s));
  LSK_CU(cudaMemsetAsync(v.ticket, 0, 256, s));
  LSK_CU(launch_accel_normalise(a, b, v, s));

  double sc[SC_COUNT];
  double ak = 0.0, Lk = o->L0, F = 0.0, plan_err = -1.0;
  int it = 0, trials = 0;
  bool converged = false;
  // The whole solve as one CUDA graph (device-side line search, DESIGN.md §6 K7): one
  // synchronisation per solve instead of one per trial; the host-driven loop below remains
  // the fallback when the graph cannot be built (tuning builds: LSK_ACCEL_HOST=1 forces it).
  const char* force_host = tuning_env("LSK_ACCEL_HOST");
  if (!(force_host && atoi(force_host) == 1)) {
    double ct[CT_COUNT] = {};
    ct[CT_LK] = o->L0;
    double* ctl = D(o_ct);
    LSK_CU(cudaMemcpyAsync(ctl, ct, sizeof(ct), cudaMemcpyHostToDevice, s));
    v.ctl = ctl;
    double* dF = D(o_tf);
    double* dL = D(o_tl);
    int* dB = reinterpret_cast<int*>(ws + o_tb);
    const cudaError_t ge = accel_solve_graph(v, Xi, n, Zeta, m, r, partA, partB, eps, o->max_iters,
                                             o->tol, dF, dL, dB, s);
    if (ge == cudaSuccess) {
      LSK_CU(cudaMemcpyAsync(ct, ctl, sizeof(ct), cudaMemcpyDeviceToHost, s));
      LSK_CU(cudaStreamSynchronize(s));
      it = (int)ct[CT_IT];
      if (it > 0) {
        if (F_trace) LSK_CU(cudaMemcpy(F_trace, dF, 8 * (size_t)it, cudaMemcpyDeviceToHost));
        if (L_trace) LSK_CU(cudaMemcpy(L_trace, dL, 8 * (size_t)it, cudaMemcpyDeviceToHost));
        if (blk_trace) LSK_CU(cudaMemcpy(blk_trace, dB, 4 * (size_t)it, cudaMemcpyDeviceToHost));
      }
      if (ct[CT_ERR] == 1.0)
        return fail(LSK_EBREAKDOWN, "zero or non-finite K e^lambda during the accelerated solve");
      if (ct[CT_ERR] != 0.0) return fail(LSK_EBREAKDOWN, "line search diverged");
      if (rep) {
        rep->iters = it;
        rep->trials = (int32_t)ct[CT_TRIALS];
        rep->converged = ct[CT_CONV] != 0.0 ? 1 : 0;
        rep->reserved = 0;
        rep->F = ct[CT_F];
        rep->L = ct[CT_LK];
        rep->plan_err = ct[CT_PERR];
      }
      if (o->tol > 0.0 && ct[CT_CONV] == 0.0) {
        g_err = "tolerance not reached within max_iters";
        return LSK_NOT_CONVERGED;
      }
      return LSK_OK;
    }
    (void)cudaGetLastError();   // the graph was not launched: the host-driven loop
    v.ctl = nullptr;
  }
  for (; it < o->max_iters;) {
    double L1 = Lk / 2.0;   // C24: one halving, then doubling on rejection
    double phi_new = 0.0;
    int blk = 1;
    for (;;) {
      const double a1 = 1.0 / (2.0 * L1) + std::sqrt(1.0 / (4.0 * L1 * L1) + ak * ak * Lk / L1);
      const double tau = 1.0 / (a1 * L1);
      ++trials;
      LSK_CU(launch_accel_lambda(tau, v, s));
      // s2 = Zeta^T e^{l2 - M2};  t1 = Xi s2 and s1 = Xi^T e^{l1 - M1};  t2 = Zeta s1
      LSK_CU(launch_accel_pass(Zeta, m, r, nullptr, v.lam2, v.scal + SC_M2, nullptr, partA, s));
      LSK_CU(launch_accel_pass(Xi, n, r, partA + (size_t)Gp * r, v.lam1, v.scal + SC_M1, v.t1, partB, s));
      LSK_CU(launch_accel_pass(Zeta, m, r, partB + (size_t)Gp * r, nullptr, nullptr, v.t2, nullptr, s));
      LSK_CU(launch_accel_stats(1, v, 0, 0, 0, s));
      LSK_CU(launch_accel_stats(2, v, 0, 0, 0, s));
      LSK_CU(launch_accel_stats(3, v, 0, 0, 0, s));
      LSK_CU(cudaMemcpyAsync(sc, v.scal, sizeof(sc), cudaMemcpyDeviceToHost, s));
      LSK_CU(cudaStreamSynchronize(s));
      const double M1 = sc[SC_M1], M2 = sc[SC_M2], S1 = sc[SC_S1], S2 = sc[SC_S2];
      const double la = sc[SC_LA], lb = sc[SC_LB], n1 = sc[SC_N1], n2 = sc[SC_N2];
      if (sc[SC_BAD] > 0.0 || !(S1 > 0.0) || !std::isfinite(S1) || !(S2 > 0.0))
        return fail(LSK_EBREAKDOWN, "zero or non-finite K e^lambda during the accelerated solve");
      blk = sc[SC_BLK] == 1.0 ? 1 : 2;                          // argmax, ties -> 1 (C27)
      // phi(lambda^k), with c from the moved block's own side (the same t as phi(eta^{k+1}),
      // so the exact block decrease stays >= 0 in floating point), and phi(eta^{k+1})
      const double phi_lam = M1 + M2 + std::log(blk == 1 ? S1 : S2) - la - lb;
      phi_new = std::log(sc[SC_E]) - (blk == 1 ? sc[SC_EW] + lb : la + sc[SC_EW]);
      if (tuning_env("LSK_ADEBUG"))   // tuning/debug only
        fprintf(stderr, "accel it %d L1 %.3g blk %d n %.3g %.3g phi %.12g -> %.12g\n", it, L1, blk,
                n1, n2, phi_lam, phi_new);
      // acceptance with an fp64 rounding allowance (reading C29)
      if (phi_new <= phi_lam - (n1 + n2) / (2.0 * L1) + 1e-13 * std::max(1.0, std::fabs(phi_lam))) {
        LSK_CU(launch_accel_stats(4, v, a1, Lk * ak * ak, L1 * a1 * a1, s));
        ak = a1;
        Lk = L1;
        break;
      }
      L1 *= 2.0;
      if (!(L1 < 1e300)) return fail(LSK_EBREAKDOWN, "line search diverged");
    }
    F = -eps * phi_new;
    if (F_trace) F_trace[it] = F;
    if (L_trace) L_trace[it] = Lk;
    if (blk_trace) blk_trace[it] = blk;
    ++it;
    if (o->tol > 0.0 || it == o->max_iters) {
      LSK_CU(cudaMemcpyAsync(&plan_err, v.scal + SC_PERR, 8, cudaMemcpyDeviceToHost, s));
      LSK_CU(cudaStreamSynchronize(s));
      if (o->tol > 0.0 && plan_err < o->tol) {
        converged = true;
        break;
      }
    }
  }
  if (rep) {
    rep->iters = it;
    rep->trials = trials;
    rep->converged = converged ? 1 : 0;
    rep->reserved = 0;
    rep->F = F;
    rep->L = Lk;
    rep->plan_err = plan_err;
  }
  if (o->tol > 0.0 && !converged) {
    g_err = "tolerance not reached within max_iters";
    return LSK_NOT_CONVERGED;
  }
  return LSK_OK;
}

// ---------------------------------------------------------------- host-buffer pipeline --
lsk_status lsk_rot_host(const float* X_host, int64_t n, const float* Y_host, int64_t m,
                        int32_t d, const float* a_host, const float* b_host, double eps,
                        int32_t r, uint64_t seed, double R, const lsk_solve_opts* o,
                        int32_t variant, float* u_host, float* v_host, lsk_report* rep) {
  LSK_TRY(check_common(n, m, r, eps));
  if (!X_host || !Y_host || !a_host || !b_host || !o) return fail(LSK_EINVAL, "NULL argument");
  if (d < 1) return fail(LSK_EINVAL, "d must be >= 1");
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  static std::map<int, std::pair<void*, size_t>> bufs;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  LSK_CU(cudaGetDevice(&dev));
  if (!streams.count(dev)) {
    cudaStream_t st;
    LSK_CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    streams[dev] = st;
  }
  cudaStream_t s = streams[dev];
  const bool impl = variant == 2 || (variant == 0 && d <= 8);
  Carve cv;
  const size_t oX = cv.take(sizeof(float) * n * d), oY = cv.take(sizeof(float) * m * d);
  const size_t oa = cv.take(sizeof(float) * n), ob = cv.take(sizeof(float) * m);
  const size_t ou = cv.take(sizeof(float) * n), ov = cv.take(sizeof(float) * m);
  const size_t oU = cv.take(sizeof(float) * r * d);
  const size_t oXi = impl ? 0 : cv.take(sizeof(float) * n * r);
  const size_t oZe = impl ? 0 : cv.take(sizeof(float) * m * r);
  auto& bb = bufs[dev];
  if (bb.second < cv.off) {
    if (bb.first) cudaFree(bb.first);
    bb.first = nullptr;
    bb.second = 0;
    if (cudaMalloc(&bb.first, cv.off) != cudaSuccess) {
      cudaGetLastError();
      return fail(LSK_ENOMEM, "lsk_rot_host: device buffers do not fit");
    }
    bb.second = cv.off;
  }
  char* base = static_cast<char*>(bb.first);
  float *X = (float*)(base + oX), *Y = (float*)(base + oY), *a = (float*)(base + oa),
        *b = (float*)(base + ob), *u = (float*)(base + ou), *v = (float*)(base + ov),
        *U = (float*)(base + oU);
  LSK_CU(cudaMemcpyAsync(X, X_host, sizeof(float) * n * d, cudaMemcpyHostToDevice, s));
  LSK_CU(cudaMemcpyAsync(Y, Y_host, sizeof(float) * m * d, cudaMemcpyHostToDevice, s));
  LSK_CU(cudaMemcpyAsync(a, a_host, sizeof(float) * n, cudaMemcpyHostToDevice, s));
  LSK_CU(cudaMemcpyAsync(b, b_host, sizeof(float) * m, cudaMemcpyHostToDevice, s));
  lsk_feature_params p;
  LSK_TRY(lsk_feature_params_init(eps, d, r, R, seed, X, n, Y, m, &p, nullptr, s));
  LSK_TRY(lsk_draw_anchors(&p, U, s));
  lsk_report local{};
  lsk_status st;
  if (impl) {
    st = lsk_factored_sinkhorn_implicit(&p, U, X, n, Y, m, a, b, o, u, v, &local, nullptr, s);
  } else {
    float* Xi = (float*)(base + oXi);
    float* Ze = (float*)(base + oZe);
    LSK_TRY(lsk_feature_map(&p, U, X, n, Xi, s));
    LSK_TRY(lsk_feature_map(&p, U, Y, m, Ze, s));
    st = lsk_factored_sinkhorn(Xi, n, Ze, m, r, a, b, eps, o, u, v, &local, nullptr, s);
  }
  if (st < 0) return st;
  if (u_host) LSK_CU(cudaMemcpyAsync(u_host, u, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
  if (v_host) LSK_CU(cudaMemcpyAsync(v_host, v, sizeof(float) * m, cudaMemcpyDeviceToHost, s));
  LSK_CU(cudaStreamSynchronize(s));
  if (rep) *rep = local;
  return st;
}

lsk_status lsk_sinkhorn_divergence(const float* Xi, int64_t n, const float* Zeta, int64_t m,
                                   int32_t r, const float* a, const float* b, double eps,
                                   const lsk_solve_opts* o, double* out4_host,
                                   lsk_report* reps3, void* stream) {
  LSK_TRY(check_common(n, m, r, eps));
  if (!Xi || !Zeta || !a || !b || !out4_host) return fail(LSK_EINVAL, "NULL argument");
  if (!aligned16(Xi) || !aligned16(Zeta)) return fail(LSK_EINVAL, "factors must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t mx = std::max(n, m);
  char* ws;
  LSK_TRY(get_ws(s, 2 * 256 + 2 * sizeof(float) * mx + solve_ws_bytes(mx, mx, 1), &ws));
  Carve cv;
  return divergence_impl(false, Xi, n, Zeta, m, r, 1, a, b, eps, nullptr, nullptr, 0.f, 0.0, o,
                         out4_host, reps3, s, ws, cv);
}

lsk_status lsk_sinkhorn_divergence_implicit(const lsk_feature_params* p, const float* U,
                                            const float* X, int64_t n, const float* Y,
                                            int64_t m, const float* a, const float* b,
                                            const lsk_solve_opts* o, double* out4_host,
                                            lsk_report* reps3, void* stream) {
  if (!p) return fail(LSK_EINVAL, "params NULL");
  LSK_TRY(check_common(n, m, p->r, p->eps));
  if (!U || !X || !Y || !a || !b || !out4_host) return fail(LSK_EINVAL, "NULL argument");
  if (p->d > 8) return fail(LSK_EDIM, "implicit variant supports d <= 8");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t mx = std::max(n, m);
  char* ws;
  Carve cv;
  const size_t oW = cv.take(sizeof(float) * p->d * p->r);
  const size_t oB = cv.take(sizeof(float) * p->r);
  LSK_TRY(get_ws(s, cv.off + 2 * 256 + 2 * sizeof(float) * mx + solve_ws_bytes(mx, mx, 1), &ws));
  float* Wt = reinterpret_cast<float*>(ws + oW);
  float* b2 = reinterpret_cast<float*>(ws + oB);
  LSK_CU(launch_anchor_prep(U, p->r, p->d, p->eps, p->q, p->log_scale, Wt, b2, nullptr, s));
  return divergence_impl(true, X, n, Y, m, p->r, p->d, a, b, p->eps, Wt, b2,
                         (float)(-2.0 * 1.4426950408889634074 / p->eps), p->R, o, out4_host, reps3, s,
                         ws, cv);
}

lsk_status lsk_rot_gradient(const lsk_feature_params* p, const float* U, const float* X,
                            int64_t n, const float* Y, int64_t m, const float* Xi,
                            const float* Zeta, const float* u, const float* v, float* gX,
                            float* gY, float* gU, void* stream) {
  if (!p || !U || !X || !Y || !Xi || !Zeta || !u || !v) return fail(LSK_EINVAL, "NULL argument");
  LSK_TRY(check_common(n, m, p->r, p->eps));
  if (p->d > 16) return fail(LSK_EDIM, "gradients support d <= 16");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws;
  LSK_TRY(get_ws(s, grad_workspace_bytes(p->r, p->d), &ws));
  LSK_CU(launch_gradients(X, n, Y, m, p->d, U, p->r, p->q, Xi, Zeta, u, v, gX, gY, gU,
                          reinterpret_cast<double*>(ws), s));
  return LSK_OK;
}

// ---------------------------------------------------------------- NCCL communicator -----
lsk_status lsk_comm_get_unique_id(void* out_host) {
  if (!out_host) return fail(LSK_EINVAL, "out is NULL");
  if (!nccl().ok) return fail(LSK_ENCCL, "NCCL not loadable");
  ncclUniqueId id;
  LSK_TRY(nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId"));
  std::memcpy(out_host, &id, sizeof(id));
  return LSK_OK;
}

lsk_status lsk_comm_init(lsk_comm** out, int32_t nranks, int32_t rank,
                         const void* unique_id_host, int32_t device) {
  if (!out || !unique_id_host || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(LSK_EINVAL, "bad communicator arguments");
  if (!nccl().ok) return fail(LSK_ENCCL, "NCCL not loadable");
  LSK_CU(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(&id, unique_id_host, sizeof(id));
  lsk_comm* c = new lsk_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  lsk_status st = nccl_check(nccl().commInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  if (st < 0) {
    delete c;
    return st;
  }
  *out = c;
  return LSK_OK;
}

lsk_status lsk_comm_enable_p2p(lsk_comm* c, int32_t r_max, void* stream) {
  if (!c || r_max < 4) return fail(LSK_EINVAL, "bad arguments");
  if (c->nranks > kMaxRanks) return fail(LSK_EUNSUPPORTED, "more ranks than kMaxRanks");
  if (!nccl().ok || !nccl().allGather) return fail(LSK_ENCCL, "NCCL (allGather) not loadable");
  if (c->p2p) return LSK_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LSK_CU(cudaSetDevice(c->device));
  const int N = c->nranks;
  const int xrs = ((r_max + kExtra + 2) + 31) & ~31;
  double* mine = nullptr;
  LSK_CU(cudaMalloc(&mine, sizeof(double) * 2 * N * xrs));
  LSK_CU(cudaMemset(mine, 0xFF, sizeof(double) * 2 * N * xrs));   // all-ones sentinel
  LSK_CU(cudaDeviceSynchronize());
  // exchange the IPC handles with one NCCL all-gather (it also orders every rank's sentinel
  // initialisation before any peer store: no rank starts a solve before the gather completes)
  cudaIpcMemHandle_t h;
  LSK_CU(cudaIpcGetMemHandle(&h, mine));
  char* dbuf = nullptr;
  LSK_CU(cudaMalloc(&dbuf, sizeof(h) * (N + 1)));
  LSK_CU(cudaMemcpyAsync(dbuf + sizeof(h) * N, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  lsk_status st = nccl_check(nccl().allGather(dbuf + sizeof(h) * N, dbuf, sizeof(h), ncclChar,
                                              c->comm, s), "ncclAllGather(ipc handles)");
  std::vector<cudaIpcMemHandle_t> all(N);
  if (st == LSK_OK) {
    LSK_CU(cudaMemcpyAsync(all.data(), dbuf, sizeof(h) * N, cudaMemcpyDeviceToHost, s));
    LSK_CU(cudaStreamSynchronize(s));
  }
  cudaFree(dbuf);
  if (st != LSK_OK) {
    cudaFree(mine);
    return st;
  }
  cudaError_t open_err = cudaSuccess;
  for (int i = 0; i < N && open_err == cudaSuccess; ++i) {
    if (i == c->rank) {
      c->xbox[i] = mine;
      continue;
    }
    void* ptr = nullptr;
    open_err = cudaIpcOpenMemHandle(&ptr, all[i], cudaIpcMemLazyEnablePeerAccess);
    if (open_err == cudaSuccess) c->xbox[i] = static_cast<double*>(ptr);
    else cudaGetLastError();
  }
  // every rank must take the same path (a rank on the in-kernel exchange would wait for peers
  // on the NCCL path until the timeout): all-gather the local outcome and agree
  int32_t* flags = nullptr;
  LSK_CU(cudaMalloc(&flags, sizeof(int32_t) * (N + 1)));
  const int32_t ok = open_err == cudaSuccess ? 1 : 0;
  std::vector<int32_t> okv(N, 0);
  LSK_CU(cudaMemcpyAsync(flags + N, &ok, sizeof(ok), cudaMemcpyHostToDevice, s));
  st = nccl_check(nccl().allGather(flags + N, flags, 1, ncclInt32, c->comm, s), "ncclAllGather(p2p flags)");
  if (st == LSK_OK) {
    LSK_CU(cudaMemcpyAsync(okv.data(), flags, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, s));
    LSK_CU(cudaStreamSynchronize(s));
  }
  bool all_ok = st == LSK_OK;
  for (int i = 0; i < N; ++i) all_ok = all_ok && okv[i] == 1;
  if (!all_ok) {
    for (int j = 0; j < N; ++j)
      if (j != c->rank && c->xbox[j]) cudaIpcCloseMemHandle(c->xbox[j]);
    // every rank has closed its mappings before any exporter frees its inbox
    if (st == LSK_OK) {
      st = nccl_check(nccl().allGather(flags + N, flags, 1, ncclInt32, c->comm, s), "ncclAllGather(p2p close)");
      cudaStreamSynchronize(s);
    }
    cudaFree(flags);
    cudaFree(mine);
    for (auto& x : c->xbox) x = nullptr;
    if (st != LSK_OK) return st;
    return fail(LSK_EUNSUPPORTED, open_err != cudaSuccess
                                      ? std::string("peer memory unavailable: ") + cudaGetErrorString(open_err)
                                      : std::string("peer memory unavailable on another rank"));
  }
  cudaFree(flags);
  c->xrs = xrs;
  c->p2p = true;
  return LSK_OK;
}

lsk_status lsk_comm_destroy(lsk_comm* comm) {
  if (!comm) return LSK_OK;
  lsk_status st = LSK_OK;
  if (comm->p2p) {
    for (int i = 0; i < comm->nranks; ++i) {
      if (!comm->xbox[i]) continue;
      if (i == comm->rank) cudaFree(comm->xbox[i]);
      else cudaIpcCloseMemHandle(comm->xbox[i]);
    }
  }
  if (comm->comm) st = nccl_check(nccl().commDestroy(comm->comm), "ncclCommDestroy");
  delete comm;
  return st;
}

}  // extern "C"
