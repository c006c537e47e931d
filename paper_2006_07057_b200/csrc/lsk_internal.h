// lsk_internal.h — internal interfaces between the host API (lsk_api.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lsk.h"

namespace lsk {

constexpr int kConsumerThreads = 256;              // 8 consumer warps per CTA
constexpr int kThreads = kConsumerThreads + 32;    // + 1 producer warp
constexpr int kExtra = 4;                          // extras appended to every r-vector:
                                                   // [0]=err, [1]=breakdown, [2]=bad weights, [3]=0
constexpr int kStateDoubles = 16;                  // per-problem solve state block
constexpr int kMaxRanks = 8;                       // GPUs of one node in the peer exchange
// state block layout (doubles)
enum StateIdx {
  ST_ERR = 3,      // latest marginal error
  ST_STOP = 4,     // 1 once the solve has finished (early stop or last pass)
  ST_ITERS = 5,    // iterations of the returned state
  ST_ROT = 6,      // W_hat of the returned state
  ST_CONV = 7,     // converged flag
  ST_BRK = 8,      // breakdown count
  ST_FINAL_A = 9,  // a^T log u of the returned state
  ST_FINAL_B = 10, // b^T log v of the returned state
  ST_XERR = 11,    // 1 if a cross-GPU peer exchange timed out
  ST_WBAD = 12     // count of weights a_i / b_j that are not finite and > 0 (LSK_EWEIGHTS)
};

// Sticky per-(device, stream) status word (device int, atomicOr'ed by the solve kernels, read
// and cleared by the synchronising calls: lsk_stream_status, lsk_rot_value, report-taking solves)
enum StickyBits { STICKY_BREAKDOWN = 1, STICKY_XERR = 2, STICKY_WEIGHTS = 4 };

// Pass schedule: p = 0 init xi-pass (s_v = xi^T 1), p = 2t-1 v-pass of iteration t,
// p = 2t u-pass of iteration t (t = 1..T), p = 2T+1 error pass (if requested).
enum PassKind { PK_INIT = 0, PK_V = 1, PK_U = 2, PK_ERR = 3, PK_NONE = 4 };

struct SinkArgs {
  // factor 0 = xi side (rows n, weights a, output u); factor 1 = zeta side (m, b, v)
  const float* F[2];       // streaming: feature matrices (rows x r); hybrid implicit: the
                           // materialised rows [0, nstream) of each side
  int64_t nstream[2];      // hybrid implicit: rows of each side streamed instead of regenerated
  const float* X[2];       // implicit: point matrices (rows x d)
  int64_t rows[2];
  int64_t fstride[2];      // per-problem element stride of F (or X) for batched
  const float* w[2];       // a, b
  float* out[2];           // u (user), v (user)
  float* vbuf1;            // second v buffer (workspace)
  int64_t wstride[2];      // per-problem stride of w / out / vbuf1 (elements)
  int r;
  int d;
  int T;                   // max iterations
  int want_err;            // append the error pass
  int tol_mode;
  double tol;
  double eps;
  int gpp;                 // CTAs per problem
  int nprob;
  int pass_begin;          // passes [pass_begin, pass_end) run in this launch
  int pass_end;            // pass_end == num_passes also finalises
  int num_passes;
  int multi_launch;        // 1: one pass per launch (NCCL all-reduce of svec between launches)
  int nstage;              // ring stages
  int stage_floats;        // floats per stage (header + TR*r for streaming)
  double* part;            // [nprob][(r+kExtra+4)/4 blocks][gpp][4] fp64 partials (lsk_sink_common.cuh)
  double* svec;            // [nprob][r+kExtra]
  unsigned int* bar;       // [nprob] monotone barrier counters (zeroed once per solve)
  double* state;           // [nprob][kStateDoubles]
  // implicit-mode anchor data (fp32, r each; W is (d, r) column groups)
  const float* Wt;         // [d][r]  W_kc = (4 log2e / eps) U_kc, transposed
  const float* beta2;      // [r]     log2e (-(2/eps)|U_k|^2 + |U_k|^2/(eps q) + log_scale)
  float c2;                // -2 log2e / eps
  // implicit factored exponent (FACT): F_jk = h_j * 2^(beta2_k + abar + sum_c W_kc p_jc),
  // h_j = 2^(alpha2_j - abar) precomputed per row; NULL = plain expanded form
  const float* hrow[2];    // FACT: h_j; stabilised (stab = 1): the per-row shifts m_j
  float abar;
  int stab;                // 1: stabilised implicit mode (reading C30)
  int dbg;                 // tuning only: 1 = consumers release stages without computing
  unsigned long long* trace;   // tuning only: [pass][cta][4] globaltimer stamps, or NULL
  float l2_resident;       // fraction of each CTA's rows per factor kept L2-resident (evict_last)
  int tr;                  // rows per tile (template dispatch)
  int nv;                  // float4 column groups per consumer thread (template dispatch)
  // cross-GPU exchange inside the persistent launch (nranks > 1; lsk_sink_common.cuh):
  // every rank's inbox [2 parity][nranks source][xrs] fp64, mapped over NVLink (peer memory)
  int nranks;
  int rank;
  int xrs;
  double* xbox[kMaxRanks];
  long long xtimeout_ns;   // a peer poll gives up after this long (ST_XERR, no hang)
  int* sticky;             // sticky status word of the (device, stream) (StickyBits)
  int cx;                  // 1: each problem's gpp CTAs are one thread-block cluster and the
                           // pass boundary runs over DSMEM (lsk_sink_common.cuh cx_*)
  // tensor-core exponent kernel (lsk_implicit_tc.cu): per side the packed 3xTF32 B image of
  // the point rows, 8 floats per row ([ph | ph | pl | 1 1 | 0 ..]); NULL = not used
  const float* bimg[2];
  int emul;                // 1: the nprob problems of this launch are the nranks ranks of ONE
                           // row-sharded solve (rank = problem index; xbox[] all on this GPU):
                           // the cross-GPU exchange emulated inside one cooperative launch
  int pingpong;            // implicit kernel, two teams: the teams' feature generations alternate
  int pre;                 // implicit team kernel: generate the next pass's first feature tile
                           // at the pass boundary (0 off, 1 after R2, 2 inside the barrier)
};

// Kernel launchers (lsk_sinkhorn.cu).  Return cudaError_t of the launch.
cudaError_t launch_sinkhorn(const SinkArgs& a, bool cooperative, int grid, size_t smem,
                            cudaStream_t s);
// Kernel configuration for a given r / mode: rows per tile and stage floats.
void sinkhorn_tile_config(int r, int max_stage_bytes, int* tr, int* nv);
size_t sinkhorn_static_smem();
int sinkhorn_max_ctas_per_sm(int nv, int tr, size_t dyn_smem);
// clusters of csize CTAs that can be resident at once (cluster-mode launches)
int sinkhorn_max_active_clusters(int nv, int tr, size_t dyn_smem, int csize);
// bytes of dynamic shared memory the cluster mode appends (partials + totals, fp64)
inline size_t cx_part_bytes(int r) { return 2 * sizeof(double) * (size_t)((r >> 2) + 1) * 4; }

// Implicit (recompute) kernel (lsk_implicit.cu): teams of recompute threads (per-team tile
// barrier; optional lag-one pipeline), optional stream warps (hybrid, LSK_HYB).
struct ImplCfg {
  int ts, teams, nv, tr, pipe;
  int warp;   // 1: warp-private kernel (lsk_implicit_warp.cu, r <= 1024)
};
ImplCfg implicit_config(int r, int d);
bool implicit_warp_config(int r, int d, int* nwarp, int* nv, int* tr);
cudaError_t launch_implicit_warp(const SinkArgs& a, bool cooperative, int grid, cudaStream_t s,
                                 int* occ);
cudaError_t launch_implicit(const SinkArgs& a, bool cooperative, int grid, cudaStream_t s);
int implicit_max_ctas_per_sm(const SinkArgs& a);
// warp-specialised hybrid (lsk_hybrid.cu): two recompute teams + one stream team per CTA
bool hybrid_supported(const SinkArgs& a);
size_t hybrid_smem(int r, int d);
cudaError_t launch_hybrid_ws(const SinkArgs& a, int grid, cudaStream_t s);
// tensor-core exponent kernel (lsk_implicit_tc.cu): r <= 1024, d <= 2, factored exponent,
// one problem over >= 2 CTAs (no cluster / multi-launch / emulation / hybrid)
bool itc_supported(const SinkArgs& a);
size_t itc_image_floats(int64_t rows);
cudaError_t launch_itc_image(const float* X, int64_t n, int d, float* img, cudaStream_t s);
cudaError_t launch_itc(const SinkArgs& a, int grid, cudaStream_t s);
// stabilised implicit mode: per-row shifts m_j (fp32) and fp64 log offsets A_j (reading C30)
cudaError_t launch_row_shift(const float* X, int64_t n, int d, const float* Wt,
                             const float* beta2, int r, float c2, float* m2, double* A,
                             cudaStream_t s);
// h_j = 2^(c2 |p_j|^2 - abar) for the factored exponent (one launch per solve and side)
cudaError_t launch_row_scale(const float* X, int64_t n, int d, float c2, float abar, float* h,
                             cudaStream_t s);

// Resident small-problem kernel (lsk_resident.cu): both factors in the shared memory of one
// cluster of G <= 8 CTAs per problem; resident_cluster returns 0 when they do not fit
size_t resident_smem_bytes(int r, int64_t n, int64_t m, int G);
int resident_cluster(int r, int64_t n, int64_t m);
cudaError_t launch_resident(const SinkArgs& a, int G, int batch, cudaStream_t s);

// Feature kernels (lsk_features.cu)
cudaError_t launch_max_sqnorm(const float* X, int64_t n, int d, unsigned long long* out,
                              cudaStream_t s);
cudaError_t launch_anchors(uint64_t seed, int r, int d, double sigma, float* U,
                           uint32_t* words, cudaStream_t s);
cudaError_t launch_anchor_prep(const float* U, int r, int d, double eps, double q,
                               double log_scale, float* Wt, float* beta2, float* betaD,
                               cudaStream_t s);
cudaError_t launch_feature_map(const float* X, int64_t n, int d, const float* U,
                               const float* Wt, const float* beta2, const float* betaD, int r,
                               double eps, float* Xi, cudaStream_t s);
// tcgen05 3xTF32 feature map (lsk_features_tc.cu), used for d > 16
size_t feature_map_tc_image_bytes(int r, int d);
// R > 0 (the Gaussian map with a max-norm bound, d <= 128): 3xFP16 operands (kind::f16)
cudaError_t launch_feature_map_tc(const float* X, int64_t n, int d, const float* U,
                                  const float* beta2, int r, double eps, float* wimg, float* Xi,
                                  cudaStream_t s, int mode = 0, int sdeg = 0, int ld = 0,
                                  double R = 0.0);
// arc-cosine features (NEXT f3)
cudaError_t launch_arccos_coef(const float* U, int r, int d, double sigma, float* coef,
                               cudaStream_t s);
cudaError_t launch_feature_map_arccos(const float* X, int64_t n, int d, const float* U,
                                      const float* coef, int r, int sdeg, double kappa,
                                      float* Xi, cudaStream_t s);
cudaError_t launch_const_cols(float* Xi, int64_t n, int ld, int col, float val, cudaStream_t s);
// envelope gradients (lsk_grad.cu)
size_t grad_workspace_bytes(int r, int d);
cudaError_t launch_gradients(const float* X, int64_t n, const float* Y, int64_t m, int d,
                             const float* U, int r, double q, const float* Xi, const float* Zeta,
                             const float* u, const float* v, float* gX, float* gY, float* gU,
                             double* ws, cudaStream_t s);
cudaError_t launch_rot_value(const float* u, const float* v, const float* a, const float* b,
                             int64_t n, int64_t m, int batch, double* partials, double* out2,
                             cudaStream_t s, const double* offA = nullptr,
                             const double* offB = nullptr);
// stabilised feature map (NEXT f4, reading C30), d <= 16
cudaError_t launch_feature_map_stab(const float* X, int64_t n, int d, const float* U,
                                    const float* betaD, int r, double eps, float* Xi,
                                    double* logoff, cudaStream_t s);

// accelerated Sinkhorn (lsk_accel.cu): fp64 device vectors of the line search
enum AccelScalar {   // device scalar block, read by the host once per trial
  SC_M1 = 0, SC_M2, SC_S1, SC_S2, SC_LA, SC_LB, SC_BAD, SC_N1, SC_N2, SC_BLK, SC_E, SC_EW,
  SC_PERR, SC_COUNT
};
struct AccelVecs {
  int64_t n, m;
  double *an, *bn;                       // simplex weights
  double *eta1, *zet1, *lam1, *p1, *t1;  // n
  double *eta2, *zet2, *lam2, *p2, *t2;  // m
  double *etan;                          // max(n, m): the moved block's minimiser
  double *part;                          // per-CTA partials (>= 6 * accel_grid())
  double *scal;                          // [SC_COUNT]
  unsigned int* ticket;                  // last-CTA counter (zero between launches)
  double* ctl;                           // device line-search state [CT_COUNT] (graph-driven
                                         // solve; NULL: the host drives the line search)
};
// device line-search state of the graph-driven accelerated solve (lsk_accel.cu)
enum AccelCtl {
  CT_AK = 0, CT_LK, CT_L1, CT_A1, CT_TAU, CT_IT, CT_TRIALS, CT_F, CT_ERR, CT_CONV, CT_PHI,
  CT_ACC, CT_AKP, CT_AK1, CT_BLK, CT_PERR, CT_COUNT
};
// The whole accelerated solve as ONE CUDA graph launch: a while-node over iterations whose
// body holds a while-node over line-search trials; the accept / double-L decision, the
// iteration count and the tolerance test run on the device (cudaGraphSetConditional), so the
// host synchronises once per solve instead of once per trial.  v.ctl must be initialised
// (CT_AK = 0, CT_LK = L0, the rest 0).  Traces (nullable) are device arrays of max_iters.
cudaError_t accel_solve_graph(const AccelVecs& v, const float* Xi, int64_t n, const float* Zeta,
                              int64_t m, int r, double* partA, double* partB, double eps,
                              int max_iters, double tol, double* Ftr, double* Ltr, int* Btr,
                              cudaStream_t s);
int accel_grid();
int accel_pass_grid();
cudaError_t launch_accel_normalise(const float* a, const float* b, const AccelVecs& v,
                                   cudaStream_t s);
cudaError_t launch_accel_lambda(double tau, const AccelVecs& v, cudaStream_t s);
cudaError_t launch_accel_pass(const float* F, int64_t rows, int r, const double* s_in,
                              const double* lam, const double* Mp, double* t_out, double* part,
                              cudaStream_t s);
// phase 1, 2, 3: statistics of the trial; phase 4: the accepted step
cudaError_t launch_accel_stats(int phase, const AccelVecs& v, double a1, double Ak, double Ak1,
                               cudaStream_t s);

// Launch counter (host, thread-local) used for the bench's gpu_launches claim.
void count_launch(int k = 1);

}  // namespace lsk
