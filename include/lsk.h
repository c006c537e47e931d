/*
 * lsk.h — C ABI of the B200 (sm_100a) linear-time Sinkhorn library ("lsk").
 *
 * Method: arXiv 2006.07057, "Linear Time Sinkhorn Divergences using Positive Features".
 * PAPER.md line numbers refer to /root/reference/PAPER.md (full paper = lines 181-1162).
 *
 *   mu = sum_i a_i delta_{x_i},  nu = sum_j b_j delta_{y_j},  eps > 0
 *   phi(x,u) = (2q)^{d/4} exp(-2|x-u|^2/eps) exp(|u|^2/(eps q))
 *   phi_theta(x) = r^{-1/2} (phi(x,u_1), ..., phi(x,u_r)),  u_k ~ N(0, q eps/4 I)
 *
 *   K_theta = xi zeta^T with xi in R_+^{n x r}, zeta in R_+^{m x r}    (
 *             the paper stores xi as r x n, we store its transpose — reading C9)
 *   Alg. 1: u^0 = 1; repeat v <- b / K^T u ; u <- a / K v
 *   W_hat  = eps (a^T log u + b^T log v)
 *
 * Conventions (all entry points):
 *   - Every array argument is a caller-owned, contiguous, row-major DEVICE pointer (e.g.
 *     from a torch CUDA tensor) unless the parameter name ends in _host; fp32 unless noted;
 *     16-byte aligned.  Inputs are never modified.  The library owns only an internal
 *     workspace cached per (device, stream): fp64 CTA partials, r-vectors, barrier
 *     counters, a second v buffer and a result block.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous, EXCEPT: lsk_feature_params_init with R <= 0, any call
 *     given a non-NULL host `lsk_report*`/`double*` result, and lsk_rot_host — these
 *     synchronise `stream` before returning.
 *   - Errors: a negative lsk_status; lsk_last_error() returns a thread-local message.  No
 *     C++ exception crosses the ABI.  On error, outputs are unspecified.
 *   - Asynchronous solve errors (a solve called with rep == NULL does not synchronise): a
 *     zero / non-finite row dot (LSK_EBREAKDOWN), a weight that is not finite and > 0
 *     (LSK_EWEIGHTS) and a cross-GPU exchange timeout (LSK_ENCCL) set a STICKY status of the
 *     (device, stream).  The next synchronising call on that stream that checks it returns the
 *     error and clears it: lsk_stream_status, lsk_rot_value, and any solve given a report.
 *   - Thread safety: calls on different streams may run concurrently; one solve at a time
 *     per (device, stream) workspace.
 */
#ifndef LSK_H
#define LSK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum lsk_status {
  LSK_OK = 0,
  LSK_NOT_CONVERGED = 1,   /* warning: tol > 0 and max_iters reached; outputs valid        */
  LSK_EINVAL = -1,         /* n,m,r,d < 1; eps <= 0; r % 4 != 0; NULL or misaligned pointer */
  LSK_EDIM = -2,           /* unsupported size combination (e.g. d > 16 for implicit)       */
  LSK_EDOMAIN = -3,        /* R given and a point lies outside B(0,R); W0 argument < -1/e   */
  LSK_EWEIGHTS = -4,       /* a weight a_i or b_j is not finite and > 0 (mu, nu are probability
                              measures with positive masses; checked by the
                              solve kernels on every row they read: report or sticky status) */
  LSK_EBREAKDOWN = -5,     /* a row dot K v or K^T u was 0 / inf / nan        */
  LSK_ECUDA = -6,          /* CUDA runtime error (message in lsk_last_error)                 */
  LSK_ENCCL = -7,          /* NCCL error or NCCL library not loadable                       */
  LSK_ENOMEM = -8,         /* workspace allocation failed                                   */
  LSK_EUNSUPPORTED = -9    /* e.g. cooperative launch unavailable                           */
} lsk_status;

/* Gaussian positive-feature parameters (Lemma decomp-RBF).
 *   z = R^2/(eps d), q = z / (2 W_0(z)), sigma = sqrt(q eps / 4),
 *   log_scale = (d/4) ln(2q) - (1/2) ln r.   All fp64, computed on the host. */
typedef struct lsk_feature_params {
  double eps;
  double R;
  double q;
  double sigma;
  double log_scale;
  int32_t d;
  int32_t r;
  uint64_t seed;
} lsk_feature_params;

/* Solve options.  tol <= 0: run exactly max_iters iterations (fixed-T mode).  tol > 0:
 * stop after the first iteration t with |v^t o K^T u^t - b|_1 < tol, at most
 * max_iters.  want_marginal_err (fixed-T mode): also evaluate |v^T o K^T u^T - b|_1 with
 * one extra half pass.  variant (implicit solver only): 0 = auto. */
typedef struct lsk_solve_opts {
  int32_t max_iters;
  int32_t want_marginal_err;
  double tol;
  int32_t ctas_per_sm;     /* 0 = library default                                         */
  int32_t flags;           /* LSK_SOLVE_STABILIZE: implicit solver in the row-normalised form;
                              LSK_SOLVE_NO_RESIDENT: no resident small-problem kernel */
  double stream_fraction;  /* implicit solver only: fraction phi of each side's rows whose
                              factor rows are materialised once and streamed from HBM in every
                              pass while the rest are regenerated on the MUFU (both units busy
                              in one launch).  0 = library default (off: within 1% of the
                              pure recompute kernel on config 2, DESIGN.md §6 K8),
                              < 0 = off (pure recompute),
                              in (0, 0.9] = that fraction.  Applies to r <= 1024, d <= 3, large
                              problems; phi (n + m) r 4 bytes of workspace. */
} lsk_solve_opts;

/* flags of lsk_solve_opts.  LSK_SOLVE_STABILIZE (lsk_factored_sinkhorn_implicit only; reading
 * C30): every row of the regenerated factors is normalised by its largest entry (a per-row
 * shift of the exponent), so no row underflows fp32 at small eps; u, v are then the scalings
 * u~ = u e^A, v~ = v e^B of the normalised problem (lsk_implicit_row_offsets returns A, B) and
 * rep->rot is the value of the original problem (the offsets are folded in). */
#define LSK_SOLVE_STABILIZE 1
/* LSK_SOLVE_NO_RESIDENT: never use the resident small-problem kernel.  By default a
 * single-GPU solve (one problem, or a batch: one cluster per problem) whose factors fit in the
 * shared memory of one thread-block cluster (<= 8 CTAs x 227 KB; r <= 512) keeps both factors on
 * chip for the whole solve (the implicit solvers then materialise them once); this flag forces
 * the persistent grid kernels (same results within the parity tolerances; for tests and
 * measurements). */
#define LSK_SOLVE_NO_RESIDENT 2

/* Report of one solve.  rot = W_hat of the returned (u, v);
 * marginal_err = |v o K^T u - b|_1 of the returned state, or -1 if not evaluated. */
typedef struct lsk_report {
  int32_t iters;
  int32_t converged;
  double marginal_err;
  double rot;
  double sum_a_log_u;      /* a^T log u (fp64)                                            */
  double sum_b_log_v;      /* b^T log v (fp64)                                            */
  int32_t breakdown;       /* 1 if a zero / non-finite row dot was seen                   */
  int32_t reserved;
} lsk_report;

typedef struct lsk_comm lsk_comm;   /* opaque NCCL communicator; NULL = single GPU */

const char* lsk_version(void);
const char* lsk_last_error(void);
/* Synchronises `stream` and returns (then clears) its sticky status: LSK_OK, or the
 * LSK_EBREAKDOWN / LSK_EWEIGHTS / LSK_ENCCL of a report-less solve enqueued on it since the
 * last check (see Conventions). */
lsk_status lsk_stream_status(void* stream);

/* ---- a1: feature parameters (host fp64) --------------------------------------------- */
/* Principal-branch Lambert W_0 ("W_0 is the Lambert function"); Halley
 * iteration from log1p(z).  z < -1/e -> LSK_EDOMAIN.  Host only, no GPU needed. */
lsk_status lsk_lambert_w0(double z, double* w);

/* Fills *out from (eps, d, r, R, seed).  R <= 0: R = max(max_i |x_i|, max_j |y_j|)
 * computed on the device from X (n x d) and Y (m x d) in fp64 (reading C3; synchronises).
 * R > 0: X/Y may be NULL; if given, a point with |p| > R gives LSK_EDOMAIN.
 * With a communicator, the auto-R max is all-reduced across ranks. */
lsk_status lsk_feature_params_init(double eps, int32_t d, int32_t r, double R, uint64_t seed,
                                   const float* X, int64_t n, const float* Y, int64_t m,
                                   lsk_feature_params* out, lsk_comm* comm, void* stream);

/* ---- a2: anchors theta = (u_1..u_r), u_k ~ N(0, sigma^2 I) ---- */
/* U (r x d, fp32, device) = fp32(sigma * z_kc); z from Philox4x32-10 with
 * key = (seed & 0xffffffff, seed >> 32), counter = (k, c/4, 0, 0), fp64 Box-Muller on word
 * pairs (w0,w1) and (w2,w3): z = sqrt(-2 ln((w0+1) 2^-32)) (cos, sin)(2 pi w1 2^-32)
 * (reading C5).  Prefix property: anchor k does not depend on r. */
lsk_status lsk_draw_anchors(const lsk_feature_params* p, float* U, void* stream);
/* Raw generator words, for bit-exact testing: out (device uint32, r x ceil(d/4) x 4). */
lsk_status lsk_philox_words(uint64_t seed, int32_t r, int32_t d, uint32_t* out, void* stream);

/* ---- a3: feature map xi = phi_theta(X) --------------------- */
/* Xi (n x r, fp32, device): Xi[i][k] = exp(-(2/eps)|x_i - U_k|^2 + |U_k|^2/(eps q)
 *   + log_scale).  d <= 16: direct difference form on FFMA; d > 16: expanded form
 * |x|^2 + |U|^2 - 2 x.U with the x.U contraction on the tcgen05 tensor cores in 3xTF32
 * (TMEM accumulators, exp epilogue).  r % 4 == 0. */
lsk_status lsk_feature_map(const lsk_feature_params* p, const float* U, const float* X,
                           int64_t n, float* Xi, void* stream);
/* Batched: X is (batch, n, d), Xi is (batch, n, r); one shared anchor draw (config 4). */
lsk_status lsk_feature_map_batched(const lsk_feature_params* p, const float* U,
                                   const float* X, int64_t n, int32_t batch, float* Xi,
                                   void* stream);

/* NEXT f3: perturbed arc-cosine positive features (Lemma decomp-arccos, PAPER.md:947-989;
 * main text PAPER.md:377-382).  Anchors u_k ~ N(0, sigma^2 I) with sigma = p->sigma > 1
 * (draw them with lsk_draw_anchors on the same p); s_degree in {0,1,2}; kappa > 0.
 * Xi is n x (r+4): Xi[i][k] = sigma^{d/2} sqrt(2) max(0, u_k.x_i)^s
 * exp(-|u_k|^2 (1 - 1/sigma^2)/4) / sqrt(r) for k < r, Xi[i][r] = sqrt(kappa), and
 * Xi[i][r+1..r+3] = 0 — the r kappa slots of phi_theta collapse into one column (same
 * k_theta), padded to a multiple of 4.  Pass r+4 as the rank to the Sinkhorn calls.  Unbiased
 * for k_s + kappa with the main-text k_s (reading C21).  d <= 16: FFMA; d > 16: tcgen05
 * 3xTF32 contraction with a relu^s epilogue. */
lsk_status lsk_feature_map_arccos(const lsk_feature_params* p, int32_t s_degree, double kappa,
                                  const float* U, const float* X, int64_t n, float* Xi,
                                  void* stream);

/* ---- a4-a9: Alg. 1 on K_theta = Xi Zeta^T, streaming the factors from HBM ---------- */
/* One persistent launch runs every iteration: per iteration a zeta-pass
 * (t_j = zeta_j . s_v, v_j = b_j / t_j, s_u += v_j zeta_j) and a xi-pass (mirror), each
 * reading its factor once (4 r (n+m) bytes / iteration); r-vectors reduced in fp64 across
 * CTAs in a fixed order (deterministic).  u^0 = 1 (reading C6).  u (n), v (m) outputs.
 * rep (host, nullable): if non-NULL the call synchronises and fills it.
 * comm: rows are sharded by the caller (n, m, Xi, Zeta, a, b, u, v are LOCAL shards; r and
 * eps global); one fp64 all-reduce of r+4 doubles per half iteration. */
lsk_status lsk_factored_sinkhorn(const float* Xi, int64_t n, const float* Zeta, int64_t m,
                                 int32_t r, const float* a, const float* b, double eps,
                                 const lsk_solve_opts* o, float* u, float* v,
                                 lsk_report* rep, lsk_comm* comm, void* stream);

/* Same iteration, but xi/zeta entries are regenerated in registers from (X, Y, U) in every
 * pass and never stored (MUFU ex2 per entry per pass).  d <= 16. */
lsk_status lsk_factored_sinkhorn_implicit(const lsk_feature_params* p, const float* U,
                                          const float* X, int64_t n, const float* Y,
                                          int64_t m, const float* a, const float* b,
                                          const lsk_solve_opts* o, float* u, float* v,
                                          lsk_report* rep, lsk_comm* comm, void* stream);

/* Batched: `batch` independent problems in ONE persistent launch.  The grid is made of
 * groups of gpp CTAs (gpp chosen from n, r and the SM count; gpp = 1: no cross-CTA exchange,
 * s stays in registers); each group loops over problems group, group + ngroups, ..., and a
 * group with gpp > 1 sums its r-vector through global memory with a group barrier per pass.
 * Xi (batch, n, r), Zeta (batch, m, r), a/u (batch, n), b/v (batch, m);
 * reps: host array of `batch` reports (nullable). */
lsk_status lsk_factored_sinkhorn_batched(const float* Xi, int64_t n, const float* Zeta,
                                         int64_t m, int32_t r, int32_t batch, const float* a,
                                         const float* b, double eps, const lsk_solve_opts* o,
                                         float* u, float* v, lsk_report* reps, void* stream);

/* Batched recompute: `batch` independent problems sharing (p, U), one CTA per problem (the
 * implicit kernel with no grid barrier), the factors regenerated in every pass.  X (batch, n,
 * d), Y (batch, m, d), a/u (batch, n), b/v (batch, m); reps: host array of `batch` reports
 * (nullable).  d <= 8.  Not with LSK_SOLVE_STABILIZE. */
lsk_status lsk_factored_sinkhorn_implicit_batched(const lsk_feature_params* p, const float* U,
                                                  const float* X, int64_t n, const float* Y,
                                                  int64_t m, int32_t batch, const float* a,
                                                  const float* b, const lsk_solve_opts* o,
                                                  float* u, float* v, lsk_report* reps,
                                                  void* stream);

/* ---- a9: read-out W_hat = eps (a^T log u + b^T log v) in fp64 ------- */
/* rot_host: host double (the call synchronises).  With comm, partial sums are all-reduced.
 * Also returns (and clears) the stream's sticky status of an earlier report-less solve. */
lsk_status lsk_rot_value(const float* u, const float* v, const float* a, const float* b,
                         int64_t n, int64_t m, double eps, double* rot_host, lsk_comm* comm,
                         void* stream);
lsk_status lsk_rot_value_batched(const float* u, const float* v, const float* a,
                                 const float* b, int64_t n, int64_t m, int32_t batch,
                                 double eps, double* rots_host, void* stream);

/* ---- NEXT f1: Sinkhorn divergence (eq. reg-sdiv) ------------------- */
/* W_bar(mu,nu) = W(mu,nu) - (W(mu,mu) + W(nu,nu)) / 2, each W the dual estimate of Alg. 1
 * on K_theta with ONE anchor draw shared by the three problems (a single cost c_theta).
 * Three persistent solves with the options o (fixed T or tolerance); out4_host (host, 4
 * doubles) = {W_bar, W_xy, W_xx, W_yy}; reps3 (host, 3 reports, nullable) in the same order
 * (xy, xx, yy).  Scalings are not returned (scratch in the workspace).  Synchronises. */
lsk_status lsk_sinkhorn_divergence(const float* Xi, int64_t n, const float* Zeta, int64_t m,
                                   int32_t r, const float* a, const float* b, double eps,
                                   const lsk_solve_opts* o, double* out4_host,
                                   lsk_report* reps3, void* stream);
lsk_status lsk_sinkhorn_divergence_implicit(const lsk_feature_params* p, const float* U,
                                            const float* X, int64_t n, const float* Y,
                                            int64_t m, const float* a, const float* b,
                                            const lsk_solve_opts* o, double* out4_host,
                                            lsk_report* reps3, void* stream);

/* ---- NEXT f2: envelope gradients (Prop. diff-gene + chain rule) ------ */
/* At the scalings (u, v) of a solve (streaming factors Xi, Zeta of X, Y under anchors U and
 * params p), with theta = U and q fixed: dW/dK = -eps u v^T gives
 *   gX_i = 4 u_i sum_k Xi_ik s_u,k (x_i - U_k),   s_u = Zeta^T v,
 *   gY_j = 4 v_j sum_k Zeta_jk s_v,k (y_j - U_k), s_v = Xi^T u,
 *   gU_k = -4 (s_u,k B_x,k + s_v,k B_y,k) - (4/q) s_u,k s_v,k U_k,
 *          B_x,k = sum_i u_i Xi_ik (x_i - U_k), B_y,k likewise.
 * gX (n x d), gY (m x d), gU (r x d): device fp32, each nullable.  d <= 16 (LSK_EDIM
 * otherwise).  Row sums are fp64 with fixed-order partials.  Asynchronous. */
lsk_status lsk_rot_gradient(const lsk_feature_params* p, const float* U, const float* X,
                            int64_t n, const float* Y, int64_t m, const float* Xi,
                            const float* Zeta, const float* u, const float* v, float* gX,
                            float* gY, float* gU, void* stream);

/* ---- NEXT f4: small-eps stabilisation (reading C30) ------------------------ */
/* The fp64 row offsets A_i = ln max_k xi_ik of the stabilised implicit solver (same arithmetic
 * as inside it): u = u~ e^{-A}.  logoff: device fp64 (n).  d <= 8.  Asynchronous. */
lsk_status lsk_implicit_row_offsets(const lsk_feature_params* p, const float* U, const float* X,
                                    int64_t n, double* logoff, void* stream);
/* Row-normalised Gaussian features: Xi (n x r) = xi / max_k xi_k (every row's largest entry
 * is 1, so no row underflows fp32 at small eps) and logoff (n, fp64) = A_i = ln max_k xi_ik,
 * i.e. xi = diag(e^A) Xi.  Alg. 1 on (Xi_x, Xi_y) returns u~ = u e^A, v~ = v e^B (it starts
 * from u~ = 1, i.e. u = e^{-A}: "any positive vector"), and
 *   W_hat = eps (a^T (log u~ - A) + b^T (log v~ - B))       (lsk_rot_value_offset).
 * d <= 16 (LSK_EDIM otherwise).  Asynchronous. */
lsk_status lsk_feature_map_stabilized(const lsk_feature_params* p, const float* U,
                                      const float* X, int64_t n, float* Xi, double* logoff,
                                      void* stream);
/* W_hat of scalings u (n), v (m) of a row-normalised problem with offsets A (n), B (m) (device
 * fp64).  rot_host: host double; synchronises. */
lsk_status lsk_rot_value_offset(const float* u, const float* v, const float* a, const float* b,
                                const double* A, const double* B, int64_t n, int64_t m,
                                double eps, double* rot_host, void* stream);

/* ---- NEXT f4: accelerated Sinkhorn (Alg. 2) ------------------------- */
/* Maximises the smooth dual (Eq. dual-smooth)
 *   F_theta(eta) = eps [<eta1,a> + <eta2,b> - log <e^{eta1}, K_theta e^{eta2}>]
 * by accelerated alternating minimisation of phi = -F/eps with the adaptive line search
 * L <- L/2, then doubling until phi(eta^{k+1}) <= phi(lambda^k) - |grad phi(lambda^k)|^2/(2L)
 * (readings C22-C28).  K_theta = Xi Zeta^T is streamed from HBM: each trial
 * applies it three times (zeta^T e^{l2}, then xi . and xi^T e^{l1} in one pass, then zeta .).
 * a, b are put on the simplex in fp64 first (C28).  Dual vectors live in fp64; e^{lambda}
 * enters the passes shifted by its maximum (fp32 weights in (0, 1]).
 *   o->max_iters  iterations (accepted steps); o->tol > 0: stop once the averaged plan's
 *                 marginal error |x_hat 1 - a|_1 + |x_hat^T 1 - b|_1 < tol;
 *   o->L0         initial smoothness estimate (> 0; 1 is a good default, phi is 2-smooth).
 * eta1 (n), eta2 (m): device fp64 outputs, the final dual point.  F_trace_host, L_trace_host
 * (host, max_iters doubles) and blk_trace_host (host, max_iters int32, the block 1/2 chosen):
 * per-iteration traces, each nullable.  rep (host, nullable).  Synchronises (the line search
 * reads four scalars per trial).  Returns LSK_NOT_CONVERGED if tol > 0 was not reached. */
typedef struct lsk_accel_opts {
  int32_t max_iters;
  int32_t reserved;
  double tol;
  double L0;
} lsk_accel_opts;

typedef struct lsk_accel_report {
  int32_t iters;        /* accepted iterations                                            */
  int32_t trials;       /* line-search trials (>= iters)                                  */
  int32_t converged;    /* tol > 0 and reached                                            */
  int32_t reserved;
  double F;             /* F_theta(eta) at the returned dual point                         */
  double L;             /* last accepted L                                                 */
  double plan_err;      /* |x_hat 1 - a|_1 + |x_hat^T 1 - b|_1 of the averaged plan        */
} lsk_accel_report;

lsk_status lsk_accelerated_sinkhorn(const float* Xi, int64_t n, const float* Zeta, int64_t m,
                                    int32_t r, const float* a, const float* b, double eps,
                                    const lsk_accel_opts* o, double* eta1, double* eta2,
                                    double* F_trace_host, double* L_trace_host,
                                    int32_t* blk_trace_host, lsk_accel_report* rep,
                                    void* stream);

/* ---- whole path with HOST buffers (end-to-end entry point) ---------------------------- */
/* X_host (n x d), Y_host (m x d), a_host, b_host (host memory, pinned or pageable).  Copies
 * inputs to the device, runs a1-a9 (variant 0 = auto, 1 = streaming, 2 = implicit), copies
 * u, v (nullable) and the report back.  Synchronous. */
lsk_status lsk_rot_host(const float* X_host, int64_t n, const float* Y_host, int64_t m,
                        int32_t d, const float* a_host, const float* b_host, double eps,
                        int32_t r, uint64_t seed, double R, const lsk_solve_opts* o,
                        int32_t variant, float* u_host, float* v_host, lsk_report* rep);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) -------------------------------- */
/* Row shard [begin, end) of `total` rows for `rank` of `nranks` (contiguous, balanced). */
lsk_status lsk_shard_range(int64_t total, int32_t nranks, int32_t rank, int64_t* begin,
                           int64_t* end);
/* 128-byte ncclUniqueId into out_host (rank 0 creates it; broadcast it yourself). */
lsk_status lsk_comm_get_unique_id(void* out_host);
lsk_status lsk_comm_init(lsk_comm** out, int32_t nranks, int32_t rank,
                         const void* unique_id_host, int32_t device);
lsk_status lsk_comm_destroy(lsk_comm* comm);
/* Collective over the communicator's ranks (all must call it): map every rank's fp64 inbox
 * ([2][nranks][~r_max + 6]) into every GPU's address space (CUDA IPC + peer access over
 * NVLink; the handles travel in one NCCL all-gather).  Afterwards single-problem solves with
 * this comm and r <= r_max run as ONE persistent launch per GPU: the per-half-iteration
 * all-rank sum of the fp64 r-vector happens inside the kernel — the owner CTA of a column
 * stores its rank's total into every peer's inbox and adds the N totals in rank order
 * (deterministic, identical on every rank) — instead of one launch plus one ncclAllReduce per
 * pass.  A peer that never arrives makes the solve fail after 20 s with LSK_ENCCL instead of
 * hanging.  LSK_EUNSUPPORTED if peer memory cannot be mapped (the NCCL path stays in use);
 * LSK_P2P=0 in the environment disables the in-kernel exchange.  Synchronises. */
lsk_status lsk_comm_enable_p2p(lsk_comm* comm, int32_t r_max, void* stream);

/* Emulated ranks (testing and timing the multi-GPU exchange on one GPU): the nranks row
 * shards of ONE problem (rank q owns rows [q n/N, (q+1) n/N) of X/Xi/a/u and of Y/Zeta/b/v;
 * n and m divisible by N, 2 <= N <= 8) run as the N problems of one cooperative launch, each
 * rank a group of CTAs with its own fp64 inbox in this GPU's memory, and the per-half-iteration
 * all-rank sum of the r-vector (the only datum the shards share) goes through
 * exactly the in-kernel exchange protocol of lsk_comm_enable_p2p (stores into every rank's
 * inbox, sentinel polls, rank-order sum, re-arm).  u (n), v (m) are the global scalings; reps
 * (host, N reports, nullable): rank q's report — every rank computes the same totals, so the
 * N reports are identical.  Synchronises iff reps != NULL. */
lsk_status lsk_factored_sinkhorn_emulated(int32_t nranks, const float* Xi, int64_t n,
                                          const float* Zeta, int64_t m, int32_t r,
                                          const float* a, const float* b, double eps,
                                          const lsk_solve_opts* o, float* u, float* v,
                                          lsk_report* reps, void* stream);
lsk_status lsk_factored_sinkhorn_implicit_emulated(int32_t nranks, const lsk_feature_params* p,
                                                   const float* U, const float* X, int64_t n,
                                                   const float* Y, int64_t m, const float* a,
                                                   const float* b, const lsk_solve_opts* o,
                                                   float* u, float* v, lsk_report* reps,
                                                   void* stream);

/* Diagnostic: the launch plan a solve of this shape would use on the current device —
 * gpp = CTAs per problem, grid = CTAs of the launch (grid / gpp = persistent groups; a batched
 * solve with batch > grid / gpp loops each group over several problems), cluster (nullable) =
 * 1 if each group is a thread-block cluster whose per-pass r-vector reduction runs over DSMEM
 * (2 <= gpp <= 8, r <= 1024), 0 if it goes through global memory.  variant 1 = factor stream
 * (lsk_factored_sinkhorn[_batched]), 2 = recompute (lsk_factored_sinkhorn_implicit*). */
lsk_status lsk_solve_plan(int64_t n, int64_t m, int32_t r, int32_t d, int32_t batch,
                          int32_t variant, int32_t* gpp, int32_t* grid, int32_t* cluster);

/* Diagnostic: the cluster size G (1, 2, 4 or 8 CTAs) of the resident small-problem kernel for a
 * single-GPU solve of this shape (per problem of a batch) (both factors held in the CTAs' shared memory
 * for the whole solve; DESIGN.md §6 K10), or 0 when the shape runs on the persistent grid
 * kernels (r > 512, or the factors exceed 8 x 227 KB).  LSK_SOLVE_NO_RESIDENT forces the grid
 * kernels; lsk_solve_plan describes those. */
lsk_status lsk_resident_plan(int64_t n, int64_t m, int32_t r, int32_t* ctas);

/* Diagnostic: the rows of each side (ns0 of X, ns1 of Y) that lsk_factored_sinkhorn_implicit
 * with these options materialises and streams from HBM (the warp-specialised hybrid kernel);
 * 0, 0 when it regenerates every row (pure recompute). */
lsk_status lsk_stream_rows(int64_t n, int64_t m, int32_t r, int32_t d, const lsk_solve_opts* o,
                           int64_t* ns0, int64_t* ns1);

/* Number of kernels the library launched on this thread since the last reset (for the
 * bench's gpu_launches claim). */
int64_t lsk_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* LSK_H */
