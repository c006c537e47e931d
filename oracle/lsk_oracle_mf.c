/* ORACLE — matrix-free fp64 application of the Gaussian positive-feature factors.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/lsk_oracle.py): only tests/, __graft_entry__ and
 * bench.py's cpu_baseline may load it.  It shares no code, header or constant with the CUDA
 * path (paper_2006_07057_b200/csrc) and includes nothing from it.
 *
 * Used where the fp64 factors do not fit in host memory (config 5: n = m = 2^23, r = 4096 —
 * 550 GB as fp64): every entry is regenerated in each product, in the direct difference form
 * of the appendix feature map (1/sqrt(r) from PAPER.md:297), paper layout
 * (xi is r x n):
 *     xi[k][i] = exp( -(2/eps) sum_c (x_ic - u_kc)^2 + |u_k|^2/(eps q) + (d/4) ln(2q) - (1/2) ln r )
 * Two products, each a plain sum in fp64:
 *     lsk_mf_apply   s_k = sum_i xi[k][i] w_i     (xi w,      r outputs)
 *     lsk_mf_apply_t t_i = sum_k xi[k][i] s_k     (xi^T s,    n outputs)
 * so K^T u = zeta^T (xi u) and K v = xi^T (zeta v) (K_theta = xi^T zeta).
 * Alg. 1 itself runs in oracle/matrix_free.py.
 *
 * Parallelism: OpenMP over rows.  lsk_mf_apply gives thread t the fixed row block
 * [t n / T, (t+1) n / T) and adds the T partial r-vectors in thread order, so the result
 * depends only on the thread count.  exp is glibc's (vectorised through libmvec when the
 * compiler maps the loop to its SIMD variant; <= 4 ulp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#pragma omp declare simd notinbranch
double exp(double);

/* per-anchor constant |u_k|^2/(eps q) + (d/4) ln(2q) - (1/2) ln r  */
static void anchor_const(const double* U, int r, int d, double eps, double q, double* beta) {
  const double log_scale = 0.25 * d * log(2.0 * q) - 0.5 * log((double)r);
  for (int k = 0; k < r; ++k) {
    double uu = 0.0;
    for (int c = 0; c < d; ++c) uu += U[(int64_t)k * d + c] * U[(int64_t)k * d + c];
    beta[k] = uu / (eps * q) + log_scale;
  }
}

/* the r entries xi[.][i] of one point x (length d) into col[r]; Ut is U transposed (d x r) */
static void point_features(const double* x, const double* Ut, const double* beta, int r, int d,
                           double c2, double* col) {
  /* col_k = sum_c (x_c - u_kc)^2, coordinate by coordinate (contiguous in k) */
  for (int k = 0; k < r; ++k) col[k] = 0.0;
  for (int c = 0; c < d; ++c) {
    const double xc = x[c];
    const double* uc = Ut + (int64_t)c * r;
#pragma omp simd
    for (int k = 0; k < r; ++k) {
      const double df = xc - uc[k];
      col[k] += df * df;
    }
  }
#pragma omp simd
  for (int k = 0; k < r; ++k) col[k] = exp(c2 * col[k] + beta[k]);
}

static double* transpose(const double* U, int r, int d) {
  double* Ut = (double*)malloc(sizeof(double) * (size_t)r * d);
  for (int k = 0; k < r; ++k)
    for (int c = 0; c < d; ++c) Ut[(int64_t)c * r + k] = U[(int64_t)k * d + c];
  return Ut;
}

/* s_k = sum_i xi[k][i] w_i   (P: np x d points, U: r x d anchors, fp64) */
void lsk_mf_apply(const double* P, int64_t np, const double* U, int r, int d, double eps,
                  double q, const double* w, double* s) {
  double* beta = (double*)malloc(sizeof(double) * r);
  anchor_const(U, r, d, eps, q, beta);
  double* Ut = transpose(U, r, d);
  const double c2 = -2.0 / eps;
  const int T = omp_get_max_threads();
  double* part = (double*)calloc((size_t)T * r, sizeof(double));
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    const int64_t i0 = np * t / T, i1 = np * (t + 1) / T;
    double* col = (double*)malloc(sizeof(double) * r);
    double* acc = part + (int64_t)t * r;
    for (int64_t i = i0; i < i1; ++i) {
      point_features(P + i * d, Ut, beta, r, d, c2, col);
      const double wi = w[i];
#pragma omp simd
      for (int k = 0; k < r; ++k) acc[k] += col[k] * wi;
    }
    free(col);
  }
  for (int k = 0; k < r; ++k) {
    double v = 0.0;
    for (int t = 0; t < T; ++t) v += part[(int64_t)t * r + k];
    s[k] = v;
  }
  free(part);
  free(Ut);
  free(beta);
}

/* t_i = sum_k xi[k][i] s_k */
void lsk_mf_apply_t(const double* P, int64_t np, const double* U, int r, int d, double eps,
                    double q, const double* s, double* out) {
  double* beta = (double*)malloc(sizeof(double) * r);
  anchor_const(U, r, d, eps, q, beta);
  double* Ut = transpose(U, r, d);
  const double c2 = -2.0 / eps;
#pragma omp parallel
  {
    double* col = (double*)malloc(sizeof(double) * r);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < np; ++i) {
      point_features(P + i * d, Ut, beta, r, d, c2, col);
      double v = 0.0;
#pragma omp simd reduction(+ : v)
      for (int k = 0; k < r; ++k) v += col[k] * s[k];
      out[i] = v;
    }
    free(col);
  }
  free(Ut);
  free(beta);
}

/* One half-iteration of Alg. 1 over the points P of one side, with the product
 * the next half-iteration needs, each regenerated entry used by both sums that contain it:
 *     t_i = sum_k xi[k][i] s_k,   out_i = c_i / t_i,   s_next_k = sum_i xi[k][i] out_i.
 * With (P, s, c) = (Y, xi u, b) this is  v <- b / K^T u  and s_next = zeta v;  with
 * (X, zeta v, a) it is  u <- a / K v  and s_next = xi u.  t (np, nullable) receives the t_i.
 * Every sum is the same fp64 sum as in lsk_mf_apply / lsk_mf_apply_t (same blocks, same
 * order); only the entries are not generated twice. */
void lsk_mf_half(const double* P, int64_t np, const double* U, int r, int d, double eps,
                 double q, const double* s, const double* c, double* out, double* t_out,
                 double* s_next) {
  double* beta = (double*)malloc(sizeof(double) * r);
  anchor_const(U, r, d, eps, q, beta);
  double* Ut = transpose(U, r, d);
  const double c2 = -2.0 / eps;
  const int T = omp_get_max_threads();
  double* part = (double*)calloc((size_t)T * r, sizeof(double));
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    const int64_t i0 = np * t / T, i1 = np * (t + 1) / T;
    double* col = (double*)malloc(sizeof(double) * r);
    double* acc = part + (int64_t)t * r;
    for (int64_t i = i0; i < i1; ++i) {
      point_features(P + i * d, Ut, beta, r, d, c2, col);
      double ti = 0.0;
#pragma omp simd reduction(+ : ti)
      for (int k = 0; k < r; ++k) ti += col[k] * s[k];
      const double oi = c[i] / ti;
      out[i] = oi;
      if (t_out) t_out[i] = ti;
#pragma omp simd
      for (int k = 0; k < r; ++k) acc[k] += col[k] * oi;
    }
    free(col);
  }
  for (int k = 0; k < r; ++k) {
    double v = 0.0;
    for (int t = 0; t < T; ++t) v += part[(int64_t)t * r + k];
    s_next[k] = v;
  }
  free(part);
  free(Ut);
  free(beta);
}

int lsk_mf_threads(void) { return omp_get_max_threads(); }
