/* ORACLE TEST INFRASTRUCTURE — CPU restatement of the reference hot path.
 * Checker only: see fmgp_oracle.h. Every function cites the reference
 * file:line (relative to /root/reference/proj) it restates.
 *
 * Built with -ffp-contract=off so the neighbour key stays the exact,
 * FMA-free sequential sum of nn_index.cpp:73-81. */
#include "fmgp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* nn_index.cpp:73-81 — s = 0; s += (a_t - b_t)^2, t ascending. */
double fmgp_oracle_dist_sq(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int t = 0; t < d; ++t) {
    double diff = a[t] - b[t];
    s += diff * diff;
  }
  return s;
}

/* kernel.cpp:55-90. The nugget sigma^2 tau^2 fires only at d == 0 exactly
 * (:58-60, :81-83). General nu (GSL lnKnu, :40-51) is not restated: no
 * BASELINE config uses it; the oracle returns NaN there. */
double fmgp_oracle_kernel_value(double dist, int kind, double sigma, double rho,
                                double nu, double tau) {
  double s2 = sigma * sigma;
  if (dist == 0.0) return s2 * (1.0 + tau * tau);
  if (kind == 1) { /* rbf_value :78-86 */
    double u = dist / rho;
    return s2 * exp(-0.5 * u * u);
  }
  double bracket;
  if (nu == 0.5) {
    bracket = exp(-dist / rho);
  } else if (nu == 1.5) {
    double a = sqrt(3.0) * dist / rho;
    bracket = (1.0 + a) * exp(-a);
  } else if (nu == 2.5) {
    double a = sqrt(5.0) * dist / rho;
    bracket = (1.0 + a + a * a / 3.0) * exp(-a);
  } else {
    return NAN;
  }
  return s2 * bracket;
}

/* (dist_sq, idx) lexicographic order: std::pair<double,int> comparison used by
 * the reference's heap (nn_index.cpp:275-281) and min (:363). */
static int pair_less(double da, int32_t ia, double db, int32_t ib) {
  return da < db || (!(db < da) && ia < ib);
}

/* nn_index.cpp:254-287, :334-341 — Exact query_knn: scan i != exclude,
 * keep the k smallest (dist_sq, i), output ascending. A sorted insertion
 * list keeps exactly the set the size-k max-heap keeps. */
int fmgp_oracle_query_knn(const double* X, int64_t n, int d, const double* q,
                          int k, int64_t exclude, int32_t* idx_out,
                          double* dsq_out) {
  int64_t available = n - (exclude >= 0 ? 1 : 0);
  if (k < 1 || k > available) return -1; /* std::domain_error :261-263 */
  int cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i == exclude) continue;
    double di = fmgp_oracle_dist_sq(q, X + i * d, d);
    int32_t ii = (int32_t)i;
    if (cnt == k && !pair_less(di, ii, dsq_out[k - 1], idx_out[k - 1])) continue;
    int pos = cnt < k ? cnt : k - 1;
    while (pos > 0 && pair_less(di, ii, dsq_out[pos - 1], idx_out[pos - 1])) {
      dsq_out[pos] = dsq_out[pos - 1];
      idx_out[pos] = idx_out[pos - 1];
      --pos;
    }
    dsq_out[pos] = di;
    idx_out[pos] = ii;
    if (cnt < k) ++cnt;
  }
  return 0;
}

/* nn_index.cpp:351-366 — min over (dist_sq, i) from (inf, -1). */
int32_t fmgp_oracle_nearest(const double* X, int64_t n, int d,
                            const double* q) {
  double bd = INFINITY;
  int32_t bi = -1;
  for (int64_t i = 0; i < n; ++i) {
    double di = fmgp_oracle_dist_sq(q, X + i * d, d);
    if (pair_less(di, (int32_t)i, bd, bi)) {
      bd = di;
      bi = (int32_t)i;
    }
  }
  return bi;
}

/* kernel.cpp:106-119 — symmetric fill; diagonal kernel_value(0); off-diagonal
 * kernel_value(||xs_i - xs_j||) (Eigen row-difference norm = sqrt of the sum
 * of squares). K_out is k*k row-major. */
void fmgp_oracle_cov_self(const double* xs, int k, int d, int kind,
                          double sigma, double rho, double nu, double tau,
                          double* K_out) {
  for (int i = 0; i < k; ++i) {
    K_out[i * k + i] = fmgp_oracle_kernel_value(0.0, kind, sigma, rho, nu, tau);
    for (int j = i + 1; j < k; ++j) {
      double dist = sqrt(fmgp_oracle_dist_sq(xs + i * d, xs + j * d, d));
      double v = fmgp_oracle_kernel_value(dist, kind, sigma, rho, nu, tau);
      K_out[i * k + j] = v;
      K_out[j * k + i] = v;
    }
  }
}

/* Eigen::LLT semantics (linalg.cpp:20-21): factor the lower triangle, fail at
 * the first pivot a_kk - sum_j L_kj^2 <= 0. In place, L in the lower
 * triangle of the row-major K. */
static int llt_inplace(double* A, int k) {
  for (int j = 0; j < k; ++j) {
    double x = A[j * k + j];
    for (int p = 0; p < j; ++p) x -= A[j * k + p] * A[j * k + p];
    if (!(x > 0.0)) return -1;
    double ljj = sqrt(x);
    A[j * k + j] = ljj;
    for (int i = j + 1; i < k; ++i) {
      double s = A[i * k + j];
      for (int p = 0; p < j; ++p) s -= A[i * k + p] * A[j * k + p];
      A[i * k + j] = s / ljj;
    }
  }
  return 0;
}

/* linalg.cpp:10-31 — jitter ladder {0, 1e-10, 1e-8, 1e-6}, applied as
 * incremental diagonal additions (jitter - previous, :14-18) to a copy that
 * accumulates across attempts. On success K holds L; returns -1 after the
 * last rung fails (NumericError, :28-30). */
int fmgp_oracle_cholesky_jitter(double* K, int k, double* applied_jitter) {
  static const double kJitters[4] = {0.0, 1e-10, 1e-8, 1e-6};
  double* work = (double*)malloc(sizeof(double) * (size_t)k * (size_t)k);
  double previous = 0.0;
  int rc = -1;
  for (int a = 0; a < 4; ++a) {
    double jitter = kJitters[a];
    if (jitter > 0.0) {
      for (int i = 0; i < k; ++i) K[i * k + i] += jitter - previous;
      previous = jitter;
    }
    memcpy(work, K, sizeof(double) * (size_t)k * (size_t)k);
    if (llt_inplace(work, k) == 0) {
      memcpy(K, work, sizeof(double) * (size_t)k * (size_t)k);
      if (applied_jitter) *applied_jitter = jitter;
      rc = 0;
      break;
    }
  }
  free(work);
  return rc;
}

/* linalg.cpp:33-36 — LLT.solve(B): forward then backward substitution, for
 * each of the m columns of B (k*m row-major, overwritten). */
static void llt_solve(const double* L, int k, double* B, int m) {
  for (int c = 0; c < m; ++c) {
    for (int j = 0; j < k; ++j) {
      double s = B[j * m + c];
      for (int p = 0; p < j; ++p) s -= L[j * k + p] * B[p * m + c];
      B[j * m + c] = s / L[j * k + j];
    }
    for (int j = k - 1; j >= 0; --j) {
      double s = B[j * m + c];
      for (int p = j + 1; p < k; ++p) s -= L[p * k + j] * B[p * m + c];
      B[j * m + c] = s / L[j * k + j];
    }
  }
}

typedef struct {
  const double* X;
  const double* Y;
  int64_t n;
  int d, m, kind, k;
  double sigma, rho, nu, tau;
  const int64_t* rows;
  int64_t begin, end;
  int32_t* S_out;
  double* C_out;
  int64_t failed_row; /* lowest failing row in this chunk, -1 if none */
  int rc;
} rows_job;

/* fast_predict.cpp:86-108 — the per-row body of precompute: S[i,0] = i;
 * S[i,1..] = query_knn(x_i, k-1, exclude=i); gather; cov_matrix_self;
 * solve_spd with context "precompute row i". */
static void* rows_worker(void* arg) {
  rows_job* j = (rows_job*)arg;
  const int k = j->k, d = j->d, m = j->m;
  double* xs = (double*)malloc(sizeof(double) * (size_t)k * (size_t)d);
  double* K = (double*)malloc(sizeof(double) * (size_t)k * (size_t)k);
  double* B = (double*)malloc(sizeof(double) * (size_t)k * (size_t)m);
  double* dsq = (double*)malloc(sizeof(double) * (size_t)k);
  j->failed_row = -1;
  j->rc = 0;
  for (int64_t r = j->begin; r < j->end; ++r) {
    int64_t i = j->rows[r];
    int32_t* S = j->S_out + r * k;
    S[0] = (int32_t)i;
    if (k > 1) {
      if (fmgp_oracle_query_knn(j->X, j->n, d, j->X + i * d, k - 1, i, S + 1, dsq) != 0) {
        j->rc = 1;
        break;
      }
    }
    for (int t = 0; t < k; ++t) {
      memcpy(xs + t * d, j->X + (int64_t)S[t] * d, sizeof(double) * (size_t)d);
      for (int c = 0; c < m; ++c) B[t * m + c] = j->Y[(int64_t)S[t] * m + c];
    }
    fmgp_oracle_cov_self(xs, k, d, j->kind, j->sigma, j->rho, j->nu, j->tau, K);
    if (fmgp_oracle_cholesky_jitter(K, k, NULL) != 0) {
      if (j->failed_row < 0) j->failed_row = i;
      j->rc = 2;
      break; /* threads=1 semantics: the first failing row throws */
    }
    llt_solve(K, k, B, m);
    memcpy(j->C_out + r * k * m, B, sizeof(double) * (size_t)k * (size_t)m);
  }
  free(xs);
  free(K);
  free(B);
  free(dsq);
  return NULL;
}

/* fast_predict.cpp:70-130 on a row subset (rows[0..nrows)), split into
 * contiguous chunks over `threads` like :110-125. Output row r of S/C is for
 * training row rows[r]. Returns 0, 1 (k out of range, :74-76) or 2
 * (NumericError; *failed_row = lowest failing row). */
int fmgp_oracle_precompute_rows(const double* X, const double* Y, int64_t n,
                                int d, int m, int kind, double sigma,
                                double rho, double nu, double tau, int k,
                                const int64_t* rows, int64_t nrows,
                                int threads, int32_t* S_out, double* C_out,
                                int64_t* failed_row) {
  if (k < 1 || k > n) return 1;
  if (threads < 1) threads = 1;
  if (nrows < 2 * threads) threads = 1;
  rows_job* jobs = (rows_job*)calloc((size_t)threads, sizeof(rows_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  int64_t chunk = (nrows + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    rows_job* j = &jobs[w];
    j->X = X; j->Y = Y; j->n = n; j->d = d; j->m = m; j->kind = kind; j->k = k;
    j->sigma = sigma; j->rho = rho; j->nu = nu; j->tau = tau;
    j->rows = rows; j->S_out = S_out; j->C_out = C_out;
    j->begin = w * chunk;
    j->end = j->begin + chunk < nrows ? j->begin + chunk : nrows;
    if (j->begin > nrows) j->begin = nrows;
    if (threads == 1) rows_worker(j);
    else pthread_create(&tids[w], NULL, rows_worker, j);
  }
  int rc = 0;
  int64_t worst = -1;
  for (int w = 0; w < threads; ++w) {
    if (threads > 1) pthread_join(tids[w], NULL);
    if (jobs[w].rc > rc) rc = jobs[w].rc;
    if (jobs[w].failed_row >= 0 && (worst < 0 || jobs[w].failed_row < worst)) worst = jobs[w].failed_row;
  }
  if (failed_row) *failed_row = worst;
  free(jobs);
  free(tids);
  return rc;
}

typedef struct {
  const double* X;
  const int32_t* S;
  const double* C;
  int64_t n;
  int d, k, m, kind;
  double sigma, rho, nu, tau, mean_offset;
  const double* Z;
  int64_t begin, end;
  double* out;
  int32_t* nn_out;
} pred_job;

/* fast_predict.cpp:132-144 — j = nearest_training_point(z);
 * acc = sum_t kernel_value(distance_to(z, S[j,t])) * C[j,t] (sequential);
 * return acc + mean_offset. distance_to = sqrt(dist_sq) (nn_index.cpp:344-349). */
static void* pred_worker(void* arg) {
  pred_job* p = (pred_job*)arg;
  const int d = p->d, k = p->k, m = p->m;
  for (int64_t t = p->begin; t < p->end; ++t) {
    const double* z = p->Z + t * d;
    int32_t j = fmgp_oracle_nearest(p->X, p->n, d, z);
    if (p->nn_out) p->nn_out[t] = j;
    for (int c = 0; c < m; ++c) {
      double acc = 0.0;
      for (int s = 0; s < k; ++s) {
        int32_t nb = p->S[(int64_t)j * k + s];
        double dist = sqrt(fmgp_oracle_dist_sq(z, p->X + (int64_t)nb * d, d));
        acc += fmgp_oracle_kernel_value(dist, p->kind, p->sigma, p->rho, p->nu, p->tau) *
               p->C[((int64_t)j * k + s) * m + c];
      }
      p->out[t * m + c] = acc + p->mean_offset;
    }
  }
  return NULL;
}

/* fast_predict.cpp:146-156 — fast_predict_batch (sequential for threads <= 1;
 * threads > 1 splits rows over fast_predict_one, documented thread-safe at
 * fast_predict.hpp:20-24). */
int fmgp_oracle_predict(const double* X, const int32_t* S, const double* C,
                        int64_t n, int d, int k, int m, int kind, double sigma,
                        double rho, double nu, double tau, double mean_offset,
                        const double* Z, int64_t nz, int threads, double* out,
                        int32_t* nn_out) {
  if (threads < 1) threads = 1;
  if (nz < 2 * threads) threads = 1;
  pred_job* jobs = (pred_job*)calloc((size_t)threads, sizeof(pred_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  int64_t chunk = (nz + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    pred_job* p = &jobs[w];
    p->X = X; p->S = S; p->C = C; p->n = n; p->d = d; p->k = k; p->m = m;
    p->kind = kind; p->sigma = sigma; p->rho = rho; p->nu = nu; p->tau = tau;
    p->mean_offset = mean_offset; p->Z = Z; p->out = out; p->nn_out = nn_out;
    p->begin = w * chunk;
    p->end = p->begin + chunk < nz ? p->begin + chunk : nz;
    if (p->begin > nz) p->begin = nz;
    if (threads == 1) pred_worker(p);
    else pthread_create(&tids[w], NULL, pred_worker, p);
  }
  if (threads > 1)
    for (int w = 0; w < threads; ++w) pthread_join(tids[w], NULL);
  free(jobs);
  free(tids);
  return 0;
}

/* muygps.cpp:32-62 local_prediction for b entries (k-neighbour lists nbr,
 * their distances dist): cross = kernel_value(dist), coeff = solve_spd(
 * cov_matrix_self(X[nbr]), Y[nbr]), pred = cross . coeff (sequential sum).
 * Returns 0, or 2 with *failed_entry = the first failing entry (the
 * reference's sequential loop order). Validation is the caller's job. */
int fmgp_oracle_local_predictions(const double* X, const double* Y, int64_t n,
                                  int d, const int32_t* nbr, const double* dist,
                                  int64_t b, int k, int kind, double sigma,
                                  double rho, double nu, double tau,
                                  double* preds, int64_t* failed_entry) {
  (void)n;
  double* xs = (double*)malloc(sizeof(double) * (size_t)k * (size_t)d);
  double* K = (double*)malloc(sizeof(double) * (size_t)k * (size_t)k);
  double* y = (double*)malloc(sizeof(double) * (size_t)k);
  int rc = 0;
  if (failed_entry) *failed_entry = -1;
  for (int64_t t = 0; t < b && rc == 0; ++t) {
    for (int j = 0; j < k; ++j) {
      const int64_t r = nbr[t * k + j];
      memcpy(xs + (size_t)j * d, X + r * d, sizeof(double) * (size_t)d);
      y[j] = Y[r];
    }
    fmgp_oracle_cov_self(xs, k, d, kind, sigma, rho, nu, tau, K);
    if (fmgp_oracle_cholesky_jitter(K, k, NULL) != 0) {
      if (failed_entry) *failed_entry = t;
      rc = 2;
      break;
    }
    llt_solve(K, k, y, 1);
    double acc = 0.0;
    for (int j = 0; j < k; ++j)
      acc += fmgp_oracle_kernel_value(dist[t * k + j], kind, sigma, rho, nu, tau) * y[j];
    preds[t] = acc;
  }
  free(xs);
  free(K);
  free(y);
  return rc;
}

/* muygps.cpp:272-295: each test point's own k exact neighbours
 * (query_knn, distances sqrt(dist_sq)), then local_prediction's arithmetic
 * + mean_offset. Returns 0 or 2 (*failed_row = first failing test point). */
int fmgp_oracle_muygps_predict(const double* X, const double* Y, int64_t n,
                               int d, double mean_offset, const double* Z,
                               int64_t nz, int k, int kind, double sigma,
                               double rho, double nu, double tau, double* out,
                               int64_t* failed_row) {
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  double* ds = (double*)malloc(sizeof(double) * (size_t)k);
  int rc = 0;
  if (failed_row) *failed_row = -1;
  for (int64_t t = 0; t < nz && rc == 0; ++t) {
    fmgp_oracle_query_knn(X, n, d, Z + t * d, k, -1, idx, ds);
    for (int j = 0; j < k; ++j) ds[j] = sqrt(ds[j]);
    int64_t fe = -1;
    if (fmgp_oracle_local_predictions(X, Y, n, d, idx, ds, 1, k, kind, sigma, rho,
                                      nu, tau, out + t, &fe) != 0) {
      if (failed_row) *failed_row = t;
      rc = 2;
      break;
    }
    out[t] += mean_offset;
  }
  free(idx);
  free(ds);
  return rc;
}
