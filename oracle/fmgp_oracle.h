/* ORACLE TEST INFRASTRUCTURE — a CPU restatement of the FastMuyGPs
 * posterior-mean path, used ONLY as the checker by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg. Nothing in the
 * product (paper_2205_10879_b200/) links, loads or calls it.
 *
 * Parity pinned: validated against the reference's own TUs compiled under
 * oracle/_ref (tests/test_oracle_vs_ref.py) and against the golden fixtures in
 * tests/golden/ generated from oracle/_ref by tests/golden/make_golden.py.
 *
 * Layout: all matrices row-major, X n*d, Y n*m, S n*k int32, C n*k*m.
 * kind: 0 = Matern, 1 = RBF (kernel.hpp:7; file tag fast_predict.cpp:179). */
#ifndef FMGP_ORACLE_H
#define FMGP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

double fmgp_oracle_dist_sq(const double* a, const double* b, int d);
double fmgp_oracle_kernel_value(double dist, int kind, double sigma, double rho,
                                double nu, double tau);
int fmgp_oracle_query_knn(const double* X, int64_t n, int d, const double* q,
                          int k, int64_t exclude, int32_t* idx_out,
                          double* dsq_out);
int32_t fmgp_oracle_nearest(const double* X, int64_t n, int d,
                            const double* q);
void fmgp_oracle_cov_self(const double* xs, int k, int d, int kind,
                          double sigma, double rho, double nu, double tau,
                          double* K_out);
int fmgp_oracle_cholesky_jitter(double* K, int k, double* applied_jitter);
int fmgp_oracle_precompute_rows(const double* X, const double* Y, int64_t n,
                                int d, int m, int kind, double sigma,
                                double rho, double nu, double tau, int k,
                                const int64_t* rows, int64_t nrows,
                                int threads, int32_t* S_out, double* C_out,
                                int64_t* failed_row);
int fmgp_oracle_predict(const double* X, const int32_t* S, const double* C,
                        int64_t n, int d, int k, int m, int kind, double sigma,
                        double rho, double nu, double tau, double mean_offset,
                        const double* Z, int64_t nz, int threads, double* out,
                        int32_t* nn_out);

int fmgp_oracle_local_predictions(const double* X, const double* Y, int64_t n,
                                  int d, const int32_t* nbr, const double* dist,
                                  int64_t b, int k, int kind, double sigma,
                                  double rho, double nu, double tau,
                                  double* preds, int64_t* failed_entry);
int fmgp_oracle_muygps_predict(const double* X, const double* Y, int64_t n,
                               int d, double mean_offset, const double* Z,
                               int64_t nz, int k, int kind, double sigma,
                               double rho, double nu, double tau, double* out,
                               int64_t* failed_row);

#ifdef __cplusplus
}
#endif
#endif
