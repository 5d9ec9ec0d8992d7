// Internal launchers shared by the C-ABI translation unit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace fmgp {

struct KParams;

// Process-wide count of kernel launches (fmgp_launch_count).
void note_launches(int n);

// Exact kNN: for each query q in [0, nq) the kk smallest (dist_sq, idx) over
// references [0, np), excluding reference q + self_offset when self_offset >= 0.
// excl_arr (nullable, nq entries) overrides self_offset with a per-query
// excluded index (-1: none). Writes nq rows of width kk (+1 when with_self, prefixed by q + self_offset).
// out_d (optional) receives the kk sorted dist_sq values.
cudaError_t knn_bruteforce(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk,
                           int64_t self_offset, const int32_t* excl_arr, int with_self, int32_t* out,
                           double* out_d, int num_sms, cudaStream_t stream);

size_t solve_smem_per_warp(int k, int d, int m, int* ld, int* dchunk);

cudaError_t fused_solve(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                        int64_t row_begin, int k, const KParams& kp, double* C, int32_t* status,
                        unsigned long long* fail_min, int num_sms, cudaStream_t stream);

cudaError_t predict_gather(const double* X, const int32_t* S, const double* C, int d, int k, int m,
                           const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz,
                           const int32_t* nn, double* out, int num_sms, cudaStream_t stream);

}  // namespace fmgp

namespace fmgp {

// solve_spd on `batch` given k x k matrices (row-major, lower triangle used).
cudaError_t spd_solve_batched(const double* K, const double* B, int64_t batch, int k, int m, double* X,
                              double* jit_out, unsigned long long* fail_min, int num_sms, cudaStream_t stream);

// cov_matrix (B != nullptr) or cov_matrix_self (B == nullptr), kernel.cpp:92-119.
cudaError_t cov_matrix_launch(const double* A, int64_t na, const double* B, int64_t nb, int d, const KParams& kp,
                              double* K, cudaStream_t stream);
cudaError_t kernel_values_launch(const double* dist, int64_t n, const KParams& kp, double* out, cudaStream_t stream);
cudaError_t sqrt_inplace_launch(double* v, int64_t n, cudaStream_t stream);
cudaError_t self_rows_launch(int32_t* S, int64_t nrows, int64_t row_begin, cudaStream_t stream);
cudaError_t nonfinite_count_launch(const double* v, int64_t n, unsigned int* count, int num_sms,
                                   cudaStream_t stream);
// ... and replace them by 0 in place (v is the caller's own device copy).
cudaError_t nonfinite_zero_launch(double* v, int64_t n, unsigned int* count, int num_sms, cudaStream_t stream);
cudaError_t distances_launch(const double* P, int d, const double* q, const int32_t* idx, int64_t cnt, double* out,
                             cudaStream_t stream);

}  // namespace fmgp

namespace fmgp {

// Exact kNN through a uniform cell grid (d <= 3, kk <= 128); same contract as
// knn_bruteforce (excl_arr only with external queries).
// Predict-walk grid of the training points, built once per model handle (d <= 3).
void* predict_grid_cache_build(const double* X, int64_t n, int d, cudaStream_t stream, cudaError_t* err);
void predict_grid_cache_free(void* cache);
// Attach a grid-ordered copy of the model (m = 1, k <= 64) that predict then
// reads in cell order (FMGP_PGRID_PERM=0 disables). Synchronous.
cudaError_t predict_grid_cache_attach(void* cache, const int32_t* S, const double* C, int k, int m,
                                      cudaStream_t stream);
cudaError_t predict_grid_cached(const void* cache, const double* X, const int32_t* S, const double* Cf, int k, int m,
                                const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz,
                                double* out, int32_t* nn_out, int num_sms, cudaStream_t stream);
bool knn_grid_supported(int d, int kk);
// Rows [0, n) of P (d <= 3) in a cell order (a processing order for the fused solve).
cudaError_t spatial_row_order(const double* P, int64_t n, int d, int32_t* order, cudaStream_t stream);
cudaError_t knn_grid(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk, int64_t self_offset,
                     const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                     cudaStream_t stream);

// Precompute's S rows (self first, then kk neighbours) for the block-cyclic
// row set of member r of g (blocks of pc rows dealt round-robin over [0, np)),
// nrows of them, written at their global rows of `out` (np x (kk + 1)).
cudaError_t knn_grid_rows_cyclic(const double* P, int64_t np, int d, int kk, int64_t nrows, int64_t pc, int g, int r,
                                 int32_t* out, int num_sms, cudaStream_t stream);

// Dispatcher used by the C ABI: the grid search where it applies, else brute
// force. FMGP_KNN=brute in the environment forces brute force (A/B checks).
cudaError_t knn_exact(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk, int64_t self_offset,
                      const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                      cudaStream_t stream);

}  // namespace fmgp

namespace fmgp {

// CTA-per-neighbourhood fallbacks with a global-memory workspace (any k).
cudaError_t fused_solve_big(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                            int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                            int num_sms, cudaStream_t stream);
cudaError_t spd_solve_big(const double* K, const double* B, int64_t batch, int k, int m, double* X, double* jit_out,
                          unsigned long long* fail_min, int num_sms, cudaStream_t stream);

}  // namespace fmgp

namespace fmgp {

// FP64 tensor-core (DMMA) blocked variant of fused_solve (k <= 128, m <= 16).
bool fused_solve_tc_supported(int k, int d, int m);
cudaError_t fused_solve_tc(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                           int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                           int num_sms, cudaStream_t stream);

}  // namespace fmgp

namespace fmgp {

// CTA-per-neighbourhood variant of fused_solve for large compile-time k.
bool fused_solve_cta_supported(int k, int d, int m);
cudaError_t fused_solve_cta(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                            int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                            int num_sms, cudaStream_t stream);

// 2-D cyclic right-looking variant for the small-d shapes (d in {2, 3},
// k in {30, 50}, m = 1, closed-form kernels); FMGP_SOLVE_2D=0 turns it off.
bool fused_solve_2d_supported(int k, int d, int m, const KParams& kp);
cudaError_t fused_solve_2d(const double* X, const double* Y, int d, const int32_t* S, int64_t nrows,
                           int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                           int num_sms, cudaStream_t stream, const int32_t* order = nullptr);

// Register-resident-row variant of fused_solve for compile-time shapes.
bool fused_solve_reg_supported(int k, int d, int m);
cudaError_t fused_solve_reg(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                            int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                            int num_sms, cudaStream_t stream, const int32_t* order = nullptr);

}  // namespace fmgp

namespace fmgp {

// Tensor-core exact kNN (d >= 4): tcgen05 fp16 distance GEMM + bounded filter +
// exact fp64 recheck. debug_G (nullable): write D~ of the first 128x256 tile and stop.
bool knn_tc_supported(int d, int kk);
cudaError_t knn_tc(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk, int64_t self_offset,
                   const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                   cudaStream_t stream, float* debug_G);

}  // namespace fmgp

namespace fmgp {

// Fused grid 1-NN + gather-kernel-dot predict for d <= 3.
cudaError_t predict_grid(const double* X, int64_t n, int d, const int32_t* S, const double* Cf, int k, int m,
                         const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz, double* out,
                         int32_t* nn_out, int num_sms, cudaStream_t stream);

}  // namespace fmgp

namespace fmgp {

// DMMA-blocked variant for the small-d shapes (d in {2, 3}, k in {30, 50},
// m = 1, closed-form kernels): the default there; FMGP_SOLVE_DM=0 falls back to the register solve.
bool fused_solve_dm_supported(int k, int d, int m, const KParams& kp);
cudaError_t fused_solve_dm(const double* X, const double* Y, int d, const int32_t* S, int64_t nrows,
                           int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                           int num_sms, cudaStream_t stream, const int32_t* order = nullptr);

}  // namespace fmgp
