// C++ facade: linalg.hpp over the C ABI (fmgp_solve_spd_batched).
#include <string>

#include "facade_common.hpp"
#include "fastmuygps/linalg.hpp"

namespace fastmuygps {

namespace {

// Solve on the GPU; returns the rung used. Throws NumericError naming context.
double gpu_solve(const Eigen::MatrixXd& K, const Eigen::MatrixXd& B, std::string_view context, Eigen::MatrixXd* X) {
  if (K.rows() != K.cols() || B.rows() != K.rows()) throw std::domain_error("solve_spd: shape mismatch");
  const auto k = static_cast<int32_t>(K.rows());
  const auto m = static_cast<int32_t>(B.cols());
  const auto kr = detail::row_major(K);
  const auto br = detail::row_major(B);
  std::vector<double> xr(br.size());
  double jitter = 0.0;
  int64_t failed = -1;
  const int rc = fmgp_solve_spd_batched(kr.data(), br.data(), 1, k, m, xr.data(), &jitter, &failed);
  if (rc == FMGP_ENUMERIC)
    throw NumericError("Cholesky factorization failed in " + std::string(context) + " after jitter escalation up to 1e-6");
  detail::check(rc);
  if (X != nullptr) *X = detail::from_row_major(xr.data(), k, m);
  return jitter;
}

}  // namespace

Eigen::MatrixXd solve_spd(const Eigen::MatrixXd& K, const Eigen::MatrixXd& B, std::string_view context) {
  Eigen::MatrixXd X;
  gpu_solve(K, B, context, &X);
  return X;
}

Eigen::LLT<Eigen::MatrixXd> cholesky_with_jitter(Eigen::MatrixXd K, std::string_view context, double* applied_jitter) {
  Eigen::MatrixXd B(K.rows(), 1);
  for (Eigen::Index i = 0; i < K.rows(); ++i) B(i, 0) = 1.0;
  const double rung = gpu_solve(K, B, context, nullptr);
  // Re-apply the ladder to the diagonal exactly as the reference does
  // (cumulative `+= jitter - previous`), then form the factor object.
  const double ladder[4] = {0.0, 1e-10, 1e-8, 1e-6};
  double previous = 0.0;
  for (double j : ladder) {
    if (j > rung) break;
    if (j > 0.0) {
      K.diagonal().array() += j - previous;
      previous = j;
    }
  }
  if (applied_jitter != nullptr) *applied_jitter = rung;
  return Eigen::LLT<Eigen::MatrixXd>(K);
}

}  // namespace fastmuygps
