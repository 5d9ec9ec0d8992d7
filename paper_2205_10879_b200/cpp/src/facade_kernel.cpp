// C++ facade: kernel.hpp over the C ABI (values computed on the GPU).
#include <cmath>
#include <stdexcept>

#include "facade_common.hpp"
#include "fastmuygps/kernel.hpp"

namespace fastmuygps {

KernelParams::KernelParams(double sigma, double rho, double nu, double tau) : sigma_(sigma), rho_(rho), nu_(nu), tau_(tau) {
  const auto positive = [](double v) { return std::isfinite(v) && v > 0.0; };
  if (!positive(sigma)) throw std::domain_error("KernelParams: sigma must be positive and finite");
  if (!positive(rho)) throw std::domain_error("KernelParams: rho must be positive and finite");
  if (!positive(nu)) throw std::domain_error("KernelParams: nu must be positive and finite");
  if (!(std::isfinite(tau) && tau >= 0.0)) throw std::domain_error("KernelParams: tau must be non-negative and finite");
}

double kernel_value(double d, KernelKind kind, const KernelParams& p) {
  const fmgp_kernel_params kp = detail::abi_params(kind, p);
  double out = 0.0;
  detail::check(fmgp_kernel_values(&d, 1, &kp, &out));
  return out;
}

double matern_value(double d, const KernelParams& p) { return kernel_value(d, KernelKind::Matern, p); }
double rbf_value(double d, const KernelParams& p) { return kernel_value(d, KernelKind::RBF, p); }

Eigen::MatrixXd cov_matrix(const Eigen::MatrixXd& A, const Eigen::MatrixXd& B, KernelKind kind, const KernelParams& p) {
  if (A.cols() != B.cols()) throw std::domain_error("cov_matrix: point sets have mismatched dimension");
  const fmgp_kernel_params kp = detail::abi_params(kind, p);
  const auto a = detail::row_major(A);
  const auto b = detail::row_major(B);
  std::vector<double> K(static_cast<std::size_t>(A.rows() * B.rows()));
  if (A.rows() > 0 && B.rows() > 0)
    detail::check(fmgp_cov_matrix(a.data(), A.rows(), b.data(), B.rows(), static_cast<int32_t>(A.cols()), &kp, K.data()));
  return detail::from_row_major(K.data(), A.rows(), B.rows());
}

Eigen::MatrixXd cov_matrix_self(const Eigen::MatrixXd& A, KernelKind kind, const KernelParams& p) {
  const fmgp_kernel_params kp = detail::abi_params(kind, p);
  const auto a = detail::row_major(A);
  std::vector<double> K(static_cast<std::size_t>(A.rows() * A.rows()));
  if (A.rows() > 0)
    detail::check(fmgp_cov_matrix(a.data(), A.rows(), nullptr, 0, static_cast<int32_t>(A.cols()), &kp, K.data()));
  return detail::from_row_major(K.data(), A.rows(), A.rows());
}

}  // namespace fastmuygps
