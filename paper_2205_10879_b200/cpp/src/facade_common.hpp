// Shared helpers of the C++ facade: Eigen <-> row-major buffers and the
// C-ABI status -> reference-exception mapping.
#pragma once

#include <Eigen/Dense>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/fmgp_b200.h"
#include "fastmuygps/errors.hpp"
#include "fastmuygps/kernel.hpp"

namespace fastmuygps::detail {

inline std::vector<double> row_major(const Eigen::MatrixXd& A) {
  std::vector<double> out(static_cast<std::size_t>(A.rows() * A.cols()));
  for (Eigen::Index i = 0; i < A.rows(); ++i)
    for (Eigen::Index j = 0; j < A.cols(); ++j) out[static_cast<std::size_t>(i * A.cols() + j)] = A(i, j);
  return out;
}

inline Eigen::MatrixXd from_row_major(const double* p, Eigen::Index rows, Eigen::Index cols) {
  Eigen::MatrixXd A(rows, cols);
  for (Eigen::Index i = 0; i < rows; ++i)
    for (Eigen::Index j = 0; j < cols; ++j) A(i, j) = p[i * cols + j];
  return A;
}

inline fmgp_kernel_params abi_params(KernelKind kind, const KernelParams& p) {
  return fmgp_kernel_params{kind == KernelKind::RBF ? FMGP_RBF : FMGP_MATERN, p.sigma(), p.rho(), p.nu(), p.tau()};
}

// Status codes of include/fmgp_b200.h -> the reference's exception types.
[[noreturn]] inline void raise(int rc) {
  std::string msg = fmgp_last_error();
  if (rc == FMGP_EINVAL) throw std::domain_error(msg);
  if (rc == FMGP_ENUMERIC) throw NumericError(msg);
  throw std::runtime_error("FastMuyGPs B200: " + msg);
}

inline void check(int rc) {
  if (rc != FMGP_OK) raise(rc);
}

}  // namespace fastmuygps::detail
