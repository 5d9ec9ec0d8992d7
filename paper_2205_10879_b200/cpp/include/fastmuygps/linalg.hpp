// Drop-in facade (B200): jitter-guarded SPD solves of the FastMuyGPs API.
// Public surface of proj/core/include/fastmuygps/linalg.hpp.
#pragma once

#include <Eigen/Dense>
#include <string_view>

namespace fastmuygps {

// Lower Cholesky factor of K under the jitter ladder {0, 1e-10, 1e-8, 1e-6}
// (added to the diagonal). The rung is decided on the GPU
// (fmgp_solve_spd_batched); the returned Eigen object is then formed from
// K + rung * I on the host. Throws NumericError naming `context` when every
// rung fails; *applied_jitter receives the rung used.
Eigen::LLT<Eigen::MatrixXd> cholesky_with_jitter(Eigen::MatrixXd K, std::string_view context,
                                                 double* applied_jitter = nullptr);

// K X = B on the GPU under the same ladder (one warp-level fused factor and
// solve per call).
Eigen::MatrixXd solve_spd(const Eigen::MatrixXd& K, const Eigen::MatrixXd& B, std::string_view context);

}  // namespace fastmuygps
