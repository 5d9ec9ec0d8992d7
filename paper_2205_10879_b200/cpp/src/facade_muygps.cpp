// Facade for muygps.hpp over the C ABI. The loss evaluations, neighbour
// searches and k x k solves run on the GPU; the host keeps what the
// reference keeps sequential for bit-stability (the residual sum in batch
// order, muygps.cpp:70-77) and the batch sampler (muygps.cpp:15-30).
#include <algorithm>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "facade_common.hpp"
#include "fastmuygps/muygps.hpp"

namespace fastmuygps {

BatchSpec BatchSpec::sample(int n, int b, std::uint64_t seed) {
  if (b < 1 || b > n) throw std::domain_error("BatchSpec: batch size out of range");
  std::vector<int> pool(static_cast<std::size_t>(n));
  std::iota(pool.begin(), pool.end(), 0);
  std::mt19937_64 rng(seed);
  for (int i = 0; i < b; ++i) {  // partial Fisher-Yates: the first b are a uniform sample
    std::uniform_int_distribution<int> pick(i, n - 1);
    std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(pick(rng))]);
  }
  pool.resize(static_cast<std::size_t>(b));
  return BatchSpec{b, seed, std::move(pool)};
}

namespace {

std::vector<double> responses(const TrainingSet& t) {
  return std::vector<double>(t.Y.data(), t.Y.data() + t.Y.size());
}

// Entries [0, b) with one common list length: one device call.
std::vector<double> predictions(const TrainingSet& train, const std::vector<int>& batch,
                                const std::vector<NeighborList>& lists, KernelKind kind, const KernelParams& p) {
  const auto b = static_cast<int64_t>(batch.size());
  const auto k = static_cast<int32_t>(lists.empty() ? 0 : lists[0].indices.size());
  std::vector<int32_t> bi(batch.begin(), batch.end());
  std::vector<int32_t> nbr(static_cast<std::size_t>(b * k));
  std::vector<double> dist(static_cast<std::size_t>(b * k));
  for (int64_t t = 0; t < b; ++t) {
    std::copy(lists[t].indices.begin(), lists[t].indices.end(), nbr.begin() + t * k);
    std::copy(lists[t].distances.begin(), lists[t].distances.end(), dist.begin() + t * k);
  }
  const fmgp_kernel_params kp = detail::abi_params(kind, p);
  const auto Y = responses(train);
  std::vector<double> out(static_cast<std::size_t>(std::max<int64_t>(b, 1)));
  int64_t failed = -1;
  detail::check(fmgp_local_predictions(detail::row_major(train.X).data(), Y.data(), train.X.rows(),
                                       static_cast<int32_t>(train.X.cols()), bi.data(), nbr.data(), dist.data(), b, k,
                                       &kp, out.data(), &failed));
  out.resize(static_cast<std::size_t>(b));
  return out;
}

}  // namespace

double local_prediction(const TrainingSet& train, int i, const NeighborList& neighbors, KernelKind kind,
                        const KernelParams& p) {
  if (neighbors.distances.size() < neighbors.indices.size())
    throw std::domain_error("local_prediction: neighbor distances missing");
  return predictions(train, {i}, {neighbors}, kind, p)[0];
}

double loocv_loss(const TrainingSet& train, const BatchSpec& batch, const std::vector<NeighborList>& neighbor_lists,
                  KernelKind kind, const KernelParams& p) {
  if (neighbor_lists.size() != batch.indices.size() || batch.indices.empty())
    throw std::domain_error("loocv_loss: batch and neighbor lists disagree");
  bool uniform = true;
  for (const auto& nl : neighbor_lists) {
    uniform &= nl.indices.size() == neighbor_lists[0].indices.size();
    if (nl.distances.size() < nl.indices.size()) throw std::domain_error("local_prediction: neighbor distances missing");
  }
  std::vector<double> preds;
  if (uniform) {
    preds = predictions(train, batch.indices, neighbor_lists, kind, p);
  } else {  // ragged lists: entry by entry, in batch order (the reference's error order)
    for (std::size_t t = 0; t < batch.indices.size(); ++t)
      preds.push_back(local_prediction(train, batch.indices[t], neighbor_lists[t], kind, p));
  }
  double sum = 0.0;
  for (std::size_t t = 0; t < batch.indices.size(); ++t) {
    const double r = train.Y(batch.indices[t]) - preds[t];
    sum += r * r;
  }
  return sum / static_cast<double>(batch.indices.size());
}

FittedParams train(const TrainingSet& data, const KernelParams& initial, const TrainConfig& config,
                   const BatchSpec& batch, const NeighborIndex& index) {
  if (config.k < 2) throw std::domain_error("train: k must be at least 2");
  if (index.size() != data.X.rows()) throw std::domain_error("train: index was not built on the training set");
  fmgp_train_config c{};
  c.k = config.k;
  c.kind = config.kind == KernelKind::RBF ? FMGP_RBF : FMGP_MATERN;
  c.has_rho = config.rho_bounds.has_value();
  c.has_nu = config.nu_bounds.has_value();
  c.has_tau = config.tau_bounds.has_value();
  if (c.has_rho) c.rho_lo = config.rho_bounds->lo, c.rho_hi = config.rho_bounds->hi;
  if (c.has_nu) c.nu_lo = config.nu_bounds->lo, c.nu_hi = config.nu_bounds->hi;
  if (c.has_tau) c.tau_lo = config.tau_bounds->lo, c.tau_hi = config.tau_bounds->hi;
  c.max_evals = config.max_evals;
  c.tol = config.tol;
  const fmgp_kernel_params kp0 = detail::abi_params(config.kind, initial);
  const auto Y = responses(data);
  std::vector<int32_t> bi(batch.indices.begin(), batch.indices.end());
  fmgp_kernel_params th{};
  double loss = 0.0;
  int32_t evals = 0, improved = 0;
  detail::check(fmgp_train(detail::row_major(data.X).data(), Y.data(), data.X.rows(),
                           static_cast<int32_t>(data.X.cols()), bi.data(), static_cast<int64_t>(bi.size()), &kp0, &c,
                           &th, &loss, &evals, &improved));
  return FittedParams{KernelParams(th.sigma, th.rho, th.nu, th.tau), config.kind, loss, evals, improved != 0};
}

Eigen::VectorXd muygps_predict(const TrainingSet& train, const Eigen::MatrixXd& Z, const FittedParams& fitted,
                               const NeighborIndex& index, int k) {
  (void)index;  // neighbours are always exact (the facade's index answers exactly)
  if (Z.cols() != train.X.cols()) throw std::domain_error("muygps_predict: test dimension mismatch");
  Eigen::VectorXd out(Z.rows());
  if (Z.rows() == 0) return out;
  const fmgp_kernel_params kp = detail::abi_params(fitted.kind, fitted.theta_hat);
  const auto Y = responses(train);
  int64_t failed = -1;
  detail::check(fmgp_muygps_predict(detail::row_major(train.X).data(), Y.data(), train.X.rows(),
                                    static_cast<int32_t>(train.X.cols()), detail::row_major(Z).data(), Z.rows(), k,
                                    &kp, train.mean_offset, out.data(), &failed));
  return out;
}

}  // namespace fastmuygps
