// Drop-in facade (B200): nearest-neighbour index of the FastMuyGPs API.
// Public surface of proj/core/include/fastmuygps/nn_index.hpp. Exact-mode
// queries run on the GPU (cell grid for d <= 3, tcgen05 filter / brute force
// otherwise) against a device-resident copy of the points. ApproxGraph mode
// builds a navigable-small-world graph on the GPU (fmgp_graph_build: the
// reference's seeded levels, each layer linked to its exact nearest
// neighbours) and answers query_knn / nearest_training_point with the
// reference's graph search, one warp per query (fmgp_graph_query_knn); graphs
// serialize in the reference's layout and reference-written graphs load.
#pragma once

#include <Eigen/Dense>
#include <cstdint>
#include <iosfwd>
#include <memory>
#include <string>
#include <vector>

struct fmgp_index;
struct fmgp_graph;

namespace fastmuygps {

enum class IndexMode : std::uint32_t { Exact = 0, ApproxGraph = 1 };

struct GraphParams {
  int max_degree = 16;
  int build_beam = 100;
  int query_beam = 0;
  std::uint64_t seed = 0;
};

// Indices into the training set with their Euclidean distances, ascending by
// (distance, index).
struct NeighborList {
  std::vector<int> indices;
  std::vector<double> distances;
};

class NeighborIndex {
 public:
  static NeighborIndex build(const Eigen::MatrixXd& points, IndexMode mode, const GraphParams& params = {});

  // k nearest stored points to q, excluding index exclude_index (>= 0) by
  // identity. dist_evals (if given) accumulates the distance evaluations
  // (Exact: the scan's count; ApproxGraph: the graph search's).
  NeighborList query_knn(const Eigen::VectorXd& q, int k, int exclude_index = -1,
                         std::size_t* dist_evals = nullptr) const;
  // Nearest stored point; ties go to the lower index.
  int nearest_training_point(const Eigen::VectorXd& q, std::size_t* dist_evals = nullptr) const;
  double distance_to(const Eigen::VectorXd& q, int j) const;

  int size() const noexcept { return n_; }
  int dim() const noexcept { return d_; }
  IndexMode mode() const noexcept { return mode_; }
  const GraphParams& params() const noexcept { return params_; }

  void serialize(std::ostream& out) const;
  static NeighborIndex deserialize(std::istream& in, const Eigen::MatrixXd& points,
                                   std::size_t* bytes_read = nullptr);

  // Facade extensions: batched queries in one device call, and the
  // row-major host copy of the points.
  std::vector<int> nearest_batch(const Eigen::MatrixXd& Q) const;
  const std::vector<double>& points_row_major() const noexcept { return pts_; }

 private:
  NeighborIndex() = default;
  int n_ = 0;
  int d_ = 0;
  IndexMode mode_ = IndexMode::Exact;
  GraphParams params_;
  std::vector<double> pts_;
  std::shared_ptr<fmgp_index> dev_;
  std::shared_ptr<fmgp_graph> graph_;  // ApproxGraph mode: the device graph (keeps dev_ alive)
};

}  // namespace fastmuygps
