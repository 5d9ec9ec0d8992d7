// C++ facade: nn_index.hpp over the C ABI's device-resident index handle.
#include <bit>
#include <cmath>
#include <istream>
#include <ostream>
#include <stdexcept>

#include "facade_common.hpp"
#include "fastmuygps/nn_index.hpp"

namespace fastmuygps {

namespace {

template <typename T>
void put_le(std::ostream& out, T v) {
  static_assert(std::endian::native == std::endian::little);
  out.write(reinterpret_cast<const char*>(&v), sizeof(v));
}

template <typename T>
T get_le(std::istream& in, std::size_t* bytes_read) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(v));
  if (!in) throw FormatError("truncated neighbor-index data", bytes_read != nullptr ? *bytes_read : 0);
  if (bytes_read != nullptr) *bytes_read += sizeof(v);
  return v;
}

std::vector<double> host_points(const Eigen::MatrixXd& P) {
  if (P.rows() < 1) throw std::domain_error("NeighborIndex: empty point set");
  if (!P.allFinite()) throw std::domain_error("NeighborIndex: non-finite coordinates");
  return detail::row_major(P);
}

std::shared_ptr<fmgp_index> device_copy(const std::vector<double>& pts, int n, int d) {
  const int dev = -1;  // the calling thread's current device
  fmgp_index* h = nullptr;
  detail::check(fmgp_index_create(pts.data(), n, d, dev, &h));
  return std::shared_ptr<fmgp_index>(h, fmgp_index_destroy);
}

}  // namespace

namespace {
std::shared_ptr<fmgp_graph> wrap_graph(fmgp_graph* g, std::shared_ptr<fmgp_index> ix) {
  return std::shared_ptr<fmgp_graph>(g, [ix](fmgp_graph* p) { fmgp_graph_destroy(p); });
}
}  // namespace

NeighborIndex NeighborIndex::build(const Eigen::MatrixXd& points, IndexMode mode, const GraphParams& params) {
  if (params.max_degree < 2 || params.build_beam < 1) throw std::domain_error("NeighborIndex: invalid graph parameters");
  NeighborIndex ix;
  ix.pts_ = host_points(points);
  ix.n_ = static_cast<int>(points.rows());
  ix.d_ = static_cast<int>(points.cols());
  ix.mode_ = mode;
  ix.params_ = params;
  ix.dev_ = device_copy(ix.pts_, ix.n_, ix.d_);
  if (mode == IndexMode::ApproxGraph) {
    fmgp_graph* g = nullptr;
    detail::check(fmgp_graph_build(ix.dev_.get(), params.max_degree, params.build_beam, params.query_beam,
                                   params.seed, &g));
    ix.graph_ = wrap_graph(g, ix.dev_);
  }
  return ix;
}

NeighborList NeighborIndex::query_knn(const Eigen::VectorXd& q, int k, int exclude_index, std::size_t* dist_evals) const {
  if (static_cast<int>(q.size()) != d_) throw std::domain_error("query_knn: query dimension mismatch");
  const int available = n_ - (exclude_index >= 0 ? 1 : 0);
  if (k < 1 || k > available) throw std::domain_error("query_knn: k out of range");
  NeighborList nl;
  nl.indices.resize(k);
  nl.distances.resize(k);
  const int32_t ex = exclude_index;
  if (graph_) {
    uint64_t ev = 0;
    detail::check(fmgp_graph_query_knn(graph_.get(), q.data(), 1, k, &ex, nl.indices.data(), nl.distances.data(), &ev));
    if (dist_evals != nullptr) *dist_evals += static_cast<std::size_t>(ev);
    return nl;
  }
  detail::check(fmgp_index_query_knn(dev_.get(), q.data(), 1, k, &ex, nl.indices.data(), nl.distances.data()));
  if (dist_evals != nullptr) *dist_evals += static_cast<std::size_t>(available);
  return nl;
}

int NeighborIndex::nearest_training_point(const Eigen::VectorXd& q, std::size_t* dist_evals) const {
  if (static_cast<int>(q.size()) != d_) throw std::domain_error("nearest_training_point: dimension mismatch");
  int32_t j = -1;
  if (graph_) {
    uint64_t ev = 0;
    detail::check(fmgp_graph_nearest(graph_.get(), q.data(), 1, &j, &ev));
    if (dist_evals != nullptr) *dist_evals += static_cast<std::size_t>(ev);
    return j;
  }
  detail::check(fmgp_index_nearest(dev_.get(), q.data(), 1, &j));
  if (dist_evals != nullptr) *dist_evals += static_cast<std::size_t>(n_);
  return j;
}

std::vector<int> NeighborIndex::nearest_batch(const Eigen::MatrixXd& Q) const {
  if (static_cast<int>(Q.cols()) != d_) throw std::domain_error("nearest_training_point: dimension mismatch");
  const auto qr = detail::row_major(Q);
  std::vector<int> out(static_cast<std::size_t>(Q.rows()));
  if (Q.rows() > 0) detail::check(fmgp_index_nearest(dev_.get(), qr.data(), Q.rows(), out.data()));
  return out;
}

double NeighborIndex::distance_to(const Eigen::VectorXd& q, int j) const {
  if (static_cast<int>(q.size()) != d_ || j < 0 || j >= n_) throw std::domain_error("distance_to: bad query or index");
  double out = 0.0;
  const int32_t jj = j;
  detail::check(fmgp_index_distances(dev_.get(), q.data(), &jj, 1, &out));
  return out;
}

// The blob is the reference's layout (nn_index.cpp:397-416): a u32 mode tag,
// then for ApproxGraph the graph parameters, entry point, maximum level and
// every node's level and layer link lists (layer 0 first).
void NeighborIndex::serialize(std::ostream& out) const {
  if (!graph_) {
    put_le<std::uint32_t>(out, 0u);
    return;
  }
  int32_t entry = 0, max_level = 0;
  int64_t counts_total = 0, ids_total = 0;
  detail::check(fmgp_graph_info(graph_.get(), &entry, &max_level, &counts_total, &ids_total));
  std::vector<int32_t> levels(static_cast<std::size_t>(n_));
  std::vector<uint32_t> counts(static_cast<std::size_t>(counts_total));
  std::vector<int32_t> ids(static_cast<std::size_t>(std::max<int64_t>(ids_total, 1)));
  detail::check(fmgp_graph_export(graph_.get(), levels.data(), counts.data(), ids.data()));
  put_le<std::uint32_t>(out, 1u);
  put_le<std::int32_t>(out, params_.max_degree);
  put_le<std::int32_t>(out, params_.build_beam);
  put_le<std::int32_t>(out, params_.query_beam);
  put_le<std::uint64_t>(out, params_.seed);
  put_le<std::int32_t>(out, entry);
  put_le<std::int32_t>(out, max_level);
  std::size_t c = 0, p = 0;
  for (int i = 0; i < n_; ++i) {
    put_le<std::int32_t>(out, levels[i]);
    for (int l = 0; l <= levels[i]; ++l) {
      const uint32_t cnt = counts[c++];
      put_le<std::uint32_t>(out, cnt);
      for (uint32_t t = 0; t < cnt; ++t) put_le<std::int32_t>(out, ids[p++]);
    }
  }
}

NeighborIndex NeighborIndex::deserialize(std::istream& in, const Eigen::MatrixXd& points, std::size_t* bytes_read) {
  const auto mode = get_le<std::uint32_t>(in, bytes_read);
  if (mode > 1) throw FormatError("unknown neighbor-index mode tag", bytes_read != nullptr ? *bytes_read : 0);
  if (mode == 0) return build(points, IndexMode::Exact);
  auto at = [&] { return bytes_read != nullptr ? *bytes_read : 0; };
  const auto n = static_cast<int>(points.rows());
  GraphParams gp;
  gp.max_degree = get_le<std::int32_t>(in, bytes_read);
  gp.build_beam = get_le<std::int32_t>(in, bytes_read);
  gp.query_beam = get_le<std::int32_t>(in, bytes_read);
  gp.seed = get_le<std::uint64_t>(in, bytes_read);
  const auto entry = get_le<std::int32_t>(in, bytes_read);
  const auto max_level = get_le<std::int32_t>(in, bytes_read);
  if (entry < 0 || entry >= n) throw FormatError("neighbor-index entry point out of range", at());
  std::vector<int32_t> levels(static_cast<std::size_t>(n));
  std::vector<uint32_t> counts;
  std::vector<int32_t> ids;
  for (int i = 0; i < n; ++i) {
    const auto lvl = get_le<std::int32_t>(in, bytes_read);
    if (lvl < 0) throw FormatError("negative node level in neighbor index", at());
    levels[i] = lvl;
    for (int l = 0; l <= lvl; ++l) {
      const auto cnt = get_le<std::uint32_t>(in, bytes_read);
      counts.push_back(cnt);
      for (std::uint32_t c = 0; c < cnt; ++c) {
        const auto u = get_le<std::int32_t>(in, bytes_read);
        if (u < 0 || u >= n) throw FormatError("neighbor id out of range", at());
        ids.push_back(u);
      }
    }
  }
  // the index itself: points on the device; the graph as read
  NeighborIndex ix;
  ix.pts_ = host_points(points);
  ix.n_ = n;
  ix.d_ = static_cast<int>(points.cols());
  ix.mode_ = IndexMode::ApproxGraph;
  ix.params_ = gp;
  ix.dev_ = device_copy(ix.pts_, ix.n_, ix.d_);
  fmgp_graph* g = nullptr;
  if (ids.empty()) ids.push_back(0);
  detail::check(fmgp_graph_load(ix.dev_.get(), gp.max_degree, gp.build_beam, gp.query_beam, gp.seed, entry, max_level,
                                levels.data(), counts.data(), ids.data(), &g));
  ix.graph_ = wrap_graph(g, ix.dev_);
  return ix;
}

}  // namespace fastmuygps
