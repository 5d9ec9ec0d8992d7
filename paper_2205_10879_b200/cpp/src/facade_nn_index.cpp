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
T get_le(std::istream& in, std::size_t* bytes_read, std::string* keep = nullptr) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(v));
  if (!in) throw FormatError("truncated neighbor-index data", bytes_read != nullptr ? *bytes_read : 0);
  if (bytes_read != nullptr) *bytes_read += sizeof(v);
  if (keep != nullptr) keep->append(reinterpret_cast<const char*>(&v), sizeof(v));
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

NeighborIndex NeighborIndex::build(const Eigen::MatrixXd& points, IndexMode mode, const GraphParams& params) {
  if (params.max_degree < 2 || params.build_beam < 1) throw std::domain_error("NeighborIndex: invalid graph parameters");
  NeighborIndex ix;
  ix.pts_ = host_points(points);
  ix.n_ = static_cast<int>(points.rows());
  ix.d_ = static_cast<int>(points.cols());
  ix.mode_ = mode;
  ix.params_ = params;
  ix.dev_ = device_copy(ix.pts_, ix.n_, ix.d_);
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
  detail::check(fmgp_index_query_knn(dev_.get(), q.data(), 1, k, &ex, nl.indices.data(), nl.distances.data()));
  if (dist_evals != nullptr) *dist_evals += static_cast<std::size_t>(available);
  return nl;
}

int NeighborIndex::nearest_training_point(const Eigen::VectorXd& q, std::size_t* dist_evals) const {
  if (static_cast<int>(q.size()) != d_) throw std::domain_error("nearest_training_point: dimension mismatch");
  int32_t j = -1;
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
// then for ApproxGraph the graph. A graph read from a reference-written file
// is kept byte for byte and written back unchanged, so such models round-trip
// bit-exactly; an index this facade built (it never builds the HNSW graph,
// queries are exact) is written with the Exact tag.
void NeighborIndex::serialize(std::ostream& out) const {
  if (mode_ == IndexMode::ApproxGraph && !graph_blob_.empty()) {
    put_le<std::uint32_t>(out, 1u);
    out.write(graph_blob_.data(), static_cast<std::streamsize>(graph_blob_.size()));
    return;
  }
  put_le<std::uint32_t>(out, 0u);
}

NeighborIndex NeighborIndex::deserialize(std::istream& in, const Eigen::MatrixXd& points, std::size_t* bytes_read) {
  const auto mode = get_le<std::uint32_t>(in, bytes_read);
  if (mode > 1) throw FormatError("unknown neighbor-index mode tag", bytes_read != nullptr ? *bytes_read : 0);
  GraphParams gp;
  std::string blob;
  if (mode == 1) {
    // A graph written by the reference: validated and kept verbatim (written
    // back by serialize); queries stay exact.
    const auto n = static_cast<int>(points.rows());
    gp.max_degree = get_le<std::int32_t>(in, bytes_read, &blob);
    gp.build_beam = get_le<std::int32_t>(in, bytes_read, &blob);
    gp.query_beam = get_le<std::int32_t>(in, bytes_read, &blob);
    gp.seed = get_le<std::uint64_t>(in, bytes_read, &blob);
    const auto entry = get_le<std::int32_t>(in, bytes_read, &blob);
    (void)get_le<std::int32_t>(in, bytes_read, &blob);  // max level
    if (entry < 0 || entry >= n)
      throw FormatError("neighbor-index entry point out of range", bytes_read != nullptr ? *bytes_read : 0);
    for (int i = 0; i < n; ++i) {
      const auto lvl = get_le<std::int32_t>(in, bytes_read, &blob);
      if (lvl < 0) throw FormatError("negative node level in neighbor index", bytes_read != nullptr ? *bytes_read : 0);
      for (int l = 0; l <= lvl; ++l) {
        const auto cnt = get_le<std::uint32_t>(in, bytes_read, &blob);
        for (std::uint32_t c = 0; c < cnt; ++c) {
          const auto u = get_le<std::int32_t>(in, bytes_read, &blob);
          if (u < 0 || u >= n) throw FormatError("neighbor id out of range", bytes_read != nullptr ? *bytes_read : 0);
        }
      }
    }
  }
  NeighborIndex ix = build(points, static_cast<IndexMode>(mode), gp.max_degree >= 2 && gp.build_beam >= 1 ? gp : GraphParams{});
  ix.graph_blob_ = std::move(blob);
  return ix;
}

}  // namespace fastmuygps
