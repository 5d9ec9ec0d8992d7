// C++ facade: fast_predict.hpp over the C ABI, plus the FMGP v1 model file.
#include <zlib.h>

#include <bit>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>

#include "facade_common.hpp"
#include "fastmuygps/fast_predict.hpp"

namespace fastmuygps {

namespace detail {

struct DeviceModelSlot {
  std::mutex mu;
  const void* x = nullptr;
  const void* s = nullptr;
  const void* c = nullptr;
  Eigen::Index n = 0, d = 0, k = 0;
  fmgp_kernel_params kp{};
  double mo = 0.0;
  std::shared_ptr<fmgp_model> h;
};

DeviceModelCache::DeviceModelCache() : slot(std::make_shared<DeviceModelSlot>()) {}
DeviceModelCache::DeviceModelCache(const DeviceModelCache&) : slot(std::make_shared<DeviceModelSlot>()) {}
DeviceModelCache& DeviceModelCache::operator=(const DeviceModelCache&) {
  slot = std::make_shared<DeviceModelSlot>();
  return *this;
}
DeviceModelCache::~DeviceModelCache() = default;

}  // namespace detail

namespace {

// The model's device replica: created once (fmgp_model_create uploads X, S, C
// and builds the predict-walk grid), then shared by every predict call.
std::shared_ptr<fmgp_model> device_model(const PrecomputedModel& model) {
  auto slot = model.device.slot;
  if (!slot) slot = std::make_shared<detail::DeviceModelSlot>();  // a moved-from model
  const fmgp_kernel_params kp = detail::abi_params(model.kind, model.params);
  std::lock_guard<std::mutex> lk(slot->mu);
  const bool same = slot->h && slot->x == model.X.data() && slot->s == model.table.S.data() &&
                    slot->c == model.C.data() && slot->n == model.X.rows() && slot->d == model.X.cols() &&
                    slot->k == model.table.S.cols() && slot->kp.kind == kp.kind && slot->kp.sigma == kp.sigma &&
                    slot->kp.rho == kp.rho && slot->kp.nu == kp.nu && slot->kp.tau == kp.tau &&
                    slot->mo == model.mean_offset;
  if (same) return slot->h;
  const auto n = static_cast<int64_t>(model.X.rows());
  const auto d = static_cast<int32_t>(model.X.cols());
  const auto k = static_cast<int32_t>(model.table.S.cols());
  if (model.C.rows() != model.X.rows() || model.C.cols() != k || model.table.S.rows() != model.X.rows())
    throw std::domain_error("fast_predict: model tables do not match the training set");
  const double mo = model.mean_offset;
  fmgp_model* h = nullptr;
  detail::check(fmgp_model_create(detail::row_major(model.X).data(), model.table.S.data(), model.C.data(), n, d, k, 1,
                                  &kp, &mo, -1, &h));
  slot->h = std::shared_ptr<fmgp_model>(h, fmgp_model_destroy);
  slot->x = model.X.data();
  slot->s = model.table.S.data();
  slot->c = model.C.data();
  slot->n = model.X.rows();
  slot->d = model.X.cols();
  slot->k = model.table.S.cols();
  slot->kp = kp;
  slot->mo = mo;
  return slot->h;
}

}  // namespace

PrecomputedModel precompute(const TrainingSet& train, const FittedParams& fitted, const NeighborIndex& index, int k,
                            int threads) {
  (void)threads;  // the device result is identical for any host thread count
  const auto n = static_cast<int64_t>(train.X.rows());
  if (k < 1 || k > n) throw std::domain_error("precompute: k out of range");
  if (index.size() != n) throw std::domain_error("precompute: index was not built on the training set");
  const auto d = static_cast<int32_t>(train.X.cols());
  const fmgp_kernel_params kp = detail::abi_params(fitted.kind, fitted.theta_hat);
  NeighborTable table;
  table.S.resize(n, k);
  Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor> C(n, k);
  std::vector<double> Y(train.Y.data(), train.Y.data() + n);
  int64_t failed = -1;
  const int rc = fmgp_precompute(detail::row_major(train.X).data(), Y.data(), n, d, 1, &kp, k, table.S.data(),
                                 C.data(), &failed);
  detail::check(rc);
  return PrecomputedModel{train.X, std::move(table), std::move(C), fitted.theta_hat, fitted.kind, train.mean_offset,
                          index};
}

Eigen::VectorXd fast_predict_batch(const PrecomputedModel& model, const Eigen::MatrixXd& Z) {
  if (Z.cols() != model.X.cols()) throw std::domain_error("fast_predict_batch: test dimension mismatch");
  Eigen::VectorXd out(Z.rows());
  if (Z.rows() == 0) return out;
  const std::shared_ptr<fmgp_model> h = device_model(model);
  if (Z.rows() == 1) {  // fast_predict_one: Eigen's column-major 1 x d is already the row
    detail::check(fmgp_model_predict(h.get(), Z.data(), 1, out.data(), nullptr));
    return out;
  }
  const auto zr = detail::row_major(Z);
  detail::check(fmgp_model_predict(h.get(), zr.data(), Z.rows(), out.data(), nullptr));
  return out;
}

double fast_predict_one(const PrecomputedModel& model, const Eigen::VectorXd& z) {
  if (z.size() != model.X.cols()) throw std::domain_error("nearest_training_point: dimension mismatch");
  double out = 0.0;
  const std::shared_ptr<fmgp_model> h = device_model(model);
  detail::check(fmgp_model_predict(h.get(), z.data(), 1, &out, nullptr));
  return out;
}

// ---------------------------------------------------------------- model file
// Layout (fast_predict.cpp:158-202): "FMGP", u32 version 1, u64 n, d, k,
// f64 sigma, rho, nu, tau, u32 kind, X row-major f64, S int32 n*k, C f64 n*k,
// f64 mean_offset, u64 index-blob size + blob, u32 CRC-32 of all prior bytes.

namespace {

static_assert(std::endian::native == std::endian::little, "the model file is little-endian");
constexpr char kMagic[4] = {'F', 'M', 'G', 'P'};
constexpr std::uint32_t kVersion = 1;

class CrcOut {
 public:
  explicit CrcOut(const std::filesystem::path& p) : f_(p, std::ios::binary) {
    if (!f_) throw std::runtime_error("cannot open model file for writing: " + p.string());
  }
  void bytes(const void* p, std::size_t n) {
    f_.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
    crc_ = crc32(crc_, static_cast<const Bytef*>(p), static_cast<uInt>(n));
  }
  template <typename T>
  void val(T v) {
    bytes(&v, sizeof(v));
  }
  void finish(const std::filesystem::path& p) {
    const auto c = static_cast<std::uint32_t>(crc_);
    f_.write(reinterpret_cast<const char*>(&c), sizeof(c));
    if (!f_) throw std::runtime_error("model write failed: " + p.string());
  }

 private:
  std::ofstream f_;
  uLong crc_ = crc32(0L, Z_NULL, 0);
};

class CrcIn {
 public:
  explicit CrcIn(const std::filesystem::path& p) : f_(p, std::ios::binary) {
    if (!f_) throw std::runtime_error("cannot open model file: " + p.string());
  }
  void bytes(void* p, std::size_t n, const char* what) {
    f_.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
    const auto got = static_cast<std::size_t>(f_.gcount());
    if (got != n) throw FormatError(std::string("truncated model file while reading ") + what, off_ + got);
    crc_ = crc32(crc_, static_cast<const Bytef*>(p), static_cast<uInt>(n));
    off_ += n;
  }
  template <typename T>
  T val(const char* what) {
    T v{};
    bytes(&v, sizeof(v), what);
    return v;
  }
  std::size_t offset() const { return off_; }
  std::uint32_t crc() const { return static_cast<std::uint32_t>(crc_); }
  std::ifstream& stream() { return f_; }

 private:
  std::ifstream f_;
  uLong crc_ = crc32(0L, Z_NULL, 0);
  std::size_t off_ = 0;
};

}  // namespace

void save_model(const PrecomputedModel& model, const std::filesystem::path& path) {
  CrcOut w(path);
  const auto n = static_cast<std::uint64_t>(model.X.rows());
  const auto d = static_cast<std::uint64_t>(model.X.cols());
  const auto k = static_cast<std::uint64_t>(model.table.S.cols());
  w.bytes(kMagic, sizeof(kMagic));
  w.val<std::uint32_t>(kVersion);
  w.val<std::uint64_t>(n);
  w.val<std::uint64_t>(d);
  w.val<std::uint64_t>(k);
  w.val<double>(model.params.sigma());
  w.val<double>(model.params.rho());
  w.val<double>(model.params.nu());
  w.val<double>(model.params.tau());
  w.val<std::uint32_t>(model.kind == KernelKind::RBF ? 1u : 0u);
  const auto xr = detail::row_major(model.X);
  w.bytes(xr.data(), xr.size() * sizeof(double));
  w.bytes(model.table.S.data(), n * k * sizeof(std::int32_t));
  w.bytes(model.C.data(), n * k * sizeof(double));
  w.val<double>(model.mean_offset);
  std::ostringstream blob;
  model.index.serialize(blob);
  const std::string b = std::move(blob).str();
  w.val<std::uint64_t>(b.size());
  w.bytes(b.data(), b.size());
  w.finish(path);
}

PrecomputedModel load_model(const std::filesystem::path& path) {
  CrcIn r(path);
  char magic[4];
  r.bytes(magic, sizeof(magic), "magic");
  if (std::memcmp(magic, kMagic, sizeof(kMagic)) != 0) throw FormatError("bad magic bytes; not a model file", 0);
  const auto version = r.val<std::uint32_t>("version");
  if (version != kVersion)
    throw FormatError("unsupported model format version " + std::to_string(version) + " (expected " +
                          std::to_string(kVersion) + ")",
                      sizeof(kMagic));
  const auto n = r.val<std::uint64_t>("n");
  const auto d = r.val<std::uint64_t>("d");
  const auto k = r.val<std::uint64_t>("k");
  if (n < 1 || d < 1 || k < 1 || k > n) throw FormatError("implausible model dimensions", r.offset());
  const double sigma = r.val<double>("sigma");
  const double rho = r.val<double>("rho");
  const double nu = r.val<double>("nu");
  const double tau = r.val<double>("tau");
  const auto tag = r.val<std::uint32_t>("kind");
  if (tag > 1) throw FormatError("unknown kernel kind tag", r.offset());
  std::vector<double> xr(n * d);
  r.bytes(xr.data(), xr.size() * sizeof(double), "X");
  Eigen::MatrixXd X = detail::from_row_major(xr.data(), static_cast<Eigen::Index>(n), static_cast<Eigen::Index>(d));
  NeighborTable table;
  table.S.resize(static_cast<Eigen::Index>(n), static_cast<Eigen::Index>(k));
  r.bytes(table.S.data(), n * k * sizeof(std::int32_t), "S");
  for (std::uint64_t i = 0; i < n; ++i)
    if (table.S(static_cast<Eigen::Index>(i), 0) != static_cast<std::int32_t>(i))
      throw FormatError("neighbor table row does not start with its own index", r.offset());
  Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor> C(static_cast<Eigen::Index>(n),
                                                                           static_cast<Eigen::Index>(k));
  r.bytes(C.data(), n * k * sizeof(double), "C");
  const double mean_offset = r.val<double>("mean_offset");
  const auto blob_size = r.val<std::uint64_t>("index blob size");
  std::string blob(blob_size, '\0');
  r.bytes(blob.data(), blob_size, "index blob");
  std::istringstream bs(blob);
  NeighborIndex index = NeighborIndex::deserialize(bs, X);
  const std::uint32_t computed = r.crc();
  std::uint32_t stored = 0;
  r.stream().read(reinterpret_cast<char*>(&stored), sizeof(stored));
  if (static_cast<std::size_t>(r.stream().gcount()) != sizeof(stored))
    throw FormatError("truncated model file while reading checksum", r.offset());
  if (stored != computed) throw FormatError("model file checksum mismatch", r.offset());
  return PrecomputedModel{std::move(X), std::move(table), std::move(C), KernelParams(sigma, rho, nu, tau),
                          tag == 1 ? KernelKind::RBF : KernelKind::Matern, mean_offset, std::move(index)};
}

}  // namespace fastmuygps
