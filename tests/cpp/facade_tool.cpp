// TEST TOOL — drives the C++ drop-in facade (paper_2205_10879_b200/cpp,
// libfastmuygps_b200.so) from tests/test_gpu_facade_model.py. Not product code.
//
//   facade_tool bench_one <n> <reps>
//       cfg2-shaped model (d = 2, n points, k = 50, Matern 1.5, rho 0.05,
//       nugget 1e-3) through precompute, then fast_predict_one timed per call
//       (steady_clock, after warm-up); prints one JSON line.
//   facade_tool save <data.bin> <model path>
//       data.bin (little-endian): i64 n, d, k, mode; u32 kind; f64 sigma, rho,
//       nu, tau, mean_offset; X row-major n*d; Y n. precompute + save_model;
//       prints the model's predictions at the data's first min(n, 64) points
//       shifted by 1e-3 (JSON).
//   facade_tool load <model path> <Z.bin> <resave path>
//       load_model, fast_predict_batch at Z.bin (i64 nz, d; f64 nz*d), save_model
//       again; prints the predictions (JSON, %.17g).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#include "fastmuygps/fast_predict.hpp"

using namespace fastmuygps;

namespace {

template <typename T>
T rd(std::ifstream& f) {
  T v{};
  f.read(reinterpret_cast<char*>(&v), sizeof(v));
  return v;
}

void print_vec(const char* key, const Eigen::VectorXd& v) {
  std::printf("{\"%s\": [", key);
  for (Eigen::Index i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v(i));
  std::printf("]}\n");
}

int bench_one(int n, int reps) {
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  Eigen::MatrixXd X(n, 2);
  Eigen::VectorXd y(n);
  for (int i = 0; i < n; ++i) {
    X(i, 0) = u(g);
    X(i, 1) = u(g);
    y(i) = std::sin(6.28 * X(i, 0)) * std::cos(6.28 * X(i, 1));
  }
  TrainingSet train = detrend(X, y);
  FittedParams f{KernelParams(1.0, 0.05, 1.5, std::sqrt(1e-3)), KernelKind::Matern, 0.0, 0, false};
  NeighborIndex index = NeighborIndex::build(train.X, IndexMode::Exact);
  PrecomputedModel model = precompute(train, f, index, 50);
  Eigen::VectorXd z(2);
  z << 0.5, 0.5;
  const auto t0 = std::chrono::steady_clock::now();
  double acc = fast_predict_one(model, z);  // first call: creates the model's device replica
  const double first_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  for (int i = 0; i < 20; ++i) acc += fast_predict_one(model, z);
  std::vector<double> us;
  for (int r = 0; r < reps; ++r) {
    z << u(g), u(g);
    const auto t = std::chrono::steady_clock::now();
    acc += fast_predict_one(model, z);
    us.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t).count());
  }
  std::sort(us.begin(), us.end());
  std::printf("{\"n\": %d, \"first_us\": %.1f, \"median_us\": %.2f, \"p90_us\": %.2f, \"checksum\": %.6g}\n", n,
              first_us, us[us.size() / 2], us[us.size() * 9 / 10], acc);
  return 0;
}

int save(const char* data, const char* path) {
  std::ifstream f(data, std::ios::binary);
  const auto n = rd<int64_t>(f), d = rd<int64_t>(f), k = rd<int64_t>(f), mode = rd<int64_t>(f);
  const auto kind = rd<uint32_t>(f);
  const double sigma = rd<double>(f), rho = rd<double>(f), nu = rd<double>(f), tau = rd<double>(f),
               mo = rd<double>(f);
  Eigen::MatrixXd X(n, d);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < d; ++j) X(i, j) = rd<double>(f);
  Eigen::VectorXd Y(n);
  for (int64_t i = 0; i < n; ++i) Y(i) = rd<double>(f);
  TrainingSet train{X, Y, mo};
  FittedParams fp{KernelParams(sigma, rho, nu, tau), kind == 1 ? KernelKind::RBF : KernelKind::Matern, 0.0, 0, false};
  NeighborIndex index = NeighborIndex::build(X, mode == 1 ? IndexMode::ApproxGraph : IndexMode::Exact);
  PrecomputedModel model = precompute(train, fp, index, static_cast<int>(k));
  save_model(model, path);
  const int64_t nz = std::min<int64_t>(n, 64);
  Eigen::MatrixXd Z = X.topRows(nz).array() + 1e-3;
  print_vec("pred", fast_predict_batch(model, Z));
  return 0;
}

int load(const char* path, const char* zfile, const char* resave) {
  PrecomputedModel model = load_model(path);
  std::ifstream f(zfile, std::ios::binary);
  const auto nz = rd<int64_t>(f), d = rd<int64_t>(f);
  Eigen::MatrixXd Z(nz, d);
  for (int64_t i = 0; i < nz; ++i)
    for (int64_t j = 0; j < d; ++j) Z(i, j) = rd<double>(f);
  print_vec("pred", fast_predict_batch(model, Z));
  save_model(model, resave);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "bench_one" && argc == 4) return bench_one(std::atoi(argv[2]), std::atoi(argv[3]));
    if (cmd == "save" && argc == 4) return save(argv[2], argv[3]);
    if (cmd == "load" && argc == 5) return load(argv[2], argv[3], argv[4]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "facade_tool: %s\n", e.what());
    return 2;
  }
  std::fprintf(stderr, "usage: facade_tool bench_one <n> <reps> | save <data.bin> <path> | load <path> <Z.bin> <out>\n");
  return 1;
}
