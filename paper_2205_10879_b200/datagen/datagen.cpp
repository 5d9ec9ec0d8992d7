// Seeded host generators for the BASELINE.json workloads
// and for the reference test suites' random sets. The same arrays feed the
// oracle and the GPU; nothing is regenerated on the device.
//
// All engines are std::mt19937_64 with libstdc++'s uniform_real_distribution
// and normal_distribution, like the reference tests
// (proj/tests/test_fast_predict.cpp:21-29, test_nn_index.cpp:16-22).
// Arrays are row-major: X n*d, Y n*m, Z nt*d. Responses are detrended per
// output column (dataset.cpp:24-36: mean_offset = mean(raw_y), Y = raw_y - mean).
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <vector>

namespace {

constexpr double kPi = std::numbers::pi;

void detrend(double* Y, int64_t n, int m, double* mean_offset) {
  for (int c = 0; c < m; ++c) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += Y[i * m + c];
    double mu = s / static_cast<double>(n);
    for (int64_t i = 0; i < n; ++i) Y[i * m + c] -= mu;
    mean_offset[c] = mu;
  }
}

}  // namespace

extern "C" {

// Static description of BASELINE.json configs[cfg-1]. kind: 0 Matern, 1 RBF.
// tau = sqrt(nugget) so the diagonal is sigma^2 (1 + nugget).
int fmgp_config_info(int cfg, int* d, int64_t* n, int64_t* nt, int* k, int* m,
                     int* kind, double* sigma, double* rho, double* nu,
                     double* tau) {
  *sigma = 1.0;
  switch (cfg) {
    case 1: *d = 2; *n = 10000; *nt = 2000; *k = 30; *m = 1; *kind = 1; *rho = 0.1; *nu = 2.5; *tau = std::sqrt(1e-4); return 0;
    case 2: *d = 2; *n = 1000000; *nt = 1000000; *k = 50; *m = 1; *kind = 0; *rho = 0.05; *nu = 1.5; *tau = std::sqrt(1e-3); return 0;
    case 3: *d = 784; *n = 60000; *nt = 10000; *k = 30; *m = 10; *kind = 0; *rho = 10.0; *nu = 0.5; *tau = std::sqrt(1e-2); return 0;
    case 4: *d = 40; *n = 2000000; *nt = 500000; *k = 100; *m = 1; *kind = 1; *rho = 3.0; *nu = 2.5; *tau = std::sqrt(1e-2); return 0;
    case 5: *d = 3; *n = 8000000; *nt = 8000000; *k = 50; *m = 1; *kind = 0; *rho = 0.02; *nu = 2.5; *tau = std::sqrt(1e-4); return 0;
    default: return 1;
  }
}

// Generates config `cfg` at sizes (n, nt) — the full BASELINE sizes or a
// smaller parity-test slice with identical distributions — from `seed`
// (SURVEY.md §8(d) proposes 20261019 + cfg). X: n*d, Y: n*m, Z: nt*d,
// mean_offset: m. Returns 0, or 1 for an unknown config.
int fmgp_generate(int cfg, int64_t n, int64_t nt, uint64_t seed, double* X,
                  double* Y, double* Z, double* mean_offset) {
  int d, k, m, kind;
  int64_t n0, nt0;
  double sigma, rho, nu, tau;
  if (fmgp_config_info(cfg, &d, &n0, &nt0, &k, &m, &kind, &sigma, &rho, &nu, &tau) != 0) return 1;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  std::normal_distribution<double> g01(0.0, 1.0);
  switch (cfg) {
    case 1: {  // y = sin(2 pi x1) cos(2 pi x2) + N(0, 0.01^2)
      for (int64_t i = 0; i < n * d; ++i) X[i] = u01(rng);
      for (int64_t i = 0; i < nt * d; ++i) Z[i] = u01(rng);
      for (int64_t i = 0; i < n; ++i)
        Y[i] = std::sin(2 * kPi * X[2 * i]) * std::cos(2 * kPi * X[2 * i + 1]) + 0.01 * g01(rng);
      break;
    }
    case 2: {  // 256 random Fourier features, lengthscale 0.05, noise 0.05
      constexpr int F = 256;
      std::vector<double> w(F * 2), b(F);
      for (int j = 0; j < F; ++j) {
        w[2 * j] = g01(rng) / 0.05;
        w[2 * j + 1] = g01(rng) / 0.05;
        b[j] = 2 * kPi * u01(rng);
      }
      for (int64_t i = 0; i < n * d; ++i) X[i] = u01(rng);
      for (int64_t i = 0; i < nt * d; ++i) Z[i] = u01(rng);
      const double amp = std::sqrt(2.0 / F);
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < F; ++j) s += std::cos(w[2 * j] * X[2 * i] + w[2 * j + 1] * X[2 * i + 1] + b[j]);
        Y[i] = amp * s + 0.05 * g01(rng);
      }
      break;
    }
    case 3: {  // sparse [0,1] features, 10-class +-1 one-hot from argmax(x^T W)
      std::vector<double> W(static_cast<size_t>(d) * m);
      for (auto& v : W) v = g01(rng);
      auto feat = [&](double* A, int64_t rows) {
        for (int64_t i = 0; i < rows * d; ++i) {
          double keep = u01(rng);
          A[i] = keep < 0.8 ? 0.0 : u01(rng);
        }
      };
      feat(X, n);
      feat(Z, nt);
      for (int64_t i = 0; i < n; ++i) {
        int best = 0;
        double bv = -INFINITY;
        for (int c = 0; c < m; ++c) {
          double s = 0.0;
          for (int t = 0; t < d; ++t) s += X[i * d + t] * W[static_cast<size_t>(t) * m + c];
          if (s > bv) { bv = s; best = c; }
        }
        for (int c = 0; c < m; ++c) Y[i * m + c] = c == best ? 1.0 : -1.0;
      }
      break;
    }
    case 4: {  // y = tanh(w.x) + 0.3 sin(v.x) + N(0, 0.1^2), w, v ~ N(0, I/40)
      std::vector<double> w(d), v(d);
      const double sc = 1.0 / std::sqrt(static_cast<double>(d));
      for (int t = 0; t < d; ++t) w[t] = g01(rng) * sc;
      for (int t = 0; t < d; ++t) v[t] = g01(rng) * sc;
      for (int64_t i = 0; i < n * d; ++i) X[i] = g01(rng);
      for (int64_t i = 0; i < nt * d; ++i) Z[i] = g01(rng);
      for (int64_t i = 0; i < n; ++i) {
        double a = 0.0, b = 0.0;
        for (int t = 0; t < d; ++t) {
          a += w[t] * X[i * d + t];
          b += v[t] * X[i * d + t];
        }
        Y[i] = std::tanh(a) + 0.3 * std::sin(b) + 0.1 * g01(rng);
      }
      break;
    }
    case 5: {  // y = sum_j sin(4 pi x_j) + N(0, 0.05^2)
      for (int64_t i = 0; i < n * d; ++i) X[i] = u01(rng);
      for (int64_t i = 0; i < nt * d; ++i) Z[i] = u01(rng);
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int t = 0; t < d; ++t) s += std::sin(4 * kPi * X[i * d + t]);
        Y[i] = s + 0.05 * g01(rng);
      }
      break;
    }
  }
  detrend(Y, n, m, mean_offset);
  return 0;
}

// The reference tests' random_set (test_fast_predict.cpp:21-29): X filled in
// Eigen column-major order from U[0,1), y = cos(4 * rowsum) + 1.5, detrended.
// Written here row-major.
void fmgp_random_set(int64_t n, int d, uint64_t seed, double* X_rm, double* Y,
                     double* mean_offset) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> cm(static_cast<size_t>(n) * d);
  for (auto& v : cm) v = u(rng);
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      X_rm[i * d + j] = cm[static_cast<size_t>(j) * n + i];
      s += X_rm[i * d + j];
    }
    Y[i] = std::cos(4.0 * s) + 1.5;
  }
  detrend(Y, n, 1, mean_offset);
}

// The MuyGPs tests' sine_set (test_muygps.cpp:17-25): x ~ U[0,1) (n x 1),
// y = sin(8x), detrended.
void fmgp_sine_set(int64_t n, uint64_t seed, double* X, double* Y, double* mean_offset) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int64_t i = 0; i < n; ++i) X[i] = u(rng);
  for (int64_t i = 0; i < n; ++i) Y[i] = std::sin(8.0 * X[i]);
  detrend(Y, n, 1, mean_offset);
}

// BatchSpec::sample (muygps.cpp:15-30): a uniform sample of b of the n
// training indices without replacement, by a partial Fisher-Yates shuffle of
// 0..n-1 driven by std::mt19937_64(seed). Returns 1 when b is out of [1, n].
int fmgp_batch_sample(int32_t n, int32_t b, uint64_t seed, int32_t* out) {
  if (b < 1 || b > n) return 1;
  std::vector<int> pool(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) pool[i] = i;
  std::mt19937_64 rng(seed);
  for (int i = 0; i < b; ++i) {
    std::uniform_int_distribution<int> pick(i, n - 1);
    const int j = pick(rng);
    const int t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  for (int i = 0; i < b; ++i) out[i] = pool[i];
  return 0;
}

}  // extern "C"
