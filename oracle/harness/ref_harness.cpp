// ORACLE TEST INFRASTRUCTURE — not product code.
//
// C-callable harness around the *reference's own* public C++ API
// (proj/core/include/fastmuygps/*.hpp), linked with the reference TUs
// compiled unmodified (oracle/Makefile `ref`). Used only by tests/ (golden
// fixture generation, cross-checks of the C restatement) and by bench.py's
// `--impl reference` / cpu_baseline legs. Every entry point makes exactly the
// public calls the reference makes:
//   fmgp_ref_precompute      -> fastmuygps::precompute            (fast_predict.cpp:70-130)
//   fmgp_ref_precompute_rows -> the do_rows body on a row subset   (fast_predict.cpp:89-107):
//                               NeighborIndex::query_knn, cov_matrix_self, solve_spd
//   fmgp_ref_predict         -> fast_predict_batch / fast_predict_one (fast_predict.cpp:132-156)
//   fmgp_ref_query_knn, fmgp_ref_nearest, fmgp_ref_kernel_value -> nn_index.cpp / kernel.cpp
//   fmgp_ref_local_predictions -> local_prediction per entry     (muygps.cpp:32-62)
//   fmgp_ref_loocv_loss      -> loocv_loss                       (muygps.cpp:64-78)
//   fmgp_ref_train           -> BatchSpec::sample + train        (muygps.cpp:15-30, :214-270)
//   fmgp_ref_muygps_predict  -> muygps_predict                   (muygps.cpp:272-295)
//   fmgp_ref_predict_session / _run / _free -> a PrecomputedModel built once,
//                               then fast_predict_batch (threads <= 1) or
//                               fast_predict_one per row (threads > 1), for timing
//   fmgp_ref_save_model / fmgp_ref_load_model -> save_model / load_model
//                               (fast_predict.cpp:158-280), for cross-build file tests
// Multi-output (BASELINE cfg3, m > 1): the reference is single-output
// (dataset.hpp:14); the harness shares S and passes the k x m right-hand
// sides to the reference's own solve_spd (linalg.hpp:19-20), which solves
// them column by column with one factorisation.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "fastmuygps/errors.hpp"
#include "fastmuygps/fast_predict.hpp"
#include "fastmuygps/kernel.hpp"
#include "fastmuygps/linalg.hpp"
#include "fastmuygps/muygps.hpp"
#include "fastmuygps/nn_index.hpp"

using namespace fastmuygps;

namespace {

thread_local std::string g_err;

Eigen::MatrixXd from_rm(const double* a, int64_t n, int d) {
  Eigen::MatrixXd X(n, d);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) X(i, j) = a[i * d + j];
  return X;
}

Eigen::VectorXd vec_from(const double* a, int64_t n) {
  Eigen::VectorXd v(n);
  for (int64_t i = 0; i < n; ++i) v(i) = a[i];
  return v;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

KernelKind kind_of(int kind) { return kind == 1 ? KernelKind::RBF : KernelKind::Matern; }

}  // namespace

extern "C" {

const char* fmgp_ref_last_error() { return g_err.c_str(); }

double fmgp_ref_kernel_value(double d, int kind, double sigma, double rho,
                             double nu, double tau) {
  return kernel_value(d, kind_of(kind), KernelParams(sigma, rho, nu, tau));
}

// Full reference precompute (single output). S_out n*k int32, C_out n*k f64.
int fmgp_ref_precompute(const double* X_rm, const double* Y, int64_t n, int d,
                        int kind, double sigma, double rho, double nu,
                        double tau, int k, int threads, int32_t* S_out,
                        double* C_out) {
  return guard([&] {
    TrainingSet train;
    train.X = from_rm(X_rm, n, d);
    train.Y = Eigen::VectorXd(n);
    for (int64_t i = 0; i < n; ++i) train.Y(i) = Y[i];
    train.mean_offset = 0.0;
    FittedParams fitted{KernelParams(sigma, rho, nu, tau), kind_of(kind), 0.0, 0, false};
    NeighborIndex index = NeighborIndex::build(train.X, IndexMode::Exact);
    PrecomputedModel model = precompute(train, fitted, index, k, threads);
    std::memcpy(S_out, model.table.S.data(), sizeof(int32_t) * n * k);
    std::memcpy(C_out, model.C.data(), sizeof(double) * n * k);
  });
}

// The do_rows body (fast_predict.cpp:89-107) for an arbitrary row subset,
// spread over `threads` std::threads in contiguous chunks like :110-125.
// Y_rm is n x m row-major; C_out is nrows x k x m. The first NumericError's
// row is reported through fmgp_ref_last_error().
int fmgp_ref_precompute_rows(const double* X_rm, const double* Y_rm, int64_t n,
                             int d, int m, int kind, double sigma, double rho,
                             double nu, double tau, int k, const int64_t* rows,
                             int64_t nrows, int threads, int32_t* S_out,
                             double* C_out) {
  return guard([&] {
    Eigen::MatrixXd X = from_rm(X_rm, n, d);
    KernelParams p(sigma, rho, nu, tau);
    KernelKind kk = kind_of(kind);
    NeighborIndex index = NeighborIndex::build(X, IndexMode::Exact);
    std::vector<std::exception_ptr> errs(std::max(1, threads));
    auto work = [&](int w, int64_t b, int64_t e) {
      try {
        Eigen::MatrixXd xs(k, d);
        Eigen::MatrixXd ys(k, m);
        std::vector<int32_t> srow(k);
        for (int64_t r = b; r < e; ++r) {
          const int64_t i = rows[r];
          srow[0] = static_cast<int32_t>(i);
          if (k > 1) {
            NeighborList nl = index.query_knn(X.row(i).transpose(), k - 1, static_cast<int>(i));
            for (int t = 0; t < k - 1; ++t) srow[t + 1] = nl.indices[t];
          }
          for (int t = 0; t < k; ++t) {
            xs.row(t) = X.row(srow[t]);
            for (int c = 0; c < m; ++c) ys(t, c) = Y_rm[static_cast<int64_t>(srow[t]) * m + c];
          }
          Eigen::MatrixXd kss = cov_matrix_self(xs, kk, p);
          Eigen::MatrixXd sol = solve_spd(kss, ys, "precompute row " + std::to_string(i));
          for (int t = 0; t < k; ++t) {
            S_out[r * k + t] = srow[t];
            for (int c = 0; c < m; ++c) C_out[(r * k + t) * m + c] = sol(t, c);
          }
        }
      } catch (...) {
        errs[w] = std::current_exception();
      }
    };
    if (threads <= 1 || nrows < 2 * threads) {
      work(0, 0, nrows);
    } else {
      std::vector<std::thread> ws;
      int64_t chunk = (nrows + threads - 1) / threads;
      for (int w = 0; w < threads; ++w) {
        int64_t b = w * chunk, e = std::min<int64_t>(nrows, b + chunk);
        if (b < e) ws.emplace_back(work, w, b, e);
      }
      for (auto& t : ws) t.join();
    }
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

// Posterior means for Z through the reference model built from X, S, C
// (m outputs: C is n x k x m, out is nz x m). threads <= 1 calls
// fast_predict_batch exactly; threads > 1 splits rows over fast_predict_one,
// which the reference documents as safe for concurrent callers
// (fast_predict.hpp:20-24). nn_out (optional) receives the 1-NN index.
int fmgp_ref_predict(const double* X_rm, const int32_t* S, const double* C,
                     int64_t n, int d, int k, int m, int kind, double sigma,
                     double rho, double nu, double tau, double mean_offset,
                     const double* Z_rm, int64_t nz, int threads, double* out,
                     int32_t* nn_out) {
  return guard([&] {
    Eigen::MatrixXd X = from_rm(X_rm, n, d);
    NeighborIndex index = NeighborIndex::build(X, IndexMode::Exact);
    NeighborTable table;
    table.S.resize(n, k);
    std::memcpy(table.S.data(), S, sizeof(int32_t) * n * k);
    std::vector<PrecomputedModel> models;
    models.reserve(m);
    for (int c = 0; c < m; ++c) {
      Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor> Cc(n, k);
      for (int64_t i = 0; i < n * k; ++i) Cc.data()[i] = C[i * m + c];
      models.push_back(PrecomputedModel{X, table, std::move(Cc), KernelParams(sigma, rho, nu, tau),
                                        kind_of(kind), mean_offset, index});
    }
    Eigen::MatrixXd Z = from_rm(Z_rm, nz, d);
    if (threads <= 1) {
      for (int c = 0; c < m; ++c) {
        Eigen::VectorXd v = fast_predict_batch(models[c], Z);
        for (int64_t t = 0; t < nz; ++t) out[t * m + c] = v(t);
      }
      if (nn_out != nullptr)
        for (int64_t t = 0; t < nz; ++t) nn_out[t] = index.nearest_training_point(Z.row(t).transpose());
      return;
    }
    std::vector<std::thread> ws;
    int64_t chunk = (nz + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
      int64_t b = w * chunk, e = std::min<int64_t>(nz, b + chunk);
      if (b >= e) continue;
      ws.emplace_back([&, b, e] {
        for (int64_t t = b; t < e; ++t) {
          Eigen::VectorXd z = Z.row(t).transpose();
          for (int c = 0; c < m; ++c) out[t * m + c] = fast_predict_one(models[c], z);
          if (nn_out != nullptr) nn_out[t] = index.nearest_training_point(z);
        }
      });
    }
    for (auto& t : ws) t.join();
  });
}

int fmgp_ref_query_knn(const double* X_rm, int64_t n, int d, const double* q,
                       int k, int exclude, int32_t* idx_out, double* dist_out) {
  return guard([&] {
    NeighborIndex index = NeighborIndex::build(from_rm(X_rm, n, d), IndexMode::Exact);
    Eigen::VectorXd qq(d);
    for (int j = 0; j < d; ++j) qq(j) = q[j];
    NeighborList nl = index.query_knn(qq, k, exclude);
    for (int t = 0; t < k; ++t) {
      idx_out[t] = nl.indices[t];
      dist_out[t] = nl.distances[t];
    }
  });
}

int fmgp_ref_nearest(const double* X_rm, int64_t n, int d, const double* Q_rm,
                     int64_t nq, int32_t* out) {
  return guard([&] {
    NeighborIndex index = NeighborIndex::build(from_rm(X_rm, n, d), IndexMode::Exact);
    Eigen::VectorXd qq(d);
    for (int64_t t = 0; t < nq; ++t) {
      for (int j = 0; j < d; ++j) qq(j) = Q_rm[t * d + j];
      out[t] = index.nearest_training_point(qq);
    }
  });
}

int fmgp_ref_local_predictions(const double* X_rm, const double* Y, int64_t n, int d, const int32_t* batch,
                               const int32_t* nbr, const double* dist, int64_t b, int k, int kind, double sigma,
                               double rho, double nu, double tau, double* preds) {
  return guard([&] {
    TrainingSet ts{from_rm(X_rm, n, d), vec_from(Y, n), 0.0};
    KernelParams p(sigma, rho, nu, tau);
    for (int64_t t = 0; t < b; ++t) {
      NeighborList nl;
      nl.indices.assign(nbr + t * k, nbr + t * k + k);
      nl.distances.assign(dist + t * k, dist + t * k + k);
      preds[t] = local_prediction(ts, batch[t], nl, static_cast<KernelKind>(kind), p);
    }
  });
}

int fmgp_ref_loocv_loss(const double* X_rm, const double* Y, int64_t n, int d, const int32_t* batch,
                        const int32_t* nbr, const double* dist, int64_t b, int k, int kind, double sigma, double rho,
                        double nu, double tau, double* loss) {
  return guard([&] {
    TrainingSet ts{from_rm(X_rm, n, d), vec_from(Y, n), 0.0};
    BatchSpec bs{static_cast<int>(b), 0, std::vector<int>(batch, batch + b)};
    std::vector<NeighborList> lists(b);
    for (int64_t t = 0; t < b; ++t) {
      lists[t].indices.assign(nbr + t * k, nbr + t * k + k);
      lists[t].distances.assign(dist + t * k, dist + t * k + k);
    }
    *loss = loocv_loss(ts, bs, lists, static_cast<KernelKind>(kind), KernelParams(sigma, rho, nu, tau));
  });
}

// bounds: [has_rho, has_nu, has_tau] flags and [rho_lo, rho_hi, nu_lo, nu_hi, tau_lo, tau_hi].
int fmgp_ref_train(const double* X_rm, const double* Y, int64_t n, int d, int batch_b, uint64_t batch_seed, int k,
                   int kind, double sigma, double rho, double nu, double tau, const int32_t* has,
                   const double* bounds, int max_evals, double tol, double* theta_out /*sigma,rho,nu,tau*/,
                   double* final_loss, int32_t* evaluations, int32_t* improved, int32_t* batch_out) {
  return guard([&] {
    TrainingSet ts{from_rm(X_rm, n, d), vec_from(Y, n), 0.0};
    NeighborIndex index = NeighborIndex::build(ts.X, IndexMode::Exact);
    BatchSpec bs = BatchSpec::sample(static_cast<int>(n), batch_b, batch_seed);
    std::copy(bs.indices.begin(), bs.indices.end(), batch_out);
    TrainConfig cfg;
    cfg.k = k;
    cfg.kind = static_cast<KernelKind>(kind);
    if (has[0]) cfg.rho_bounds = Bounds{bounds[0], bounds[1]};
    if (has[1]) cfg.nu_bounds = Bounds{bounds[2], bounds[3]};
    if (has[2]) cfg.tau_bounds = Bounds{bounds[4], bounds[5]};
    cfg.max_evals = max_evals;
    cfg.tol = tol;
    FittedParams f = train(ts, KernelParams(sigma, rho, nu, tau), cfg, bs, index);
    theta_out[0] = f.theta_hat.sigma();
    theta_out[1] = f.theta_hat.rho();
    theta_out[2] = f.theta_hat.nu();
    theta_out[3] = f.theta_hat.tau();
    *final_loss = f.final_loss;
    *evaluations = f.evaluations;
    *improved = f.improved ? 1 : 0;
  });
}

int fmgp_ref_muygps_predict(const double* X_rm, const double* Y, int64_t n, int d, double mean_offset,
                            const double* Z_rm, int64_t nz, int k, int kind, double sigma, double rho, double nu,
                            double tau, double* out) {
  return guard([&] {
    TrainingSet ts{from_rm(X_rm, n, d), vec_from(Y, n), mean_offset};
    NeighborIndex index = NeighborIndex::build(ts.X, IndexMode::Exact);
    FittedParams f{KernelParams(sigma, rho, nu, tau), static_cast<KernelKind>(kind), 0.0, 0, false};
    Eigen::VectorXd r = muygps_predict(ts, from_rm(Z_rm, nz, d), f, index, k);
    for (int64_t t = 0; t < nz; ++t) out[t] = r(t);
  });
}

// A reference PrecomputedModel per output column, built once (the copies
// and the index build are outside whatever the caller times).
struct RefPredictSession {
  std::vector<PrecomputedModel> models;
  int d = 0, m = 0;
};

void* fmgp_ref_predict_session(const double* X_rm, const int32_t* S, const double* C, int64_t n, int d, int k, int m,
                               int kind, double sigma, double rho, double nu, double tau, double mean_offset) {
  RefPredictSession* out = nullptr;
  const int rc = guard([&] {
    auto* ss = new RefPredictSession();
    ss->d = d;
    ss->m = m;
    Eigen::MatrixXd X = from_rm(X_rm, n, d);
    NeighborIndex index = NeighborIndex::build(X, IndexMode::Exact);
    NeighborTable table;
    table.S.resize(n, k);
    std::memcpy(table.S.data(), S, sizeof(int32_t) * n * k);
    for (int c = 0; c < m; ++c) {
      Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor> Cc(n, k);
      for (int64_t i = 0; i < n * k; ++i) Cc.data()[i] = C[i * m + c];
      ss->models.push_back(PrecomputedModel{X, table, std::move(Cc), KernelParams(sigma, rho, nu, tau),
                                            kind_of(kind), mean_offset, index});
    }
    out = ss;
  });
  return rc == 0 ? out : nullptr;
}

int fmgp_ref_predict_run(void* session, const double* Z_rm, int64_t nz, int threads, double* out) {
  return guard([&] {
    auto* ss = static_cast<RefPredictSession*>(session);
    const int m = ss->m;
    Eigen::MatrixXd Z = from_rm(Z_rm, nz, ss->d);
    if (threads <= 1) {
      for (int c = 0; c < m; ++c) {
        Eigen::VectorXd v = fast_predict_batch(ss->models[c], Z);
        for (int64_t t = 0; t < nz; ++t) out[t * m + c] = v(t);
      }
      return;
    }
    std::vector<std::thread> ws;
    const int64_t chunk = (nz + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
      const int64_t b = w * chunk, e = std::min<int64_t>(nz, b + chunk);
      if (b >= e) continue;
      ws.emplace_back([&, b, e] {
        for (int64_t t = b; t < e; ++t) {
          Eigen::VectorXd z = Z.row(t).transpose();
          for (int c = 0; c < m; ++c) out[t * m + c] = fast_predict_one(ss->models[c], z);
        }
      });
    }
    for (auto& t : ws) t.join();
  });
}

void fmgp_ref_predict_free(void* session) { delete static_cast<RefPredictSession*>(session); }

// save_model of a reference model assembled from the given arrays; mode 1
// builds the index as IndexMode::ApproxGraph with the given graph parameters
// (its HNSW blob is written by the reference, nn_index.cpp:397-416).
int fmgp_ref_save_model(const double* X_rm, const int32_t* S, const double* C, int64_t n, int d, int k, int kind,
                        double sigma, double rho, double nu, double tau, double mean_offset, int mode, int max_degree,
                        int build_beam, uint64_t seed, const char* path) {
  return guard([&] {
    Eigen::MatrixXd X = from_rm(X_rm, n, d);
    GraphParams gp;
    gp.max_degree = max_degree;
    gp.build_beam = build_beam;
    gp.seed = seed;
    NeighborIndex index = NeighborIndex::build(X, mode == 1 ? IndexMode::ApproxGraph : IndexMode::Exact, gp);
    NeighborTable table;
    table.S.resize(n, k);
    std::memcpy(table.S.data(), S, sizeof(int32_t) * n * k);
    Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor> Cc(n, k);
    std::memcpy(Cc.data(), C, sizeof(double) * n * k);
    PrecomputedModel model{X, table, std::move(Cc), KernelParams(sigma, rho, nu, tau), kind_of(kind), mean_offset,
                           index};
    save_model(model, path);
  });
}

// load_model, then fast_predict_batch of Z; dims_out = {n, d, k, mode}.
int fmgp_ref_load_model(const char* path, const double* Z_rm, int64_t nz, int64_t* dims_out, double* pred_out) {
  return guard([&] {
    PrecomputedModel model = load_model(path);
    dims_out[0] = model.X.rows();
    dims_out[1] = model.X.cols();
    dims_out[2] = model.table.S.cols();
    dims_out[3] = model.index.mode() == IndexMode::ApproxGraph ? 1 : 0;
    if (nz > 0) {
      Eigen::VectorXd v = fast_predict_batch(model, from_rm(Z_rm, nz, static_cast<int>(model.X.cols())));
      for (int64_t t = 0; t < nz; ++t) pred_out[t] = v(t);
    }
  });
}

// load_model then save_model (the reference re-writing a file it read).
int fmgp_ref_resave(const char* path_in, const char* path_out) {
  return guard([&] { save_model(load_model(path_in), path_out); });
}

}  // extern "C"
